// FP64 issue-rate microbenchmark (profiling tool, not product code): the
// FP64 pipe peak on this GPU for DADD, DMUL and DFMA (explicit intrinsics, so
// -fmad=false does not matter), many independent accumulators per thread,
// grid = 8 x SMs x 1024 threads.  Prints JSON: op/s per instruction kind and
// flop/s (DFMA = 2 flops).  The FP64 roofline denominator of the simulation,
// inter-reorder and search kernels (SURVEY.md §7 hard part 4).
#include <cstdio>
#include <cuda_runtime.h>

template <int KIND>
__global__ void __launch_bounds__(256) fp64_loop(double* out, int iters, double a, double b) {
  constexpr int N = 8;  // independent chains per thread
  double x[N];
#pragma unroll
  for (int k = 0; k < N; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < N; ++k) {
      if (KIND == 0) x[k] = __dadd_rn(x[k], a);
      if (KIND == 1) x[k] = __dmul_rn(x[k], b);
      if (KIND == 2) x[k] = __fma_rn(x[k], b, a);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < N; ++k) s += x[k];
  if (s == 1.2345) out[blockIdx.x] = s;  // keep the work
}

int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaMalloc(&out, 1 << 20);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  const double ops = static_cast<double>(blocks) * threads * iters * 8;
  const char* names[3] = {"dadd", "dmul", "dfma"};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::printf("{\"sms\": %d", sms);
  for (int kind = 0; kind < 3; ++kind) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      if (kind == 0) fp64_loop<0><<<blocks, threads>>>(out, iters, 1e-12, 1.0000001);
      if (kind == 1) fp64_loop<1><<<blocks, threads>>>(out, iters, 1e-12, 1.0000001);
      if (kind == 2) fp64_loop<2><<<blocks, threads>>>(out, iters, 1e-12, 1.0000001);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
    }
    const double rate = ops / (best * 1e-3);
    std::printf(", \"%s_ops_per_s\": %.4e", names[kind], rate);
    if (kind == 2) std::printf(", \"dfma_flops_per_s\": %.4e", 2 * rate);
  }
  std::printf(", \"how\": \"8 independent chains x 256 threads x 8 blocks/SM, 4096 iterations, "
              "best of 4 timed runs, CUDA events\"}\n");
  return 0;
}

// Microbenchmark: warp peer masks by MATCH.ANY vs 7 ballots (debug tool).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE, unsigned DIV>
__global__ void k(const unsigned* in, unsigned* out, int iters) {
  unsigned d = in[threadIdx.x + blockIdx.x * blockDim.x] & 127;
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
    unsigned peers;
    if (MODE == 0) {
      peers = __match_any_sync(0xffffffffu, d);
    } else {
      peers = 0xffffffffu;
#pragma unroll
      for (int b = 0; b < 7; ++b) {
        const bool set = (d >> b) & 1u;
        const unsigned bal = __ballot_sync(0xffffffffu, set);
        peers &= set ? bal : ~bal;
      }
    }
    acc += __popc(peers);
    d = (d * 37u + acc + threadIdx.x * DIV) & 127u;
  }
  out[threadIdx.x + blockIdx.x * blockDim.x] = acc;
}
int main() {
  const int blocks = 148 * 4, threads = 512, iters = 4096;
  unsigned *in, *out;
  cudaMalloc(&in, 4ull * blocks * threads);
  cudaMalloc(&out, 4ull * blocks * threads);
  cudaMemset(in, 7, 4ull * blocks * threads);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 6; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) k<0, 0><<<blocks, threads>>>(in, out, iters);
      else if (mode == 1) k<1, 0><<<blocks, threads>>>(in, out, iters);
      else if (mode == 2) k<0, 1><<<blocks, threads>>>(in, out, iters);
      else if (mode == 3) k<1, 1><<<blocks, threads>>>(in, out, iters);
      else if (mode == 4) k<0, 8><<<blocks, threads>>>(in, out, iters);
      else k<1, 8><<<blocks, threads>>>(in, out, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double per = ms * 1e-3 / (double(blocks) * threads / 32 * iters) * 148;
      if (rep == 2)
        printf("%s distinct=%s: %.3f ms, %.2f SM-cycles per warp-op at 1.965 GHz\n",
               (mode & 1) ? "ballot7" : "match.any",
               mode < 2 ? "1" : mode < 4 ? "32" : "16", ms, per * 1.965e9);
    }
  }
  return 0;
}

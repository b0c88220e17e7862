// Exhaustive ordering scorer (reference: the optimality oracle of
// tests/test_reorder.cpp:215-239 — sim_time(t, perm) for every
// std::next_permutation of the identity; StageTimes::permuted,
// src/pipeline_sim.cpp:201-212).
//
// One thread per ordering: rank r in [0, l!) decodes to the r-th permutation
// in lexicographic (= next_permutation) order through the factorial number
// system, its makespan is the tick program (vpp == 1) or the readiness sweep
// (vpp > 1) over the permuted rows — the same evaluators and doubles as
// dtb_schedule.  A makespan evaluation is one serial max/add chain, so a
// thread per ordering keeps every lane busy (32 lanes on one ordering would
// idle).  The winner is the lexicographic min over (makespan, rank): the
// reference's `it < best` scan keeps the first ordering attaining the
// minimum.
#include "kernels.cuh"
#include "sched.cuh"

namespace dtb {

constexpr int kExMaxL = 12;
constexpr int kExMaxP = 16;
constexpr int kExT = 128;

__device__ __forceinline__ void decode_perm(unsigned long long r, int l, int* perm) {
  unsigned long long fact[kExMaxL + 1];
  fact[0] = 1;
  for (int i = 1; i <= l; ++i) fact[i] = fact[i - 1] * i;
  unsigned used = 0u;
  for (int i = 0; i < l; ++i) {
    const unsigned long long f = fact[l - 1 - i];
    int d = static_cast<int>(r / f);
    r -= static_cast<unsigned long long>(d) * f;
    int e = 0;  // d-th unused element
    for (;; ++e) {
      if (used >> e & 1u) continue;
      if (d == 0) break;
      --d;
    }
    used |= 1u << e;
    perm[i] = e;
  }
}

__device__ __forceinline__ bool ex_better(double t, unsigned long long r, double bt,
                                          unsigned long long br) {
  return t < bt || (t == bt && r < br);
}

__global__ void __launch_bounds__(kExT)
exhaustive_kernel(const double* __restrict__ fwd, const double* __restrict__ bwd, int l, int p,
                  int vpp, unsigned long long total, double* all, double* blk_t,
                  unsigned long long* blk_r, DevErr* err) {
  __shared__ double s_t[kExT / 32];
  __shared__ unsigned long long s_r[kExT / 32];
  double bt = 1e300;
  unsigned long long br = ~0ull;
  const int devices = p / vpp;
  for (unsigned long long r = blockIdx.x * static_cast<unsigned long long>(kExT) + threadIdx.x;
       r < total; r += static_cast<unsigned long long>(gridDim.x) * kExT) {
    int perm[kExMaxL];
    decode_perm(r, l, perm);
    auto dur = [&](int mb, int st, int ph) {
      const int row = perm[mb];
      return ph == DTB_FORWARD ? fwd[row * p + st] : bwd[row * p + st];
    };
    double iter = 0.0;
    auto visit = [&](int, Op, double, double end) { iter = smax(iter, end); };
    if (vpp == 1) {
      double prev[kExMaxP], cur[kExMaxP], avail[kExMaxP];
      tick_1f1b(l, p, dur, prev, cur, avail, visit);
    } else {
      double f_end[kExMaxL * kExMaxP], b_end[kExMaxL * kExMaxP], avail[kExMaxP];
      int next[kExMaxP];
      const int e = dataflow_schedule(l, p, vpp, dur, f_end, b_end, next, avail, visit);
      if (e) dev_fail(err, e);
    }
    (void)devices;
    if (all != nullptr) all[r] = iter;
    if (ex_better(iter, r, bt, br)) {
      bt = iter;
      br = r;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double t2 = __shfl_xor_sync(0xffffffffu, bt, o);
    const unsigned long long r2 = __shfl_xor_sync(0xffffffffu, br, o);
    if (ex_better(t2, r2, bt, br)) {
      bt = t2;
      br = r2;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    s_t[threadIdx.x >> 5] = bt;
    s_r[threadIdx.x >> 5] = br;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kExT / 32; ++w)
      if (ex_better(s_t[w], s_r[w], bt, br)) {
        bt = s_t[w];
        br = s_r[w];
      }
    blk_t[blockIdx.x] = bt;
    blk_r[blockIdx.x] = br;
  }
}

__global__ void exhaustive_final(int n_blocks, const double* blk_t,
                                 const unsigned long long* blk_r, int l, double* best_t,
                                 int* best_order) {
  if (threadIdx.x != 0) return;
  double bt = 1e300;
  unsigned long long br = ~0ull;
  for (int i = 0; i < n_blocks; ++i)
    if (ex_better(blk_t[i], blk_r[i], bt, br)) {
      bt = blk_t[i];
      br = blk_r[i];
    }
  *best_t = bt;
  int perm[kExMaxL];
  decode_perm(br, l, perm);
  for (int i = 0; i < l; ++i) best_order[i] = perm[i];
}

int exhaustive_max_l() { return kExMaxL; }
int exhaustive_max_p() { return kExMaxP; }

size_t exhaustive_scratch(int n_blocks) {
  return static_cast<size_t>(n_blocks) * 16 + 256;
}

cudaError_t launch_exhaustive(const double* fwd, const double* bwd, int l, int p, int vpp,
                              double* all, double* best_t, int* best_order, void* scratch,
                              int n_blocks, DevErr* err, cudaStream_t stream) {
  unsigned long long total = 1;
  for (int i = 2; i <= l; ++i) total *= i;
  auto* blk_t = static_cast<double*>(scratch);
  auto* blk_r = reinterpret_cast<unsigned long long*>(blk_t + n_blocks);
  exhaustive_kernel<<<n_blocks, kExT, 0, stream>>>(fwd, bwd, l, p, vpp, total, all, blk_t, blk_r,
                                                   err);
  exhaustive_final<<<1, 32, 0, stream>>>(n_blocks, blk_t, blk_r, l, best_t, best_order);
  return cudaGetLastError();
}

}  // namespace dtb

// Intra-microbatch reordering kernels (Alg. 2).
//
//  * intra_generic_kernel  — intra_partition(sizes, m, order, equal_counts)
//    for arbitrary doubles (reference: src/reorder.cpp:30-90).  One CTA per
//    problem; keys/values in global scratch.
//  * intra_fused_kernel    — the disaggregated hot path, one CTA per global
//    batch, everything staged in shared memory: per-sample cost from the CSR
//    (Sample::cost_size, core.hpp:160-167) -> stable radix sort by cost ->
//    greedy equal-count partition -> block_group_loads of greedy and identity
//    orders -> keep-greedy-if-no-worse decision (src/reorder.cpp:340-354) ->
//    output order, both load vectors and the per-position token keys the
//    microbatch stage consumes.
#include <cub/cub.cuh>

#include "block_ops.cuh"
#include "greedy.cuh"
#include "kernels.cuh"

namespace dtb {

// Orderable bits of a double: -0.0 folds onto +0.0 (the reference
// comparator treats them as equal, src/reorder.cpp:34-40).
__device__ __forceinline__ unsigned long long ord_bits(double x) {
  if (x == 0.0) x = 0.0;
  const unsigned long long b = __double_as_longlong(x);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

// ------------------------------------------------------------------ generic
constexpr int kGenT = 1024;
constexpr int kGenEmax = 4;    // m <= 4096

__global__ void __launch_bounds__(kGenT)
intra_keys_kernel(const double* __restrict__ sizes, int n, int order,
                  unsigned long long* __restrict__ keys, int* __restrict__ vals) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += gridDim.x * blockDim.x) {
    const unsigned long long k = ord_bits(sizes[i]);
    keys[i] = order == DTB_DESCENDING ? ~k : k;
    vals[i] = i;
  }
}

__global__ void __launch_bounds__(kGenT)
intra_generic_kernel(const double* __restrict__ sizes, int n, int m, int order,
                     int equal_counts, const int* __restrict__ vals,
                     int* __restrict__ g_of, int* __restrict__ slot_of,
                     int* __restrict__ flat_out, long long* __restrict__ offsets_out,
                     GreedyState<double> st) {
  __shared__ int s_tmp[kGenT / 32 + 2];
  // zero run in sorted order
  int below = 0, zeros = 0;
  for (int i = threadIdx.x; i < n; i += kGenT) {
    const double x = sizes[i];
    zeros += x == 0.0;
    below += order == DTB_DESCENDING ? (x > 0.0) : (x < 0.0);
  }
  int tot_below, tot_zeros;
  block_excl_scan<kGenT>(below, s_tmp, &tot_below);
  block_excl_scan<kGenT>(zeros, s_tmp, &tot_zeros);
  const int cap = equal_counts ? (n + m - 1) / m : n;
  auto size_at = [&](int k) { return sizes[vals[k]]; };
  auto assign = [&](int k, int g, int slot) {
    g_of[k] = g;
    slot_of[k] = slot;
  };
  greedy_rounds<kGenT, kGenEmax, double>(n, m, cap, tot_below,
                                         tot_below + tot_zeros, size_at, assign,
                                         st);
  // group offsets (exclusive scan of counts) and the flat order
  const int E = (m + kGenT - 1) / kGenT;
  int local = 0;
  for (int e = 0; e < E; ++e) {
    const int g = threadIdx.x * E + e;
    if (g < m) local += st.cnt[g];
  }
  int total;
  int pre = block_excl_scan<kGenT>(local, s_tmp, &total);
  for (int e = 0; e < E; ++e) {
    const int g = threadIdx.x * E + e;
    if (g < m) {
      st.TG[g] = pre;
      offsets_out[g] = pre;
      pre += st.cnt[g];
    }
  }
  if (threadIdx.x == 0) offsets_out[m] = total;
  __syncthreads();
  for (int k = threadIdx.x; k < n; k += kGenT) {
    flat_out[st.TG[g_of[k]] + slot_of[k]] = vals[k];
  }
}

// -------------------------------------------------------------------- fused
// One CTA per global batch of n <= kFusedT * kFusedItems samples.
constexpr int kFusedT = 512;
constexpr int kFusedItems = 32;
constexpr int kFusedMaxN = kFusedT * kFusedItems;  // 16384
constexpr int kFusedEmax = 1;                      // m <= 512

struct FusedSmem {
  unsigned int keys[kFusedMaxN];        // cost (asc) or ~cost (desc)
  unsigned short vals[kFusedMaxN];      // batch-local sample index
  unsigned int asg[kFusedMaxN];         // (group << 16) | slot per sorted item
  int radix_cnt[256 * (kFusedT / 32)];
  long long AL[kFusedT], TL[kFusedT];
  int AG[kFusedT], TG[kFusedT], cnt[kFusedT], off[kFusedT];
  unsigned long long blk_greedy[kFusedT], blk_ident[kFusedT];
  int tmp[kFusedT / 32 + 2];
  long long tmpll[kFusedT / 32 + 1];
};

size_t fused_smem_bytes() { return sizeof(FusedSmem); }
int fused_max_n() { return kFusedMaxN; }
int fused_max_m() { return kFusedT; }

__global__ void __launch_bounds__(kFusedT, 1)
intra_fused_kernel(FusedArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FusedSmem& S = *reinterpret_cast<FusedSmem*>(smem_raw);
  const int n = a.n;
  const int m = a.m;
  const long long b = blockIdx.x;
  const long long first = b * n;
  const int tid = threadIdx.x;

  // ---- 1. per-sample cost (Sample::cost_size) and sort keys
  unsigned int kand = ~0u, kor = 0u;
  int zeros = 0;
  long long maxc = 0;
  for (int i = tid; i < n; i += kFusedT) {
    const long long g = first + i;
    long long t = 0;
    for (int q = a.img_off[g]; q < a.img_off[g + 1]; ++q) t += a.img_tok[q];
    if (a.aud_off != nullptr)
      for (int q = a.aud_off[g]; q < a.aud_off[g + 1]; ++q) t += a.aud_tok[q];
    const long long cost = t + t;
    maxc = cost > maxc ? cost : maxc;
    if (cost < 0) maxc = 0x100000000ll;  // negative tokens: out of key range
    const unsigned int c = static_cast<unsigned int>(cost);
    const unsigned int key = a.order == DTB_DESCENDING ? ~c : c;
    S.keys[i] = key;
    S.vals[i] = static_cast<unsigned short>(i);
    kand &= key;
    kor |= key;
    zeros += cost == 0;
    if (a.orig_tok != nullptr) a.orig_tok[first + i] = static_cast<int>(t);
    if (a.mb_orig != nullptr && i < a.pg * a.dp_me)
      a.mb_orig[(b * a.pg + i % a.pg) * a.dp_me + i / a.pg] = static_cast<int>(t);
  }
  const long long bmax = block_max_ll<kFusedT>(maxc, S.tmpll);
  if (bmax > 0xffffffffll) {
    if (tid == 0) dev_fail(a.err, E_COST_RANGE, static_cast<int>(b));
    return;
  }
  int tot_zeros;
  block_excl_scan<kFusedT>(zeros, S.tmp, &tot_zeros);
  {
    __shared__ unsigned int s_and, s_or;
    if (tid == 0) {
      s_and = ~0u;
      s_or = 0u;
    }
    __syncthreads();
    atomicAnd(&s_and, kand);
    atomicOr(&s_or, kor);
    __syncthreads();
    const unsigned int varying = s_and ^ s_or;
    const int lo = varying ? __ffs(static_cast<int>(varying)) - 1 : 0;
    const int hi = varying ? 32 - __clz(static_cast<int>(varying)) : 0;
    // ---- 2. stable LSD radix sort by cost (index order breaks ties)
    // digit width: split the varying window into the fewest <=8-bit passes
    const int width = hi - lo;
    const int passes = (width + 7) / 8;
    const int rb = passes ? (width + passes - 1) / passes : 8;
    if (rb <= 7)
      tile_radix_sort<kFusedT, kFusedItems, 7>(S.keys, S.vals, n, lo, hi,
                                               S.radix_cnt, S.tmp);
    else
      tile_radix_sort<kFusedT, kFusedItems, 8>(S.keys, S.vals, n, lo, hi,
                                               S.radix_cnt, S.tmp);
  }

  // ---- 3. greedy equal-count partition
  const bool desc = a.order == DTB_DESCENDING;
  const int z0 = desc ? n - tot_zeros : 0;
  const int z1 = desc ? n : tot_zeros;
  const int cap = (n + m - 1) / m;
  GreedyState<long long> st{S.AL, S.AG, S.cnt, S.TL, S.TG, S.tmp};
  auto size_at = [&](int k) -> long long {
    const unsigned int key = S.keys[k];
    return static_cast<long long>(desc ? ~key : key);
  };
  auto assign = [&](int k, int g, int slot) {
    S.asg[k] = (static_cast<unsigned int>(g) << 16) | static_cast<unsigned int>(slot);
  };
  if (a.intra) {
    greedy_rounds<kFusedT, kFusedEmax, long long>(n, m, cap, z0, z1, size_at,
                                                  assign, st);
  }

  // ---- 4. block_group_loads of the greedy and the identity order
  const int pg = n / m;  // block size (src/reorder.cpp:113)
  for (int g = tid; g < m; g += kFusedT) {
    S.blk_greedy[g] = 0ull;
    S.blk_ident[g] = 0ull;
  }
  int pre_local = (tid < m && a.intra) ? S.cnt[tid] : 0;
  int total;
  const int pre = block_excl_scan<kFusedT>(pre_local, S.tmp, &total);
  if (tid < m) S.off[tid] = pre;
  __syncthreads();
  for (int k = tid; k < n; k += kFusedT) {
    const unsigned int key = S.keys[k];
    const unsigned long long sz = desc ? ~key : key;
    const int idx = S.vals[k];
    atomicAdd(&S.blk_ident[min(idx / pg, m - 1)], sz);
    if (a.intra) {
      const unsigned int as = S.asg[k];
      const int pos = S.off[as >> 16] + static_cast<int>(as & 0xffffu);
      atomicAdd(&S.blk_greedy[min(pos / pg, m - 1)], sz);
    }
  }
  __syncthreads();
  long long mg = 0, mi = 0;
  for (int g = tid; g < m; g += kFusedT) {
    mg = max(mg, static_cast<long long>(S.blk_greedy[g]));
    mi = max(mi, static_cast<long long>(S.blk_ident[g]));
  }
  // src/reorder.cpp:350-353: keep the greedy split when its max block load
  // is no worse than the incoming order's.
  mg = block_max_ll<kFusedT>(mg, S.tmpll);
  mi = block_max_ll<kFusedT>(mi, S.tmpll);
  const bool keep = a.intra && mg <= mi;
  if (tid == 0 && a.kept != nullptr) a.kept[b] = keep ? 1 : 0;
  for (int g = tid; g < m; g += kFusedT) {
    if (a.load_before) a.load_before[b * m + g] = static_cast<double>(S.blk_ident[g]);
    if (a.load_after)
      a.load_after[b * m + g] =
          static_cast<double>(keep ? S.blk_greedy[g] : S.blk_ident[g]);
  }

  // ---- 5. the intra order (batch-local indices) and staged token keys
  const int mb_span = a.pg * a.dp_me;
  auto put_staged = [&](int pos, unsigned int key) {
    const int tok = static_cast<int>((desc ? ~key : key) >> 1);  // cost_size / 2
    if (a.staged_tok != nullptr) a.staged_tok[first + pos] = tok;
    if (a.mb_staged != nullptr && pos < mb_span)
      a.mb_staged[(b * a.pg + pos % a.pg) * a.dp_me + pos / a.pg] = tok;
  };
  if (keep) {
    for (int k = tid; k < n; k += kFusedT) {
      const unsigned int as = S.asg[k];
      const int pos = S.off[as >> 16] + static_cast<int>(as & 0xffffu);
      a.order_out[first + pos] = S.vals[k];
      put_staged(pos, S.keys[k]);
    }
  } else {
    for (int i = tid; i < n; i += kFusedT) a.order_out[first + i] = i;
    for (int k = tid; k < n; k += kFusedT) put_staged(S.vals[k], S.keys[k]);
  }
}

// ------------------------------------------------------------- host glue
cudaError_t launch_intra_fused(const FusedArgs& a, long long n_batches,
                               cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(intra_fused_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sizeof(FusedSmem)));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  intra_fused_kernel<<<static_cast<unsigned>(n_batches), kFusedT,
                       sizeof(FusedSmem), stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_intra_generic(const double* sizes, int n, int m, int order,
                                 int equal_counts, void* scratch,
                                 size_t scratch_bytes, int* flat_out,
                                 long long* offsets_out, cudaStream_t stream) {
  // scratch layout: keys[n] u64, keys_alt[n] u64, vals[n], vals_alt[n],
  // g_of[n], slot_of[n], greedy state (5 * m words), cub temp.
  char* p = static_cast<char*>(scratch);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) & ~size_t(255);
    return r;
  };
  auto* keys = reinterpret_cast<unsigned long long*>(take(sizeof(unsigned long long) * n));
  auto* keys2 = reinterpret_cast<unsigned long long*>(take(sizeof(unsigned long long) * n));
  auto* vals = reinterpret_cast<int*>(take(sizeof(int) * n));
  auto* vals2 = reinterpret_cast<int*>(take(sizeof(int) * n));
  auto* g_of = reinterpret_cast<int*>(take(sizeof(int) * n));
  auto* slot_of = reinterpret_cast<int*>(take(sizeof(int) * n));
  GreedyState<double> st;
  st.AL = reinterpret_cast<double*>(take(sizeof(double) * m));
  st.TL = reinterpret_cast<double*>(take(sizeof(double) * m));
  st.AG = reinterpret_cast<int*>(take(sizeof(int) * m));
  st.TG = reinterpret_cast<int*>(take(sizeof(int) * m));
  st.cnt = reinterpret_cast<int*>(take(sizeof(int) * m));
  st.tmp = reinterpret_cast<int*>(take(sizeof(int) * (kGenT / 32 + 2)));
  const size_t used = static_cast<size_t>(p - static_cast<char*>(scratch));
  if (used > scratch_bytes) return cudaErrorMemoryAllocation;
  const int grid = (n + kGenT - 1) / kGenT;
  intra_keys_kernel<<<grid > 0 ? grid : 1, kGenT, 0, stream>>>(sizes, n, order, keys, vals);
  // Stable device-wide radix sort of (orderable key, index) pairs: ties keep
  // index order, i.e. the reference's (size, index) comparator.
  size_t temp = scratch_bytes - used;
  cub::DoubleBuffer<unsigned long long> dk(keys, keys2);
  cub::DoubleBuffer<int> dv(vals, vals2);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(p, temp, dk, dv, n, 0, 64, stream);
  if (e != cudaSuccess) return e;
  intra_generic_kernel<<<1, kGenT, 0, stream>>>(sizes, n, m, order, equal_counts,
                                                dv.Current(), g_of, slot_of,
                                                flat_out, offsets_out, st);
  return cudaGetLastError();
}

size_t intra_generic_scratch(int n, int m) {
  size_t b = 0;
  auto add = [&](size_t x) { b += (x + 255) & ~size_t(255); };
  add(8ull * n); add(8ull * n); add(4ull * n); add(4ull * n); add(4ull * n); add(4ull * n);
  add(8ull * m); add(8ull * m); add(4ull * m); add(4ull * m); add(4ull * m);
  add(4ull * (kGenT / 32 + 2));
  size_t temp = 0;
  cub::DoubleBuffer<unsigned long long> dk(nullptr, nullptr);
  cub::DoubleBuffer<int> dv(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, temp, dk, dv, n, 0, 64);
  return b + temp + 1024;
}

int intra_generic_max_m() { return kGenT * kGenEmax; }

}  // namespace dtb

// Block-wide primitives (scan / reduce / stable radix ranking) used by the
// intra-partition kernels.  T = threads per block, a multiple of 32.
#pragma once

#include <cstdint>

#include "dtb_internal.cuh"

namespace dtb {

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Exclusive scan of one int per thread; returns the prefix, writes the block
// total to *total.  `s` needs T/32 + 1 ints.  Contains two __syncthreads.
template <int T>
__device__ __forceinline__ int block_excl_scan(int v, int* s, int* total) {
  constexpr int W = T / 32;
  const int lane = lane_id(), w = warp_id();
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();  // readers of the previous result in `s` are done
  if (lane == 31) s[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = lane < W ? s[lane] : 0;
    int u = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, u, o);
      if (lane >= o) u += y;
    }
    if (lane < W) s[lane] = u - t;
    if (lane == W - 1) s[W] = u;
  }
  __syncthreads();
  const int r = x - v + s[w];
  *total = s[W];
  return r;
}

// Inclusive scan of one 64-bit integer per thread (exact: integer adds are
// associative); *total gets the block sum.  `s` needs T/32 + 1 long longs.
template <int T>
__device__ __forceinline__ long long block_incl_scan_ll(long long v, long long* s,
                                                        long long* total) {
  constexpr int W = T / 32;
  const int lane = lane_id(), w = warp_id();
  long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) s[w] = x;
  __syncthreads();
  if (w == 0) {
    long long t = lane < W ? s[lane] : 0;
    long long u = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(kFull, u, o);
      if (lane >= o) u += y;
    }
    if (lane < W) s[lane] = u - t;
    if (lane == W - 1) s[W] = u;
  }
  __syncthreads();
  const long long r = x + s[w];
  *total = s[W];
  return r;
}

// Block minimum of one int per thread (all threads get the result).
template <int T>
__device__ __forceinline__ int block_min(int v, int* s) {
  constexpr int W = T / 32;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(kFull, v, o));
  __syncthreads();
  if (lane_id() == 0) s[warp_id()] = v;
  __syncthreads();
  int r = s[0];
#pragma unroll 1
  for (int i = 1; i < W; ++i) r = min(r, s[i]);
  return r;
}

template <int T>
__device__ __forceinline__ long long block_max_ll(long long v, long long* s) {
  constexpr int W = T / 32;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long y = __shfl_xor_sync(kFull, v, o);
    v = v < y ? y : v;
  }
  __syncthreads();
  if (lane_id() == 0) s[warp_id()] = v;
  __syncthreads();
  long long r = s[0];
#pragma unroll 1
  for (int i = 1; i < W; ++i) r = r < s[i] ? s[i] : r;
  return r;
}

template <int T>
__device__ __forceinline__ unsigned block_or(unsigned v, unsigned* s) {
  constexpr int W = T / 32;
  v = __reduce_or_sync(kFull, v);
  __syncthreads();
  if (lane_id() == 0) s[warp_id()] = v;
  __syncthreads();
  unsigned r = 0;
#pragma unroll 1
  for (int i = 0; i < W; ++i) r |= s[i];
  return r;
}

// Stable in-place LSD radix sort of n <= T*ITEMS (key, value) pairs held in
// (shared) memory, by key bits [lo_bit, hi_bit).  Warp-striped tiles:
// warp w owns positions [w*32*ITEMS, (w+1)*32*ITEMS), item i of a lane is at
// w*32*ITEMS + i*32 + lane, so ranking slot by slot with __match_any_sync
// keeps equal digits in input order (stability); per-(digit, warp) counts
// are then scanned digit-major.  `cnt` needs (1<<RB) * (T/32) ints.
template <int T, int ITEMS, int RB, typename K, typename V>
__device__ void tile_radix_sort(K* keys, V* vals, int n, int lo_bit,
                                int hi_bit, int* cnt, int* scan_tmp) {
  constexpr int W = T / 32;
  constexpr int D = 1 << RB;
  const int lane = lane_id(), w = warp_id();
  const unsigned lt = lanemask_lt();
  for (int shift = lo_bit; shift < hi_bit; shift += RB) {
    const int bits = min(RB, hi_bit - shift);
    const unsigned mask = (1u << bits) - 1u;
    for (int i = threadIdx.x; i < D * W; i += T) cnt[i] = 0;
    K k[ITEMS];
    V v[ITEMS];
    unsigned short rank[ITEMS];
    unsigned char dig[ITEMS];
    __syncthreads();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int pos = w * 32 * ITEMS + i * 32 + lane;
      const bool ok = pos < n;
      k[i] = ok ? keys[pos] : K(0);
      v[i] = ok ? vals[pos] : V(0);
      const unsigned d = ok ? static_cast<unsigned>(k[i] >> shift) & mask : D;
      dig[i] = static_cast<unsigned char>(d & 0xff);
      const unsigned peers = __match_any_sync(kFull, d);
      int before = 0;
      if (ok) before = cnt[w * D + d];
      __syncwarp();
      if (ok && (peers & lt) == 0) cnt[w * D + d] = before + __popc(peers);
      __syncwarp();
      rank[i] = static_cast<unsigned short>(before + __popc(peers & lt));
    }
    __syncthreads();
    // exclusive scan of cnt in (digit, warp) order: each thread scans a
    // contiguous chunk of D*W / T entries.
    constexpr int PER = (D * W + T - 1) / T;
    int local[PER];
    int sum = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int idx = threadIdx.x * PER + j;
      local[j] = idx < D * W ? cnt[(idx % W) * D + idx / W] : 0;
      sum += local[j];
    }
    int total;
    int base = block_excl_scan<T>(sum, scan_tmp, &total);
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int idx = threadIdx.x * PER + j;
      if (idx < D * W) cnt[(idx % W) * D + idx / W] = base;
      base += local[j];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int pos = w * 32 * ITEMS + i * 32 + lane;
      if (pos < n) {
        const int dst = cnt[w * D + dig[i]] + rank[i];
        keys[dst] = k[i];
        vals[dst] = v[i];
      }
    }
    __syncthreads();
  }
}

// Lanes of the warp whose RB-bit digit equals this lane's, among lanes with
// `ok` set: RB + 1 ballots instead of MATCH.ANY (a low-throughput
// instruction; the ballots issue at full rate).
template <int RB>
__device__ __forceinline__ unsigned digit_peers(unsigned d, bool ok) {
  unsigned peers = __ballot_sync(kFull, ok);
#pragma unroll
  for (int bit = 0; bit < RB; ++bit) {
    const bool set = (d >> bit) & 1u;
    const unsigned bal = __ballot_sync(kFull, set);
    peers &= set ? bal : ~bal;
  }
  return peers;
}

// One stable counting pass over n <= T*ITEMS 32-bit items in place, digit
// given by digit(pos, item) in [0, 1 << RB).  Same warp-striped ranking as
// tile_radix_sort; used both for the cost-key passes (digit = key bits) and
// for the group partition after the greedy (digit = group id).
template <int T, int ITEMS, int RB, typename DigitFn>
__device__ void tile_pass_u32(unsigned int* items, int n, const DigitFn& digit, int* cnt,
                              int* scan_tmp) {
  constexpr int W = T / 32;
  constexpr int D = 1 << RB;
  const int lane = lane_id(), w = warp_id();
  const unsigned lt = lanemask_lt();
  for (int i = threadIdx.x; i < D * W; i += T) cnt[i] = 0;
  static_assert(ITEMS % 2 == 0, "ranks are packed in pairs");
  unsigned int k[ITEMS];
  unsigned int rk[ITEMS / 2];  // two 16-bit ranks per register; digits recomputed
  // all item loads first: the ranking chain below then only waits on the
  // per-digit counters, not on item loads
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int pos = w * 32 * ITEMS + i * 32 + lane;
    k[i] = pos < n ? items[pos] : 0u;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int pos = w * 32 * ITEMS + i * 32 + lane;
    const bool ok = pos < n;
    const unsigned d = ok ? static_cast<unsigned>(digit(pos, k[i])) : 0u;
    const unsigned peers = digit_peers<RB>(d, ok);
    int before = 0;
    if (ok) before = cnt[w * D + d];
    __syncwarp();
    if (ok && (peers & lt) == 0) cnt[w * D + d] = before + __popc(peers);
    __syncwarp();
    const unsigned r = static_cast<unsigned>(before + __popc(peers & lt));
    if (i & 1) rk[i >> 1] |= r << 16;
    else rk[i >> 1] = r;
  }
  __syncthreads();
  constexpr int PER = (D * W + T - 1) / T;
  int local[PER];
  int sum = 0;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int idx = threadIdx.x * PER + j;
    local[j] = idx < D * W ? cnt[(idx % W) * D + idx / W] : 0;
    sum += local[j];
  }
  int total;
  int base = block_excl_scan<T>(sum, scan_tmp, &total);
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int idx = threadIdx.x * PER + j;
    if (idx < D * W) cnt[(idx % W) * D + idx / W] = base;
    base += local[j];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int pos = w * 32 * ITEMS + i * 32 + lane;
    if (pos < n) {
      const unsigned d = static_cast<unsigned>(digit(pos, k[i]));
      const unsigned r = (i & 1) ? (rk[i >> 1] >> 16) : (rk[i >> 1] & 0xffffu);
      items[cnt[w * D + d] + r] = k[i];
    }
  }
  __syncthreads();
}

}  // namespace dtb

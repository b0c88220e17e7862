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

// Barrier of the first T threads: BAR == 0 is __syncthreads (T = the whole
// block); BAR > 0 is the named barrier BAR over threads [0, T) only, so a
// subset of a larger block can run a block-wide primitive on its own.
template <int BAR, int T>
__device__ __forceinline__ void bar_sync() {
  if constexpr (BAR == 0) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(T) : "memory");
  }
}

// Exclusive scan of one int per thread; returns the prefix, writes the block
// total to *total.  `s` needs T/32 + 1 ints.  Contains two __syncthreads.
template <int T, int BAR = 0>
__device__ __forceinline__ int block_excl_scan(int v, int* s, int* total) {
  constexpr int W = T / 32;
  const int lane = lane_id(), w = warp_id();
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  bar_sync<BAR, T>();  // readers of the previous result in `s` are done
  if (lane == 31) s[w] = x;
  bar_sync<BAR, T>();
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
  bar_sync<BAR, T>();
  const int r = x - v + s[w];
  *total = s[W];
  return r;
}

// Inclusive scan of one 64-bit integer per thread (exact: integer adds are
// associative); *total gets the block sum.  `s` needs T/32 + 1 long longs.
template <int T, int BAR = 0>
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
  bar_sync<BAR, T>();
  if (lane == 31) s[w] = x;
  bar_sync<BAR, T>();
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
  bar_sync<BAR, T>();
  const long long r = x + s[w];
  *total = s[W];
  return r;
}

// Block minimum of one int per thread (all threads get the result).
template <int T, int BAR = 0>
__device__ __forceinline__ int block_min(int v, int* s) {
  constexpr int W = T / 32;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(kFull, v, o));
  bar_sync<BAR, T>();
  if (lane_id() == 0) s[warp_id()] = v;
  bar_sync<BAR, T>();
  int r = s[0];
#pragma unroll 1
  for (int i = 1; i < W; ++i) r = min(r, s[i]);
  return r;
}

template <int T, int BAR = 0>
__device__ __forceinline__ long long block_max_ll(long long v, long long* s) {
  constexpr int W = T / 32;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long y = __shfl_xor_sync(kFull, v, o);
    v = v < y ? y : v;
  }
  bar_sync<BAR, T>();
  if (lane_id() == 0) s[warp_id()] = v;
  bar_sync<BAR, T>();
  long long r = s[0];
#pragma unroll 1
  for (int i = 1; i < W; ++i) r = r < s[i] ? s[i] : r;
  return r;
}

template <int T, int BAR = 0>
__device__ __forceinline__ unsigned block_or(unsigned v, unsigned* s) {
  constexpr int W = T / 32;
  v = __reduce_or_sync(kFull, v);
  bar_sync<BAR, T>();
  if (lane_id() == 0) s[warp_id()] = v;
  bar_sync<BAR, T>();
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

// Bijective in-block swizzle of sorted positions (stays inside its 32-item
// block): strided gathers of sorted items (stride r = active groups in the
// greedy, consecutive slots of one group in the write-out) spread over banks.
__device__ __forceinline__ int swz(int k) {
  const int x = k >> 5;
  return k ^ ((x ^ (x >> 2) ^ (x >> 4)) & 31);
}

// One stable counting pass (per-THREAD counters, blocked arrangement) of a
// block radix sort of u16 sample indices by the u16 keys key[idx], in place.
// Thread t owns slots [t*ITEMS, (t+1)*ITEMS) — contiguous, so the stable
// order is (digit, thread, item) — and counts its digits in private u16
// counters c(d, t), packed two per 32-bit word, digit-major, one pad word
// per 16 (conflict-free raking scan).  Counting and the scatter's
// position reservation are shared-memory atomics on the counter words: no
// load -> add -> store chain between a thread's items (same-thread atomics
// on one address retire in program order, which is exactly the stable
// order), no warp votes or matches (their throughput bounded the
// warp-striped variant), no per-item rank storage.  The caller pads past n
// with indices whose key has the largest digit in every pass.
// ITEMS % 4 == 0 (64-bit loads of a thread's slots).  Counter storage:
// blocked_cnt_words(T, RB) 32-bit words.
__host__ __device__ constexpr int blocked_cnt_words(int T, int RB) {
  return (1 << RB) * T / 2 + (1 << RB) * T / 32;
}

template <int T, int ITEMS, int RB, bool SWZ, typename DigitFn>
__device__ void tile_pass_blocked(unsigned short* idx, const unsigned short* key,
                                  const DigitFn& digit, unsigned* cntw, int* scan_tmp) {
  constexpr int D = 1 << RB;
  constexpr int WORDS = D * T / 2;
  constexpr int PER = WORDS / T;  // raking segment (16 words for RB = 5)
  constexpr int G = 4;
  static_assert(ITEMS % G == 0 && WORDS % T == 0 && PER % 16 == 0, "shape");
  const int t = threadIdx.x;
  // counter (d, t): logical u16 e = d*T + t -> padded word (e>>1) + (e>>5)
  auto word_of = [&](unsigned d) -> int {
    const int e = static_cast<int>(d) * T + t;
    return (e >> 1) + (e >> 5);
  };
  const unsigned half = (t & 1) * 16;  // e and t have the same parity (T even)
  for (int i = t; i < blocked_cnt_words(T, RB); i += T) cntw[i] = 0u;
  __syncthreads();
  const uint2* mine = reinterpret_cast<const uint2*>(idx + t * ITEMS);
#pragma unroll 2
  for (int g = 0; g < ITEMS / G; ++g) {
    const uint2 p = mine[g];
    const unsigned v[G] = {p.x & 0xffffu, p.x >> 16, p.y & 0xffffu, p.y >> 16};
    unsigned d[G];
#pragma unroll
    for (int j = 0; j < G; ++j) d[j] = static_cast<unsigned>(digit(key[v[j]]));
#pragma unroll
    for (int j = 0; j < G; ++j) atomicAdd(cntw + word_of(d[j]), 1u << half);
  }
  // this thread's items, two per register, held across the scan (the
  // scatter is in place)
  uint2 it[ITEMS / G];
#pragma unroll
  for (int g = 0; g < ITEMS / G; ++g) {
    it[g] = mine[g];
    asm volatile("" : "+r"(it[g].x), "+r"(it[g].y));  // keep them packed
  }
  __syncthreads();
  // raking exclusive scan over (d, t) = logical word order: thread t owns
  // logical words [t*PER, (t+1)*PER) = padded words t*(PER + PER/16) + ...
  unsigned* seg = cntw + t * (PER + PER / 16);
  unsigned local[PER];
  int sum = 0;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    local[j] = seg[j + j / 16];
    sum += static_cast<int>((local[j] & 0xffffu) + (local[j] >> 16));
  }
  int total;
  int base = block_excl_scan<T>(sum, scan_tmp, &total);
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const unsigned lo = local[j] & 0xffffu, hi = local[j] >> 16;
    seg[j + j / 16] = static_cast<unsigned>(base) | (static_cast<unsigned>(base + lo) << 16);
    base += static_cast<int>(lo + hi);
  }
  __syncthreads();
#pragma unroll
  for (int g = 0; g < ITEMS / G; ++g) {
    const unsigned v[G] = {it[g].x & 0xffffu, it[g].x >> 16, it[g].y & 0xffffu, it[g].y >> 16};
    unsigned d[G];
#pragma unroll
    for (int j = 0; j < G; ++j) d[j] = static_cast<unsigned>(digit(key[v[j]]));
    unsigned old[G];
#pragma unroll
    for (int j = 0; j < G; ++j) old[j] = atomicAdd(cntw + word_of(d[j]), 1u << half);
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const int dst = static_cast<int>((old[j] >> half) & 0xffffu);
      DTB_CHECK(dst < T * ITEMS);
      idx[SWZ ? swz(dst) : dst] = static_cast<unsigned short>(v[j]);
    }
  }
  __syncthreads();
}

// The same stable blocked pass over packed (key << 16 | index) items: the
// digit comes from the item itself (no indirect key lookups in shared
// memory), the scatter moves the 32-bit item.  ITEMS % 4 == 0 (128-bit loads
// of a thread's slots).
template <int T, int ITEMS, int RB, bool SWZ, typename DigitFn>
__device__ void tile_pass_kv(unsigned* kv, const DigitFn& digit, unsigned* cntw, int* scan_tmp) {
  constexpr int D = 1 << RB;
  constexpr int WORDS = D * T / 2;
  constexpr int PER = WORDS / T;
  constexpr int G = 4;
  static_assert(ITEMS % G == 0 && WORDS % T == 0 && PER % 16 == 0, "shape");
  const int t = threadIdx.x;
  auto word_of = [&](unsigned d) -> int {
    const int e = static_cast<int>(d) * T + t;
    return (e >> 1) + (e >> 5);
  };
  const unsigned half = (t & 1) * 16;
  for (int i = t; i < blocked_cnt_words(T, RB); i += T) cntw[i] = 0u;
  uint4 it[ITEMS / G];
  const uint4* mine = reinterpret_cast<const uint4*>(kv + t * ITEMS);
#pragma unroll
  for (int g = 0; g < ITEMS / G; ++g) it[g] = mine[g];
  __syncthreads();
#pragma unroll
  for (int g = 0; g < ITEMS / G; ++g) {
    const unsigned v[G] = {it[g].x, it[g].y, it[g].z, it[g].w};
#pragma unroll
    for (int j = 0; j < G; ++j) atomicAdd(cntw + word_of(static_cast<unsigned>(digit(v[j] >> 16))), 1u << half);
  }
  __syncthreads();
  // (the thread's counter words are re-read after the scan instead of held:
  // the items already occupy 16 registers)
  unsigned* seg = cntw + t * (PER + PER / 16);
  int sum = 0;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const unsigned c = seg[j + j / 16];
    sum += static_cast<int>((c & 0xffffu) + (c >> 16));
  }
  int total;
  int base = block_excl_scan<T>(sum, scan_tmp, &total);
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const unsigned c = seg[j + j / 16];
    const unsigned lo = c & 0xffffu, hi = c >> 16;
    seg[j + j / 16] = static_cast<unsigned>(base) | (static_cast<unsigned>(base + lo) << 16);
    base += static_cast<int>(lo + hi);
  }
  __syncthreads();
#pragma unroll
  for (int g = 0; g < ITEMS / G; ++g) {
    const unsigned v[G] = {it[g].x, it[g].y, it[g].z, it[g].w};
    unsigned old[G];
#pragma unroll
    for (int j = 0; j < G; ++j)
      old[j] = atomicAdd(cntw + word_of(static_cast<unsigned>(digit(v[j] >> 16))), 1u << half);
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const int dst = static_cast<int>((old[j] >> half) & 0xffffu);
      DTB_CHECK(dst < T * ITEMS);
      kv[SWZ ? swz(dst) : dst] = v[j];
    }
  }
  __syncthreads();
}

}  // namespace dtb

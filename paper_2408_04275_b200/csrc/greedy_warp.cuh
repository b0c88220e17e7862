// Equal-count greedy on ONE warp (reference: src/reorder.cpp:70-90,
// intra_partition with equal_counts) for the narrow path's m <= 128 groups.
//
// Same round decomposition as greedy_fused.cuh — a round gives the next R
// sorted items to the R lowest (load, gid) active groups, R the longest
// prefix for which every item's group is still the minimum when its turn
// comes — but with the active list A held in REGISTERS: 4 consecutive
// entries per lane as one 64-bit key (load << 8 | gid; unique, so the
// (load, gid) order is the key order).  A round is then a binary search per
// entry (upper bound of its new key in A, a shared-memory copy of A), one
// warp min, the emission, and a warp bitonic sort of the 128 keys — no
// block barriers.  Rounds whose new loads come out unsorted (descending
// sizes: the LPT snake) cost a sort either way; the block version pays
// ~8 barriers plus a quadratic rank per round there.
#pragma once

#include "block_ops.cuh"

namespace dtb {

struct WarpGreedySmem {
  unsigned long long key[128];  // A at the start of the round (sorted; u32 keys use the low half)
  int cnt[128];                 // items assigned per gid
  int pre[128];                 // zero run: capacity prefix over A
};

template <typename K>
__device__ __forceinline__ K wg_cmpx(K a, K b, bool take_min) {
  return take_min ? (a < b ? a : b) : (a < b ? b : a);
}

// Ascending bitonic sort of 128 keys, lane l holding positions 4l .. 4l+3.
template <typename K>
__device__ __forceinline__ void wg_sort128(K (&v)[4]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 128; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 4) {
        const int lj = j >> 2;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int i = 4 * lane + e;
          const K o = __shfl_xor_sync(0xffffffffu, v[e], lj);
          const bool up = (i & k) == 0;
          const bool lower = (i & j) == 0;
          v[e] = wg_cmpx(v[e], o, lower == up);
        }
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (e & j) continue;
          const int i = 4 * lane + e;
          const bool up = (i & k) == 0;
          const K a = v[e], b = v[e | j];
          const bool swap = up ? (b < a) : (a < b);
          v[e] = swap ? b : a;
          v[e | j] = swap ? a : b;
        }
      }
    }
  }
}

// sizes(k): size of sorted item k; emit(k, g, slot).  Zero run = [z0, z1).
// Outputs gload[g], gcnt[g].  K = u32 when every load stays below 2^24 (the
// caller checks cap x max size), else u64.  Called by all 32 lanes of one
// warp.
template <typename K, typename SizeFn, typename EmitFn>
__device__ void greedy_warp(int n, int m, int cap, int z0, int z1, const SizeFn& sizes,
                            const EmitFn& emit, WarpGreedySmem& W, unsigned* gload, int* gcnt,
                            unsigned long long* prof = nullptr) {
  constexpr K kNone = static_cast<K>(~static_cast<K>(0));
  K* key = reinterpret_cast<K*>(W.key);
  const int lane = threadIdx.x & 31;
  K v[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int t = 4 * lane + e;
    v[e] = t < m ? static_cast<K>(t) : kNone;  // load 0, gid t
    W.cnt[t] = 0;
  }
  int r = m;
  unsigned long long n_rounds = 0;
  __syncwarp();
  int k = 0;
  while (k < n) {
    if (k >= z0 && k < z1) {
      // ---- zero run: items of size 0 fill A[0], A[1], ... to cap in order
      // (no load changes, ties stay with the lowest entry)
      const int z = z1 - k;
      int capl[4], sum = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int t = 4 * lane + e;
        capl[e] = t < r ? cap - W.cnt[static_cast<int>(v[e] & 0xffu)] : 0;
        sum += capl[e];
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int pre = incl - sum;
      int take[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        W.pre[4 * lane + e] = pre;
        key[4 * lane + e] = v[e];
        take[e] = max(0, min(capl[e], z - pre));
        pre += capl[e];
      }
      __syncwarp();
      for (int q = lane; q < z; q += 32) {
        int lo = 0, hi = r - 1;  // last entry whose capacity prefix is <= q
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (W.pre[mid] <= q) lo = mid;
          else hi = mid - 1;
        }
        DTB_CHECK(lo >= 0 && lo < r);
        const int g = static_cast<int>(key[lo] & 0xffu);
        emit(k + q, g, W.cnt[g] + (q - W.pre[lo]));
      }
      __syncwarp();
      int removed = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int t = 4 * lane + e;
        if (t < r && take[e] > 0) {
          const int g = static_cast<int>(v[e] & 0xffu);
          const int c = W.cnt[g] + take[e];
          if (take[e] == capl[e]) {  // filled: leaves A
            gload[g] = static_cast<unsigned>(v[e] >> 8);
            gcnt[g] = c;
            v[e] = kNone;
            ++removed;
          }
          W.cnt[g] = c;
        }
      }
      r -= static_cast<int>(__reduce_add_sync(0xffffffffu, static_cast<unsigned>(removed)));
      wg_sort128(v);
      k = z1;
      __syncwarp();
      if (prof && lane == 0) {
        unsigned long long tnow;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
        prof[0] = tnow;
      }
      continue;
    }
    const int lim = k < z0 ? min(n, z0) : n;  // non-zero items [k, lim)
    // ---- general round
#pragma unroll
    for (int e = 0; e < 4; ++e) key[4 * lane + e] = v[e];
    __syncwarp();
    const int R_lim = min(r, lim - k);
    K nk[4];
    int bmin = 0x7fffffff;
    bool room[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int t = 4 * lane + e;
      nk[e] = kNone;
      room[e] = false;
      if (t < R_lim) {
        const int g = static_cast<int>(v[e] & 0xffu);
        nk[e] = v[e] + (static_cast<K>(sizes(k + t)) << 8);
        room[e] = W.cnt[g] + 1 < cap;
      }
    }
    // upper bound of every new key in A (128 slots, kNone-padded: a fixed
    // 7-step search, the four entries interleaved)
    int ub[4] = {0, 0, 0, 0};
#pragma unroll
    for (int step = 64; step > 0; step >>= 1) {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (key[ub[e] + step - 1] <= nk[e]) ub[e] += step;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int t = 4 * lane + e;
      if (ub[e] == 127 && key[127] <= nk[e]) ub[e] = 128;
      if (t < R_lim && room[e]) bmin = min(bmin, max(t + 1, ub[e]));
    }
    const int R = min(R_lim, static_cast<int>(__reduce_min_sync(0xffffffffu, static_cast<unsigned>(bmin))));
    int removed = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int t = 4 * lane + e;
      if (t < R) {
        const int g = static_cast<int>(v[e] & 0xffu);
        const int c = W.cnt[g];
        emit(k + t, g, c);
        W.cnt[g] = c + 1;
        if (room[e]) {
          v[e] = nk[e];
        } else {  // full: leaves A
          gload[g] = static_cast<unsigned>(nk[e] >> 8);
          gcnt[g] = c + 1;
          v[e] = kNone;
          ++removed;
        }
      }
    }
    r -= static_cast<int>(__reduce_add_sync(0xffffffffu, static_cast<unsigned>(removed)));
    wg_sort128(v);
    k += R;
    ++n_rounds;
    __syncwarp();
  }
  if (prof && lane == 0) prof[1] = n_rounds;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    if (v[e] != kNone) {
      const int g = static_cast<int>(v[e] & 0xffu);
      gload[g] = static_cast<unsigned>(v[e] >> 8);
      gcnt[g] = W.cnt[g];
    }
  }
  __syncwarp();
}

}  // namespace dtb

// Equal-count greedy of the fused intra kernel's shared-memory path
// (reference: src/reorder.cpp:70-90, intra_partition with equal_counts).
//
// Same round decomposition as greedy.cuh (a round assigns the next R sorted
// items to the R lowest (load, gid) active groups), specialised for the
// narrow layout — m <= 128 groups, integer sizes <= 65534, n <= 16384, so
// every load is an exact u32 — and organised so that the BULK of the work is
// block-parallel:
//
//   * zero run: items of size 0 fill A[0], A[1], ... to cap in order; the
//     emission of those items is spread over all threads (binary search of
//     the capacity prefix);
//   * full rounds (ascending sizes): tstar rounds that keep A's order are
//     found with two block prefix scans (greedy.cuh), then committed by all
//     threads at once — column j of the tstar x r block of items goes to
//     entry j, the per-entry load is a sum of integer sizes (exact in any
//     order, combined with shared-memory atomics);
//   * general rounds (ties, full groups, descending sizes): as greedy.cuh.
//
// Items are EMITTED as (sorted position k, group, slot); the caller scatters
// them straight into the flat order (IntraPartition::flat) — no partition
// pass over the sorted items is needed.
#pragma once

#include "block_ops.cuh"

namespace dtb {

constexpr int kFG = 128;  // max groups of the narrow path

struct FusedGreedySmem {
  unsigned AL[kFG];  // active entries sorted by (load, gid)
  int AG[kFG];
  int AC[kFG];       // items assigned to the entry's group
  unsigned TL[kFG];  // merge / staging scratch
  int TG[kFG];
  int TC[kFG];
  int pre[kFG];       // zero-run capacity prefix
  unsigned gload[kFG];  // final load per gid
  int gcnt[kFG];        // final item count per gid
};

__device__ __forceinline__ bool fkey_lt(unsigned a, int ga, unsigned b, int gb) {
  return a < b || (a == b && ga < gb);
}

// Block inclusive scan of one u32 per thread (sums here stay < 2^31).
template <int T, int BAR = 0>
__device__ __forceinline__ unsigned block_incl_scan_u32(unsigned v, int* s, unsigned* total) {
  int tot;
  const int ex = block_excl_scan<T, BAR>(static_cast<int>(v), s, &tot);
  *total = static_cast<unsigned>(tot);
  return static_cast<unsigned>(ex) + v;
}

// sizes(k): size of sorted item k; emit(k, g, slot).  Zero run = [z0, z1).
// prof (debug, may be null): [0] globaltimer after the zero run, [1] round
// counts (full-round segments << 32 | general rounds).
template <int T, bool ASC, int BAR = 0, typename SizeFn, typename EmitFn>
__device__ void greedy_fused(int n, int m, int cap, int z0, int z1, const SizeFn& sizes,
                             const EmitFn& emit, FusedGreedySmem& G, int* tmp,
                             long long* tmpll, unsigned long long* prof = nullptr) {
  unsigned long long n_full = 0, n_general = 0;
  static_assert(T >= 2 * kFG && T % kFG == 0, "one entry per thread, two in a merge");
  const int tid = threadIdx.x;
  if (tid < m) {
    G.AL[tid] = 0u;
    G.AG[tid] = tid;
    G.AC[tid] = 0;
  }
  bar_sync<BAR, T>();
  int r = m;
  int k = 0;
  while (k < n) {
    // ------------------------------------------------------------ zero run
    if (k >= z0 && k < z1) {
      const int z = z1 - k;
      const int capl = tid < r ? cap - G.AC[tid] : 0;
      int tot;
      const int pre = block_excl_scan<T, BAR>(capl, tmp, &tot);
      int take = 0;
      unsigned L = 0u;
      int g = 0, c = 0;
      if (tid < r) {
        take = max(0, min(capl, z - pre));
        L = G.AL[tid];
        g = G.AG[tid];
        c = G.AC[tid];
        G.pre[tid] = pre;
        G.TC[tid] = c;
      }
      const bool full = tid < r && take == capl && take > 0;
      if (full) {
        G.gload[g] = L;
        G.gcnt[g] = cap;
      }
      int nfull;  // filled entries are a prefix of A
      block_excl_scan<T, BAR>(full ? 1 : 0, tmp, &nfull);
      if (k == 0) {
        // first run of the batch: every entry is empty (capacity cap, in gid
        // order), so the entry of item q is q / cap — no search
        // (a warp per entry: no division per item)
        const int lane = tid & 31, nfill = (z + cap - 1) / cap;
        for (int j = tid >> 5; j < nfill; j += T / 32) {
          const int g = G.AG[j], lim = min(cap, z - j * cap);
          for (int sl = lane; sl < lim; sl += 32) emit(k + j * cap + sl, g, sl);
        }
      } else {
        for (int q = tid; q < z; q += T) {
          int lo = 0, hi = r - 1;  // last entry whose capacity prefix is <= q
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (G.pre[mid] <= q) lo = mid;
            else hi = mid - 1;
          }
          emit(k + q, G.AG[lo], G.TC[lo] + (q - G.pre[lo]));
        }
      }
      bar_sync<BAR, T>();
      if (tid < r && tid >= nfull) {
        G.AL[tid - nfull] = L;
        G.AG[tid - nfull] = g;
        G.AC[tid - nfull] = c + take;
      }
      r -= nfull;
      k = z1;
      bar_sync<BAR, T>();
      if (prof && tid == 0) {
        unsigned long long tnow;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
        prof[0] = tnow;
      }
      continue;
    }
    const int lim = k < z0 ? min(n, z0) : n;  // non-zero items [k, lim)

    // --------------------------------------------------------- full rounds
    if (ASC) {
      int room = tid < r ? cap - 1 - G.AC[tid] : 0x7fffffff;
      room = block_min<T, BAR>(room, tmp);
      const int Tr = r > 0 ? min(room, (lim - k) / r) : 0;
      if (Tr >= 1) {
        int tstar = Tr;
        if (r >= 2) {
          // full round t keeps A's order iff newkey_0 > A[r-1] at its start
          const unsigned l0 = G.AL[0], ll = G.AL[r - 1];
          const int g0 = G.AG[0], gl = G.AG[r - 1];
          unsigned c0 = 0u, cl = 0u;
          for (int t0 = 0; t0 < Tr; t0 += T) {
            const int t = t0 + tid;
            const bool ok = t < Tr;
            const unsigned s0 = ok ? sizes(k + t * r) : 0u;
            const unsigned sl = ok ? sizes(k + t * r + r - 1) : 0u;
            // both columns in one 64-bit scan: each half's sum stays < 2^31
            // (loads of <= 16384 items of <= 65534), so no carry crosses
            long long tot;
            const unsigned long long inc = static_cast<unsigned long long>(block_incl_scan_ll<T, BAR>(
                static_cast<long long>((static_cast<unsigned long long>(sl) << 32) | s0),
                tmpll, &tot));
            const unsigned inc0 = static_cast<unsigned>(inc), incl = static_cast<unsigned>(inc >> 32);
            const unsigned tot0 = static_cast<unsigned>(tot),
                           totl = static_cast<unsigned>(static_cast<unsigned long long>(tot) >> 32);
            const unsigned new0 = l0 + c0 + inc0;
            const unsigned last = ll + cl + (incl - sl);
            const int f = ok && !fkey_lt(last, gl, new0, g0) ? t : 0x7fffffff;
            const int first = block_min<T, BAR>(f, tmp);
            if (first != 0x7fffffff) {
              tstar = first;
              break;
            }
            c0 += tot0;
            cl += totl;
          }
        }
        if (tstar > 0) {
          // column j of the tstar x r block goes to entry j, slots AC + t
          constexpr int kRows = T / kFG;
          const int j = tid % kFG;
          unsigned part = 0u;
          if (j < r) {
            const int g = G.AG[j], c = G.AC[j];
#pragma unroll 4
            for (int t = tid / kFG; t < tstar; t += kRows) {
              const int item = k + t * r + j;
              part += sizes(item);
              emit(item, g, c + t);
            }
          }
          bar_sync<BAR, T>();
          if (j < r && part) atomicAdd(&G.AL[j], part);
          if (tid < r) G.AC[tid] += tstar;
          k += tstar * r;
          ++n_full;
          bar_sync<BAR, T>();
          continue;
        }
      }
    }

    // ------------------------------------------------------- general round
    const int R_lim = min(r, lim - k);
    int bmin = 0x7fffffff;
    if (tid < R_lim && G.AC[tid] + 1 < cap) {
      const int g = G.AG[tid];
      const unsigned nl = G.AL[tid] + sizes(k + tid);
      int lo = 0, hi = r;  // upper_bound of (nl, g) in A
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (fkey_lt(nl, g, G.AL[mid], G.AG[mid])) hi = mid;
        else lo = mid + 1;
      }
      bmin = max(tid + 1, lo);
    }
    const int R = min(R_lim, block_min<T, BAR>(bmin, tmp));
    const bool keep = tid < R && G.AC[tid] + 1 < cap;
    int nkeep;
    const int keep_pre = block_excl_scan<T, BAR>(keep ? 1 : 0, tmp, &nkeep);
    if (tid < R) {
      const int g = G.AG[tid], c = G.AC[tid];
      const unsigned nl = G.AL[tid] + sizes(k + tid);
      emit(k + tid, g, c);
      if (keep) {
        G.TL[keep_pre] = nl;
        G.TG[keep_pre] = g;
        G.TC[keep_pre] = c + 1;
      } else {
        G.gload[g] = nl;
        G.gcnt[g] = c + 1;
      }
    }
    bar_sync<BAR, T>();
    unsigned unsorted = 0u;
    if (!ASC && tid + 1 < nkeep)
      unsorted = fkey_lt(G.TL[tid], G.TG[tid], G.TL[tid + 1], G.TG[tid + 1]) ? 0u : 1u;
    if (!ASC) unsorted = block_or<T, BAR>(unsorted, reinterpret_cast<unsigned*>(tmp));
    // final ranks of the merged order; written after a barrier
    unsigned oL = 0u;
    int oG = 0, oC = 0, oP = -1;
    if (tid < nkeep) {  // new key
      const unsigned kl = G.TL[tid];
      const int kg = G.TG[tid];
      int lo = R, hi = r;  // A[R..r) entries below it
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (fkey_lt(G.AL[mid], G.AG[mid], kl, kg)) lo = mid + 1;
        else hi = mid;
      }
      int rank_new = tid;
      if (unsorted) {
        rank_new = 0;
        for (int c2 = 0; c2 < nkeep; ++c2) rank_new += fkey_lt(G.TL[c2], G.TG[c2], kl, kg);
      }
      oL = kl;
      oG = kg;
      oC = G.TC[tid];
      oP = rank_new + (lo - R);
    }
    unsigned pL = 0u;
    int pG = 0, pC = 0, pP = -1;
    if (R + tid < r) {  // kept old entry
      const int j = R + tid;
      const unsigned al = G.AL[j];
      const int ag = G.AG[j];
      int below = 0;
      if (!unsorted) {
        int lo = 0, hi = nkeep;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (fkey_lt(G.TL[mid], G.TG[mid], al, ag)) lo = mid + 1;
          else hi = mid;
        }
        below = lo;
      } else {
        for (int c2 = 0; c2 < nkeep; ++c2) below += fkey_lt(G.TL[c2], G.TG[c2], al, ag);
      }
      pL = al;
      pG = ag;
      pC = G.AC[j];
      pP = tid + below;
    }
    bar_sync<BAR, T>();
    if (oP >= 0) {
      G.AL[oP] = oL;
      G.AG[oP] = oG;
      G.AC[oP] = oC;
    }
    if (pP >= 0) {
      G.AL[pP] = pL;
      G.AG[pP] = pG;
      G.AC[pP] = pC;
    }
    r = nkeep + (r - R);
    k += R;
    ++n_general;
    bar_sync<BAR, T>();
  }
  if (prof && tid == 0) prof[1] = (n_full << 32) | n_general;
  if (tid < r) {
    G.gload[G.AG[tid]] = G.AL[tid];
    G.gcnt[G.AG[tid]] = G.AC[tid];
  }
  bar_sync<BAR, T>();
}

}  // namespace dtb

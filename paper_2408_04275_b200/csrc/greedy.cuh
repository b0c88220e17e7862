// Exact block-parallel restatement of the intra-microbatch greedy
// (reference: src/reorder.cpp:70-90, intra_partition).
//
// The reference assigns sorted items one by one to argmin_(load, gid) over
// groups with count < cap — an n-step dependency chain.  Here the same
// assignment is produced in ROUNDS (SURVEY.md §7 hard part 2):
//
//   state A = active groups sorted by (load, gid)        (a priority queue)
//   round: item k+j goes to A[j] for j < R, where R is the first j at which a
//          group re-inserted earlier in the round, (A[i].load + s[k+i], A[i].gid),
//          would precede A[j]; R = min_i max(i+1, upper_bound(A, newkey_i)).
//          Groups reaching cap are not re-inserted.  New state = merge of the
//          re-inserted keys and A[R..r).
//   zero run: items of size 0 leave loads unchanged, so a run of them fills
//          A[0], A[1], ... to cap in order (closed form).
//   fast path: speculate that the next T rounds are full and keep A's order;
//          round t is exact iff its new keys stay sorted and
//          newkey_0 > A[r-1]; the first failing t* is found with one block
//          min-reduction and rounds < t* are committed at once.  For
//          ascending input the speculation only fails when a group fills.
//
// Loads are accumulated per group in assignment order with the same IEEE
// adds as the reference (`load[target] += sizes[idx]`), and every comparison
// is the reference's lexicographic (load, gid) order, so the result is
// identical for any input, not just integer sizes.
#pragma once

#include "block_ops.cuh"

namespace dtb {

template <typename L>
struct GreedyState {
  L* AL;      // [m] loads of active groups, sorted by (load, gid)
  int* AG;    // [m] their group ids
  int* cnt;   // [m] items assigned per group id
  L* TL;      // [m] merge scratch
  int* TG;    // [m]
  int* tmp;   // [T/32 + 2] reduction scratch
  L* gload;   // [m] final load per group id (null: not recorded)
  long long* tmpll;  // [T/32 + 1] 64-bit scan scratch (ASC_INT fast path)
};

template <typename L>
__device__ __forceinline__ bool key_lt(L a, int ga, L b, int gb) {
  return a < b || (a == b && ga < gb);
}

// Block-uniform greedy driver.  sizes(k): size of the k-th sorted item;
// assign(k, g, slot): record the assignment.  Items [z0, z1) are the zero run
// (size == 0).  m <= T * E_MAX.
//
// ASC_INT: integer sizes in ascending order.  Then a full round keeps A's
// order automatically: L_j <= L_j+1 and s_j <= s_j+1 give
// L_j + s_j <= L_j+1 + s_j+1, with equality only if both loads were equal
// (so g_j < g_j+1 still orders them) — integer adds are exact.  Only
// condition (b), newkey_0 > A[r-1], remains, and because integer sums are
// associative it is evaluated for all speculative rounds at once from two
// block-wide prefix scans (columns 0 and r-1), not by one thread per round.
template <int T, int E_MAX, typename L, bool ASC_INT = false, typename SizeFn,
          typename AssignFn>
__device__ void greedy_rounds(int n, int m, int cap, int z0, int z1,
                              const SizeFn& sizes, const AssignFn& assign,
                              GreedyState<L> st) {
  const int tid = threadIdx.x;
  constexpr int E = E_MAX;  // entries per thread (blocked; compile-time so
                            // per-entry arrays stay in registers)
  for (int j = tid; j < m; j += T) {
    st.AL[j] = L(0);
    st.AG[j] = j;
    st.cnt[j] = 0;
  }
  __syncthreads();
  int r = m;
  int k = 0;
  while (k < n) {
    // ---------------------------------------------------------- zero run
    if (k >= z0 && k < z1) {
      const int z = z1 - k;
      // capacity prefix over entries in A order (blocked: thread owns E).
      int cap_local[E_MAX];
      int sum = 0;
      for (int e = 0; e < E; ++e) {
        const int j = tid * E + e;
        cap_local[e] = j < r ? cap - st.cnt[st.AG[j]] : 0;
        sum += cap_local[e];
      }
      int total;
      int pre = block_excl_scan<T>(sum, st.tmp, &total);
      int full_here = 0;
      for (int e = 0; e < E; ++e) {
        const int j = tid * E + e;
        if (j < r) {
          const int take = max(0, min(cap_local[e], z - pre));
          const int g = st.AG[j];
          const int c0 = st.cnt[g];
          for (int t = 0; t < take; ++t) assign(k + pre + t, g, c0 + t);
          st.cnt[g] = c0 + take;
          if (take == cap_local[e] && take > 0) {
            ++full_here;
            if (st.gload) st.gload[g] = st.AL[j];
          }
        }
        pre += cap_local[e];
      }
      int nfull;
      block_excl_scan<T>(full_here, st.tmp, &nfull);
      // drop the filled prefix of A
      if (nfull > 0) {
        for (int j = tid; j < r - nfull; j += T) {
          st.TL[j] = st.AL[j + nfull];
          st.TG[j] = st.AG[j + nfull];
        }
        __syncthreads();
        for (int j = tid; j < r - nfull; j += T) {
          st.AL[j] = st.TL[j];
          st.AG[j] = st.TG[j];
        }
      }
      r -= nfull;
      k = z1;
      __syncthreads();
      continue;
    }
    const int lim = k < z0 ? min(n, z0) : n;  // non-zero items [k, lim)

    // --------------------------------------------------------- fast path
    {
      int room = 0x7fffffff;
      for (int e = 0; e < E; ++e) {
        const int j = tid * E + e;
        if (j < r) room = min(room, cap - 1 - st.cnt[st.AG[j]]);
      }
      room = block_min<T>(room, st.tmp);
      const int T_rounds = r > 0 ? min(room, (lim - k) / r) : 0;
      if (ASC_INT && T_rounds >= 1) {
        int tstar = T_rounds;
        if (r >= 2) {
          const long long l0 = static_cast<long long>(st.AL[0]);
          const long long ll = static_cast<long long>(st.AL[r - 1]);
          const int g0 = st.AG[0], gl = st.AG[r - 1];
          long long c0 = 0, cl = 0;  // column sums of earlier chunks
          for (int t0 = 0; t0 < T_rounds; t0 += T) {
            const int t = t0 + tid;
            const bool ok = t < T_rounds;
            const long long s0 = ok ? static_cast<long long>(sizes(k + t * r)) : 0;
            const long long sl = ok ? static_cast<long long>(sizes(k + t * r + r - 1)) : 0;
            long long tot0, totl;
            const long long inc0 = block_incl_scan_ll<T>(s0, st.tmpll, &tot0);
            const long long incl = block_incl_scan_ll<T>(sl, st.tmpll, &totl);
            // round t: newkey_0 = L0 + sum_{t'<=t} s0, A[r-1] = Llast + sum_{t'<t} sl
            const long long new0 = l0 + c0 + inc0;
            const long long last = ll + cl + (incl - sl);
            const int f = ok && !key_lt(last, gl, new0, g0) ? t : 0x7fffffff;
            const int first = block_min<T>(f, st.tmp);
            if (first != 0x7fffffff) {
              tstar = first;
              break;
            }
            c0 += tot0;
            cl += totl;
          }
        }
        if (tstar > 0) {
          for (int e = 0; e < E; ++e) {
            const int j = tid * E + e;
            if (j >= r) break;
            const int g = st.AG[j];
            const int cs = st.cnt[g];
            L l = st.AL[j];
#pragma unroll 4
            for (int t = 0; t < tstar; ++t) {
              const int item = k + t * r + j;
              l = l + sizes(item);
              assign(item, g, cs + t);
            }
            st.AL[j] = l;
            st.cnt[g] = cs + tstar;
          }
          k += tstar * r;
          __syncthreads();
          continue;
        }
      } else if (T_rounds >= 1) {
        int fail = T_rounds;
        // columns owned: j = tid*E .. tid*E+E-1 plus j+1 for the pair check
        for (int e = 0; e < E; ++e) {
          const int j = tid * E + e;
          if (j >= r) break;
          const int gj = st.AG[j];
          L lj = st.AL[j];
          const bool pair = j + 1 < r;
          const int gj1 = pair ? st.AG[j + 1] : 0;
          L lj1 = pair ? st.AL[j + 1] : L(0);
          const bool last = (j == 0) && r >= 2;
          const int glast = last ? st.AG[r - 1] : 0;
          L llast = last ? st.AL[r - 1] : L(0);
          for (int t = 0; t < fail; ++t) {
            const int base = k + t * r;
            const L nj = lj + sizes(base + j);
            if (pair) {
              const L nj1 = lj1 + sizes(base + j + 1);
              if (!key_lt(nj, gj, nj1, gj1)) {
                fail = t;
                break;
              }
              lj1 = nj1;
            }
            if (last) {
              // newkey_0 of round t must exceed A[r-1] at the start of t
              if (!key_lt(llast, glast, nj, gj)) {
                fail = t;
                break;
              }
              llast = llast + sizes(base + r - 1);
            }
            lj = nj;
          }
        }
        const int tstar = block_min<T>(fail, st.tmp);
        if (tstar > 0) {
          for (int e = 0; e < E; ++e) {
            const int j = tid * E + e;
            if (j >= r) break;
            const int g = st.AG[j];
            const int c0 = st.cnt[g];
            L l = st.AL[j];
            for (int t = 0; t < tstar; ++t) {
              const int item = k + t * r + j;
              l = l + sizes(item);
              assign(item, g, c0 + t);
            }
            st.AL[j] = l;
            st.cnt[g] = c0 + tstar;
          }
          k += tstar * r;
          __syncthreads();
          continue;
        }
      }
    }

    // ------------------------------------------------------ general round
    const int R_lim = min(r, lim - k);
    int bmin = 0x7fffffff;
    for (int e = 0; e < E; ++e) {
      const int i = tid * E + e;
      if (i >= R_lim) break;
      const int g = st.AG[i];
      if (st.cnt[g] + 1 >= cap) continue;  // becomes full: not re-inserted
      const L nl = st.AL[i] + sizes(k + i);
      int lo = 0, hi = r;  // upper_bound of (nl, g) in A
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (key_lt(nl, g, st.AL[mid], st.AG[mid])) hi = mid;
        else lo = mid + 1;
      }
      bmin = min(bmin, max(i + 1, lo));
    }
    const int R = min(R_lim, block_min<T>(bmin, st.tmp));
    // New keys of the R popped entries (full ones dropped), A[R..r) kept.
    // Positions by rank: NK sorted among themselves? check, else count.
    int keep_local = 0;
    unsigned unsorted = 0;
    for (int e = 0; e < E; ++e) {
      const int i = tid * E + e;
      if (i >= R) break;
      const int g = st.AG[i];
      const bool full = st.cnt[g] + 1 >= cap;
      keep_local += full ? 0 : 1;
    }
    int nkeep;
    int keep_pre = block_excl_scan<T>(keep_local, st.tmp, &nkeep);
    // Stage new keys compacted into TL/TG[0..nkeep) and record slots.
    for (int e = 0; e < E; ++e) {
      const int i = tid * E + e;
      if (i >= R) break;
      const int g = st.AG[i];
      const int c0 = st.cnt[g];
      assign(k + i, g, c0);
      const L nl = st.AL[i] + sizes(k + i);
      if (c0 + 1 < cap) {
        st.TL[keep_pre] = nl;
        st.TG[keep_pre] = g;
        ++keep_pre;
      } else if (st.gload) {
        st.gload[g] = nl;
      }
    }
    __syncthreads();
    for (int e = 0; e < E; ++e) {
      const int i = tid * E + e;
      if (i >= R) break;
      st.cnt[st.AG[i]] += 1;
    }
    for (int c = tid; c + 1 < nkeep; c += T) {
      if (!key_lt(st.TL[c], st.TG[c], st.TL[c + 1], st.TG[c + 1])) unsorted = 1;
    }
    unsorted = block_or<T>(unsorted, reinterpret_cast<unsigned*>(st.tmp));
    // Each element computes its final rank in the merged order; results are
    // written after a barrier (AL/AG and TL/TG are both read during ranking).
    const int rest = r - R;
    const int total_new = nkeep + rest;
    L outL[E_MAX * 2];
    int outG[E_MAX * 2];
    int outP[E_MAX * 2];
    int nout = 0;
    for (int e = 0; e < E; ++e) {
      const int c = tid * E + e;
      if (c < nkeep) {  // new key c
        const L kl = st.TL[c];
        const int kg = st.TG[c];
        int lo = R, hi = r;  // A[R..r) elements below it
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (key_lt(st.AL[mid], st.AG[mid], kl, kg)) lo = mid + 1;
          else hi = mid;
        }
        int rank_new = c;
        if (unsorted) {
          rank_new = 0;
          for (int c2 = 0; c2 < nkeep; ++c2)
            rank_new += key_lt(st.TL[c2], st.TG[c2], kl, kg) ? 1 : 0;
        }
        outL[nout] = kl;
        outG[nout] = kg;
        outP[nout++] = rank_new + (lo - R);
      }
      const int j = R + tid * E + e;  // kept old entry
      if (j < r) {
        const L al = st.AL[j];
        const int ag = st.AG[j];
        int below = 0;
        if (!unsorted) {
          int lo = 0, hi = nkeep;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (key_lt(st.TL[mid], st.TG[mid], al, ag)) lo = mid + 1;
            else hi = mid;
          }
          below = lo;
        } else {
          for (int c2 = 0; c2 < nkeep; ++c2)
            below += key_lt(st.TL[c2], st.TG[c2], al, ag) ? 1 : 0;
        }
        outL[nout] = al;
        outG[nout] = ag;
        outP[nout++] = (j - R) + below;
      }
    }
    __syncthreads();
    for (int q = 0; q < nout; ++q) {
      st.AL[outP[q]] = outL[q];
      st.AG[outP[q]] = outG[q];
    }
    r = total_new;
    k += R;
    __syncthreads();
  }
  if (st.gload)
    for (int j = tid; j < r; j += T) st.gload[st.AG[j]] = st.AL[j];
  __syncthreads();
}

}  // namespace dtb

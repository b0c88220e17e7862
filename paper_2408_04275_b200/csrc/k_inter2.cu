// Inter-microbatch reordering on the disaggregated stream path (Alg. 3;
// reference src/reorder.cpp:238-298, candidate_times / windows_for
// :182-234, select_min / select_closest :121-175), plain 1F1B (vpp == 1).
//
// One thread per problem (a coupled group's l microbatches).  The reference
// algorithm is O(l^2) per problem — every step re-derives the pending-row
// means as a SEQUENTIAL sum in ascending index order and scans the pending
// keys — so its operands must live on chip: each thread owns a column of
// shared memory ([i][thread] layout, bank-conflict free) holding, per
// microbatch, the forward stage value of the encoder and generator units,
// the forward key and the token sum; placed rows' backward values come from
// the token-indexed cost table.  Compared with the generic kernel
// (k_inter.cu, global scratch):
//   * the pending means are formed per UNIT, not per stage (all stages of a
//     unit carry the unit's value, src/cost_model.cpp:334-362); backbone
//     rows are the constant seq_len row, whose sequential sums of k copies
//     are tabulated once per CTA;
//   * the stage -> unit layout is a template parameter (as in the tiled
//     simulations), the tick state lives in registers;
//   * the schedule work per step is the speculative frontier only (ticks
//     from the committed frontier to B(step-1, 0)), as in k_inter.cu.
// Every value is produced by the reference's operation sequence: sums in
// ascending index order, then one division; start = max(avail, dep),
// end = start + dur; picks by the (key, index) / (|r - key|, key > r,
// index) total orders.
#include "kernels.cuh"

namespace dtb {

namespace {

constexpr int kInterMaxL = 256;  // mask words below

struct Row4 {
  double ef, eb, gf, gb;
};

// Cold path: token sums outside the cost table (32-bit batches).
__device__ __noinline__ Row4 inter_row_direct(const InterArgs* a, long long te, double* key,
                                              int* err) {
  Row4 r{0.0, 0.0, 0.0, 0.0};
  if (te < 0) {
    *err = E_NEG_LOAD;
    return r;
  }
  UnitEval ue, ug;
  ue.init(a->cm, a->plan, DTB_ENCODER);
  ug.init(a->cm, a->plan, DTB_GENERATOR);
  const double x = mb_mean_fast(te, a->span);
  ue.eval(x, &r.ef, &r.eb);
  ug.eval(x, &r.gf, &r.gb);
  const int e = dev_fwd_key(a->cm, a->plan, x, x, key);
  if (e) *err = e;
  return r;
}

}  // namespace

// Backward rows of recently placed positions, kept on chip: the windows
// only ever read backward cells of positions within kBRing of the frontier.
constexpr int kBRing = 16;

// Shared memory per thread (bytes).
// Pending list row stride (bytes): l rounded up to whole words, plus one
// word so the stride in words is odd (bank-conflict-free row starts).
__host__ __device__ inline int inter_pl_stride(int l) {
  int w = (l + 3) / 4;
  if ((w & 1) == 0) ++w;
  return 4 * w;
}

__host__ __device__ inline size_t inter_tok_bytes_per_thread(int l, bool gather) {
  return static_cast<size_t>(l) * ((gather ? 0 : 3 * 8) + 2 + 1) + (gather ? 0 : 2 * 8 * kBRing) +
         inter_pl_stride(l);
}

// GATHER: forward values and keys are read from the (L1-resident) cost table
// through the token sums instead of being kept in shared memory — 0.77 KB of
// on-chip state per problem instead of 3.8 KB, so ~4x the problems per SM.
// Problems whose sums fall outside the table (or beyond u16) are flagged in
// a.redo and solved by the shared-memory variant (a.redo_only).
template <int PE, int PB, int PG, bool GATHER>
__global__ void __launch_bounds__(128)
inter_tok_kernel(const __grid_constant__ InterArgs a) {
  constexpr int P = PE + PB + PG;
  constexpr int DEV = P;  // vpp == 1: one stage per device
  extern __shared__ __align__(16) unsigned char smem[];
  const int T = blockDim.x, t = threadIdx.x, l = a.l;
  // shared tables: sequential sums of k copies of the backbone forward value
  double* sb_sum = reinterpret_cast<double*>(smem);  // [l + 1]
  double* colF = sb_sum + (l + 1);                   // [l][T] encoder F
  double* colG = colF + (GATHER ? 0 : static_cast<size_t>(l) * T);  // [l][T] generator F
  double* colK = colG + (GATHER ? 0 : static_cast<size_t>(l) * T);  // [l][T] forward keys
  auto* colT = reinterpret_cast<unsigned short*>(colK + (GATHER ? 0 : static_cast<size_t>(l) * T));
  // backward ring [kBRing][T] (encoder, generator), 8-byte aligned after the u16 tokens
  double* colBE = reinterpret_cast<double*>(
      (reinterpret_cast<size_t>(colT + static_cast<size_t>(l) * T) + 7) & ~size_t(7));
  constexpr int RING = GATHER ? 0 : kBRing;  // the gather variant reads the table instead
  double* colBG = colBE + static_cast<size_t>(RING) * T;
  unsigned char* colR = reinterpret_cast<unsigned char*>(colBG + static_cast<size_t>(RING) * T);
  // per-thread pending list (ascending indices), row-contiguous: [T][stride]
  const int pls = inter_pl_stride(l);
  unsigned char* colPL = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<size_t>(colR + static_cast<size_t>(l) * T) + 3) & ~size_t(3));

  UnitEval ub;
  ub.init(a.cm, a.plan, DTB_BACKBONE);
  double fB, bB;
  ub.eval(a.cm.seq_len, &fB, &bB);
  if (t == 0) {
    double acc = 0.0;
    sb_sum[0] = 0.0;
    for (int k = 1; k <= l; ++k) {
      acc += fB;
      sb_sum[k] = acc;
    }
  }
  __syncthreads();
  const long long prob = blockIdx.x * static_cast<long long>(T) + t;
  if (prob >= a.batch) return;
  if (!GATHER && a.redo_only && a.redo[prob] == 0) return;
  int* out = a.orders + prob * l;
  auto F = [&](int i) -> double& { return colF[static_cast<size_t>(i) * T + t]; };
  auto G = [&](int i) -> double& { return colG[static_cast<size_t>(i) * T + t]; };
  auto K = [&](int i) -> double& { return colK[static_cast<size_t>(i) * T + t]; };
  // u16 / u8 columns: the 32 lanes of a warp read 32 different rows, so each
  // lane's element gets its own bank — lane j of warp w at column 2j + (w & 1)
  // (u16) / 4j + (w & 3) (u8) of its 64- / 128-thread block (T % 128 == 0)
  const bool swz_ok = (T & 127) == 0;
  const int ct = swz_ok ? (t & ~63) + 2 * (t & 31) + ((t >> 5) & 1) : t;
  const int cr = swz_ok ? (t & ~127) + 4 * (t & 31) + ((t >> 5) & 3) : t;
  auto TK = [&](int i) -> unsigned short& { return colT[static_cast<size_t>(i) * T + ct]; };
  auto RET = [&](int i) -> unsigned char& { return colR[static_cast<size_t>(i) * T + cr]; };
  auto BE = [&](int pos) -> double& { return colBE[static_cast<size_t>(pos % kBRing) * T + t]; };
  auto BG = [&](int pos) -> double& { return colBG[static_cast<size_t>(pos % kBRing) * T + t]; };
  auto Fv = [&](int i) -> double {
    if constexpr (GATHER) return __ldg(a.table.fz + TK(i)).x;
    else return F(i);
  };
  auto Gv = [&](int i) -> double {
    if constexpr (GATHER) return __ldg(a.table.fz + TK(i)).y;
    else return G(i);
  };
  auto Kv = [&](int i) -> double {
    if constexpr (GATHER) return __ldg(a.table.key + TK(i));
    else return K(i);
  };

  // ---- fill: rows of the problem's microbatches (staged order)
  const long long bb = prob / a.groups;
  const int grp = static_cast<int>(prob - bb * a.groups);
  int err = 0;
  bool direct_rows = false;
  if constexpr (GATHER) {
    for (int i = 0; i < l; ++i) {
      const long long v = a.span == 1 ? a.tok.get(bb, grp * l + i, true)
                                      : a.mbsum[prob * static_cast<long long>(l) + i];
      if (v < 0 || v >= a.table.size || v > 0xffff) {
        a.redo[prob] = 1;
        return;
      }
      TK(i) = static_cast<unsigned short>(v);
    }
  } else for (int i = 0; i < l; ++i) {
    const long long v = a.span == 1 ? a.tok.get(bb, grp * l + i, true)
                                    : a.mbsum[prob * static_cast<long long>(l) + i];
    // TK is u16: larger sums (span >= 3) take the direct rows
    if (v >= 0 && v < a.table.size && v <= 0xffff) {
      const double4 r = ld_row(a.table.eg + v);
      F(i) = r.x;
      G(i) = r.z;
      K(i) = __ldg(a.table.key + v);
      TK(i) = static_cast<unsigned short>(v);
    } else {
      double key = 0.0;
      const Row4 r = inter_row_direct(&a, v, &key, &err);
      F(i) = r.ef;
      G(i) = r.gf;
      K(i) = key;
      TK(i) = 0;
      direct_rows = true;
    }
  }
  if (err) {
    dev_fail(a.err, err);
    return;
  }
  // backward values of a placed row (table, or direct for 32-bit batches)
  auto bwd_row = [&](int idx, double* eb, double* gb) {
    if (!direct_rows) {
      const double4 r = ld_row(a.table.eg + TK(idx));
      *eb = r.y;
      *gb = r.w;
    } else {
      const long long v = a.span == 1 ? a.tok.get(bb, grp * l + idx, true)
                                      : a.mbsum[prob * static_cast<long long>(l) + idx];
      double key;
      int e2 = 0;
      const Row4 r = inter_row_direct(&a, v, &key, &e2);
      *eb = r.eb;
      *gb = r.gb;
    }
  };

  for (int i = 0; i < l; ++i) out[i] = i;
  if (l <= 1 || DEV == 1) return;

  // pending set as a bit mask over indices (ascending iteration = index order)
  constexpr int MW = kInterMaxL / 32;
  unsigned pend[MW];
#pragma unroll
  for (int w = 0; w < MW; ++w) {
    const int lo = w * 32;
    pend[w] = lo >= l ? 0u : (l - lo >= 32 ? 0xffffffffu : ((1u << (l - lo)) - 1u));
  }
  int npend = l;
  // the same set as a compacted ascending list: the hot O(npend) loops then
  // run exactly npend iterations in every lane (npend is uniform across the
  // warp) instead of l predicated ones
  unsigned char* PL = colPL + static_cast<size_t>(t) * pls;
  for (int q = 0; q < l; ++q) PL[q] = static_cast<unsigned char>(q);
  // removes list position `pos` four bytes per step (rows are word aligned;
  // little-endian byte order)
  auto list_remove = [&](int pos) {
    unsigned* W = reinterpret_cast<unsigned*>(PL);
    const int k0 = pos >> 2, nw = (npend + 3) >> 2;
    const unsigned keep = (1u << (8 * (pos & 3))) - 1u;
    unsigned w = W[k0];
    for (int k = k0; k < nw; ++k) {
      const unsigned nx = k + 1 < nw ? W[k + 1] : 0u;
      unsigned v = __funnelshift_r(w, nx, 8);
      if (k == k0) v = (w & keep) | (v & ~keep);
      W[k] = v;
      w = nx;
    }
  };
  auto list_find = [&](int idx) -> int {  // position of idx (ascending list)
    int lo = 0, hi = npend - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (PL[mid] < idx) lo = mid + 1;
      else hi = mid;
    }
    return lo;
  };
  auto pend_word = [&](int w) -> unsigned {
    unsigned r = 0u;
#pragma unroll
    for (int z = 0; z < MW; ++z)
      if (z == w) r = pend[z];
    return r;
  };
  auto clear = [&](int idx) {
#pragma unroll
    for (int w = 0; w < MW; ++w)
      if (w == (idx >> 5)) pend[w] &= ~(1u << (idx & 31));
  };
  // select_min, one pick: smallest (key, index)
  auto pick_min = [&]() -> int {
    int best = -1;
    double kb = 0.0;
#pragma unroll
    for (int w = 0; w < MW; ++w) {
      unsigned m = pend[w];
      while (m) {
        const int idx = w * 32 + __ffs(m) - 1;
        m &= m - 1;
        const double k = Kv(idx);
        if (best < 0 || k < kb) {
          best = idx;
          kb = k;
        }
      }
    }
    return best;
  };
  // select_closest, one pick: smallest (|r - key|, key > r, index) over the
  // pending list (ascending, so the incumbent always has the lower index);
  // *pos gets the list position of the pick
  auto pick_closest = [&](double residual, int* pos) -> int {
    int best = -1, bq = 0;
    double db = 0.0;
    bool bover = false;
#pragma unroll 4
    for (int q = 0; q < npend; ++q) {
      const int idx = PL[q];
      const double k = Kv(idx);
      const double da = fabs(residual - k);
      const bool over = !(k <= residual);
      const bool take = best < 0 || da < db || (da == db && !over && bover);
      best = take ? idx : best;
      bq = take ? q : bq;
      db = take ? da : db;
      bover = take ? over : bover;
    }
    *pos = bq;
    return best;
  };

  int nret = 0;
  auto place = [&](int idx) {
    if constexpr (!GATHER) {
      double eb, gb;
      bwd_row(idx, &eb, &gb);
      BE(nret) = eb;
      BG(nret) = gb;
    }
    RET(nret++) = static_cast<unsigned char>(idx);
  };
  const int first = pick_min();
  place(first);
  clear(first);
  list_remove(list_find(first));
  --npend;
  const int tail_n = min(DEV - 1, npend);
  int rear[DEV > 1 ? DEV - 1 : 1];
#pragma unroll
  for (int q = 0; q < (DEV > 1 ? DEV - 1 : 1); ++q) rear[q] = 0;
  for (int q = 0; q < tail_n; ++q) {
    const int r = pick_min();
#pragma unroll
    for (int z = 0; z < (DEV > 1 ? DEV - 1 : 1); ++z)
      if (z == q) rear[z] = r;
    clear(r);
    list_remove(list_find(r));
    --npend;
  }

  // ---- committed tick state (ticks < Tc) and the speculative frontier
  double av[P], pv[P];
#pragma unroll
  for (int s = 0; s < P; ++s) av[s] = pv[s] = 0.0;
  int Tc = 0;
  double f00_end = 0.0, last_b0_end = 0.0;
  int np = nret;
  double meanE = 0.0, meanG = 0.0, meanB = 0.0;
  // backward pending means, formed lazily (pending backward cells enter a
  // window only at the first step)
  bool have_bmean = false;
  double bmeanE = 0.0, bmeanG = 0.0, bmeanB = 0.0;
  auto rear_row = [&](int q) -> int {
    int r = 0;
#pragma unroll
    for (int z = 0; z < (DEV > 1 ? DEV - 1 : 1); ++z)
      if (z == q) r = rear[z];
    return r;
  };
  // forward duration of candidate position r at stage s
  auto candF = [&](int r, int s) -> double {
    if (s >= PE && s < PE + PB) {
      if (r >= np && r < np + npend) return meanB;
      return fB;
    }
    const bool enc = s < PE;
    if (r < np) {
      const int row = RET(r);
      return enc ? Fv(row) : Gv(row);
    }
    if (r < np + npend) return enc ? meanE : meanG;
    const int row = rear_row(r - np - npend);
    return enc ? Fv(row) : Gv(row);
  };
  auto candB = [&](int r, int s) -> double {
    if (r >= np && r < np + npend) {
      if (!have_bmean) {
        double sE = 0.0, sG = 0.0, sB = 0.0;
#pragma unroll
        for (int w = 0; w < MW; ++w) {
          unsigned m = pend[w];
          while (m) {
            const int idx = w * 32 + __ffs(m) - 1;
            m &= m - 1;
            double eb, gb;
            bwd_row(idx, &eb, &gb);
            sE += eb;
            sG += gb;
            sB += bB;
          }
        }
        const double c = static_cast<double>(npend);
        bmeanE = sE / c;
        bmeanG = sG / c;
        bmeanB = sB / c;
        have_bmean = true;
      }
      return s < PE ? bmeanE : s < PE + PB ? bmeanB : bmeanG;
    }
    if (s >= PE && s < PE + PB) return bB;
    if constexpr (!GATHER)
      if (r < np && r + kBRing >= nret) return s < PE ? BE(r) : BG(r);
    const int row = r < np ? static_cast<int>(RET(r)) : rear_row(r - np - npend);
    double eb, gb;
    bwd_row(row, &eb, &gb);
    return s < PE ? eb : gb;
  };
  // ticks [t0, t1] of 1F1B on state (x, y); visit(s, i, fwd, start, end)
  auto run_ticks = [&](int t0, int t1, double* x, double* y, auto&& visit) {
    for (int tk = t0; tk <= t1; ++tk) {
      double cur[P];
#pragma unroll
      for (int s = 0; s < P; ++s) cur[s] = y[s];
#pragma unroll
      for (int s = 0; s < P; ++s) {
        const int q = tk - s;
        if (q < 0) continue;
        if ((q & 1) == 0) {
          const int i = q >> 1;
          if (i >= l) continue;
          const double dep = s > 0 ? y[s - 1] : 0.0;
          const double start = smax(x[s], dep);
          const double end = start + candF(i, s);
          x[s] = end;
          cur[s] = end;
          visit(s, i, true, start, end);
        } else {
          const int qb = tk - 2 * P + 1 + s;
          if (qb < 0) continue;
          const int j = qb >> 1;
          if (j >= l) continue;
          const double dep = s + 1 < P ? y[s + 1] : y[s];
          const double start = smax(x[s], dep);
          const double end = start + candB(j, s);
          x[s] = end;
          cur[s] = end;
          visit(s, j, false, start, end);
        }
      }
#pragma unroll
      for (int s = 0; s < P; ++s) y[s] = cur[s];
    }
  };

  int step = 1;
  while (npend > 0) {
    const int wi = step - 1;
    const int t_target = 2 * wi + 2 * P - 1;  // tick of B(wi, 0)
    // pending means per unit: sequential sums in ascending index order
    {
      // sequential over the ascending pending list (src/reorder.cpp:191-201)
      double sE = 0.0, sG = 0.0;
#pragma unroll 4
      for (int q = 0; q < npend; ++q) {
        const int idx = PL[q];
        if constexpr (GATHER) {
          const double2 r = __ldg(a.table.fz + TK(idx));
          sE += r.x;
          sG += r.y;
        } else {
          sE += F(idx);
          sG += G(idx);
        }
      }
      const double c = static_cast<double>(npend);
      meanE = sE / c;
      meanG = sG / c;
      meanB = sb_sum[npend] / c;
    }
    have_bmean = false;
    double sx[P], sy[P];
#pragma unroll
    for (int s = 0; s < P; ++s) {
      sx[s] = av[s];
      sy[s] = pv[s];
    }
    double sf00 = f00_end, sb0 = last_b0_end, b_start = 0.0;
    run_ticks(Tc, t_target, sx, sy, [&](int s, int i, bool fwd, double start, double end) {
      if (s != 0) return;
      if (fwd) {
        if (i == 0) sf00 = end;
      } else if (i == wi) {
        b_start = start;
      } else if (i < wi) {
        sb0 = end;
      }
    });
    const double anchor = wi == 0 ? sf00 : sb0;
    const double target = 0.0 + (b_start - anchor);
    const int take = step == 1 ? min(DEV - 1, npend) : 1;
    double residual = target;
    for (int q = 0; q < take; ++q) {
      int ppos;
      const int pick = pick_closest(residual, &ppos);
      residual -= Kv(pick);
      place(pick);
      clear(pick);
      list_remove(ppos);
      --npend;
    }
    np = nret;
    const int Tc_new = 2 * np;
    if (Tc_new > Tc) {
      run_ticks(Tc, Tc_new - 1, av, pv, [&](int s, int i, bool fwd, double, double end) {
        if (s != 0) return;
        if (fwd) {
          if (i == 0) f00_end = end;
        } else {
          last_b0_end = end;
        }
      });
      Tc = Tc_new;
    }
    ++step;
  }
  for (int q = 0; q < tail_n; ++q) RET(nret++) = static_cast<unsigned char>(rear_row(q));
  for (int i = 0; i < l; ++i) out[i] = RET(i);
}

using InterTokFn = void (*)(InterArgs);
template <bool GATHER>
static InterTokFn inter_tok_for(int pe, int pb, int pg) {
#define DTB_ITOK(E, B, G) \
  if (pe == E && pb == B && pg == G) return inter_tok_kernel<E, B, G, GATHER>;
  DTB_ITOK(1, 1, 1)
  DTB_ITOK(1, 2, 1)
  DTB_ITOK(2, 1, 1)
  DTB_ITOK(1, 1, 2)
  DTB_ITOK(1, 3, 1)
  DTB_ITOK(1, 4, 1)
  DTB_ITOK(2, 2, 1)
  DTB_ITOK(1, 2, 2)
  DTB_ITOK(2, 2, 2)
  DTB_ITOK(1, 6, 1)
#undef DTB_ITOK
  return nullptr;
}

// The shared-memory kernel applies to the stream token form with vpp == 1,
// a compiled stage layout and l <= 255 (u8 positions).
bool inter_tok_applies(const InterArgs& a) {
  return a.stream && a.fwd == nullptr && a.vpp == 1 && a.l >= 1 && a.l <= 255 &&
         a.table.size > 0 &&
         inter_tok_for<false>(a.plan.unit[0].pp, a.plan.unit[1].pp, a.plan.unit[2].pp) != nullptr;
}

static cudaError_t launch_inter_tok_one(InterTokFn fn, const InterArgs& a, bool gather,
                                        cudaStream_t stream) {
  int dev = 0, max_smem = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t fixed = 8 * static_cast<size_t>(a.l + 1) + 64 + 8;
  const size_t per = inter_tok_bytes_per_thread(a.l, gather);
  int T = 128;
  while (T > 1 && fixed + per * T + 64 > static_cast<size_t>(max_smem)) --T;
  const size_t bytes = fixed + per * T + 64;  // + alignment slack of the ring
  if (bytes > static_cast<size_t>(max_smem)) return cudaErrorNotSupported;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(bytes));
  if (e != cudaSuccess) return e;
#ifndef DTB_INTER_CARVEOUT
#define DTB_INTER_CARVEOUT 60
#endif
  // gather variant: two blocks per SM and the rest of the unified L1 for the
  // cost-table rows it gathers (measured: 3 blocks + ~50 KB L1 10.2 ms,
  // 2 blocks + ~90 KB L1 9.3 ms, 1 block 12.1 ms)
  if (gather) cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, DTB_INTER_CARVEOUT);
  if (a.batch == 0) return cudaSuccess;
  fn<<<static_cast<unsigned>((a.batch + T - 1) / T), T, bytes, stream>>>(a);
  return cudaGetLastError();
}

__global__ void table_fz_kernel(const double4* __restrict__ eg, double2* __restrict__ fz, int n) {
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i < n) {
    const double4 r = eg[i];
    fz[i] = make_double2(r.x, r.z);
  }
}

cudaError_t launch_table_fz(const double4* eg, double2* fz, int size, cudaStream_t stream) {
  if (size > 0) table_fz_kernel<<<(size + 255) / 256, 256, 0, stream>>>(eg, fz, size);
  return cudaGetLastError();
}

// With a.redo (a zeroed byte per problem) and a.table.fz: the gather variant for every
// problem, then the shared-memory variant for the flagged ones only.
cudaError_t launch_inter_tok(const InterArgs& a, cudaStream_t stream) {
  if (!inter_tok_applies(a)) return cudaErrorNotSupported;
  const int pe = a.plan.unit[0].pp, pb = a.plan.unit[1].pp, pg = a.plan.unit[2].pp;
  if (a.redo == nullptr || a.table.fz == nullptr)
    return launch_inter_tok_one(inter_tok_for<false>(pe, pb, pg), a, false, stream);
  InterArgs g = a;
  g.redo_only = false;
  cudaError_t e = launch_inter_tok_one(inter_tok_for<true>(pe, pb, pg), g, true, stream);
  if (e != cudaSuccess) return e;
  InterArgs r = a;
  r.redo_only = true;
  return launch_inter_tok_one(inter_tok_for<false>(pe, pb, pg), r, false, stream);
}

}  // namespace dtb

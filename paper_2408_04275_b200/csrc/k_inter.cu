// Inter-microbatch reordering (Alg. 3; reference src/reorder.cpp:121-298).
//
// One thread per independent problem (a coupled group's microbatch
// sequence).  The reference rebuilds the whole candidate stage matrix and
// re-simulates the whole 1F1B schedule at every step only to read ONE
// window: window i = B(i,0).start - (i ? B(i-1,0).end : F(0,0).end).  With
// the tick evaluation of sched.cuh, cells at ticks < 2*np (np = placed rows)
// depend on placed rows only and never change again, so they are COMMITTED
// once; each step only evaluates the speculative ticks from the committed
// frontier to B(i,0) with the candidate rows (placed | pending-mean | rear,
// src/reorder.cpp:182-225).  Values are the same doubles the reference
// computes; per-problem work drops from O(l^2 p) to O(l p) for the schedule.
// vpp > 1 keeps the full re-simulation (interleaved order, dataflow sweep).
#include "kernels.cuh"
#include "sched.cuh"

namespace dtb {

// Stage-time access: explicit row-major matrices...
// col(s): the column class of stage s — stages of one class hold the same
// value in every row, so the pending-row means of a step are per class.
struct ExplicitTimes {
  const double* f;
  const double* b;
  int p;
  __device__ double F(int i, int s) const { return f[static_cast<size_t>(i) * p + s]; }
  __device__ double B(int i, int s) const { return b[static_cast<size_t>(i) * p + s]; }
  __device__ int col(int s) const { return s; }
  __device__ int ncols() const { return p; }
};
// ...or per-microbatch unit rows (build_stage_times: every stage of a unit
// carries the unit's value).
struct RowTimes {
  const double* rows;  // [l][6] = f[3], b[3]
  dtb_plan plan;
  __device__ double F(int i, int s) const { return rows[i * 6 + stage_unit(plan, s)]; }
  __device__ double B(int i, int s) const { return rows[i * 6 + 3 + stage_unit(plan, s)]; }
  __device__ int col(int s) const { return stage_unit(plan, s); }
  __device__ int ncols() const { return 3; }
};

// select_closest (reorder.cpp:136-175) over the pending flags, one pick.
__device__ __forceinline__ int pick_closest(const double* keys, const unsigned char* pend,
                                            int l, double residual) {
  int best = -1;
  double db = 0.0, kb = 0.0;
  for (int idx = 0; idx < l; ++idx) {
    if (!pend[idx]) continue;
    const double k = keys[idx];
    if (best < 0) {
      best = idx;
      kb = k;
      db = fabs(residual - k);
      continue;
    }
    const double da = fabs(residual - k);
    if (da != db) {
      if (da < db) {
        best = idx;
        kb = k;
        db = da;
      }
      continue;
    }
    const bool a_under = k <= residual;
    const bool b_under = kb <= residual;
    if (a_under != b_under) {
      if (a_under) {
        best = idx;
        kb = k;
        db = da;
      }
      continue;
    }
    // idx ascends, so the incumbent already has the lower index
  }
  return best;
}

// select_min (reorder.cpp:121-134), one pick: smallest (key, index).
__device__ __forceinline__ int pick_min(const double* keys, const unsigned char* pend, int l) {
  int best = -1;
  for (int idx = 0; idx < l; ++idx) {
    if (!pend[idx]) continue;
    if (best < 0 || keys[idx] < keys[best]) best = idx;
  }
  return best;
}

struct InterScratch {
  unsigned char* pend;  // [l]
  int* ret;             // [l]  placed order then rear
  int* rear;            // [l]
  double* st;           // state: vpp==1: 8p ; vpp>1: 2lp + 4 l vpp + 3 dev
  int* ist;             // int state: vpp>1: devices
};

template <typename Times>
__device__ int inter_one(const Times& tm, const double* keys, int l, int p,
                         int vpp, InterScratch sc, int* out) {
  for (int i = 0; i < l; ++i) out[i] = i;
  if (l <= 1) return 0;
  const int devices = p / vpp;
  if (devices == 1) return 0;
  unsigned char* pend = sc.pend;
  for (int i = 0; i < l; ++i) pend[i] = 1;
  int npend = l;
  int nret = 0;
  const int first = pick_min(keys, pend, l);
  sc.ret[nret++] = first;
  pend[first] = 0;
  --npend;
  const int tail_n = min(devices - 1, npend);
  for (int t = 0; t < tail_n; ++t) {
    const int r = pick_min(keys, pend, l);
    sc.rear[t] = r;
    pend[r] = 0;
    --npend;
  }
  if (npend > 0) {
    // the reference validates the candidate matrix inside every schedule
    // (pipeline_sim.cpp:214-230); invalid inputs surface at the first step
    for (int i = 0; i < l; ++i)
      for (int s = 0; s < p; ++s) {
        if (!(tm.F(i, s) >= 0.0)) return E_BAD_TIMES;
        if (!(tm.B(i, s) >= 0.0)) return E_BAD_TIMES;
      }
  }

  if (vpp == 1) {
    // committed tick state (after ticks < Tc) and a speculative copy
    double* avail = sc.st;
    double* prev = avail + p;
    double* cur = prev + p;
    double* s_avail = cur + p;
    double* s_prev = s_avail + p;
    double* s_cur = s_prev + p;
    // pending-row means of the current step, per column class (NaN = not
    // yet computed; valid times are never NaN): [0, ncols) forward,
    // [ncols, 2 ncols) backward — at most 2p doubles
    double* mean_c = s_cur + p;
    const int nc = tm.ncols();
    int Tc = 0;
    double f00_end = 0.0, last_b0_end = 0.0;
    for (int s = 0; s < p; ++s) avail[s] = prev[s] = cur[s] = 0.0;
    int np = nret;
    // candidate row accessors for the current step
    auto mean_of = [&](int s, bool fwd) -> double {
      // sequential mean over pending rows in ascending index order
      // (src/reorder.cpp:191-201), once per class and step
      double* slot = mean_c + (fwd ? 0 : nc) + tm.col(s);
      if (isnan(*slot)) {
        double acc = 0.0;
        for (int idx = 0; idx < l; ++idx)
          if (pend[idx]) acc += fwd ? tm.F(idx, s) : tm.B(idx, s);
        *slot = acc / static_cast<double>(npend);
      }
      return *slot;
    };
    auto cand = [&](int r, int s, int ph) -> double {
      if (r < np) {
        const int row = sc.ret[r];
        return ph == DTB_FORWARD ? tm.F(row, s) : tm.B(row, s);
      }
      if (r < np + npend) return mean_of(s, ph == DTB_FORWARD);
      const int row = sc.rear[r - np - npend];
      return ph == DTB_FORWARD ? tm.F(row, s) : tm.B(row, s);
    };
    // run ticks [t0, t1] on (av, pv, cv) with row accessor `dur`
    auto run_ticks = [&](int t0, int t1, double* av, double* pv, double* cv,
                         auto&& dur, auto&& visit) {
      for (int t = t0; t <= t1; ++t) {
        for (int s = 0; s < p; ++s) {
          const int a = t - s;
          if (a < 0) continue;
          if ((a & 1) == 0) {
            const int i = a >> 1;
            if (i >= l) continue;
            const double dep = s > 0 ? pv[s - 1] : 0.0;
            const double start = smax(av[s], dep);
            const double end = start + dur(i, s, DTB_FORWARD);
            av[s] = end;
            cv[s] = end;
            visit(s, i, DTB_FORWARD, start, end);
          } else {
            const int q = t - 2 * p + 1 + s;
            if (q < 0) continue;
            const int j = q >> 1;
            if (j >= l) continue;
            const double dep = s + 1 < p ? pv[s + 1] : pv[s];
            const double start = smax(av[s], dep);
            const double end = start + dur(j, s, DTB_BACKWARD);
            av[s] = end;
            cv[s] = end;
            visit(s, j, DTB_BACKWARD, start, end);
          }
        }
        for (int s = 0; s < p; ++s) pv[s] = cv[s];
      }
    };
    auto placed_dur = [&](int r, int s, int ph) -> double {
      const int row = sc.ret[r];
      return ph == DTB_FORWARD ? tm.F(row, s) : tm.B(row, s);
    };
    auto commit_visit = [&](int s, int i, int ph, double start, double end) {
      if (s != 0) return;
      if (ph == DTB_FORWARD) {
        if (i == 0) f00_end = end;
      } else {
        last_b0_end = end;
      }
    };
    int step = 1;
    while (npend > 0) {
      const int wi = step - 1;  // window index (vpp == 1)
      const int t_target = 2 * wi + 2 * p - 1;  // tick of B(wi, 0)
      // speculative ticks [Tc, t_target] on a copy of the committed state
      for (int s = 0; s < p; ++s) {
        s_avail[s] = avail[s];
        s_prev[s] = prev[s];
        s_cur[s] = cur[s];
      }
      for (int c = 0; c < 2 * nc; ++c) mean_c[c] = __longlong_as_double(0x7ff8000000000000ll);
      double sf00 = f00_end, sb0 = last_b0_end, b_start = 0.0;
      auto spec_visit = [&](int s, int i, int ph, double start, double end) {
        if (s != 0) return;
        if (ph == DTB_FORWARD) {
          if (i == 0) sf00 = end;
        } else if (i == wi) {
          b_start = start;
        } else if (i < wi) {
          sb0 = end;
        }
      };
      run_ticks(Tc, t_target, s_avail, s_prev, s_cur, cand, spec_visit);
      const double anchor = wi == 0 ? sf00 : sb0;
      const double target = 0.0 + (b_start - anchor);
      const int take = step == 1 ? min(devices - 1, npend) : 1;
      double residual = target;
      for (int t = 0; t < take; ++t) {
        const int pick = pick_closest(keys, pend, l, residual);
        residual -= keys[pick];
        sc.ret[nret++] = pick;
        pend[pick] = 0;
        --npend;
      }
      // commit ticks now fully determined by placed rows
      const int np_new = nret;
      const int Tc_new = 2 * np_new;
      np = np_new;
      if (Tc_new > Tc) {
        run_ticks(Tc, Tc_new - 1, avail, prev, cur, placed_dur, commit_visit);
        Tc = Tc_new;
      }
      ++step;
    }
  } else {
    // full re-simulation per step on the interleaved order
    const size_t cells = static_cast<size_t>(l) * p;
    double* f_end = sc.st;
    double* b_end = f_end + cells;
    double* b0s = b_end + cells;            // device-0 backward starts [l*vpp]
    double* b0e = b0s + l * vpp;            // ends
    double* b0k = b0e + l * vpp;            // (mb, stage) packed as double
    double* avail = b0k + l * vpp;
    double* mean = avail + devices;         // [2p] per step
    int* next = sc.ist;
    int step = 1;
    while (npend > 0) {
      int np = nret;
      for (int s = 0; s < p; ++s) {
        double af = 0.0, ab = 0.0;
        for (int idx = 0; idx < l; ++idx)
          if (pend[idx]) {
            af += tm.F(idx, s);
            ab += tm.B(idx, s);
          }
        mean[s] = af / static_cast<double>(npend);
        mean[p + s] = ab / static_cast<double>(npend);
      }
      auto cand = [&](int r, int s, int ph) -> double {
        if (r < np) {
          const int row = sc.ret[r];
          return ph == DTB_FORWARD ? tm.F(row, s) : tm.B(row, s);
        }
        if (r < np + npend) return ph == DTB_FORWARD ? mean[s] : mean[p + s];
        const int row = sc.rear[r - np - npend];
        return ph == DTB_FORWARD ? tm.F(row, s) : tm.B(row, s);
      };
      int nb = 0;
      double f00 = 0.0;
      auto visit = [&](int d, Op op, double start, double end) {
        if (d != 0) return;
        if (op.phase == DTB_FORWARD) {
          if (op.mb == 0 && op.stage == 0) f00 = end;
        } else {
          b0s[nb] = start;
          b0e[nb] = end;
          b0k[nb] = static_cast<double>(op.mb) * 65536.0 + op.stage;
          ++nb;
        }
      };
      const int e = dataflow_schedule(l, p, vpp, cand, f_end, b_end, next, avail, visit);
      if (e) return e;
      // Timeline order on device 0: stable insertion sort by (start, mb, stage)
      for (int a = 1; a < nb; ++a) {
        const double s0 = b0s[a], e0 = b0e[a], k0 = b0k[a];
        int c = a - 1;
        while (c >= 0 && (b0s[c] > s0 || (b0s[c] == s0 && b0k[c] > k0))) {
          b0s[c + 1] = b0s[c];
          b0e[c + 1] = b0e[c];
          b0k[c + 1] = b0k[c];
          --c;
        }
        b0s[c + 1] = s0;
        b0e[c + 1] = e0;
        b0k[c + 1] = k0;
      }
      double target = 0.0;
      for (int w = 0; w < vpp; ++w) {
        const int wi = (step - 1) * vpp + w;
        if (wi < nb) {
          const double anchor = wi == 0 ? f00 : b0e[wi - 1];
          target += b0s[wi] - anchor;
        }
      }
      const int take = step == 1 ? min(devices - 1, npend) : 1;
      double residual = target;
      for (int t = 0; t < take; ++t) {
        const int pick = pick_closest(keys, pend, l, residual);
        residual -= keys[pick];
        sc.ret[nret++] = pick;
        pend[pick] = 0;
        --npend;
      }
      ++step;
    }
  }
  for (int t = 0; t < tail_n; ++t) sc.ret[nret++] = sc.rear[t];
  for (int i = 0; i < l; ++i) out[i] = sc.ret[i];
  return 0;
}

static __host__ __device__ size_t inter_state_doubles(int l, int p, int vpp) {
  const int devices = p / vpp;
  return vpp == 1 ? static_cast<size_t>(8 * p)
                  : 2 * static_cast<size_t>(l) * p + 3 * static_cast<size_t>(l) * vpp +
                        devices + 2 * p;
}

static __host__ __device__ size_t inter_bytes_per_problem(int l, int p, int vpp) {
  size_t b = inter_state_doubles(l, p, vpp) * 8;
  b += 4 * static_cast<size_t>(l) * 2 + static_cast<size_t>(l) + 4 * (p / vpp);
  b += 6 * 8 * static_cast<size_t>(l) + 8 * static_cast<size_t>(l);  // rows + keys (token form)
  return (b + 63) & ~size_t(63);
}

__global__ void inter_kernel(InterArgs a, char* scratch, long long begin,
                             long long count) {
  const long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (q >= count) return;
  const long long prob = begin + q;
  const int l = a.l, p = a.p, vpp = a.vpp;
  char* base = scratch + q * inter_bytes_per_problem(l, p, vpp);
  InterScratch sc;
  sc.st = reinterpret_cast<double*>(base);
  char* c = base + inter_state_doubles(l, p, vpp) * 8;
  double* rows = reinterpret_cast<double*>(c);
  c += 6 * 8 * static_cast<size_t>(l);
  double* tkeys = reinterpret_cast<double*>(c);
  c += 8 * static_cast<size_t>(l);
  sc.ret = reinterpret_cast<int*>(c);
  c += 4 * static_cast<size_t>(l);
  sc.rear = reinterpret_cast<int*>(c);
  c += 4 * static_cast<size_t>(l);
  sc.ist = reinterpret_cast<int*>(c);
  c += 4 * (p / vpp);
  sc.pend = reinterpret_cast<unsigned char*>(c);
  int* out = a.orders + prob * l;
  int e = 0;
  if (a.fwd != nullptr) {
    ExplicitTimes tm{a.fwd + prob * l * p, a.bwd + prob * l * p, p};
    e = inter_one(tm, a.keys + prob * l, l, p, vpp, sc, out);
  } else {
    // token form: build_stage_times rows and microbatch_fwd_keys per microbatch
    const long long bb = prob / a.groups;
    const int grp = static_cast<int>(prob % a.groups);
    for (int i = 0; i < l && !e; ++i) {
      const long long v = a.span == 1 ? a.tok.get(bb, grp * l + i, true)
                                      : a.mbsum[(bb * a.groups + grp) * static_cast<long long>(l) + i];
      const double me = mb_mean(v, a.span);
      const double mg = me;
      StageRow r;
      e = dev_stage_row(a.cm, a.plan, me, mg, &r);
      if (!e) e = dev_fwd_key(a.cm, a.plan, me, mg, &tkeys[i]);
      for (int u = 0; u < 3; ++u) {
        rows[i * 6 + u] = r.f[u];
        rows[i * 6 + 3 + u] = r.b[u];
      }
    }
    if (!e) {
      RowTimes tm{rows, a.plan};
      e = inter_one(tm, tkeys, l, p, vpp, sc, out);
    }
  }
  if (e) dev_fail(a.err, e);
}

size_t inter_scratch(const InterArgs& a) {
  const long long chunk = a.batch < 32768 ? a.batch : 32768;
  return static_cast<size_t>(chunk) * inter_bytes_per_problem(a.l, a.p, a.vpp) + 256;
}

cudaError_t launch_inter(const InterArgs& a, void* scratch, size_t bytes,
                         cudaStream_t stream) {
  const size_t per = inter_bytes_per_problem(a.l, a.p, a.vpp);
  long long chunk = static_cast<long long>(bytes / per);
  if (chunk < 1) return cudaErrorMemoryAllocation;
  const int T = 64;
  for (long long begin = 0; begin < a.batch; begin += chunk) {
    const long long count = a.batch - begin < chunk ? a.batch - begin : chunk;
    inter_kernel<<<static_cast<unsigned>((count + T - 1) / T), T, 0, stream>>>(
        a, static_cast<char*>(scratch), begin, count);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace dtb

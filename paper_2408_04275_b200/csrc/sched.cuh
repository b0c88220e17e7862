// Pipeline-schedule evaluation on the device (reference:
// src/pipeline_sim.cpp:36-183).
//
// Event times depend only on each device's op order and the dependency edges
// (start = max(device availability, dependency end); end = start + dur), so
// any evaluation order that respects the edges yields identical doubles
// (SURVEY.md §3.4).  Two evaluators:
//
//  * Tick1F1B — plain 1F1B.  Device s runs F(i,s) at tick 2i+s and B(j,s) at
//    tick 2j+2p-1-s.  Every edge (F(i,s-1)->F(i,s), B(j,s+1)->B(j,s),
//    F(j,p-1)->B(j,p-1) and each device's sequence order, warm-up
//    min(p-s,l)) points from tick T-1 or earlier to tick T, and each (tick,
//    device) holds at most one op, so a loop over ticks evaluates the
//    schedule with a p-entry state and no readiness checks.
//  * dataflow_schedule — any vpp (interleaved op order of
//    src/pipeline_sim.cpp:58-99): the reference's readiness sweep over
//    per-device op cursors, used where vpp > 1.
#pragma once

#include "dtb_internal.cuh"

namespace dtb {

struct Op {
  int mb, stage, phase;
};

// The q-th op of device s (src/pipeline_sim.cpp:36-52 for vpp == 1,
// :58-99 otherwise).  2*l*vpp ops per device.
__host__ __device__ __forceinline__ Op device_op(int l, int p, int vpp, int s,
                                                 int q) {
  if (vpp == 1) {
    const int w = (p - s) < l ? (p - s) : l;
    if (q < w) return {q, s, DTB_FORWARD};
    const int r = q - w;
    const int steady = l - w;
    if (r < 2 * steady)
      return (r & 1) ? Op{w + (r >> 1), s, DTB_FORWARD} : Op{r >> 1, s, DTB_BACKWARD};
    return {steady + (r - 2 * steady), s, DTB_BACKWARD};
  }
  const int devices = p / vpp;
  const int total = l * vpp;
  int w = 2 * (devices - 1 - s) + (vpp - 1) * devices;
  if (w > total) w = total;
  auto virt = [&](int idx, bool bwd) {
    const int group = idx / (devices * vpp);
    const int within = idx % (devices * vpp);
    int chunk = within / devices;
    if (bwd) chunk = vpp - 1 - chunk;
    return Op{group * devices + within % devices, chunk * devices + s,
              bwd ? DTB_BACKWARD : DTB_FORWARD};
  };
  if (q < w) return virt(q, false);
  const int r = q - w;
  const int steady = total - w;
  if (r < 2 * steady) return (r & 1) ? virt(r >> 1, true) : virt(w + (r >> 1), false);
  return virt(steady + (r - 2 * steady), true);
}

// Generic readiness-sweep evaluation (run_schedule, pipeline_sim.cpp:108-183).
// f_end/b_end: [l*p] scratch, overwritten.  Calls visit(d, op, start, end)
// for every op in per-device execution order.  Returns 0 or E_DEADLOCK.
template <typename TimeFn, typename Visit>
__device__ int dataflow_schedule(int l, int p, int vpp, const TimeFn& dur,
                                 double* f_end, double* b_end, int* next,
                                 double* avail, const Visit& visit) {
  const int devices = p / vpp;
  const int per = 2 * l * vpp;
  for (int i = 0; i < l * p; ++i) f_end[i] = b_end[i] = -1.0;
  for (int d = 0; d < devices; ++d) {
    next[d] = 0;
    avail[d] = 0.0;
  }
  long long remaining = static_cast<long long>(per) * devices;
  while (remaining > 0) {
    bool progressed = false;
    for (int d = 0; d < devices; ++d) {
      while (next[d] < per) {
        const Op op = device_op(l, p, vpp, d, next[d]);
        const int me = op.mb * p + op.stage;
        double dep = 0.0;
        if (op.phase == DTB_FORWARD) {
          if (op.stage > 0) {
            dep = f_end[me - 1];
            if (dep == -1.0) break;
          }
        } else {
          dep = op.stage + 1 < p ? b_end[me + 1] : f_end[me];
          if (dep == -1.0) break;
        }
        const double start = smax(avail[d], dep);
        const double end = start + dur(op.mb, op.stage, op.phase);
        (op.phase == DTB_FORWARD ? f_end : b_end)[me] = end;
        avail[d] = end;
        visit(d, op, start, end);
        ++next[d];
        --remaining;
        progressed = true;
      }
    }
    if (!progressed) return E_DEADLOCK;
  }
  return 0;
}

// Plain 1F1B by ticks.  prev/cur: [p] scratch.  visit(s, op, start, end) is
// called per op in per-device execution order (ticks ascending).
template <typename TimeFn, typename Visit>
__device__ void tick_1f1b(int l, int p, const TimeFn& dur, double* prev,
                          double* cur, double* avail, const Visit& visit) {
  for (int s = 0; s < p; ++s) avail[s] = 0.0;
  const int last_tick = 2 * l + 2 * p - 3;
  for (int t = 0; t <= last_tick; ++t) {
    for (int s = 0; s < p; ++s) {
      const int a = t - s;
      if (a < 0) continue;
      if ((a & 1) == 0) {
        const int i = a >> 1;
        if (i >= l) continue;
        const double dep = s > 0 ? prev[s - 1] : 0.0;
        const double start = smax(avail[s], dep);
        const double end = start + dur(i, s, DTB_FORWARD);
        avail[s] = end;
        cur[s] = end;
        visit(s, Op{i, s, DTB_FORWARD}, start, end);
      } else {
        const int q = t - 2 * p + 1 + s;
        if (q < 0 || (q & 1)) continue;
        const int j = q >> 1;
        if (j >= l) continue;
        const double dep = s + 1 < p ? prev[s + 1] : prev[s];
        const double start = smax(avail[s], dep);
        const double end = start + dur(j, s, DTB_BACKWARD);
        avail[s] = end;
        cur[s] = end;
        visit(s, Op{j, s, DTB_BACKWARD}, start, end);
      }
    }
    for (int s = 0; s < p; ++s) prev[s] = cur[s];
  }
}

}  // namespace dtb

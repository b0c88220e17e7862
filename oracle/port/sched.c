/* ORACLE restatement of the pipeline simulator: src/pipeline_sim.cpp,
 * src/simulate.cpp. */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "port.h"

typedef struct {
  int mb, stage, phase;
} op_t;

/* ops_1f1b — src/pipeline_sim.cpp:36-52. */
static int ops_1f1b(int l, int p, int s, op_t* ops) {
  int n = 0;
  const int warmup = (p - s) < l ? (p - s) : l;
  for (int i = 0; i < warmup; ++i) ops[n++] = (op_t){i, s, DTB_FORWARD};
  for (int j = 0; j + warmup < l; ++j) {
    ops[n++] = (op_t){j, s, DTB_BACKWARD};
    ops[n++] = (op_t){j + warmup, s, DTB_FORWARD};
  }
  for (int j = (l - warmup > 0 ? l - warmup : 0); j < l; ++j)
    ops[n++] = (op_t){j, s, DTB_BACKWARD};
  return n;
}

/* virtual_at / ops_interleaved — src/pipeline_sim.cpp:58-99. */
static op_t virtual_op(int idx, int devices, int vpp, int backward, int s) {
  const int group = idx / (devices * vpp);
  const int within = idx % (devices * vpp);
  int chunk = within / devices;
  if (backward) chunk = vpp - 1 - chunk;
  const int mb = group * devices + within % devices;
  return (op_t){mb, chunk * devices + s, backward ? DTB_BACKWARD : DTB_FORWARD};
}

static int ops_interleaved(int l, int p, int vpp, int s, op_t* ops) {
  const int devices = p / vpp;
  const int total = l * vpp;
  int warmup = 2 * (devices - 1 - s) + (vpp - 1) * devices;
  if (warmup > total) warmup = total;
  int n = 0;
  for (int i = 0; i < warmup; ++i) ops[n++] = virtual_op(i, devices, vpp, 0, s);
  for (int j = 0; j + warmup < total; ++j) {
    ops[n++] = virtual_op(warmup + j, devices, vpp, 0, s);
    ops[n++] = virtual_op(j, devices, vpp, 1, s);
  }
  for (int j = (total - warmup > 0 ? total - warmup : 0); j < total; ++j)
    ops[n++] = virtual_op(j, devices, vpp, 1, s);
  return n;
}

/* StageTimes::valid — src/pipeline_sim.cpp:214-230. */
int port_check_times(const double* fwd, const double* bwd, int l, int p) {
  const char* why = NULL;
  if (l < 1) why = "microbatch count must be >= 1";
  else if (p < 1) why = "stage count must be >= 1";
  else {
    const int64_t n = (int64_t)l * p;
    for (int64_t i = 0; i < n && !why; ++i)
      if (!(fwd[i] >= 0.0)) why = "negative or NaN forward time";
    for (int64_t i = 0; i < n && !why; ++i)
      if (!(bwd[i] >= 0.0)) why = "negative or NaN backward time";
  }
  if (why) return port_fail(DTB_ERR_INTERNAL, "bad stage times: %s", why);
  return 0;
}

static int cmp_event(const void* pa, const void* pb) {
  const port_event* a = pa;
  const port_event* b = pb;
  if (a->start != b->start) return a->start < b->start ? -1 : 1;
  if (a->device != b->device) return a->device < b->device ? -1 : 1;
  if (a->mb != b->mb) return a->mb < b->mb ? -1 : 1;
  if (a->stage != b->stage) return a->stage < b->stage ? -1 : 1;
  return a->phase - b->phase;
}

/* run_schedule — src/pipeline_sim.cpp:108-183 (round-robin device sweep). */
int port_schedule(const double* fwd, const double* bwd, int l, int p, int vpp,
                  port_timeline* tl) {
  memset(tl, 0, sizeof *tl);
  TRY(port_check_times(fwd, bwd, l, p));
  if (vpp < 1) return port_fail(DTB_ERR_INDIVISIBLE_VPP, "vpp must be >= 1");
  if (vpp > 1) {
    if (p % vpp != 0)
      return port_fail(DTB_ERR_INDIVISIBLE_VPP,
                       "stage count %d is not divisible by vpp %d", p, vpp);
    if (l % (p / vpp) != 0)
      return port_fail(DTB_ERR_INDIVISIBLE_VPP,
                       "microbatch count %d is not divisible by the device "
                       "count %d",
                       l, p / vpp);
  }
  const int devices = p / vpp;
  const int per = 2 * l * vpp;
  op_t* ops = malloc(sizeof(op_t) * (size_t)per * devices);
  int* nops = calloc(devices, sizeof(int));
  int* next = calloc(devices, sizeof(int));
  double* avail = calloc(devices, sizeof(double));
  const size_t cells = (size_t)l * p;
  double* f_end = malloc(sizeof(double) * cells);
  double* b_end = malloc(sizeof(double) * cells);
  for (size_t i = 0; i < cells; ++i) f_end[i] = b_end[i] = -1.0;
  tl->events = malloc(sizeof(port_event) * 2 * cells);
  tl->busy = calloc(devices, sizeof(double));
  tl->devices = devices;
  int64_t remaining = 0;
  for (int d = 0; d < devices; ++d) {
    nops[d] = vpp == 1 ? ops_1f1b(l, p, d, ops + (size_t)d * per)
                       : ops_interleaved(l, p, vpp, d, ops + (size_t)d * per);
    remaining += nops[d];
  }
  int64_t ne = 0;
  while (remaining > 0) {
    int progressed = 0;
    for (int d = 0; d < devices; ++d) {
      while (next[d] < nops[d]) {
        const op_t op = ops[(size_t)d * per + next[d]];
        double dep = 0.0;
        const size_t me = (size_t)op.mb * p + op.stage;
        if (op.phase == DTB_FORWARD) {
          if (op.stage > 0) {
            dep = f_end[me - 1];
            if (dep == -1.0) break;
          }
        } else {
          dep = op.stage + 1 < p ? b_end[me + 1] : f_end[me];
          if (dep == -1.0) break;
        }
        const double start = port_max(avail[d], dep);
        const double dur = op.phase == DTB_FORWARD ? fwd[me] : bwd[me];
        const double end = start + dur;
        (op.phase == DTB_FORWARD ? f_end : b_end)[me] = end;
        avail[d] = end;
        tl->busy[d] += dur;
        tl->events[ne++] = (port_event){d, op.mb, op.stage, op.phase, start, end};
        ++next[d];
        --remaining;
        progressed = 1;
      }
    }
    if (!progressed) {
      free(ops); free(nops); free(next); free(avail); free(f_end); free(b_end);
      port_timeline_free(tl);
      return port_fail(DTB_ERR_INTERNAL,
                       "pipeline schedule deadlocked; op order is invalid");
    }
  }
  tl->n_events = ne;
  qsort(tl->events, (size_t)ne, sizeof(port_event), cmp_event);
  tl->iteration_time = 0.0;
  for (int64_t i = 0; i < ne; ++i)
    tl->iteration_time = port_max(tl->iteration_time, tl->events[i].end);
  free(ops); free(nops); free(next); free(avail); free(f_end); free(b_end);
  return 0;
}

void port_timeline_free(port_timeline* tl) {
  free(tl->events);
  free(tl->busy);
  tl->events = NULL;
  tl->busy = NULL;
}

/* get_intervals — src/pipeline_sim.cpp:264-289. */
int64_t port_get_intervals(const port_event* ev, int64_t n, double* starts,
                           double* ends, int64_t* fill_off, int32_t* fill_mb) {
  int64_t nf = 0, nb = 0;
  const port_event** f0 = malloc(sizeof(*f0) * (size_t)(n ? n : 1));
  const port_event** b0 = malloc(sizeof(*b0) * (size_t)(n ? n : 1));
  for (int64_t i = 0; i < n; ++i) {
    if (ev[i].device != 0) continue;
    if (ev[i].phase == DTB_FORWARD) f0[nf++] = &ev[i];
    else b0[nb++] = &ev[i];
  }
  int64_t k = 0, filled = 0;
  if (fill_off) fill_off[0] = 0;
  if (nf > 0 && nb > 0) {
    double anchor = f0[0]->end;
    int64_t fill = 0;
    for (int64_t i = 0; i < nb; ++i) {
      const double s = anchor, e = b0[i]->start;
      while (fill < nf && f0[fill]->start < s) ++fill;
      while (fill < nf && f0[fill]->start < e) {
        if (fill_mb) fill_mb[filled] = f0[fill]->mb;
        ++filled;
        ++fill;
      }
      if (starts) starts[k] = s;
      if (ends) ends[k] = e;
      ++k;
      if (fill_off) fill_off[k] = filled;
      anchor = b0[i]->end;
    }
  }
  free(f0);
  free(b0);
  return k;
}

/* simulate_iteration — src/simulate.cpp:23-48 (iteration_stats,
 * src/pipeline_sim.cpp:355-366). */
int port_simulate_iteration(const port_cm* cm, const dtb_plan* plan,
                            int n_groups, const int64_t* group_off,
                            const port_mb* mbs, double* t_iter,
                            double* group_times, int32_t* slowest,
                            double* slowest_time, double* bubble) {
  if (n_groups <= 0)
    return port_fail(DTB_ERR_INTERNAL, "no microbatch groups to simulate");
  const int p = (plan->unit[0].pp + plan->unit[1].pp + plan->unit[2].pp) *
                plan->vpp;
  double bubble_sum = 0.0, worst = 0.0;
  int worst_g = 0;
  for (int g = 0; g < n_groups; ++g) {
    const int64_t l = group_off[g + 1] - group_off[g];
    const size_t cells = (size_t)(l > 0 ? l : 1) * (size_t)(p > 0 ? p : 1);
    double* f = malloc(sizeof(double) * cells);
    double* b = malloc(sizeof(double) * cells);
    int st = port_build_stage_times(cm, plan, mbs + group_off[g], l, f, b);
    port_timeline tl;
    if (st == 0) st = port_schedule(f, b, (int)l, p, plan->vpp, &tl);
    free(f);
    free(b);
    if (st != 0) return st;
    double bub = 0.0;
    if (tl.iteration_time > 0.0 && tl.devices > 0) {
      double idle = 0.0;
      for (int d = 0; d < tl.devices; ++d) idle += tl.iteration_time - tl.busy[d];
      bub = idle / (tl.devices * tl.iteration_time);
    }
    bubble_sum += bub;
    if (group_times) group_times[g] = tl.iteration_time;
    if (tl.iteration_time > worst) {
      worst = tl.iteration_time;
      worst_g = g;
    }
    port_timeline_free(&tl);
  }
  if (bubble) *bubble = bubble_sum / (double)n_groups;
  if (slowest) *slowest = worst_g;
  if (slowest_time) *slowest_time = worst;
  if (t_iter) *t_iter = worst + cm->model.dp_sync_seconds;
  return 0;
}

/* ORACLE restatement of Alg. 1: src/orchestrator.cpp. */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "port.h"

static const int kTp[4] = {1, 2, 4, 8};

/* divisors — src/orchestrator.cpp:30-40 (ascending). */
static int64_t divisors(int64_t n, int64_t* out) {
  int64_t k = 0;
  for (int64_t d = 1; d * d <= n; ++d) {
    if (n % d == 0) {
      out[k++] = d;
      if (d != n / d) out[k++] = n / d;
    }
  }
  for (int64_t i = 1; i < k; ++i) /* insertion sort */
    for (int64_t j = i; j > 0 && out[j - 1] > out[j]; --j) {
      const int64_t t = out[j];
      out[j] = out[j - 1];
      out[j - 1] = t;
    }
  return k;
}

static int cmp_tuple(const void* pa, const void* pb) {
  const int32_t* a = pa;
  const int32_t* b = pb;
  for (int i = 0; i < 6; ++i)
    if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
  return 0;
}

/* enumerate_parallelism — src/orchestrator.cpp:268-301. */
int64_t port_enumerate(const dtb_cluster_spec* c, int64_t bs, dtb_tuple** out) {
  const int n = c->total_gpus;
  int64_t* dl = malloc(sizeof(int64_t) * 4096);
  int64_t* dm = malloc(sizeof(int64_t) * 4096);
  const int64_t nd = divisors(bs, dl);
  int64_t cap = 1024, k = 0;
  dtb_tuple* v = malloc(sizeof(dtb_tuple) * cap);
  for (int a = 0; a < 4; ++a)
    for (int bb = 0; bb < 4; ++bb)
      for (int cc = 0; cc < 4; ++cc)
        for (int64_t i = 0; i < nd; ++i) {
          const int64_t dp_lm = dl[i];
          if (kTp[bb] * dp_lm > n) continue;
          const int64_t nm = divisors(dp_lm, dm);
          for (int64_t j = 0; j < nm; ++j) {
            if (kTp[a] * dm[j] > n) continue;
            for (int64_t q = 0; q < nm; ++q) {
              dtb_tuple t = {kTp[a], (int32_t)dm[j], kTp[bb], (int32_t)dp_lm,
                             kTp[cc], (int32_t)dm[q]};
              if ((int64_t)t.tp_me * t.dp_me + (int64_t)t.tp_lm * t.dp_lm +
                      (int64_t)t.tp_mg * t.dp_mg > n)
                continue;
              if (k == cap) v = realloc(v, sizeof(dtb_tuple) * (cap *= 2));
              v[k++] = t;
            }
          }
        }
  qsort(v, (size_t)k, sizeof(dtb_tuple), cmp_tuple);
  free(dl);
  free(dm);
  *out = v;
  return k;
}

static dtb_plan plan_from(const dtb_tuple* t, int pe, int pl, int pg,
                          int64_t bs, int vpp) {
  dtb_plan p;
  memset(&p, 0, sizeof p);
  p.unit[0] = (dtb_parallelism){t->tp_me, t->dp_me, pe};
  p.unit[1] = (dtb_parallelism){t->tp_lm, t->dp_lm, pl};
  p.unit[2] = (dtb_parallelism){t->tp_mg, t->dp_mg, pg};
  p.global_batch = bs;
  p.vpp = vpp;
  return p;
}

static double stats_load(const port_cm* cm, int kind,
                         const dtb_workload_stats* s) {
  if (kind == DTB_ENCODER) return s->mean_encoder_tokens;
  if (kind == DTB_GENERATOR) return s->mean_generator_tokens;
  return (double)cm->model.seq_len;
}

static int fwdbwd(const port_cm* cm, int kind, int tp, double load,
                  double* out) {
  double f, b;
  TRY(port_unit_forward(cm, kind, tp, load, &f));
  TRY(port_unit_backward(cm, kind, tp, load, &b));
  *out = f + b;
  return 0;
}

/* predict_times — src/orchestrator.cpp:237-266. */
int port_predict_times(const port_cm* cm, const dtb_plan* plan,
                       const dtb_workload_stats* stats,
                       dtb_predicted_times* out) {
  const int64_t mbs = plan->global_batch / plan->unit[DTB_BACKBONE].dp;
  if (mbs < 1)
    return port_fail(DTB_ERR_INTERNAL, "plan yields no microbatches per iteration");
  out->t_warm = out->t_steady = out->t_iter = 0.0;
  double stage_max = 0.0;
  for (int kind = 0; kind < 3; ++kind) {
    const dtb_parallelism* pc = &plan->unit[kind];
    const double coupling =
        kind == DTB_BACKBONE ? 1.0 : (double)plan->unit[DTB_BACKBONE].dp / pc->dp;
    const double load = stats_load(cm, kind, stats);
    double cfb;
    TRY(fwdbwd(cm, kind, pc->tp, load, &cfb));
    const double comm = port_pp_boundary_seconds(
        plan, kind, &cm->cluster, port_boundary_bytes(cm, kind, plan, load));
    out->t_warm += coupling * cfb / plan->vpp + pc->pp * 2.0 * comm;
    stage_max = port_max(stage_max, coupling * cfb / pc->pp + plan->vpp * 2.0 * comm);
  }
  out->t_steady = stage_max * (double)(mbs - 1);
  out->t_iter = out->t_warm + out->t_steady + cm->model.dp_sync_seconds;
  return 0;
}

typedef struct {
  double coupling[3], cfb[3], comm[3], floor_gpus[3];
  int q[3];
  int64_t microbatches;
  int feasible, reason;
} tuple_costs_t;

/* tuple_costs — src/orchestrator.cpp:65-113. */
static int tuple_costs(const port_cm* cm, const dtb_tuple* t,
                       const dtb_workload_stats* stats, int64_t bs,
                       tuple_costs_t* tc) {
  memset(tc, 0, sizeof *tc);
  tc->feasible = 1;
  if (bs % t->dp_lm != 0) {
    tc->feasible = 0;
    tc->reason = DTB_REASON_DP_NOT_DIVIDING;
    return 0;
  }
  tc->microbatches = bs / t->dp_lm;
  const dtb_plan probe = plan_from(t, 1, 1, 1, bs, 1);
  const int tps[3] = {t->tp_me, t->tp_lm, t->tp_mg};
  const int dps[3] = {t->dp_me, t->dp_lm, t->dp_mg};
  for (int u = 0; u < 3; ++u) {
    tc->coupling[u] = (double)t->dp_lm / dps[u];
    const double load = stats_load(cm, u, stats);
    TRY(fwdbwd(cm, u, tps[u], load, &tc->cfb[u]));
    tc->comm[u] = port_pp_boundary_seconds(
        &probe, u, &cm->cluster, port_boundary_bytes(cm, u, &probe, load));
    tc->q[u] = tps[u] * dps[u];
    const dtb_module_memory* mem = &cm->model.unit[u].mem;
    const double act_const =
        (double)t->dp_lm * mem->activation_bytes_per_mb / tc->q[u];
    const double headroom = cm->cluster.gpu_mem_bytes - act_const;
    if (headroom <= 0.0) {
      tc->feasible = 0;
      tc->reason = DTB_REASON_ACTIVATION_ENCODER + u;
      return 0;
    }
    const double mem_floor =
        (dps[u] * mem->param_grad_bytes + mem->optimizer_bytes) / headroom;
    tc->floor_gpus[u] = port_max((double)tc->q[u], mem_floor);
  }
  double floor_sum = 0.0;
  for (int u = 0; u < 3; ++u) floor_sum += tc->floor_gpus[u];
  if (floor_sum > cm->cluster.total_gpus) {
    tc->feasible = 0;
    tc->reason = DTB_REASON_MEMORY_FLOOR;
  }
  return 0;
}

typedef struct {
  double a[3], b[3], c[3], floor[3], w0, steady_mult, dp_sync;
} cont_t;

static double gpus_at(const cont_t* k, double bound, double* g) {
  double sum = 0.0;
  for (int u = 0; u < 3; ++u) {
    const double need = bound > k->c[u] ? k->b[u] / (bound - k->c[u]) : INFINITY;
    g[u] = port_max(k->floor[u], need);
    sum += g[u];
  }
  return sum;
}

static double objective(const cont_t* k, double bound, double* g) {
  gpus_at(k, bound, g);
  double warm_comm = 0.0, stage_max = 0.0;
  for (int u = 0; u < 3; ++u) {
    warm_comm += k->a[u] * g[u];
    stage_max = port_max(stage_max, k->b[u] / g[u] + k->c[u]);
  }
  return k->w0 + warm_comm + stage_max * k->steady_mult + k->dp_sync;
}

/* solve_continuous — src/orchestrator.cpp:130-209. */
static int solve_continuous(const tuple_costs_t* tc, double total, int vpp,
                            double dp_sync, double* gpus, double* t_iter) {
  cont_t k;
  k.w0 = 0.0;
  for (int u = 0; u < 3; ++u) {
    k.b[u] = tc->coupling[u] * tc->cfb[u] * tc->q[u];
    k.c[u] = 2.0 * vpp * tc->comm[u];
    k.a[u] = 2.0 * tc->comm[u] / tc->q[u];
    k.w0 += tc->coupling[u] * tc->cfb[u];
    k.floor[u] = tc->floor_gpus[u];
  }
  k.w0 /= vpp;
  k.steady_mult = (double)(tc->microbatches - 1);
  k.dp_sync = dp_sync;
  double hi = 0.0, cmax = 0.0;
  for (int u = 0; u < 3; ++u) {
    hi = port_max(hi, k.b[u] / k.floor[u] + k.c[u]);
    cmax = port_max(cmax, k.c[u]);
  }
  double lo = cmax + 1e-300;
  double g[3];
  if (gpus_at(&k, hi, g) > total) return 0;
  double bad = lo, good = hi;
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (bad + good);
    if (gpus_at(&k, mid, g) <= total) good = mid;
    else bad = mid;
  }
  lo = good;
  double t_lo = lo, t_hi = hi;
  for (int it = 0; it < 200; ++it) {
    const double m1 = t_lo + (t_hi - t_lo) / 3.0;
    const double m2 = t_hi - (t_hi - t_lo) / 3.0;
    if (objective(&k, m1, g) <= objective(&k, m2, g)) t_hi = m2;
    else t_lo = m1;
  }
  const double best = 0.5 * (t_lo + t_hi);
  *t_iter = objective(&k, best, gpus);
  return 1;
}

/* BestTracker key comparison — src/orchestrator.cpp:211-233.  Returns 1
 * when candidate c should replace the incumbent b. */
static int key_less(const dtb_candidate* a, const dtb_candidate* b) {
  const int ga = a->plan.unit[0].tp * a->plan.unit[0].dp * a->plan.unit[0].pp +
                 a->plan.unit[1].tp * a->plan.unit[1].dp * a->plan.unit[1].pp +
                 a->plan.unit[2].tp * a->plan.unit[2].dp * a->plan.unit[2].pp;
  const int gb = b->plan.unit[0].tp * b->plan.unit[0].dp * b->plan.unit[0].pp +
                 b->plan.unit[1].tp * b->plan.unit[1].dp * b->plan.unit[1].pp +
                 b->plan.unit[2].tp * b->plan.unit[2].dp * b->plan.unit[2].pp;
  if (ga != gb) return ga < gb;
  const int c = cmp_tuple(&a->tuple, &b->tuple);
  if (c != 0) return c < 0;
  for (int u = 0; u < 3; ++u)
    if (a->plan.unit[u].pp != b->plan.unit[u].pp)
      return a->plan.unit[u].pp < b->plan.unit[u].pp;
  return 0;
}

int port_offer(int has, dtb_candidate* best, const dtb_candidate* cand) {
  if (!cand->feasible) return has;
  if (has) {
    if (cand->times.t_iter > best->times.t_iter) return has;
    if (cand->times.t_iter == best->times.t_iter && !key_less(cand, best))
      return has;
  }
  *best = *cand;
  return 1;
}

static int cmp_int(const void* a, const void* b) {
  return *(const int*)a - *(const int*)b;
}

/* solve_subproblem — src/orchestrator.cpp:303-378. */
int port_solve_subproblem(const port_cm* cm, const dtb_workload_stats* stats,
                          const dtb_tuple* t, int64_t bs, int vpp,
                          dtb_candidate* out) {
  memset(out, 0, sizeof *out);
  out->tuple = *t;
  /* CandidateResult::plan default-constructs to Plan{} (core.hpp:115-121). */
  for (int u = 0; u < 3; ++u) out->plan.unit[u] = (dtb_parallelism){1, 1, 1};
  out->plan.global_batch = 1;
  out->plan.vpp = 1;
  tuple_costs_t tc;
  TRY(tuple_costs(cm, t, stats, bs, &tc));
  if (!tc.feasible) {
    out->reason = tc.reason;
    return 0;
  }
  const int n = cm->cluster.total_gpus;
  double gpus[3], t_iter;
  if (!solve_continuous(&tc, (double)n, vpp, cm->model.dp_sync_seconds, gpus,
                        &t_iter)) {
    out->reason = DTB_REASON_MEMORY_FLOOR;
    return 0;
  }
  out->cont_x = gpus[0];
  out->cont_y = gpus[1];
  out->cont_z = gpus[2];
  out->cont_t_iter = t_iter;

  int cands[3][6], nc[3];
  const int q_sum = tc.q[0] + tc.q[1] + tc.q[2];
  for (int u = 0; u < 3; ++u) {
    const double cont_pp = gpus[u] / tc.q[u];
    const int pp_max = (n - (q_sum - tc.q[u])) / tc.q[u];
    const int fl = (int)floor(cont_pp), ce = (int)ceil(cont_pp);
    const int raw[6] = {fl - 1, fl, ce, ce + 1, 1, pp_max};
    int k = 0;
    for (int i = 0; i < 6; ++i) {
      if (raw[i] < 1 || raw[i] > pp_max) continue;
      int dup = 0;
      for (int j = 0; j < k; ++j) dup |= cands[u][j] == raw[i];
      if (!dup) cands[u][k++] = raw[i];
    }
    qsort(cands[u], (size_t)k, sizeof(int), cmp_int);
    nc[u] = k;
  }
  int has = 0;
  dtb_candidate best;
  for (int a = 0; a < nc[0]; ++a)
    for (int b = 0; b < nc[1]; ++b)
      for (int c = 0; c < nc[2]; ++c) {
        const long g = (long)tc.q[0] * cands[0][a] + (long)tc.q[1] * cands[1][b] +
                       (long)tc.q[2] * cands[2][c];
        if (g > n) continue;
        dtb_candidate cand;
        memset(&cand, 0, sizeof cand);
        cand.tuple = *t;
        cand.feasible = 1;
        cand.plan = plan_from(t, cands[0][a], cands[1][b], cands[2][c], bs, vpp);
        if (vpp > 1 && tc.microbatches % (cands[0][a] + cands[1][b] + cands[2][c]) != 0)
          continue;
        dtb_memory_report mr;
        port_memory_check(&cand.plan, &cm->model, &cm->cluster, &mr);
        if (!mr.pass) continue;
        TRY(port_predict_times(cm, &cand.plan, stats, &cand.times));
        has = port_offer(has, &best, &cand);
      }
  if (!has) {
    out->reason = DTB_REASON_NO_INTEGER_SPLIT;
    return 0;
  }
  out->feasible = 1;
  out->reason = DTB_REASON_NONE;
  out->plan = best.plan;
  out->times = best.times;
  return 0;
}

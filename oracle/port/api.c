/* ORACLE — `mmport_` C ABI over the restatement (same signatures as
 * include/disttrain_b200.h).  Test infrastructure only. */
#include <stdlib.h>
#include <string.h>

#include "port.h"

#define API(name) mmport_##name

struct dtb_context {
  int device;
};

static int64_t modality(const dtb_samples* s, int64_t i) {
  int64_t t = 0;
  for (int32_t k = s->image_offsets[i]; k < s->image_offsets[i + 1]; ++k)
    t += s->image_tokens[k];
  if (s->audio_offsets)
    for (int32_t k = s->audio_offsets[i]; k < s->audio_offsets[i + 1]; ++k)
      t += s->audio_tokens[k];
  return t;
}

static port_mb* to_mbs(const dtb_microbatches* m) {
  port_mb* v = malloc(sizeof(port_mb) * (size_t)(m->n ? m->n : 1));
  for (int64_t i = 0; i < m->n; ++i)
    v[i] = (port_mb){m->encoder_tokens[i], m->generator_tokens[i], m->sample_count[i]};
  return v;
}

const char* API(last_error)(void) { return port_msg; }
int API(abi_version)(void) { return DTB_ABI_VERSION; }

dtb_status API(context_create)(int32_t device, dtb_context** out) {
  *out = malloc(sizeof(dtb_context));
  (*out)->device = device;
  return DTB_OK;
}
dtb_status API(context_destroy)(dtb_context* ctx) {
  free(ctx);
  return DTB_OK;
}

/* CostProfile::add_row — src/cost_model.cpp:37-60. */
static int add_row(port_cm* cm, const dtb_profile_row* r) {
  const int ti = port_tp_index(r->tp);
  if (ti < 0)
    return port_fail(DTB_ERR_CONFIG, "profile TP size %d is not one of {1,2,4,8}", r->tp);
  if (!(r->fwd_s > 0.0) || (r->has_bwd && !(r->bwd_s > 0.0)))
    return port_fail(DTB_ERR_CONFIG, "profile times must be strictly positive");
  if (r->token_load < 0.0)
    return port_fail(DTB_ERR_CONFIG, "profile token load must be non-negative");
  if (r->module < 0 || r->module > 2)
    return port_fail(DTB_ERR_CONFIG, "bad module index %d", r->module);
  int n = cm->nrows[r->module][ti];
  port_row* rows = realloc(cm->rows[r->module][ti], sizeof(port_row) * (n + 1));
  cm->rows[r->module][ti] = rows;
  const port_row pt = {r->token_load, r->fwd_s, r->has_bwd ? r->bwd_s : 2.0 * r->fwd_s};
  int pos = 0;
  while (pos < n && rows[pos].load < r->token_load) ++pos;
  if (pos < n && rows[pos].load == r->token_load) {
    rows[pos] = pt;
  } else {
    memmove(rows + pos + 1, rows + pos, sizeof(port_row) * (n - pos));
    rows[pos] = pt;
    cm->nrows[r->module][ti] = n + 1;
  }
  cm->nonempty[r->module] = 1;
  return 0;
}

dtb_status API(cost_model_destroy)(port_cm* cm) {
  if (!cm) return DTB_OK;
  for (int u = 0; u < 3; ++u)
    for (int t = 0; t < 4; ++t) free(cm->rows[u][t]);
  free(cm);
  return DTB_OK;
}

dtb_status API(cost_model_create)(dtb_context* ctx, const dtb_model_spec* model,
                                  const dtb_cluster_spec* cluster,
                                  const dtb_costbook* book, port_cm** out) {
  port_cm* cm = calloc(1, sizeof(port_cm));
  cm->model = *model;
  cm->cluster = *cluster;
  cm->eff = book->analytic_efficiency;
  cm->ratio = book->analytic_bwd_fwd_ratio;
  for (int64_t i = 0; i < book->n_rows; ++i) {
    if (add_row(cm, &book->rows[i]) != 0) {
      API(cost_model_destroy)(cm);
      return port_status;
    }
  }
  *out = cm;
  return DTB_OK;
}

dtb_status API(cost_sizes)(dtb_context* ctx, const dtb_samples* s, int64_t* out) {
  for (int64_t i = 0; i < s->n; ++i) out[i] = 2 * modality(s, i);
  return DTB_OK;
}

dtb_status API(unit_times)(dtb_context* ctx, const port_cm* cm, int32_t module,
                           int32_t tp, int64_t n, const double* loads,
                           double* fwd, double* bwd) {
  for (int64_t i = 0; i < n; ++i) {
    if (fwd) TRY(port_unit_forward(cm, module, tp, loads[i], &fwd[i]));
    if (bwd) TRY(port_unit_backward(cm, module, tp, loads[i], &bwd[i]));
  }
  return DTB_OK;
}

dtb_status API(memory_check)(dtb_context* ctx, const port_cm* cm,
                             const dtb_plan* plan, dtb_memory_report* out) {
  port_memory_check(plan, &cm->model, &cm->cluster, out);
  return DTB_OK;
}

dtb_status API(build_stage_times)(dtb_context* ctx, const port_cm* cm,
                                  const dtb_plan* plan,
                                  const dtb_microbatches* m, double* fwd,
                                  double* bwd) {
  port_mb* v = to_mbs(m);
  const int st = port_build_stage_times(cm, plan, v, m->n, fwd, bwd);
  free(v);
  return st;
}

dtb_status API(microbatch_fwd_keys)(dtb_context* ctx, const port_cm* cm,
                                    const dtb_plan* plan,
                                    const dtb_microbatches* m, double* keys) {
  port_mb* v = to_mbs(m);
  const int st = port_fwd_keys(cm, plan, v, m->n, keys);
  free(v);
  return st;
}

/* compute_stats — src/workload.cpp:206-220. */
dtb_status API(compute_stats)(dtb_context* ctx, const dtb_samples* s,
                              int64_t seq_len, dtb_workload_stats* out) {
  out->seq_len = seq_len;
  out->mean_encoder_tokens = out->mean_generator_tokens = 0.0;
  if (s->n == 0) return DTB_OK;
  double enc = 0.0, gen = 0.0;
  for (int64_t i = 0; i < s->n; ++i) {
    const double t = (double)modality(s, i);
    enc += t;
    gen += t;
  }
  out->mean_encoder_tokens = enc / (double)s->n;
  out->mean_generator_tokens = gen / (double)s->n;
  return DTB_OK;
}

dtb_status API(intra_partition)(dtb_context* ctx, const double* sizes,
                                int64_t n, int32_t m, int32_t order,
                                int32_t equal_counts, int32_t* flat,
                                int64_t* offsets) {
  return port_intra_partition(sizes, n, m, order, equal_counts, flat, offsets);
}

dtb_status API(block_group_loads)(dtb_context* ctx, const double* sizes,
                                  const int32_t* order, int64_t n, int32_t m,
                                  double* loads) {
  return port_block_group_loads(sizes, order, n, m, loads);
}

dtb_status API(select_min)(dtb_context* ctx, const double* keys, int64_t nk,
                           const int32_t* pending, int64_t np, int32_t k,
                           int32_t* out) {
  return port_select_min(keys, pending, np, k, out);
}

dtb_status API(select_closest)(dtb_context* ctx, const double* keys,
                               int64_t nk, const int32_t* pending, int64_t np,
                               int32_t k, double target, int32_t* out) {
  return port_select_closest(keys, pending, np, k, target, out);
}

dtb_status API(schedule)(dtb_context* ctx, const double* fwd,
                         const double* bwd, int32_t l, int32_t p, int32_t vpp,
                         int32_t* ev_device, int32_t* ev_mb, int32_t* ev_stage,
                         int32_t* ev_phase, double* ev_start, double* ev_end,
                         double* iteration_time, double* device_busy) {
  port_timeline tl;
  TRY(port_schedule(fwd, bwd, l, p, vpp, &tl));
  for (int64_t i = 0; i < tl.n_events; ++i) {
    const port_event* e = &tl.events[i];
    if (ev_device) ev_device[i] = e->device;
    if (ev_mb) ev_mb[i] = e->mb;
    if (ev_stage) ev_stage[i] = e->stage;
    if (ev_phase) ev_phase[i] = e->phase;
    if (ev_start) ev_start[i] = e->start;
    if (ev_end) ev_end[i] = e->end;
  }
  if (iteration_time) *iteration_time = tl.iteration_time;
  if (device_busy) memcpy(device_busy, tl.busy, sizeof(double) * tl.devices);
  port_timeline_free(&tl);
  return DTB_OK;
}

dtb_status API(get_intervals)(dtb_context* ctx, int64_t n,
                              const int32_t* dev, const int32_t* mb,
                              const int32_t* stage, const int32_t* phase,
                              const double* start, const double* end,
                              int64_t* n_int, double* starts, double* ends,
                              int64_t* fill_off, int32_t* fill_mb) {
  port_event* ev = malloc(sizeof(port_event) * (size_t)(n ? n : 1));
  for (int64_t i = 0; i < n; ++i)
    ev[i] = (port_event){dev[i], mb[i], stage[i], phase[i], start[i], end[i]};
  *n_int = port_get_intervals(ev, n, starts, ends, fill_off, fill_mb);
  free(ev);
  return DTB_OK;
}

dtb_status API(interval_windows)(dtb_context* ctx, const double* fwd,
                                 const double* bwd, int32_t l, int32_t p,
                                 double* volumes) {
  port_timeline tl;
  TRY(port_schedule(fwd, bwd, l, p, 1, &tl));
  double* s = malloc(sizeof(double) * (size_t)2 * l);
  const int64_t k = port_get_intervals(tl.events, tl.n_events, s, s + l, NULL, NULL);
  for (int64_t i = 0; i < k; ++i) volumes[i] = s[l + i] - s[i];
  free(s);
  port_timeline_free(&tl);
  return DTB_OK;
}

dtb_status API(schedule_batch)(dtb_context* ctx, int64_t batch,
                               const double* fwd, const double* bwd, int32_t l,
                               int32_t p, int32_t vpp, double* it,
                               double* busy) {
  const size_t cells = (size_t)l * p;
  for (int64_t b = 0; b < batch; ++b) {
    port_timeline tl;
    TRY(port_schedule(fwd + b * cells, bwd + b * cells, l, p, vpp, &tl));
    it[b] = tl.iteration_time;
    if (busy) memcpy(busy + b * tl.devices, tl.busy, sizeof(double) * tl.devices);
    port_timeline_free(&tl);
  }
  return DTB_OK;
}

/* std::next_permutation over ints (lexicographic successor; 0 at the end). */
static int next_perm(int32_t* a, int n) {
  int i = n - 2;
  while (i >= 0 && a[i] >= a[i + 1]) --i;
  if (i < 0) {
    for (int x = 0, y = n - 1; x < y; ++x, --y) {
      const int32_t t = a[x];
      a[x] = a[y];
      a[y] = t;
    }
    return 0;
  }
  int j = n - 1;
  while (a[j] <= a[i]) --j;
  int32_t t = a[i];
  a[i] = a[j];
  a[j] = t;
  for (int x = i + 1, y = n - 1; x < y; ++x, --y) {
    t = a[x];
    a[x] = a[y];
    a[y] = t;
  }
  return 1;
}

/* tests/test_reorder.cpp:215-239: sim_time of every ordering. */
dtb_status API(exhaustive_order)(dtb_context* ctx, const double* fwd, const double* bwd,
                                 int32_t l, int32_t p, int32_t vpp, double* best_time,
                                 int32_t* best_order, double* all_times) {
  if (l < 1 || l > 12) return port_fail(DTB_ERR_INTERNAL, "exhaustive_order needs 1 <= l <= 12");
  const size_t cells = (size_t)l * p;
  int32_t perm[12];
  double* pf = malloc(sizeof(double) * cells);
  double* pb = malloc(sizeof(double) * cells);
  for (int i = 0; i < l; ++i) perm[i] = i;
  double best = 1e300;
  int64_t k = 0;
  dtb_status st = DTB_OK;
  do {
    for (int i = 0; i < l; ++i)
      for (int s = 0; s < p; ++s) {
        pf[(size_t)i * p + s] = fwd[(size_t)perm[i] * p + s];
        pb[(size_t)i * p + s] = bwd[(size_t)perm[i] * p + s];
      }
    port_timeline tl;
    st = port_schedule(pf, pb, l, p, vpp, &tl);
    if (st != DTB_OK) break;
    const double it = tl.iteration_time;
    port_timeline_free(&tl);
    if (all_times) all_times[k] = it;
    if (it < best) {
      best = it;
      memcpy(best_order, perm, sizeof(int32_t) * l);
    }
    ++k;
  } while (next_perm(perm, l));
  free(pf);
  free(pb);
  if (st != DTB_OK) return st;
  *best_time = best;
  return DTB_OK;
}

dtb_status API(simulate_iteration)(dtb_context* ctx, const port_cm* cm,
                                   const dtb_plan* plan, int32_t n_groups,
                                   const int64_t* goff,
                                   const dtb_microbatches* m, double* t_iter,
                                   double* group_times, int32_t* slowest,
                                   double* slowest_time, double* bubble) {
  port_mb* v = to_mbs(m);
  const int st = port_simulate_iteration(cm, plan, n_groups, goff, v, t_iter,
                                         group_times, slowest, slowest_time,
                                         bubble);
  free(v);
  return st;
}

dtb_status API(inter_reorder)(dtb_context* ctx, const double* fwd,
                              const double* bwd, int32_t l, int32_t p,
                              const double* keys, int32_t vpp, int32_t* out) {
  return port_inter_reorder(fwd, bwd, l, p, keys, vpp, out);
}

dtb_status API(inter_reorder_batch)(dtb_context* ctx, int64_t batch,
                                    const double* fwd, const double* bwd,
                                    int32_t l, int32_t p, const double* keys,
                                    int32_t vpp, int32_t* orders) {
  const size_t cells = (size_t)l * p;
  for (int64_t b = 0; b < batch; ++b)
    TRY(port_inter_reorder(fwd + b * cells, bwd + b * cells, l, p, keys + b * l,
                           vpp, orders + b * l));
  return DTB_OK;
}

dtb_status API(disaggregated_reorder)(dtb_context* ctx, const port_cm* cm,
                                      const dtb_plan* plan,
                                      const dtb_reorder_mode* mode,
                                      const dtb_samples* batch,
                                      dtb_reorder_report* rep) {
  if (batch->n != plan->global_batch)
    return port_fail(DTB_ERR_BATCH_SIZE_MISMATCH,
                     "batch has %lld samples, plan expects %lld",
                     (long long)batch->n, (long long)plan->global_batch);
  const dtb_reorder_mode def = {1, 1, DTB_ASCENDING};
  return port_disaggregated_reorder(cm, plan, mode ? mode : &def, batch, 0, rep);
}

dtb_status API(reorder_stream)(dtb_context* ctx, const port_cm* cm,
                               const dtb_plan* plan,
                               const dtb_reorder_mode* mode,
                               const dtb_samples* s, int64_t n_batches,
                               int32_t* order, double* lb, double* la,
                               double* tb, double* ta, uint8_t* kept) {
  const int64_t bs = plan->global_batch;
  const int dp = plan->unit[DTB_BACKBONE].dp;
  if (n_batches < 0 || s->n != n_batches * bs)
    return port_fail(DTB_ERR_BATCH_SIZE_MISMATCH,
                     "stream has %lld samples, plan expects %lld batches of %lld",
                     (long long)s->n, (long long)n_batches, (long long)bs);
  const dtb_reorder_mode def = {1, 1, DTB_ASCENDING};
  for (int64_t b = 0; b < n_batches; ++b) {
    dtb_reorder_report rep = {order + b * bs, lb + b * dp, la + b * dp, 0, 0};
    TRY(port_disaggregated_reorder(cm, plan, mode ? mode : &def, s, b * bs, &rep));
    tb[b] = rep.t_iter_before;
    ta[b] = rep.t_iter_after;
    if (kept) kept[b] = 0xff; /* not derivable from the report */
  }
  return DTB_OK;
}

dtb_status API(predict_times)(dtb_context* ctx, const port_cm* cm,
                              const dtb_workload_stats* stats,
                              const dtb_plan* plans, int64_t n,
                              dtb_predicted_times* out) {
  for (int64_t i = 0; i < n; ++i)
    TRY(port_predict_times(cm, &plans[i], stats, &out[i]));
  return DTB_OK;
}

dtb_status API(enumerate_parallelism)(dtb_context* ctx,
                                      const dtb_cluster_spec* c, int64_t bs,
                                      int64_t* count, dtb_tuple* tuples,
                                      int64_t capacity) {
  dtb_tuple* v;
  *count = port_enumerate(c, bs, &v);
  if (tuples)
    memcpy(tuples, v, sizeof(dtb_tuple) * (size_t)(capacity < *count ? capacity : *count));
  free(v);
  return DTB_OK;
}

dtb_status API(solve_subproblem)(dtb_context* ctx, const port_cm* cm,
                                 const dtb_workload_stats* stats,
                                 const dtb_tuple* tuples, int64_t n,
                                 int64_t bs, int32_t vpp, dtb_candidate* out) {
  for (int64_t i = 0; i < n; ++i)
    TRY(port_solve_subproblem(cm, stats, &tuples[i], bs, vpp, &out[i]));
  return DTB_OK;
}

int port_offer(int has, dtb_candidate* best, const dtb_candidate* cand);

static dtb_plan plan_of(const dtb_tuple* t, int pe, int pl, int pg, int64_t bs, int vpp) {
  dtb_plan p;
  p.unit[0].tp = t->tp_me;
  p.unit[0].dp = t->dp_me;
  p.unit[0].pp = pe;
  p.unit[1].tp = t->tp_lm;
  p.unit[1].dp = t->dp_lm;
  p.unit[1].pp = pl;
  p.unit[2].tp = t->tp_mg;
  p.unit[2].dp = t->dp_mg;
  p.unit[2].pp = pg;
  p.vpp = vpp;
  p.global_batch = bs;
  return p;
}

/* brute_force_oracle — src/orchestrator.cpp:433-491. */
dtb_status API(brute_force_oracle)(dtb_context* ctx, const port_cm* cm,
                                   const dtb_workload_stats* stats, int64_t bs, int32_t vpp,
                                   int32_t gpu_cap, dtb_orchestration_result* res) {
  const int n = cm->cluster.total_gpus;
  if (n > gpu_cap)
    return port_fail(DTB_ERR_CAP_EXCEEDED, "exhaustive search capped at %d GPUs, got %d",
                     gpu_cap, n);
  dtb_tuple* v;
  const int64_t nt = port_enumerate(&cm->cluster, bs, &v);
  int has = 0;
  int64_t evaluated = 0;
  dtb_candidate best, c;
  for (int64_t i = 0; i < nt; ++i) {
    const dtb_tuple* t = &v[i];
    const int q_me = t->tp_me * t->dp_me, q_lm = t->tp_lm * t->dp_lm, q_mg = t->tp_mg * t->dp_mg;
    for (int pe = 1; q_me * pe + q_lm + q_mg <= n; ++pe)
      for (int pl = 1; q_me * pe + q_lm * pl + q_mg <= n; ++pl)
        for (int pg = 1; q_me * pe + q_lm * pl + q_mg * pg <= n; ++pg) {
          const dtb_plan plan = plan_of(t, pe, pl, pg, bs, vpp);
          if (vpp > 1 && (bs / t->dp_lm) % (pe + pl + pg) != 0) continue;
          dtb_memory_report mem;
          port_memory_check(&plan, &cm->model, &cm->cluster, &mem);
          if (!mem.pass) continue;
          memset(&c, 0, sizeof c);
          c.tuple = *t;
          c.feasible = 1;
          c.plan = plan;
          if (port_predict_times(cm, &plan, stats, &c.times) != 0) {
            free(v);
            return port_status;
          }
          ++evaluated;
          has = port_offer(has, &best, &c);
        }
  }
  free(v);
  res->candidates_evaluated = evaluated;
  res->solve_seconds = 0.0;
  if (!has) return port_fail(DTB_ERR_INFEASIBLE, "no feasible plan in the exhaustive search");
  res->best = best.plan;
  res->times = best.times;
  return DTB_OK;
}

/* rigid_baseline — src/orchestrator.cpp:407-431 (validate_plan reduces to
 * the memory check here: every other rule holds by construction). */
dtb_status API(rigid_baseline)(dtb_context* ctx, const port_cm* cm,
                               const dtb_workload_stats* stats, int64_t bs, int32_t vpp,
                               dtb_plan* out) {
  static const int tps[4] = {1, 2, 4, 8};
  int64_t divs[4096];
  int64_t nd = 0;
  for (int64_t d = 1; d <= bs && nd < 4096; ++d)
    if (bs % d == 0) divs[nd++] = d;
  int has = 0;
  dtb_candidate best, c;
  for (int a = 0; a < 4; ++a)
    for (int64_t j = 0; j < nd; ++j) {
      const long q = (long)tps[a] * divs[j];
      const int pl = (int)((cm->cluster.total_gpus - 2 * q) / q);
      if (pl < 1) continue;
      dtb_tuple t = {tps[a], (int32_t)divs[j], tps[a], (int32_t)divs[j], tps[a], (int32_t)divs[j]};
      const dtb_plan plan = plan_of(&t, 1, pl, 1, bs, vpp);
      if (vpp > 1 && (bs / divs[j]) % (pl + 2) != 0) continue;
      dtb_memory_report mem;
      port_memory_check(&plan, &cm->model, &cm->cluster, &mem);
      if (!mem.pass) continue;
      memset(&c, 0, sizeof c);
      c.tuple = t;
      c.feasible = 1;
      c.plan = plan;
      if (port_predict_times(cm, &plan, stats, &c.times) != 0) return port_status;
      has = port_offer(has, &best, &c);
    }
  if (!has) return port_fail(DTB_ERR_INFEASIBLE, "no feasible rigid configuration");
  *out = best.plan;
  return DTB_OK;
}

/* model_orchestration — src/orchestrator.cpp:380-405. */
dtb_status API(model_orchestration)(dtb_context* ctx, const port_cm* cm,
                                    const dtb_workload_stats* stats,
                                    int64_t bs, int32_t vpp,
                                    dtb_orchestration_result* res,
                                    dtb_candidate* cands, int64_t capacity) {
  dtb_tuple* v;
  const int64_t n = port_enumerate(&cm->cluster, bs, &v);
  int has = 0;
  dtb_candidate best, c;
  for (int64_t i = 0; i < n; ++i) {
    if (port_solve_subproblem(cm, stats, &v[i], bs, vpp, &c) != 0) {
      free(v);
      return port_status;
    }
    if (cands && i < capacity) cands[i] = c;
    has = port_offer(has, &best, &c);
  }
  free(v);
  res->candidates_evaluated = n;
  res->solve_seconds = 0.0;
  if (!has)
    return port_fail(DTB_ERR_INFEASIBLE, "no feasible plan for this model and cluster");
  res->best = best.plan;
  res->times = best.times;
  return DTB_OK;
}

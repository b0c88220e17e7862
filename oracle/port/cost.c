/* ORACLE restatement of the cost model: src/cost_model.cpp, src/core.cpp. */
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "port.h"

_Thread_local int port_status = 0;
_Thread_local char port_msg[512];

int port_fail(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(port_msg, sizeof port_msg, fmt, ap);
  va_end(ap);
  port_status = status;
  return status;
}

static const char* kind_name(int k) {
  return k == 0 ? "encoder" : k == 1 ? "backbone" : "generator";
}

int port_tp_index(int tp) {
  switch (tp) {
    case 1: return 0;
    case 2: return 1;
    case 4: return 2;
    case 8: return 3;
  }
  return -1;
}

/* std::max / std::min: return the first argument unless the second compares
 * strictly greater / smaller. */
double port_max(double a, double b) { return a < b ? b : a; }
double port_min(double a, double b) { return b < a ? b : a; }

/* ArchDesc::param_count — src/core.cpp:40-49. */
double port_param_count(const dtb_arch* a) {
  const double h = (double)a->hidden;
  const double f = (double)a->ffn_hidden;
  const double kv = a->heads > 0 ? (double)a->groups / (double)a->heads : 1.0;
  const double attn = h * h * (2.0 + 2.0 * kv);
  const double ffn = 3.0 * h * f;
  return (double)a->layers * (attn + ffn);
}

/* interpolate — src/cost_model.cpp:79-106; which = 0 fwd, 1 bwd. */
static double interpolate(const port_row* rows, int n, double x, int which) {
#define VAL(r) (which ? (r).bwd : (r).fwd)
  if (x <= rows[0].load) return VAL(rows[0]);
  if (x >= rows[n - 1].load) return VAL(rows[n - 1]);
  int hi = 0;
  while (hi < n && rows[hi].load < x) ++hi; /* lower_bound */
  if (rows[hi].load == x) return VAL(rows[hi]);
  const int lo = hi - 1;
  const double t = (x - rows[lo].load) / (rows[hi].load - rows[lo].load);
  return VAL(rows[lo]) + t * (VAL(rows[hi]) - VAL(rows[lo]));
#undef VAL
}

static int rows_for(const port_cm* cm, int kind, int tp, const port_row** rows,
                    int* n) {
  const int ti = port_tp_index(tp);
  if (ti < 0 || cm->nrows[kind][ti] == 0) {
    return port_fail(DTB_ERR_EMPTY_PROFILE, "no profile rows for tp=%d", tp);
  }
  *rows = cm->rows[kind][ti];
  *n = cm->nrows[kind][ti];
  return 0;
}

/* CostModel::analytic_forward — src/cost_model.cpp:240-253. */
static int analytic_forward(const port_cm* cm, int kind, double load,
                            double* out) {
  if (!(cm->eff > 0.0) || !(cm->cluster.peak_flops > 0.0)) {
    return port_fail(DTB_ERR_EMPTY_PROFILE,
                     "no profile rows for module '%s' and no usable analytic "
                     "fallback",
                     kind_name(kind));
  }
  const double flops =
      2.0 * port_param_count(&cm->model.unit[kind].arch) * load;
  *out = flops / (cm->cluster.peak_flops * cm->eff);
  return 0;
}

/* CostModel::unit_forward_time — src/cost_model.cpp:255-264. */
int port_unit_forward(const port_cm* cm, int kind, int tp, double load,
                      double* out) {
  if (port_tp_index(tp) < 0) {
    return port_fail(DTB_ERR_INTERNAL, "tp size %d not allowed", tp);
  }
  if (load < 0.0) return port_fail(DTB_ERR_INTERNAL, "negative token load");
  if (!cm->nonempty[kind]) return analytic_forward(cm, kind, load, out);
  const port_row* rows = NULL;
  int n = 0;
  TRY(rows_for(cm, kind, tp, &rows, &n));
  *out = interpolate(rows, n, load, 0);
  return 0;
}

/* CostModel::unit_backward_time — src/cost_model.cpp:266-276. */
int port_unit_backward(const port_cm* cm, int kind, int tp, double load,
                       double* out) {
  double bwd;
  if (!cm->nonempty[kind]) {
    double f;
    TRY(analytic_forward(cm, kind, load, &f));
    bwd = cm->ratio * f;
  } else {
    const port_row* rows = NULL;
    int n = 0;
    TRY(rows_for(cm, kind, tp, &rows, &n));
    bwd = interpolate(rows, n, load, 1);
  }
  const double factor =
      cm->model.unit[kind].frozen ? cm->model.frozen_backward_factor : 1.0;
  *out = bwd * factor;
  return 0;
}

/* pp_boundary_seconds — src/cost_model.cpp:191-199. */
double port_pp_boundary_seconds(const dtb_plan* plan, int unit,
                                const dtb_cluster_spec* c, double bytes) {
  const dtb_parallelism* pc = &plan->unit[unit];
  const int intra = 2 * pc->tp * pc->dp <= c->gpus_per_node;
  const double bw = intra ? c->intra_node_bw : c->inter_node_bw;
  return bytes / bw;
}

static double coupling_of(const dtb_plan* plan, int unit) {
  return unit == DTB_BACKBONE
             ? 1.0
             : (double)plan->unit[DTB_BACKBONE].dp / (double)plan->unit[unit].dp;
}

/* CostModel::boundary_bytes — src/cost_model.cpp:322-332. */
double port_boundary_bytes(const port_cm* cm, int unit, const dtb_plan* plan,
                           double tokens) {
  const double coupling = coupling_of(plan, unit);
  const double hidden = (double)cm->model.unit[unit].arch.hidden;
  return 2.0 * hidden * tokens * coupling;
}

/* memory_check — src/cost_model.cpp:167-189. */
void port_memory_check(const dtb_plan* plan, const dtb_model_spec* model,
                       const dtb_cluster_spec* cluster,
                       dtb_memory_report* out) {
  out->capacity_bytes = cluster->gpu_mem_bytes;
  out->pass = 1;
  const double dp_lm = (double)plan->unit[DTB_BACKBONE].dp;
  for (int u = 0; u < 3; ++u) {
    const dtb_parallelism* pc = &plan->unit[u];
    const dtb_module_memory* mem = &model->unit[u].mem;
    const double gpus = (double)(pc->tp * pc->dp * pc->pp);
    const double bytes = ((double)pc->dp * mem->param_grad_bytes +
                          mem->optimizer_bytes +
                          dp_lm * mem->activation_bytes_per_mb * pc->pp) /
                         gpus;
    out->bytes_per_gpu[u] = bytes;
    out->fits[u] = bytes <= cluster->gpu_mem_bytes;
    out->pass = out->pass && out->fits[u];
  }
}

/* Microbatch::mean_*_tokens — include/core.hpp:183-192. */
double port_mb_mean_enc(const port_mb* mb) {
  return mb->count == 0 ? 0.0 : (double)mb->enc / (double)mb->count;
}
double port_mb_mean_gen(const port_mb* mb) {
  return mb->count == 0 ? 0.0 : (double)mb->gen / (double)mb->count;
}

/* CostModel::token_load(kind, mb) — src/cost_model.cpp:284-295. */
static double token_load_mb(const port_cm* cm, int kind, const port_mb* mb) {
  if (kind == DTB_ENCODER) return port_mb_mean_enc(mb);
  if (kind == DTB_GENERATOR) return port_mb_mean_gen(mb);
  return (double)cm->model.seq_len;
}

/* CostModel::stage_time — src/cost_model.cpp:308-320. */
static int stage_time(const port_cm* cm, int kind, const dtb_plan* plan,
                      const port_mb* mb, int phase, double* out) {
  const dtb_parallelism* pc = &plan->unit[kind];
  const double coupling = coupling_of(plan, kind);
  const double load = token_load_mb(cm, kind, mb);
  double whole;
  if (phase == DTB_FORWARD) {
    TRY(port_unit_forward(cm, kind, pc->tp, load, &whole));
  } else {
    TRY(port_unit_backward(cm, kind, pc->tp, load, &whole));
  }
  *out = coupling * whole / (double)pc->pp;
  return 0;
}

/* CostModel::build_stage_times — src/cost_model.cpp:334-362. */
int port_build_stage_times(const port_cm* cm, const dtb_plan* plan,
                           const port_mb* mbs, int64_t l, double* fwd,
                           double* bwd) {
  const int p = (plan->unit[0].pp + plan->unit[1].pp + plan->unit[2].pp) *
                plan->vpp;
  for (int64_t i = 0; i < l; ++i) {
    int stage = 0;
    for (int kind = 0; kind < 3; ++kind) {
      const dtb_parallelism* pc = &plan->unit[kind];
      const double comm = port_pp_boundary_seconds(
          plan, kind, &cm->cluster,
          port_boundary_bytes(cm, kind, plan, token_load_mb(cm, kind, &mbs[i])));
      double sf, sb;
      TRY(stage_time(cm, kind, plan, &mbs[i], DTB_FORWARD, &sf));
      TRY(stage_time(cm, kind, plan, &mbs[i], DTB_BACKWARD, &sb));
      const double f = sf / plan->vpp + comm;
      const double b = sb / plan->vpp + comm;
      for (int k = 0; k < pc->pp * plan->vpp; ++k, ++stage) {
        fwd[i * p + stage] = f;
        bwd[i * p + stage] = b;
      }
    }
  }
  return 0;
}

/* microbatch_fwd_keys — src/reorder.cpp:300-317. */
int port_fwd_keys(const port_cm* cm, const dtb_plan* plan, const port_mb* mbs,
                  int64_t l, double* keys) {
  const double k_me = (double)plan->unit[DTB_BACKBONE].dp / plan->unit[DTB_ENCODER].dp;
  const double k_mg = (double)plan->unit[DTB_BACKBONE].dp / plan->unit[DTB_GENERATOR].dp;
  for (int64_t i = 0; i < l; ++i) {
    double enc, gen;
    TRY(port_unit_forward(cm, DTB_ENCODER, plan->unit[DTB_ENCODER].tp,
                          port_mb_mean_enc(&mbs[i]), &enc));
    TRY(port_unit_forward(cm, DTB_GENERATOR, plan->unit[DTB_GENERATOR].tp,
                          port_mb_mean_gen(&mbs[i]), &gen));
    keys[i] = k_me * enc + k_mg * gen;
  }
  return 0;
}

// Internal shared definitions for the sm_100a implementation of the
// DistTrain reorder + orchestration hot path.  Device functions here restate
// the reference cost model (proj/core/src/cost_model.cpp) with the SAME
// IEEE operation order so every value is bit-identical to the CPU reference
// (the library is compiled with -fmad=false; no fast-math).
#pragma once

#include <cstdio>

#include <cstdint>
#include <cuda_runtime.h>

#include "disttrain_b200.h"

namespace dtb {

// Debug bounds checks (the pool has no compute-sanitizer): built with
// DTB_DEFINES=DTB_DEBUG_CHECKS, every DTB_CHECK traps the kernel when its
// condition fails — the GPU suite run against that build then fails loudly
// (tools/gpu_run_checks.sh).  Compiled out otherwise.
#ifdef DTB_DEBUG_CHECKS
#define DTB_CHECK(cond)                                                         \
  do {                                                                          \
    if (!(cond)) {                                                              \
      printf("DTB_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond,        \
             __FILE__, __LINE__, static_cast<int>(blockIdx.x),                  \
             static_cast<int>(threadIdx.x));                                    \
      __trap();                                                                 \
    }                                                                           \
  } while (0)
#else
#define DTB_CHECK(cond) \
  do {                  \
  } while (0)
#endif


constexpr int kFull = 0xffffffff;

// ------------------------------------------------------------------ errors
// First device-side failure wins (atomicCAS on `code`).  The host maps the
// record onto dtb_status + the reference's message text.
enum DevErrCode : int {
  E_NONE = 0,
  E_EMPTY_TP = 1,        // EmptyProfileError "no profile rows for tp=%d"
  E_ANALYTIC = 2,        // EmptyProfileError "no profile rows for module ..."
  E_TP_NOT_ALLOWED = 3,  // InternalError "tp size %d not allowed"
  E_NEG_LOAD = 4,        // InternalError "negative token load"
  E_BAD_TIMES = 5,       // InternalError "bad stage times: <a>"
  E_DEADLOCK = 6,        // InternalError (schedule deadlock)
  E_COST_RANGE = 7,      // InvalidArgument: sample cost exceeds the kernel's key width
  E_NO_MICROBATCH = 8,   // InternalError "plan yields no microbatches per iteration"
};

struct DevErr {
  int code;  // -1: an ordered failure is recorded in `ordered`
  int a;
  int b;
  int pad;
  // min over (evaluation-order key << 8 | code): the failure the sequential
  // reference would have raised first.  ~0 = none.
  unsigned long long ordered;
};

__device__ __forceinline__ void dev_fail_ordered(DevErr* e, unsigned long long order,
                                                 int code) {
  atomicMin(&e->ordered, (order << 8) | static_cast<unsigned long long>(code));
  atomicCAS(&e->code, 0, -1);
}

__device__ __forceinline__ void dev_fail(DevErr* e, int code, int a = 0,
                                         int b = 0) {
  if (atomicCAS(&e->code, 0, code) == 0) {
    e->a = a;
    e->b = b;
  }
}

// std::max / std::min semantics (first argument unless the second compares
// strictly greater / smaller) — never fmax/fmin, whose NaN rules differ.
__host__ __device__ __forceinline__ double smax(double a, double b) {
  return a < b ? b : a;
}
__host__ __device__ __forceinline__ double smin(double a, double b) {
  return b < a ? b : a;
}

// Division by a runtime-invariant divisor 1 <= d < 2^31 for 0 <= n < 2^31
// with one mul-hi (round-up method): q = (umulhi(n, mul) + n) >> shift.
struct FastDiv {
  unsigned d, mul, shift;
  __host__ __device__ static FastDiv make(unsigned d) {
    FastDiv f;
    f.d = d;
    f.shift = 0;
    while ((1u << f.shift) < d) ++f.shift;
    f.mul = static_cast<unsigned>(((1ull << 32) * ((1ull << f.shift) - d)) / d + 1);
    return f;
  }
  __device__ __forceinline__ unsigned div(unsigned n) const {
    const unsigned t = __umulhi(n, mul);
    return (t + n) >> shift;
  }
  __device__ __forceinline__ unsigned mod(unsigned n) const { return n - div(n) * d; }
};

__host__ __device__ __forceinline__ int tp_index(int tp) {
  return tp == 1 ? 0 : tp == 2 ? 1 : tp == 4 ? 2 : tp == 8 ? 3 : -1;
}

// -------------------------------------------------------------- cost model
// Flattened CostBook (cost_model.hpp:72-83) + the model/cluster scalars the
// hot path reads.  Rows for (module u, tp index t) live at
// [off[u][t], off[u][t] + cnt[u][t]) of load/fwd/bwd, sorted by load, with
// bwd already resolved to "measured or 2 x fwd" (cost_model.cpp:117-121).
struct DevCM {
  const double* load;
  const double* fwd;
  const double* bwd;
  int off[3][4];
  int cnt[3][4];
  int nonempty[3];
  int analytic_ok;           // efficiency > 0 && peak_flops > 0
  double analytic_denom;     // peak_flops * efficiency
  double analytic_ratio;     // bwd_fwd_ratio
  double param_count[3];     // ArchDesc::param_count (host, same op order)
  double hidden[3];
  double bwd_factor[3];      // ModelSpec::backward_factor
  double seq_len;            // static_cast<double>(seq_len)
  double dp_sync;
  double mem_pg[3], mem_opt[3], mem_act[3];
  dtb_cluster_spec cluster;
};

// interpolate (cost_model.cpp:79-106) over rows [0, n).
__device__ __forceinline__ double dev_interp(const double* xs, const double* ys,
                                             int n, double x) {
  if (x <= xs[0]) return ys[0];
  if (x >= xs[n - 1]) return ys[n - 1];
  int lo = 0, hi = n;  // lower_bound: first xs[i] >= x
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (xs[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  if (xs[lo] == x) return ys[lo];
  const int a = lo - 1;
  const double t = (x - xs[a]) / (xs[lo] - xs[a]);
  return ys[a] + t * (ys[lo] - ys[a]);
}

// CostModel::unit_forward_time (cost_model.cpp:255-264).  Returns an
// E_* code (0 on success).
__device__ __forceinline__ int dev_unit_fwd(const DevCM& cm, int kind, int tp,
                                            double load, double* out) {
  const int ti = tp_index(tp);
  if (ti < 0) return E_TP_NOT_ALLOWED;
  if (load < 0.0) return E_NEG_LOAD;
  if (!cm.nonempty[kind]) {
    if (!cm.analytic_ok) return E_ANALYTIC;
    const double flops = 2.0 * cm.param_count[kind] * load;
    *out = flops / cm.analytic_denom;
    return 0;
  }
  const int n = cm.cnt[kind][ti];
  if (n == 0) return E_EMPTY_TP;
  const int o = cm.off[kind][ti];
  *out = dev_interp(cm.load + o, cm.fwd + o, n, load);
  return 0;
}

// CostModel::unit_backward_time (cost_model.cpp:266-276).
__device__ __forceinline__ int dev_unit_bwd(const DevCM& cm, int kind, int tp,
                                            double load, double* out) {
  double bwd;
  if (!cm.nonempty[kind]) {
    if (!cm.analytic_ok) return E_ANALYTIC;
    const double flops = 2.0 * cm.param_count[kind] * load;
    bwd = cm.analytic_ratio * (flops / cm.analytic_denom);
  } else {
    const int ti = tp_index(tp);
    const int n = ti < 0 ? 0 : cm.cnt[kind][ti];
    if (n == 0) return E_EMPTY_TP;
    const int o = cm.off[kind][ti];
    bwd = dev_interp(cm.load + o, cm.bwd + o, n, load);
  }
  *out = bwd * cm.bwd_factor[kind];
  return 0;
}

__host__ __device__ __forceinline__ double coupling_of(const dtb_plan& p,
                                                       int unit) {
  return unit == DTB_BACKBONE
             ? 1.0
             : static_cast<double>(p.unit[DTB_BACKBONE].dp) /
                   static_cast<double>(p.unit[unit].dp);
}

// pp_boundary_seconds (cost_model.cpp:191-199) of boundary_bytes
// (cost_model.cpp:322-332).
__device__ __forceinline__ double dev_comm(const DevCM& cm, const dtb_plan& p,
                                           int unit, double tokens) {
  const double bytes = 2.0 * cm.hidden[unit] * tokens * coupling_of(p, unit);
  const dtb_parallelism& pc = p.unit[unit];
  const bool intra = 2 * pc.tp * pc.dp <= cm.cluster.gpus_per_node;
  return bytes / (intra ? cm.cluster.intra_node_bw : cm.cluster.inter_node_bw);
}

// Token load of a unit for a microbatch (cost_model.cpp:284-295).
__device__ __forceinline__ double mb_load(const DevCM& cm, int unit,
                                          double mean_enc, double mean_gen) {
  return unit == DTB_ENCODER ? mean_enc
         : unit == DTB_GENERATOR ? mean_gen
                                 : cm.seq_len;
}

// The build_stage_times entries (cost_model.cpp:334-362) of ONE unit at a
// token load: f = stage_time/vpp + comm, b likewise, where stage_time =
// coupling * whole / pp (cost_model.cpp:308-320).
__device__ __forceinline__ int dev_unit_stage(const DevCM& cm, const dtb_plan& p, int u,
                                              double load, bool want_f, bool want_b,
                                              double* f, double* b) {
  const dtb_parallelism& pc = p.unit[u];
  const double comm = dev_comm(cm, p, u, load);
  const double coupling = coupling_of(p, u);
  double wf = 0.0, wb = 0.0;
  int e = dev_unit_fwd(cm, u, pc.tp, load, &wf);
  if (e) return e;
  if (want_b) {
    e = dev_unit_bwd(cm, u, pc.tp, load, &wb);
    if (e) return e;
  }
  if (want_f) *f = coupling * wf / static_cast<double>(pc.pp) / p.vpp + comm;
  if (want_b) *b = coupling * wb / static_cast<double>(pc.pp) / p.vpp + comm;
  return 0;
}

// build_stage_times entries of one unit with every microbatch-independent
// quantity hoisted: the plan/profile constants are read once per thread,
// the interpolation parameter t is shared between the forward and backward
// columns (the reference computes the same t twice from the same inputs),
// and divisions by exactly 1.0 (pp == 1, vpp == 1, one sample per
// microbatch) are skipped since x / 1.0 == x in IEEE arithmetic.
struct UnitEval {
  const double* xs;
  const double* yf;
  const double* yb;
  int n;            // profile rows at the unit's TP (0: analytic)
  int analytic;
  double two_pc;    // 2.0 * param_count (analytic)
  double denom;     // peak * efficiency
  double ratio;     // analytic bwd/fwd
  double bfac;      // backward factor
  double two_hidden;
  double coupling;
  double bw;
  double pp;
  double vpp;
  bool pp1, vpp1;

  __device__ __forceinline__ void init(const DevCM& cm, const dtb_plan& p, int u) {
    const dtb_parallelism& pc = p.unit[u];
    const int ti = tp_index(pc.tp);
    analytic = !cm.nonempty[u];
    n = (analytic || ti < 0) ? 0 : cm.cnt[u][ti];
    const int o = (analytic || ti < 0) ? 0 : cm.off[u][ti];
    xs = cm.load + o;
    yf = cm.fwd + o;
    yb = cm.bwd + o;
    two_pc = 2.0 * cm.param_count[u];
    denom = cm.analytic_denom;
    ratio = cm.analytic_ratio;
    bfac = cm.bwd_factor[u];
    two_hidden = 2.0 * cm.hidden[u];
    coupling = coupling_of(p, u);
    const bool intra = 2 * pc.tp * pc.dp <= cm.cluster.gpus_per_node;
    bw = intra ? cm.cluster.intra_node_bw : cm.cluster.inter_node_bw;
    pp = static_cast<double>(pc.pp);
    vpp = static_cast<double>(p.vpp);
    pp1 = pc.pp == 1;
    vpp1 = p.vpp == 1;
  }

  // (f, b) of build_stage_times at token load x (host-validated book).
  __device__ __forceinline__ void eval(double x, double* f, double* b) const {
    const double comm = two_hidden * x * coupling / bw;
    double wf, wb;
    if (analytic) {
      wf = two_pc * x / denom;
      wb = ratio * wf;
    } else if (x <= xs[0]) {
      wf = yf[0];
      wb = yb[0];
    } else if (x >= xs[n - 1]) {
      wf = yf[n - 1];
      wb = yb[n - 1];
    } else {
      int lo = 0, hi = n;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (xs[mid] < x) lo = mid + 1;
        else hi = mid;
      }
      if (xs[lo] == x) {
        wf = yf[lo];
        wb = yb[lo];
      } else {
        const int a = lo - 1;
        const double t = (x - xs[a]) / (xs[lo] - xs[a]);
        wf = yf[a] + t * (yf[lo] - yf[a]);
        wb = yb[a] + t * (yb[lo] - yb[a]);
      }
    }
    wb = wb * bfac;
    double sf = coupling * wf, sb = coupling * wb;
    if (!pp1) {
      sf = sf / pp;
      sb = sb / pp;
    }
    if (!vpp1) {
      sf = sf / vpp;
      sb = sb / vpp;
    }
    *f = sf + comm;
    *b = sb + comm;
  }
};

// One 32-byte cost-table row in a single 256-bit load (sm_100: LDG.256).
__device__ __forceinline__ double4 ld_row(const double4* p) {
  double4 r;
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
      : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w)
      : "l"(p));
  return r;
}

__device__ __forceinline__ double mb_mean_fast(long long tokens, int count) {
  return count == 1   ? static_cast<double>(tokens)
         : count == 0 ? 0.0
                      : static_cast<double>(tokens) / static_cast<double>(count);
}

// One microbatch row of build_stage_times (cost_model.cpp:334-362): the
// per-unit forward/backward entry shared by all of a unit's stages.
struct StageRow {
  double f[3];
  double b[3];
};

__device__ __forceinline__ int dev_stage_row(const DevCM& cm, const dtb_plan& p,
                                             double mean_enc, double mean_gen,
                                             StageRow* row) {
  for (int u = 0; u < 3; ++u) {
    const dtb_parallelism& pc = p.unit[u];
    const double load = mb_load(cm, u, mean_enc, mean_gen);
    const double comm = dev_comm(cm, p, u, load);
    const double coupling = coupling_of(p, u);
    double wf, wb;
    int e = dev_unit_fwd(cm, u, pc.tp, load, &wf);
    if (e) return e;
    e = dev_unit_bwd(cm, u, pc.tp, load, &wb);
    if (e) return e;
    const double sf = coupling * wf / static_cast<double>(pc.pp);
    const double sb = coupling * wb / static_cast<double>(pc.pp);
    row->f[u] = sf / p.vpp + comm;
    row->b[u] = sb / p.vpp + comm;
  }
  return 0;
}

// microbatch_fwd_keys (reorder.cpp:300-317) for one microbatch.
__device__ __forceinline__ int dev_fwd_key(const DevCM& cm, const dtb_plan& p,
                                           double mean_enc, double mean_gen,
                                           double* key) {
  const double k_me = static_cast<double>(p.unit[DTB_BACKBONE].dp) /
                      static_cast<double>(p.unit[DTB_ENCODER].dp);
  const double k_mg = static_cast<double>(p.unit[DTB_BACKBONE].dp) /
                      static_cast<double>(p.unit[DTB_GENERATOR].dp);
  double enc, gen;
  int e = dev_unit_fwd(cm, DTB_ENCODER, p.unit[DTB_ENCODER].tp, mean_enc, &enc);
  if (e) return e;
  e = dev_unit_fwd(cm, DTB_GENERATOR, p.unit[DTB_GENERATOR].tp, mean_gen, &gen);
  if (e) return e;
  *key = k_me * enc + k_mg * gen;
  return 0;
}

// Microbatch::mean_*_tokens (core.hpp:183-192).
__host__ __device__ __forceinline__ double mb_mean(int64_t tokens, int count) {
  return count == 0 ? 0.0
                    : static_cast<double>(tokens) / static_cast<double>(count);
}

__host__ __device__ __forceinline__ int plan_stages(const dtb_plan& p) {
  return (p.unit[0].pp + p.unit[1].pp + p.unit[2].pp) * p.vpp;
}

// Global stage -> unit map of build_stage_times (stages are encoder | backbone
// | generator, each pp * vpp long).
__host__ __device__ __forceinline__ int stage_unit(const dtb_plan& p, int s) {
  const int e = p.unit[0].pp * p.vpp;
  const int b = e + p.unit[1].pp * p.vpp;
  return s < e ? 0 : s < b ? 1 : 2;
}

}  // namespace dtb

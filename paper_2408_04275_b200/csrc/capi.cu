// C-ABI layer of libdisttrain_b200.so (include/disttrain_b200.h).
//
// Host code here only validates inputs (in the reference's order, with the
// reference's messages), stages buffers and launches kernels; every value of
// the hot path is computed on the device.  Host-pointer entry points copy in,
// run on the context stream and synchronise; `_dev` entry points enqueue on
// the caller's stream.
#include <algorithm>
#include <array>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "jsonl.cuh"
#include "kernels.cuh"

using namespace dtb;

namespace dtb {
size_t enumerate_scratch(long long bs);
}

// ------------------------------------------------------------------ errors
namespace {
thread_local std::string g_err;

dtb_status fail(dtb_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

const char* kind_name(int k) {
  return k == 0 ? "encoder" : k == 1 ? "backbone" : "generator";
}

#define CU(expr)                                                          \
  do {                                                                    \
    cudaError_t _e = (expr);                                              \
    if (_e != cudaSuccess)                                                \
      return fail(DTB_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(_e)); \
  } while (0)

#define TRY(expr)                      \
  do {                                 \
    dtb_status _s = (expr);            \
    if (_s != DTB_OK) return _s;       \
  } while (0)

}  // namespace

struct dtb_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_in = nullptr, copy_out = nullptr;  // host-buffer pipelines (lazy)
  cudaStream_t side = nullptr;  // partition kernel next to the simulations
  cudaStream_t xchg = nullptr;  // peer exchange of the final order
  DevErr* err = nullptr;  // device
  // warning log (dtb_warnings_enable): the strings the reference's CostModel
  // appends to its sink, in the reference's query order
  bool warn_on = false;
  std::vector<std::string> warnings;
};

struct dtb_peer_group {
  int device = 0, rank = 0, world = 1;
  int64_t n_samples = 0;
  uint16_t* replica[dtb::kMaxPeers] = {};  // [rank] = local, others IPC-mapped
  unsigned* flags[dtb::kMaxPeers] = {};
  bool opened[dtb::kMaxPeers] = {};
  unsigned* done = nullptr;  // device: [0] CTA counter, [1] call counter (epoch)
};

struct dtb_cost_model {
  dtb_model_spec model;
  dtb_cluster_spec cluster;
  double eff = 0.45, ratio = 2.0;
  struct Row {
    double load, fwd, bwd;
  };
  std::vector<Row> rows[3][4];
  bool nonempty[3] = {false, false, false};
  double* d_rows = nullptr;  // device: load | fwd | bwd
  DevCM dev{};
};

namespace {

// Device allocation tied to a stream (stream-ordered pool).
struct DBuf {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() {
    if (p) cudaFreeAsync(p, s);
  }
  cudaError_t alloc(size_t bytes, cudaStream_t st) {
    s = st;
    return cudaMallocAsync(&p, bytes ? bytes : 16, st);
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

dtb_status set_device(dtb_context* ctx) {
  if (ctx == nullptr) return fail(DTB_ERR_INVALID_ARGUMENT, "null context");
  CU(cudaSetDevice(ctx->device));
  return DTB_OK;
}

dtb_status reset_err(dtb_context* ctx) {
  DevErr init{0, 0, 0, 0, ~0ull};
  CU(cudaMemcpyAsync(ctx->err, &init, sizeof init, cudaMemcpyHostToDevice, ctx->stream));
  return DTB_OK;
}

template <typename T>
dtb_status upload(DBuf& b, const T* host, size_t count, cudaStream_t s) {
  CU(b.alloc(sizeof(T) * count, s));
  if (count) CU(cudaMemcpyAsync(b.p, host, sizeof(T) * count, cudaMemcpyHostToDevice, s));
  return DTB_OK;
}

template <typename T>
dtb_status download(T* host, const DBuf& b, size_t count, cudaStream_t s) {
  if (count && host) CU(cudaMemcpyAsync(host, b.p, sizeof(T) * count, cudaMemcpyDeviceToHost, s));
  return DTB_OK;
}

// Maps the device error record onto the reference's exception + message.
// `ctx_tp[u]` gives the TP of unit u when the record carries only a unit.
dtb_status dev_status(const DevErr& e, const int* tp_of_unit = nullptr) {
  int code = e.code, a = e.a;
  int unit = -1;
  if (code == 0) return DTB_OK;
  if (code == -1) {
    code = static_cast<int>(e.ordered & 0xff);
    unit = static_cast<int>((e.ordered >> 8) % 3);
  }
  switch (code) {
    case E_EMPTY_TP:
      return fail(DTB_ERR_EMPTY_PROFILE, "no profile rows for tp=%d",
                  tp_of_unit && unit >= 0 ? tp_of_unit[unit] : a);
    case E_ANALYTIC:
      return fail(DTB_ERR_EMPTY_PROFILE,
                  "no profile rows for module '%s' and no usable analytic fallback",
                  kind_name(unit >= 0 ? unit : a));
    case E_TP_NOT_ALLOWED:
      return fail(DTB_ERR_INTERNAL, "tp size %d not allowed",
                  tp_of_unit && unit >= 0 ? tp_of_unit[unit] : a);
    case E_NEG_LOAD:
      return fail(DTB_ERR_INTERNAL, "negative token load");
    case E_BAD_TIMES:
      return fail(DTB_ERR_INTERNAL, "bad stage times: %s",
                  a == 2 ? "negative or NaN backward time" : "negative or NaN forward time");
    case E_DEADLOCK:
      return fail(DTB_ERR_INTERNAL, "pipeline schedule deadlocked; op order is invalid");
    case E_COST_RANGE:
      return fail(DTB_ERR_INVALID_ARGUMENT,
                  "sample cost outside the kernel's 32-bit key range (batch %d)", a);
    case E_NO_MICROBATCH:
      return fail(DTB_ERR_INTERNAL, "plan yields no microbatches per iteration");
  }
  return fail(DTB_ERR_INTERNAL, "device error %d", code);
}

dtb_status sync_and_check(dtb_context* ctx, const int* tp_of_unit = nullptr,
                          DevErr* out = nullptr) {
  DevErr e;
  CU(cudaMemcpyAsync(&e, ctx->err, sizeof e, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  if (out) *out = e;
  return dev_status(e, tp_of_unit);
}

bool tp_allowed(int tp) { return tp == 1 || tp == 2 || tp == 4 || tp == 8; }

// The reference raises cost-model errors from the first query it makes;
// these checks depend only on (kind, tp) and the book, so they are evaluated
// up front in the same query order.
dtb_status check_fwd_query(const dtb_cost_model* cm, int kind, int tp) {
  if (!tp_allowed(tp)) return fail(DTB_ERR_INTERNAL, "tp size %d not allowed", tp);
  if (!cm->nonempty[kind]) {
    if (!(cm->eff > 0.0) || !(cm->cluster.peak_flops > 0.0))
      return fail(DTB_ERR_EMPTY_PROFILE,
                  "no profile rows for module '%s' and no usable analytic fallback",
                  kind_name(kind));
    return DTB_OK;
  }
  if (cm->rows[kind][tp_index(tp)].empty())
    return fail(DTB_ERR_EMPTY_PROFILE, "no profile rows for tp=%d", tp);
  return DTB_OK;
}

dtb_status check_bwd_query(const dtb_cost_model* cm, int kind, int tp) {
  if (!cm->nonempty[kind]) {
    if (!(cm->eff > 0.0) || !(cm->cluster.peak_flops > 0.0))
      return fail(DTB_ERR_EMPTY_PROFILE,
                  "no profile rows for module '%s' and no usable analytic fallback",
                  kind_name(kind));
    return DTB_OK;
  }
  const int ti = tp_index(tp);
  if (ti < 0 || cm->rows[kind][ti].empty())
    return fail(DTB_ERR_EMPTY_PROFILE, "no profile rows for tp=%d", tp);
  return DTB_OK;
}

// build_stage_times queries, per unit: forward then backward.
dtb_status check_stage_queries(const dtb_cost_model* cm, const dtb_plan& p) {
  for (int u = 0; u < 3; ++u) {
    TRY(check_fwd_query(cm, u, p.unit[u].tp));
    TRY(check_bwd_query(cm, u, p.unit[u].tp));
  }
  return DTB_OK;
}

dtb_status check_key_queries(const dtb_cost_model* cm, const dtb_plan& p) {
  TRY(check_fwd_query(cm, DTB_ENCODER, p.unit[DTB_ENCODER].tp));
  return check_fwd_query(cm, DTB_GENERATOR, p.unit[DTB_GENERATOR].tp);
}

// ---- warning log.  One unit_forward_time / unit_backward_time query at
// `load` appends what the reference appends (src/cost_model.cpp:84-95 via
// CostProfile::forward_seconds / backward_seconds — both interpolate over
// rows_for(tp), so the clamp condition is the same — and :248-251 via
// analytic_forward): "token load X below|above profile range; clamped" with
// X = std::to_string(load), or "module 'K' has no profile; using analytic
// estimate".  Called on successful calls only (a query that throws appends
// nothing in the reference either).
void warn_query(dtb_context* ctx, const dtb_cost_model* cm, int kind, int tp, double load) {
  if (!cm->nonempty[kind]) {
    ctx->warnings.push_back(std::string("module '") + kind_name(kind) +
                            "' has no profile; using analytic estimate");
    return;
  }
  const int ti = tp_index(tp);
  if (ti < 0 || cm->rows[kind][ti].empty()) return;
  const auto& rows = cm->rows[kind][ti];
  if (load < rows.front().load)
    ctx->warnings.push_back("token load " + std::to_string(load) + " below profile range; clamped");
  else if (load > rows.back().load)
    ctx->warnings.push_back("token load " + std::to_string(load) + " above profile range; clamped");
}

// build_stage_times (src/cost_model.cpp:334-362) over microbatches given by
// their encoder / generator token sums and sample counts: per microbatch,
// per unit (encoder, backbone, generator), forward then backward.
template <typename TokFn>
void warn_stage_times(dtb_context* ctx, const dtb_cost_model* cm, const dtb_plan& p, long long l,
                      const TokFn& mb) {
  for (long long i = 0; i < l; ++i) {
    int64_t te, tg;
    int cnt;
    mb(i, &te, &tg, &cnt);
    const double loads[3] = {mb_mean(te, cnt), static_cast<double>(cm->model.seq_len),
                             mb_mean(tg, cnt)};
    for (int u = 0; u < 3; ++u) {
      warn_query(ctx, cm, u, p.unit[u].tp, loads[u]);
      warn_query(ctx, cm, u, p.unit[u].tp, loads[u]);
    }
  }
}

// microbatch_fwd_keys (src/reorder.cpp:300-317): per microbatch, the
// encoder then the generator forward query.
template <typename TokFn>
void warn_fwd_keys(dtb_context* ctx, const dtb_cost_model* cm, const dtb_plan& p, long long l,
                   const TokFn& mb) {
  for (long long i = 0; i < l; ++i) {
    int64_t te, tg;
    int cnt;
    mb(i, &te, &tg, &cnt);
    warn_query(ctx, cm, DTB_ENCODER, p.unit[DTB_ENCODER].tp, mb_mean(te, cnt));
    warn_query(ctx, cm, DTB_GENERATOR, p.unit[DTB_GENERATOR].tp, mb_mean(tg, cnt));
  }
}

auto host_mbs(const dtb_microbatches* m, long long first = 0) {
  return [m, first](long long i, int64_t* te, int64_t* tg, int* cnt) {
    *te = m->encoder_tokens[first + i];
    *tg = m->generator_tokens[first + i];
    *cnt = m->sample_count[first + i];
  };
}

// schedule_interleaved's divisibility checks (pipeline_sim.cpp:237-253).
dtb_status check_vpp(int l, int p, int vpp) {
  if (l < 1) return fail(DTB_ERR_INTERNAL, "bad stage times: microbatch count must be >= 1");
  if (p < 1) return fail(DTB_ERR_INTERNAL, "bad stage times: stage count must be >= 1");
  if (vpp < 1) return fail(DTB_ERR_INDIVISIBLE_VPP, "vpp must be >= 1");
  if (vpp == 1) return DTB_OK;
  if (p % vpp != 0)
    return fail(DTB_ERR_INDIVISIBLE_VPP, "stage count %d is not divisible by vpp %d", p, vpp);
  if (l % (p / vpp) != 0)
    return fail(DTB_ERR_INDIVISIBLE_VPP,
                "microbatch count %d is not divisible by the device count %d", l, p / vpp);
  return DTB_OK;
}

long long total_subseqs(const dtb_samples* s, bool audio) {
  return 0 * audio + 0 * s->n;
}

// Uploads a CSR span of samples [0, n) (offsets absolute).
struct DevSamples {
  DBuf io, it, ao, at;
  const int* img_off = nullptr;
  const int* img_tok = nullptr;
  const int* aud_off = nullptr;
  const int* aud_tok = nullptr;
};

dtb_status upload_samples(const dtb_samples* s, cudaStream_t st, DevSamples* d) {
  if (s == nullptr || s->image_offsets == nullptr)
    return fail(DTB_ERR_INVALID_ARGUMENT, "samples need image_offsets");
  const long long n = s->n;
  const long long ni = s->image_offsets[n];
  TRY(upload(d->io, s->image_offsets, n + 1, st));
  TRY(upload(d->it, s->image_tokens, ni, st));
  d->img_off = d->io.as<int>();
  d->img_tok = d->it.as<int>();
  if (s->audio_offsets != nullptr) {
    const long long na = s->audio_offsets[n];
    TRY(upload(d->ao, s->audio_offsets, n + 1, st));
    TRY(upload(d->at, s->audio_tokens, na, st));
    d->aud_off = d->ao.as<int>();
    d->aud_tok = d->at.as<int>();
  }
  return DTB_OK;
}

}  // namespace

extern "C" {

const char* dtb_last_error(void) { return g_err.c_str(); }
int dtb_abi_version(void) { return DTB_ABI_VERSION; }

const char* dtb_infeasible_reason_text(int32_t r) {
  switch (r) {
    case DTB_REASON_NONE: return "";
    case DTB_REASON_DP_NOT_DIVIDING: return "dp does not divide the global batch";
    case DTB_REASON_ACTIVATION_ENCODER:
      return "activation memory of encoder exceeds GPU capacity at any allocation";
    case DTB_REASON_ACTIVATION_BACKBONE:
      return "activation memory of backbone exceeds GPU capacity at any allocation";
    case DTB_REASON_ACTIVATION_GENERATOR:
      return "activation memory of generator exceeds GPU capacity at any allocation";
    case DTB_REASON_MEMORY_FLOOR: return "memory floor exceeds the cluster";
    case DTB_REASON_NO_INTEGER_SPLIT: return "no integer stage split is feasible";
  }
  return "?";
}

dtb_status dtb_context_create(int32_t device, dtb_context** out) {
  if (out == nullptr) return fail(DTB_ERR_INVALID_ARGUMENT, "null out");
  int count = 0;
  CU(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count)
    return fail(DTB_ERR_CUDA, "CUDA device %d not present (%d visible)", device, count);
  auto* ctx = new dtb_context;
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->xchg, cudaStreamNonBlocking);
  if (e == cudaSuccess) {
    // keep stream-ordered scratch cached across calls (no per-call cudaMalloc)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      unsigned long long keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  if (e == cudaSuccess) e = cudaMalloc(&ctx->err, sizeof(DevErr));
  if (e != cudaSuccess) {
    delete ctx;
    return fail(DTB_ERR_CUDA, "context init: %s", cudaGetErrorString(e));
  }
  *out = ctx;
  return DTB_OK;
}

dtb_status dtb_context_destroy(dtb_context* ctx) {
  if (!ctx) return DTB_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  cudaFree(ctx->err);
  cudaStreamDestroy(ctx->stream);
  if (ctx->copy_in) cudaStreamDestroy(ctx->copy_in);
  if (ctx->copy_out) cudaStreamDestroy(ctx->copy_out);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->xchg) cudaStreamDestroy(ctx->xchg);
  delete ctx;
  return DTB_OK;
}

// ---------------------------------------------------------------- cost model
static double param_count(const dtb_arch& a) {  // src/core.cpp:40-49
  const double h = static_cast<double>(a.hidden);
  const double f = static_cast<double>(a.ffn_hidden);
  const double kv = a.heads > 0 ? static_cast<double>(a.groups) / static_cast<double>(a.heads) : 1.0;
  const double attn = h * h * (2.0 + 2.0 * kv);
  const double ffn = 3.0 * h * f;
  return static_cast<double>(a.layers) * (attn + ffn);
}

dtb_status dtb_cost_model_create(dtb_context* ctx, const dtb_model_spec* model,
                                 const dtb_cluster_spec* cluster, const dtb_costbook* book,
                                 dtb_cost_model** out) {
  TRY(set_device(ctx));
  if (!model || !cluster || !book || !out) return fail(DTB_ERR_INVALID_ARGUMENT, "null argument");
  auto* cm = new dtb_cost_model;
  cm->model = *model;
  cm->cluster = *cluster;
  cm->eff = book->analytic_efficiency;
  cm->ratio = book->analytic_bwd_fwd_ratio;
  // CostProfile::add_row (cost_model.cpp:37-60)
  for (int64_t i = 0; i < book->n_rows; ++i) {
    const dtb_profile_row& r = book->rows[i];
    dtb_status st = DTB_OK;
    if (!tp_allowed(r.tp))
      st = fail(DTB_ERR_CONFIG, "profile TP size %d is not one of {1,2,4,8}", r.tp);
    else if (!(r.fwd_s > 0.0) || (r.has_bwd && !(r.bwd_s > 0.0)))
      st = fail(DTB_ERR_CONFIG, "profile times must be strictly positive");
    else if (r.token_load < 0.0)
      st = fail(DTB_ERR_CONFIG, "profile token load must be non-negative");
    else if (r.module < 0 || r.module > 2)
      st = fail(DTB_ERR_CONFIG, "bad module index %d", r.module);
    if (st != DTB_OK) {
      delete cm;
      return st;
    }
    auto& rows = cm->rows[r.module][tp_index(r.tp)];
    const dtb_cost_model::Row pt{r.token_load, r.fwd_s, r.has_bwd ? r.bwd_s : 2.0 * r.fwd_s};
    auto it = std::lower_bound(rows.begin(), rows.end(), r.token_load,
                               [](const dtb_cost_model::Row& p, double v) { return p.load < v; });
    if (it != rows.end() && it->load == r.token_load) *it = pt;
    else rows.insert(it, pt);
    cm->nonempty[r.module] = true;
  }
  // flatten + upload
  std::vector<double> flat;
  DevCM& d = cm->dev;
  int off = 0;
  for (int u = 0; u < 3; ++u)
    for (int t = 0; t < 4; ++t) {
      d.off[u][t] = off;
      d.cnt[u][t] = static_cast<int>(cm->rows[u][t].size());
      off += d.cnt[u][t];
    }
  flat.resize(3 * static_cast<size_t>(off > 0 ? off : 1));
  for (int u = 0; u < 3; ++u)
    for (int t = 0; t < 4; ++t)
      for (size_t k = 0; k < cm->rows[u][t].size(); ++k) {
        const auto& r = cm->rows[u][t][k];
        flat[d.off[u][t] + k] = r.load;
        flat[off + d.off[u][t] + k] = r.fwd;
        flat[2 * off + d.off[u][t] + k] = r.bwd;
      }
  cudaError_t e = cudaMalloc(&cm->d_rows, sizeof(double) * flat.size());
  if (e == cudaSuccess)
    e = cudaMemcpy(cm->d_rows, flat.data(), sizeof(double) * flat.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    delete cm;
    return fail(DTB_ERR_CUDA, "cost model upload: %s", cudaGetErrorString(e));
  }
  d.load = cm->d_rows;
  d.fwd = cm->d_rows + off;
  d.bwd = cm->d_rows + 2 * off;
  for (int u = 0; u < 3; ++u) {
    d.nonempty[u] = cm->nonempty[u] ? 1 : 0;
    d.param_count[u] = param_count(model->unit[u].arch);
    d.hidden[u] = static_cast<double>(model->unit[u].arch.hidden);
    d.bwd_factor[u] = model->unit[u].frozen ? model->frozen_backward_factor : 1.0;
    d.mem_pg[u] = model->unit[u].mem.param_grad_bytes;
    d.mem_opt[u] = model->unit[u].mem.optimizer_bytes;
    d.mem_act[u] = model->unit[u].mem.activation_bytes_per_mb;
  }
  d.analytic_ok = (cm->eff > 0.0 && cluster->peak_flops > 0.0) ? 1 : 0;
  d.analytic_denom = cluster->peak_flops * cm->eff;
  d.analytic_ratio = cm->ratio;
  d.seq_len = static_cast<double>(model->seq_len);
  d.dp_sync = model->dp_sync_seconds;
  d.cluster = *cluster;
  *out = cm;
  return DTB_OK;
}

dtb_status dtb_cost_model_destroy(dtb_cost_model* cm) {
  if (!cm) return DTB_OK;
  cudaFree(cm->d_rows);
  delete cm;
  return DTB_OK;
}

dtb_status dtb_cost_sizes(dtb_context* ctx, const dtb_samples* s, int64_t* out) {
  TRY(set_device(ctx));
  if (s->n == 0) return DTB_OK;
  DevSamples d;
  TRY(upload_samples(s, ctx->stream, &d));
  DBuf o;
  CU(o.alloc(sizeof(long long) * s->n, ctx->stream));
  CU(launch_cost_sizes(d.img_off, d.img_tok, d.aud_off, d.aud_tok, s->n, o.as<long long>(),
                       ctx->stream));
  TRY(download(reinterpret_cast<long long*>(out), o, s->n, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return DTB_OK;
}

dtb_status dtb_unit_times(dtb_context* ctx, const dtb_cost_model* cm, int32_t module, int32_t tp,
                          int64_t n, const double* loads, double* fwd, double* bwd) {
  TRY(set_device(ctx));
  if (module < 0 || module > 2) return fail(DTB_ERR_INVALID_ARGUMENT, "bad module");
  if (n == 0) return DTB_OK;
  TRY(reset_err(ctx));
  DBuf dl, df, db;
  TRY(upload(dl, loads, n, ctx->stream));
  CU(df.alloc(8 * n, ctx->stream));
  CU(db.alloc(8 * n, ctx->stream));
  // one query stream per output, in the reference's order for element 0
  if (fwd) TRY(check_fwd_query(cm, module, tp));
  if (bwd && !fwd) TRY(check_bwd_query(cm, module, tp));
  if (fwd && bwd) TRY(check_bwd_query(cm, module, tp));
  CU(launch_unit_times(cm->dev, module, tp, n, dl.as<double>(), fwd ? df.as<double>() : nullptr,
                       bwd ? db.as<double>() : nullptr, ctx->err, ctx->stream));
  TRY(download(fwd, df, n, ctx->stream));
  TRY(download(bwd, db, n, ctx->stream));
  TRY(sync_and_check(ctx));
  if (ctx->warn_on)  // per load: the forward query, then the backward one
    for (int64_t i = 0; i < n; ++i) {
      if (fwd) warn_query(ctx, cm, module, tp, loads[i]);
      if (bwd) warn_query(ctx, cm, module, tp, loads[i]);
    }
  return DTB_OK;
}

dtb_status dtb_memory_check(dtb_context* ctx, const dtb_cost_model* cm, const dtb_plan* plan,
                            dtb_memory_report* out) {
  TRY(set_device(ctx));
  DBuf o;
  CU(o.alloc(sizeof(dtb_memory_report), ctx->stream));
  CU(launch_memory_check(cm->dev, *plan, o.as<dtb_memory_report>(), ctx->stream));
  TRY(download(out, o, 1, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return DTB_OK;
}

static dtb_status upload_mbs(const dtb_microbatches* m, cudaStream_t s, DBuf& e, DBuf& g,
                             DBuf& c) {
  TRY(upload(e, m->encoder_tokens, m->n, s));
  TRY(upload(g, m->generator_tokens, m->n, s));
  TRY(upload(c, m->sample_count, m->n, s));
  return DTB_OK;
}

dtb_status dtb_build_stage_times(dtb_context* ctx, const dtb_cost_model* cm,
                                 const dtb_plan* plan, const dtb_microbatches* mbs, double* fwd,
                                 double* bwd) {
  TRY(set_device(ctx));
  if (mbs->n == 0) return DTB_OK;
  TRY(check_stage_queries(cm, *plan));
  TRY(reset_err(ctx));
  const int p = plan_stages(*plan);
  DBuf e, g, c, f, b;
  TRY(upload_mbs(mbs, ctx->stream, e, g, c));
  CU(f.alloc(8ull * mbs->n * p, ctx->stream));
  CU(b.alloc(8ull * mbs->n * p, ctx->stream));
  CU(launch_stage_times(cm->dev, *plan, mbs->n, e.as<long long>(), g.as<long long>(),
                        c.as<int>(), f.as<double>(), b.as<double>(), ctx->err, ctx->stream));
  TRY(download(fwd, f, mbs->n * p, ctx->stream));
  TRY(download(bwd, b, mbs->n * p, ctx->stream));
  TRY(sync_and_check(ctx));
  if (ctx->warn_on) warn_stage_times(ctx, cm, *plan, mbs->n, host_mbs(mbs));
  return DTB_OK;
}

dtb_status dtb_microbatch_fwd_keys(dtb_context* ctx, const dtb_cost_model* cm,
                                   const dtb_plan* plan, const dtb_microbatches* mbs,
                                   double* keys) {
  TRY(set_device(ctx));
  if (mbs->n == 0) return DTB_OK;
  TRY(check_key_queries(cm, *plan));
  TRY(reset_err(ctx));
  DBuf e, g, c, k;
  TRY(upload_mbs(mbs, ctx->stream, e, g, c));
  CU(k.alloc(8ull * mbs->n, ctx->stream));
  CU(launch_fwd_keys(cm->dev, *plan, mbs->n, e.as<long long>(), g.as<long long>(), c.as<int>(),
                     k.as<double>(), ctx->err, ctx->stream));
  TRY(download(keys, k, mbs->n, ctx->stream));
  TRY(sync_and_check(ctx));
  if (ctx->warn_on) warn_fwd_keys(ctx, cm, *plan, mbs->n, host_mbs(mbs));
  return DTB_OK;
}

dtb_status dtb_compute_stats(dtb_context* ctx, const dtb_samples* s, int64_t seq_len,
                             dtb_workload_stats* out) {
  TRY(set_device(ctx));
  out->seq_len = seq_len;
  DevSamples d;
  if (s->n > 0) TRY(upload_samples(s, ctx->stream, &d));
  DBuf o;
  CU(o.alloc(64, ctx->stream));
  CU(launch_compute_stats(d.img_off, d.img_tok, d.aud_off, d.aud_tok, s->n, o.as<double>(),
                          ctx->stream));
  double r[2];
  TRY(download(r, o, 2, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  out->mean_encoder_tokens = r[0];
  out->mean_generator_tokens = r[1];
  return DTB_OK;
}

// ------------------------------------------------------------------- intra
dtb_status dtb_intra_partition(dtb_context* ctx, const double* sizes, int64_t n, int32_t m,
                               int32_t order, int32_t equal_counts, int32_t* flat_out,
                               int64_t* offsets_out) {
  TRY(set_device(ctx));
  if (m < 1) return fail(DTB_ERR_INTERNAL, "group count must be >= 1");
  if (n == 0) return fail(DTB_ERR_INTERNAL, "cannot reorder an empty batch");
  if (m > intra_generic_max_m())
    return fail(DTB_ERR_INVALID_ARGUMENT, "group count %d exceeds the kernel limit %d", m,
                intra_generic_max_m());
  if (n >= (1LL << 31)) return fail(DTB_ERR_INVALID_ARGUMENT, "n exceeds 2^31");
  DBuf ds, scratch, flat, offs;
  TRY(upload(ds, sizes, n, ctx->stream));
  const size_t sb = intra_generic_scratch(static_cast<int>(n), m);
  CU(scratch.alloc(sb, ctx->stream));
  CU(flat.alloc(4ull * n, ctx->stream));
  CU(offs.alloc(8ull * (m + 1), ctx->stream));
  CU(launch_intra_generic(ds.as<double>(), static_cast<int>(n), m, order, equal_counts,
                          scratch.p, sb, flat.as<int>(), offs.as<long long>(), ctx->stream));
  TRY(download(flat_out, flat, n, ctx->stream));
  TRY(download(reinterpret_cast<long long*>(offsets_out), offs, m + 1, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return DTB_OK;
}

dtb_status dtb_block_group_loads(dtb_context* ctx, const double* sizes, const int32_t* order,
                                 int64_t n, int32_t m, double* loads) {
  TRY(set_device(ctx));
  if (m < 1) return fail(DTB_ERR_INTERNAL, "group count must be >= 1");
  if (n > 0 && n / m == 0) return fail(DTB_ERR_INTERNAL, "fewer samples than groups");
  DBuf ds, dord, dl;
  // sizes is indexed by order entries: upload the span that covers them
  int32_t max_idx = -1;
  for (int64_t i = 0; i < n; ++i) max_idx = std::max(max_idx, order[i]);
  TRY(upload(ds, sizes, static_cast<size_t>(max_idx + 1), ctx->stream));
  TRY(upload(dord, order, n, ctx->stream));
  CU(dl.alloc(8ull * m, ctx->stream));
  if (n == 0) CU(cudaMemsetAsync(dl.p, 0, 8ull * m, ctx->stream));
  else CU(launch_block_loads(ds.as<double>(), dord.as<int>(), static_cast<int>(n), m,
                             dl.as<double>(), ctx->stream));
  TRY(download(loads, dl, m, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return DTB_OK;
}

static dtb_status select_common(dtb_context* ctx, const double* keys, int64_t n_keys,
                                const int32_t* pending, int64_t np, int32_t k, int closest,
                                double target, int32_t* out) {
  TRY(set_device(ctx));
  if (k < 0 || k > np)
    return fail(DTB_ERR_K_TOO_LARGE, "%s asked for %d of %lld",
                closest ? "select_closest" : "select_min", k, static_cast<long long>(np));
  if (k == 0) return DTB_OK;
  DBuf dk, dp, dout;
  TRY(upload(dk, keys, n_keys, ctx->stream));
  TRY(upload(dp, pending, np, ctx->stream));
  CU(dout.alloc(4ull * (k + 1) + np + 16, ctx->stream));
  CU(launch_select(dk.as<double>(), dp.as<int>(), static_cast<int>(np), k, closest, target,
                   dout.as<int>(), ctx->stream));
  TRY(download(out, dout, k, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return DTB_OK;
}

dtb_status dtb_select_min(dtb_context* ctx, const double* keys, int64_t n_keys,
                          const int32_t* pending, int64_t n_pending, int32_t k, int32_t* out) {
  return select_common(ctx, keys, n_keys, pending, n_pending, k, 0, 0.0, out);
}

dtb_status dtb_select_closest(dtb_context* ctx, const double* keys, int64_t n_keys,
                              const int32_t* pending, int64_t n_pending, int32_t k,
                              double target, int32_t* out) {
  return select_common(ctx, keys, n_keys, pending, n_pending, k, 1, target, out);
}

// --------------------------------------------------------------- simulator
dtb_status dtb_schedule(dtb_context* ctx, const double* fwd, const double* bwd, int32_t l,
                        int32_t p, int32_t vpp, int32_t* ev_device, int32_t* ev_mb,
                        int32_t* ev_stage, int32_t* ev_phase, double* ev_start, double* ev_end,
                        double* iteration_time, double* device_busy) {
  TRY(set_device(ctx));
  // schedule_interleaved: check_times first (in-kernel for values), vpp rules
  if (l < 1) return fail(DTB_ERR_INTERNAL, "bad stage times: microbatch count must be >= 1");
  if (p < 1) return fail(DTB_ERR_INTERNAL, "bad stage times: stage count must be >= 1");
  TRY(reset_err(ctx));
  const size_t cells = static_cast<size_t>(l) * p;
  DBuf df, db;
  TRY(upload(df, fwd, cells, ctx->stream));
  TRY(upload(db, bwd, cells, ctx->stream));
  // values are validated before the vpp rules, as check_times runs first
  CU(launch_check_times(df.as<double>(), db.as<double>(), static_cast<long long>(cells), ctx->err,
                        ctx->stream));
  TRY(sync_and_check(ctx));
  TRY(check_vpp(l, p, vpp));
  const int devices = p / vpp;
  const size_t ne = 2 * cells;
  DBuf dev, mb, st, ph, s, e, busy, it, scr, sort_scr;
  CU(dev.alloc(4 * ne, ctx->stream));
  CU(mb.alloc(4 * ne, ctx->stream));
  CU(st.alloc(4 * ne, ctx->stream));
  CU(ph.alloc(4 * ne, ctx->stream));
  CU(s.alloc(8 * ne, ctx->stream));
  CU(e.alloc(8 * ne, ctx->stream));
  CU(busy.alloc(8ull * devices, ctx->stream));
  CU(it.alloc(8, ctx->stream));
  CU(scr.alloc(8 * (2 * cells + 4 * static_cast<size_t>(p) + 8), ctx->stream));
  CU(launch_schedule_events(df.as<double>(), db.as<double>(), l, p, vpp, dev.as<int>(),
                            mb.as<int>(), st.as<int>(), ph.as<int>(), s.as<double>(),
                            e.as<double>(), busy.as<double>(), it.as<double>(), scr.p, ctx->err,
                            ctx->stream));
  const size_t sbytes = sort_events_scratch(static_cast<int>(ne));
  CU(sort_scr.alloc(sbytes, ctx->stream));
  CU(launch_sort_events(static_cast<int>(ne), dev.as<int>(), mb.as<int>(), st.as<int>(),
                        ph.as<int>(), s.as<double>(), e.as<double>(), sort_scr.p, sbytes,
                        ctx->stream));
  TRY(download(ev_device, dev, ne, ctx->stream));
  TRY(download(ev_mb, mb, ne, ctx->stream));
  TRY(download(ev_stage, st, ne, ctx->stream));
  TRY(download(ev_phase, ph, ne, ctx->stream));
  TRY(download(ev_start, s, ne, ctx->stream));
  TRY(download(ev_end, e, ne, ctx->stream));
  TRY(download(device_busy, busy, devices, ctx->stream));
  TRY(download(iteration_time, it, 1, ctx->stream));
  return sync_and_check(ctx);
}

dtb_status dtb_get_intervals(dtb_context* ctx, int64_t n, const int32_t* dev,
                             const int32_t* mb, const int32_t* stage, const int32_t* phase,
                             const double* start, const double* end, int64_t* n_intervals,
                             double* starts, double* ends, int64_t* fill_offsets,
                             int32_t* fill_mb) {
  TRY(set_device(ctx));
  (void)stage;
  DBuf dd, dm, dp, ds, de, ni, os, oe, fo, fm;
  TRY(upload(dd, dev, n, ctx->stream));
  TRY(upload(dm, mb, n, ctx->stream));
  TRY(upload(dp, phase, n, ctx->stream));
  TRY(upload(ds, start, n, ctx->stream));
  TRY(upload(de, end, n, ctx->stream));
  CU(ni.alloc(8, ctx->stream));
  CU(os.alloc(8 * (n + 1), ctx->stream));
  CU(oe.alloc(8 * (n + 1), ctx->stream));
  CU(fo.alloc(8 * (n + 2), ctx->stream));
  CU(fm.alloc(4 * (n + 1), ctx->stream));
  CU(launch_get_intervals(n, dd.as<int>(), dm.as<int>(), dp.as<int>(), ds.as<double>(),
                          de.as<double>(), ni.as<long long>(), os.as<double>(), oe.as<double>(),
                          fo.as<long long>(), fm.as<int>(), ctx->stream));
  long long k = 0;
  TRY(download(&k, ni, 1, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  *n_intervals = k;
  TRY(download(starts, os, k, ctx->stream));
  TRY(download(ends, oe, k, ctx->stream));
  TRY(download(reinterpret_cast<long long*>(fill_offsets), fo, k + 1, ctx->stream));
  long long nf = 0;
  CU(cudaMemcpyAsync(&nf, fo.as<long long>() + k, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  TRY(download(fill_mb, fm, nf, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return DTB_OK;
}

dtb_status dtb_interval_windows(dtb_context* ctx, const double* fwd, const double* bwd,
                                int32_t l, int32_t p, double* volumes) {
  TRY(set_device(ctx));
  const size_t cells = static_cast<size_t>(l) * p;
  const size_t ne = 2 * cells;
  std::vector<int32_t> dev(ne), mb(ne), st(ne), ph(ne);
  std::vector<double> s(ne), e(ne), busy(p > 0 ? p : 1);
  double it;
  TRY(dtb_schedule(ctx, fwd, bwd, l, p, 1, dev.data(), mb.data(), st.data(), ph.data(),
                   s.data(), e.data(), &it, busy.data()));
  std::vector<double> a(ne + 1), b(ne + 1);
  std::vector<int64_t> fo(ne + 2);
  std::vector<int32_t> fm(ne + 1);
  int64_t k = 0;
  TRY(dtb_get_intervals(ctx, static_cast<int64_t>(ne), dev.data(), mb.data(), st.data(),
                        ph.data(), s.data(), e.data(), &k, a.data(), b.data(), fo.data(),
                        fm.data()));
  for (int64_t i = 0; i < k; ++i) volumes[i] = b[i] - a[i];  // Interval::volume
  return DTB_OK;
}

dtb_status dtb_schedule_batch_dev(dtb_context* ctx, int64_t batch, const double* fwd,
                                  const double* bwd, int32_t l, int32_t p, int32_t vpp,
                                  double* iteration_time, double* device_busy, void* stream) {
  TRY(set_device(ctx));
  TRY(check_vpp(l, p, vpp));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  TRY(reset_err(ctx));
  CU(cudaStreamSynchronize(ctx->stream));
  DBuf scr;
  CU(scr.alloc(schedule_batch_scratch(batch, l, p, vpp), s));
  CU(launch_schedule_batch(batch, fwd, bwd, l, p, vpp, iteration_time, device_busy, scr.p,
                           ctx->err, s));
  return DTB_OK;
}

dtb_status dtb_exhaustive_order(dtb_context* ctx, const double* fwd, const double* bwd,
                                int32_t l, int32_t p, int32_t vpp, double* best_time,
                                int32_t* best_order, double* all_times) {
  TRY(set_device(ctx));
  if (l < 1 || l > exhaustive_max_l())
    return fail(DTB_ERR_INTERNAL, "exhaustive_order needs 1 <= l <= %d", exhaustive_max_l());
  if (p < 1 || p > exhaustive_max_p())
    return fail(DTB_ERR_INVALID_ARGUMENT, "exhaustive_order supports 1 <= p <= %d",
                exhaustive_max_p());
  TRY(check_vpp(l, p, vpp));
  long long total = 1;
  for (int i = 2; i <= l; ++i) total *= i;
  if (all_times != nullptr && total > (1ll << 26))
    return fail(DTB_ERR_INVALID_ARGUMENT, "all_times of %lld orderings not supported", total);
  const size_t cells = static_cast<size_t>(l) * p;
  cudaStream_t s = ctx->stream;
  TRY(reset_err(ctx));
  DBuf df, db, all, bt, bo, scr;
  TRY(upload(df, fwd, cells, s));
  TRY(upload(db, bwd, cells, s));
  CU(launch_check_times(df.as<double>(), db.as<double>(), static_cast<long long>(cells), ctx->err,
                        s));
  if (all_times != nullptr) CU(all.alloc(8ull * total, s));
  CU(bt.alloc(8, s));
  CU(bo.alloc(4ull * l, s));
  const int n_blocks = static_cast<int>(std::min<long long>(148 * 16, (total + 127) / 128));
  CU(scr.alloc(exhaustive_scratch(n_blocks), s));
  CU(launch_exhaustive(df.as<double>(), db.as<double>(), l, p, vpp,
                       all_times ? all.as<double>() : nullptr, bt.as<double>(), bo.as<int>(),
                       scr.p, n_blocks, ctx->err, s));
  TRY(download(best_time, bt, 1, s));
  TRY(download(best_order, bo, l, s));
  if (all_times != nullptr) TRY(download(all_times, all, total, s));
  return sync_and_check(ctx);
}

dtb_status dtb_schedule_batch(dtb_context* ctx, int64_t batch, const double* fwd,
                              const double* bwd, int32_t l, int32_t p, int32_t vpp,
                              double* iteration_time, double* device_busy) {
  TRY(set_device(ctx));
  TRY(check_vpp(l, p, vpp));
  const size_t cells = static_cast<size_t>(batch) * l * p;
  DBuf df, db, it, busy;
  TRY(upload(df, fwd, cells, ctx->stream));
  TRY(upload(db, bwd, cells, ctx->stream));
  CU(it.alloc(8ull * batch, ctx->stream));
  CU(busy.alloc(8ull * batch * (p / vpp), ctx->stream));
  TRY(reset_err(ctx));
  DBuf scr;
  CU(scr.alloc(schedule_batch_scratch(batch, l, p, vpp), ctx->stream));
  CU(launch_schedule_batch(batch, df.as<double>(), db.as<double>(), l, p, vpp, it.as<double>(),
                           device_busy ? busy.as<double>() : nullptr, scr.p, ctx->err,
                           ctx->stream));
  TRY(download(iteration_time, it, batch, ctx->stream));
  TRY(download(device_busy, busy, batch * (p / vpp), ctx->stream));
  return sync_and_check(ctx);
}

dtb_status dtb_simulate_iteration(dtb_context* ctx, const dtb_cost_model* cm,
                                  const dtb_plan* plan, int32_t n_groups,
                                  const int64_t* group_offsets, const dtb_microbatches* mbs,
                                  double* t_iter, double* group_times, int32_t* slowest_group,
                                  double* slowest_group_time, double* mean_bubble) {
  TRY(set_device(ctx));
  if (n_groups <= 0) return fail(DTB_ERR_INTERNAL, "no microbatch groups to simulate");
  const int p = plan_stages(*plan);
  // groups may have different sizes: one launch per distinct size run
  std::vector<double> tg(n_groups), bub(n_groups);
  DBuf e, g, c;
  TRY(upload_mbs(mbs, ctx->stream, e, g, c));
  for (int32_t gi = 0; gi < n_groups; ++gi) {
    const long long l = group_offsets[gi + 1] - group_offsets[gi];
    if (l > 0) TRY(check_stage_queries(cm, *plan));
    // simulate.cpp:31: build_stage_times of the group, then its simulation
    if (ctx->warn_on) warn_stage_times(ctx, cm, *plan, l, host_mbs(mbs, group_offsets[gi]));
    TRY(check_vpp(static_cast<int>(l), p, plan->vpp));
    TRY(reset_err(ctx));
    GroupSimArgs a{};
    a.cm = cm->dev;
    a.plan = *plan;
    a.n_batches = 1;
    a.groups = 1;
    a.l = static_cast<int>(l);
    a.enc = e.as<long long>() + group_offsets[gi];
    a.gen = g.as<long long>() + group_offsets[gi];
    a.count = c.as<int>() + group_offsets[gi];
    a.span = 1;
    DBuf tgd, bd, scr;
    CU(tgd.alloc(8, ctx->stream));
    CU(bd.alloc(8, ctx->stream));
    a.t_group = tgd.as<double>();
    a.busy = bd.as<double>();
    a.err = ctx->err;
    CU(scr.alloc(group_sims_scratch(a), ctx->stream));
    CU(launch_group_sims(a, scr.p, ctx->stream));
    TRY(download(&tg[gi], tgd, 1, ctx->stream));
    TRY(download(&bub[gi], bd, 1, ctx->stream));
    TRY(sync_and_check(ctx));
  }
  // simulate.cpp:31-46 fold (sequential over groups, as the reference)
  double bubble_sum = 0.0, worst = 0.0;
  int worst_g = 0;
  for (int32_t gi = 0; gi < n_groups; ++gi) {
    bubble_sum += bub[gi];
    if (tg[gi] > worst) {
      worst = tg[gi];
      worst_g = gi;
    }
  }
  if (group_times) std::copy(tg.begin(), tg.end(), group_times);
  if (slowest_group) *slowest_group = worst_g;
  if (slowest_group_time) *slowest_group_time = worst;
  if (mean_bubble) *mean_bubble = bubble_sum / static_cast<double>(n_groups);
  if (t_iter) *t_iter = worst + cm->model.dp_sync_seconds;
  return DTB_OK;
}

// ------------------------------------------------------------------- inter
static dtb_status inter_checks(int32_t l, int32_t p, int32_t vpp) {
  if (l <= 1) return DTB_OK;
  if (vpp < 1) return fail(DTB_ERR_INDIVISIBLE_VPP, "vpp must be >= 1");
  if (p % vpp != 0) return fail(DTB_ERR_INDIVISIBLE_VPP, "stage count not divisible by vpp");
  const int devices = p / vpp;
  if (devices == 1) return DTB_OK;
  const int pending = l - 1 - std::min(devices - 1, l - 1);
  if (pending > 0 && vpp > 1 && l % devices != 0)
    return fail(DTB_ERR_INDIVISIBLE_VPP,
                "microbatch count %d is not divisible by the device count %d", l, devices);
  return DTB_OK;
}

dtb_status dtb_inter_reorder_batch_dev(dtb_context* ctx, int64_t batch, const double* fwd,
                                       const double* bwd, int32_t l, int32_t p,
                                       const double* keys, int32_t vpp, int32_t* orders,
                                       void* stream) {
  TRY(set_device(ctx));
  TRY(inter_checks(l, p, vpp));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  InterArgs a{};
  a.batch = batch;
  a.l = l;
  a.p = p;
  a.vpp = vpp;
  a.fwd = fwd;
  a.bwd = bwd;
  a.keys = keys;
  a.orders = orders;
  a.err = ctx->err;
  const size_t bytes = inter_scratch(a);
  DBuf scr;
  CU(scr.alloc(bytes, s));
  CU(launch_inter(a, scr.p, bytes, s));
  return DTB_OK;
}

dtb_status dtb_inter_reorder_batch(dtb_context* ctx, int64_t batch, const double* fwd,
                                   const double* bwd, int32_t l, int32_t p, const double* keys,
                                   int32_t vpp, int32_t* orders) {
  TRY(set_device(ctx));
  TRY(inter_checks(l, p, vpp));
  if (batch == 0 || l == 0) return DTB_OK;
  const size_t cells = static_cast<size_t>(batch) * l * p;
  DBuf df, db, dk, dord;
  TRY(upload(df, fwd, cells, ctx->stream));
  TRY(upload(db, bwd, cells, ctx->stream));
  TRY(upload(dk, keys, static_cast<size_t>(batch) * l, ctx->stream));
  CU(dord.alloc(4ull * batch * l, ctx->stream));
  TRY(reset_err(ctx));
  TRY(dtb_inter_reorder_batch_dev(ctx, batch, df.as<double>(), db.as<double>(), l, p,
                                  dk.as<double>(), vpp, dord.as<int>(), ctx->stream));
  TRY(download(orders, dord, static_cast<size_t>(batch) * l, ctx->stream));
  return sync_and_check(ctx);
}

dtb_status dtb_inter_reorder(dtb_context* ctx, const double* fwd, const double* bwd, int32_t l,
                             int32_t p, const double* keys, int32_t vpp, int32_t* order_out) {
  if (l <= 1) {
    for (int i = 0; i < l; ++i) order_out[i] = i;
    return DTB_OK;
  }
  return dtb_inter_reorder_batch(ctx, 1, fwd, bwd, l, p, keys, vpp, order_out);
}

// --------------------------------------------------------- disaggregated
static dtb_status stream_checks(const dtb_cost_model* cm, const dtb_plan* plan,
                                const dtb_reorder_mode* mode, long long n_total,
                                long long n_batches) {
  const long long bs = plan->global_batch;
  if (n_batches < 1 || n_total != n_batches * bs) {
    if (n_batches == 1)
      return fail(DTB_ERR_BATCH_SIZE_MISMATCH, "batch has %lld samples, plan expects %lld",
                  n_total, bs);
    return fail(DTB_ERR_BATCH_SIZE_MISMATCH,
                "stream has %lld samples, plan expects %lld batches of %lld", n_total, n_batches,
                bs);
  }
  const int dp_lm = plan->unit[DTB_BACKBONE].dp;
  const int dp_me = plan->unit[DTB_ENCODER].dp;
  if (mode->intra && dp_lm < 1) return fail(DTB_ERR_INTERNAL, "group count must be >= 1");
  if (bs == 0) return fail(DTB_ERR_INTERNAL, "cannot reorder an empty batch");
  if (dp_lm < 1 || dp_me < 1 || plan->unit[DTB_GENERATOR].dp < 1)
    return fail(DTB_ERR_INTERNAL, "parallel sizes must be >= 1");
  if (bs / dp_lm == 0) return fail(DTB_ERR_INTERNAL, "fewer samples than groups");
  if ((bs > fused_max_n() || dp_lm > fused_max_m()) && dp_lm > intra_generic_max_m())
    return fail(DTB_ERR_INVALID_ARGUMENT, "more than %d DP groups", intra_generic_max_m());
  if (bs > 0x7fffffffLL) return fail(DTB_ERR_INVALID_ARGUMENT, "global batch beyond int32");
  // simulate_iteration(identity) is the first cost-model consumer
  TRY(check_stage_queries(cm, *plan));
  const int per_group = static_cast<int>(bs / dp_lm);
  TRY(check_vpp(per_group, plan_stages(*plan), plan->vpp));
  if (mode->inter) TRY(inter_checks(per_group, plan_stages(*plan), plan->vpp));
  return DTB_OK;
}

// Sort/partition path of a stream of global batches: the streaming cost pass
// (k_cost.cu: tokens, identity order and loads, batches the averaging bound
// decides), then the partition kernel on the rest (k_intra.cu).  `fa` holds
// everything but the cost-pass outputs; `cscr` receives its scratch.
// Global batches beyond the fused kernels' limits (more than 16,384 samples
// or 512 groups): per batch, the per-sample costs, a stable device radix
// sort of (orderable cost, index) and the one-CTA equal-count greedy
// (launch_intra_generic, any n, m <= 4096), the block loads of both orders
// and the keep decision; consumers read the 32-bit tokens.
static cudaError_t launch_sort_partition_generic(FusedArgs& fa, long long n_batches,
                                                 cudaStream_t s) {
  const int n = fa.n, m = fa.m;
  DBuf sizes, flat, offs, li, lg, scr;
  const size_t sb = intra_generic_scratch(n, m);
  cudaError_t e = sizes.alloc(8ull * n, s);
  if (e == cudaSuccess) e = flat.alloc(4ull * n, s);
  if (e == cudaSuccess) e = offs.alloc(8ull * (m + 1), s);
  if (e == cudaSuccess) e = li.alloc(8ull * m, s);
  if (e == cudaSuccess) e = lg.alloc(8ull * m, s);
  if (e == cudaSuccess) e = scr.alloc(sb, s);
  for (long long b = 0; b < n_batches && e == cudaSuccess; ++b) {
    e = launch_batch_tokens(fa.img_off, fa.img_tok, fa.aud_off, fa.aud_tok, b * n, n,
                            fa.tok32_orig, sizes.as<double>(), fa.err, static_cast<int>(b), s);
    if (e == cudaSuccess) e = launch_block_loads(sizes.as<double>(), nullptr, n, m, li.as<double>(), s);
    if (e == cudaSuccess && fa.intra) {
      e = launch_intra_generic(sizes.as<double>(), n, m, fa.order, 1, scr.p, sb, flat.as<int>(),
                               offs.as<long long>(), s);
      if (e == cudaSuccess)
        e = launch_block_loads(sizes.as<double>(), flat.as<int>(), n, m, lg.as<double>(), s);
    }
    if (e == cudaSuccess)
      e = launch_generic_decide(li.as<double>(), fa.intra ? lg.as<double>() : li.as<double>(), m,
                                n, b, fa.intra, flat.as<int>(), fa.tok32_orig, fa.order_out,
                                fa.tok32_staged, fa.load_before, fa.load_after, fa.kept,
                                fa.wide_flag, s);
  }
  return e;
}

// side != null: the partition kernel runs on `side` after the cost pass
// (event `fork`), so work that needs only the cost pass's outputs can proceed
// on `s` meanwhile; the caller joins `side` back.
static cudaError_t launch_sort_partition(FusedArgs& fa, long long n_batches, DBuf& cscr,
                                         cudaStream_t s, cudaStream_t side = nullptr,
                                         cudaEvent_t fork = nullptr) {
  if (fa.n > fused_max_n() || fa.m > fused_max_m())
    return launch_sort_partition_generic(fa, n_batches, s);
  cudaError_t e = cscr.alloc(cost_scratch_bytes(n_batches, fa.m), s);
  if (e != cudaSuccess) return e;
  CostArgs ca{};
  ca.n = fa.n;
  ca.m = fa.m;
  ca.order = fa.order;
  ca.intra = fa.intra;
  ca.n_batches = n_batches;
  ca.img_off = fa.img_off;
  ca.img_tok = fa.img_tok;
  ca.aud_off = fa.aud_off;
  ca.aud_tok = fa.aud_tok;
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  ca.staged = al(fa.img_off) && al(fa.img_tok) &&
              (fa.aud_off == nullptr || (al(fa.aud_off) && al(fa.aud_tok))) && fa.n % 4 == 0;
  ca.tok16 = const_cast<unsigned short*>(fa.tok16);
  ca.order_out = fa.order_out;
  ca.tok16_staged = fa.tok16_staged;
  ca.blk_ident = cscr.as<unsigned>();
  ca.bstat = ca.blk_ident + n_batches * fa.m;
  ca.list = ca.bstat + 4 * n_batches;
  ca.state = ca.list + 1 + n_batches;
  ca.wide_flag = fa.wide_flag;
  ca.tok32_orig = fa.tok32_orig;
  ca.load_before = fa.load_before;
  ca.load_after = fa.load_after;
  ca.kept = fa.kept;
  ca.div_pg = fa.div_pg;
  ca.err = fa.err;
  e = launch_cost_stream(ca, s);
  if (e != cudaSuccess) return e;
  fa.state = ca.state;
  fa.blk_ident = ca.blk_ident;
  fa.list = ca.list;
  if (side != nullptr) {
    e = cudaEventRecord(fork, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(side, fork, 0);
    if (e != cudaSuccess) return e;
    return launch_intra_fused(fa, n_batches, side);
  }
  return launch_intra_fused(fa, n_batches, s, true);
}

// Warning log of a stream call: the queries disaggregated_reorder makes per
// batch (src/reorder.cpp:319-396), in order — build_stage_times of every
// coupled group in the input order (simulate_iteration, t_iter_before); with
// inter, per group build_stage_times then microbatch_fwd_keys in the intra
// order; build_stage_times of every group in the final order (t_iter_after).
// The microbatch token sums of each phase come from the device
// (launch_mb_tokens), the strings are built here.
static dtb_status warn_stream(dtb_context* ctx, const dtb_cost_model* cm, const dtb_plan* plan,
                              const dtb_reorder_mode* mode, const GroupSimArgs& base,
                              const int* mb0, const int* mb1, const int* inter_orders,
                              cudaStream_t s) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  CU(cudaStreamIsCapturing(s, &cap));
  if (cap != cudaStreamCaptureStatusNone) return DTB_OK;  // graphs: no warning log
  const long long n_batches = base.n_batches, groups = base.groups, l = base.l;
  const long long n_mb = n_batches * groups * l;
  const int phases = mode->inter ? 3 : 2;
  DBuf d;
  CU(d.alloc(4ull * n_mb * phases, s));
  for (int ph = 0; ph < phases; ++ph) {
    GroupSimArgs a = base;
    const bool last = ph == phases - 1;
    a.staged = ph > 0;
    a.mbsum = base.span > 1 ? (ph == 0 ? mb0 : mb1) : nullptr;
    a.order = last && mode->inter ? inter_orders : nullptr;
    CU(launch_mb_tokens(a, d.as<int>() + ph * n_mb, s));
  }
  std::vector<int> h(static_cast<size_t>(n_mb) * phases);
  TRY(download(h.data(), d, n_mb * phases, s));
  CU(cudaStreamSynchronize(s));
  const int cnt = base.span;
  for (long long b = 0; b < n_batches; ++b) {
    for (int ph = 0; ph < phases; ++ph) {
      for (long long e = 0; e < groups; ++e) {
        const int* t = h.data() + ph * n_mb + (b * groups + e) * l;
        auto mb = [t, cnt](long long i, int64_t* te, int64_t* tg, int* c) {
          *te = *tg = t[i];
          *c = cnt;
        };
        warn_stage_times(ctx, cm, *plan, l, mb);
        if (mode->inter && ph == 1) warn_fwd_keys(ctx, cm, *plan, l, mb);
      }
    }
  }
  return DTB_OK;
}

// Device pipeline for n_batches global batches (all pointers device):
//   cost pass (k_cost.cu) -> partition kernel on the side stream (intra_fused:
//   greedy / decision / kept orders of the batches the cost pass left open),
//   concurrently with: cost table -> group sims on the input order
//   (t_iter_before) — then, joined: [inter_reorder per coupled group] ->
//   compose -> group sims on the reordered groups (t_iter_after).
static dtb_status run_stream(dtb_context* ctx, const dtb_cost_model* cm, const dtb_plan* plan,
                             const dtb_reorder_mode* mode, const int* io, const int* it,
                             const int* ao, const int* at, long long n_batches, int* order_out,
                             double* lb, double* la, double* tb, double* ta, unsigned char* kept,
                             cudaStream_t s, const PeerBcast* peer = nullptr) {
  // Peer exchange of the final order on its own stream, joined at the end:
  // it overlaps everything after the order is final (the simulations).
  // `after`: the stream on which the order became final.
  cudaEvent_t ev_ready = nullptr, ev_done = nullptr;
  // phase 0: the whole range, then the flag barrier; phase 1: the batches
  // the cost pass decided (after the cost pass, next to the partition
  // kernel); phase 2: the rest and the barrier.
  auto exchange = [&](cudaStream_t after, int phase, const unsigned* state) -> cudaError_t {
    if (peer == nullptr) return cudaSuccess;
    cudaError_t e = cudaSuccess;
    if (ev_ready == nullptr) e = cudaEventCreateWithFlags(&ev_ready, cudaEventDisableTiming);
    if (e == cudaSuccess && ev_done == nullptr)
      e = cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(ev_ready, after);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->xchg, ev_ready, 0);
    PeerBcast pb = *peer;
    pb.src = order_out;
    pb.phase = phase;
    pb.state = state;
    if (e == cudaSuccess) e = launch_peer_broadcast(pb, ctx->xchg);
    if (e == cudaSuccess && phase != 1) e = cudaEventRecord(ev_done, ctx->xchg);
    return e;
  };
  cudaEvent_t ev_fork = nullptr, ev_part = nullptr;  // partition kernel on ctx->side
  cudaEvent_t ev_table = nullptr, ev_after = nullptr;  // t_iter_after sims on ctx->side
  struct EvGuard {
    cudaEvent_t* e[6];
    ~EvGuard() {
      for (cudaEvent_t* x : e)
        if (*x) cudaEventDestroy(*x);
    }
  } ev_guard{{&ev_ready, &ev_done, &ev_fork, &ev_part, &ev_table, &ev_after}};
  const int n = static_cast<int>(plan->global_batch);
  const int dp_lm = plan->unit[DTB_BACKBONE].dp;
  const int dp_me = plan->unit[DTB_ENCODER].dp;
  const int per_group = n / dp_lm;
  const int span = dp_lm / dp_me;
  const long long n_mb = n_batches * dp_me * static_cast<long long>(per_group);
  const long long total = n_batches * static_cast<long long>(n);
  DBuf intra, tok16, tok16s, tok32, tok32s, wflag, kept_buf, wide, mb0, mb1, tgrp, inter, scr;
  DBuf tgrp2, scr2, tab_eg, tab_k;  // side-stream simulations, cost table
  // without inter the intra order is the output order whenever every
  // position belongs to a microbatch
  const bool compose_needed = mode->inter || dp_me * span * per_group != n;
  int* intra_out = order_out;
  if (compose_needed) {
    CU(intra.alloc(4ull * total, s));
    intra_out = intra.as<int>();
  }
  unsigned char* kept_dev = kept;
  if (kept_dev == nullptr) {
    CU(kept_buf.alloc(n_batches, s));
    kept_dev = kept_buf.as<unsigned char>();
  }
  CU(tok16.alloc(2ull * total + 16, s));
  CU(tok16s.alloc(2ull * total + 16, s));
  CU(tok32.alloc(4ull * total, s));
  CU(tok32s.alloc(4ull * total, s));
  CU(wflag.alloc(4ull * n_batches, s));
  CU(wide.alloc(fused_wide_scratch_bytes(n_batches), s));
  FusedArgs fa{};
  fa.n = n;
  fa.m = dp_lm;
  fa.order = mode->sort_order;
  fa.intra = mode->intra;
  fa.img_off = io;
  fa.img_tok = it;
  fa.aud_off = ao;
  fa.aud_tok = at;
  fa.order_out = intra_out;
  fa.load_before = lb;
  fa.load_after = la;
  fa.kept = kept_dev;
  fa.tok16_staged = tok16s.as<unsigned short>();
  fa.tok32_orig = tok32.as<int>();
  fa.tok32_staged = tok32s.as<int>();
  fa.pg = per_group;
  fa.dp_me = dp_me;
  fa.wide_scratch = wide.as<unsigned char>();
  fa.tok16 = tok16.as<unsigned short>();
  fa.wide_flag = wflag.as<unsigned int>();
  fa.div_pg = FastDiv::make(static_cast<unsigned>(per_group));
  fa.err = ctx->err;
  DBuf cscr;
  // joins the side stream back into `s` on every exit, before the scratch
  // above is freed (stream-ordered frees on `s`)
  struct Join {
    cudaStream_t s;
    cudaEvent_t* e[3];
    ~Join() {
      for (cudaEvent_t* x : e)
        if (*x) cudaStreamWaitEvent(s, *x, 0);
    }
  } join{s, {&ev_part, &ev_done, &ev_after}};
  CU(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&ev_part, cudaEventDisableTiming));
  CU(launch_sort_partition(fa, n_batches, cscr, s, ctx->side, ev_fork));
  CU(cudaEventRecord(ev_part, ctx->side));
  // the intra order is the output order: the batches the cost pass decided
  // are exchanged right after it (their order is the identity, final), the
  // rest right after the partition kernel — both next to the simulations
  if (!compose_needed) {
    if (fa.state != nullptr) {
      CU(exchange(s, 1, fa.state));
      CU(exchange(ctx->side, 2, fa.state));
    } else {
      CU(exchange(ctx->side, 0, nullptr));
    }
  }
  const TokSrc tok{tok16.as<unsigned short>(), tok16s.as<unsigned short>(), tok32.as<int>(),
                   tok32s.as<int>(), kept_dev, wflag.as<unsigned int>(), n};
  if (span > 1) {  // assembled microbatch sums [b][e][i] (input order: cost pass only)
    CU(mb0.alloc(4ull * n_mb, s));
    CU(mb1.alloc(4ull * n_mb, s));
    CU(launch_assemble(n_batches, n, dp_lm, dp_me, tok, false, mb0.as<int>(), s));
  }
  // token-indexed cost table shared by both simulations and the inter kernel
  // (built on the side stream before the cost pass it measured slower: its
  // CTAs delay the cost pass's first wave)
  const int tsize = static_cast<int>(std::min<long long>(
      static_cast<long long>(span) * 0x8000, static_cast<long long>(kCostTableMax)));
  CU(tab_eg.alloc(sizeof(double4) * tsize, s));
  CU(tab_k.alloc(sizeof(double) * tsize, s));
  CU(launch_cost_table(cm->dev, *plan, span, tsize, tab_eg.as<double4>(), tab_k.as<double>(),
                       ctx->err, s));
  CostTable table{tab_eg.as<double4>(), tab_k.as<double>(), tsize, span};
  GroupSimArgs ga{};
  ga.cm = cm->dev;
  ga.plan = *plan;
  ga.n_batches = n_batches;
  ga.groups = dp_me;
  ga.l = per_group;
  ga.stream = true;
  ga.tok = tok;
  ga.staged = false;
  ga.mbsum = span > 1 ? mb0.as<int>() : nullptr;
  ga.span = span;
  ga.table = table;
  CU(tgrp.alloc(8ull * n_batches * dp_me, s));
  ga.t_group = tgrp.as<double>();
  ga.busy = nullptr;
  ga.err = ctx->err;
  const size_t sim_bytes = group_sims_scratch(ga);
  InterArgs ia{};
  ia.batch = n_batches * dp_me;
  ia.l = per_group;
  ia.p = plan_stages(*plan);
  ia.vpp = plan->vpp;
  ia.cm = cm->dev;
  ia.plan = *plan;
  ia.stream = true;
  ia.tok = tok;
  ia.mbsum = span > 1 ? mb1.as<int>() : nullptr;
  ia.groups = dp_me;
  ia.span = span;
  ia.table = table;
  ia.err = ctx->err;
  const bool inter_tok = mode->inter && inter_tok_applies(ia);
  // many stages / long sequences: warp per problem, problem in shared memory
  const bool inter_warp = mode->inter && !inter_tok && inter_warp_applies(ia);
  const size_t inter_bytes = mode->inter && !inter_tok && !inter_warp ? inter_scratch(ia) : 0;
  CU(scr.alloc(std::max(sim_bytes, inter_bytes), s));
  // intra only: a batch whose greedy split was not kept runs the identity
  // order again, so its t_iter_after IS its t_iter_before (same microbatches,
  // same operation sequence) — only kept batches are re-simulated.  Those
  // simulations need the partition kernel but not the t_iter_before ones:
  // with small simulation scratch they run on the side stream, after the
  // partition kernel, concurrently with the t_iter_before simulations.
  const unsigned char* only_kept = mode->inter ? nullptr : kept_dev;
  const bool after_on_side = !mode->inter && !compose_needed && sim_bytes <= 4096;
  if (after_on_side) {
    CU(cudaEventCreateWithFlags(&ev_table, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&ev_after, cudaEventDisableTiming));
    CU(tgrp2.alloc(8ull * n_batches * dp_me, s));
    CU(scr2.alloc(sim_bytes, s));
    CU(cudaEventRecord(ev_table, s));  // table and scratch ready
    GroupSimArgs gb = ga;
    gb.staged = true;
    gb.mbsum = span > 1 ? mb1.as<int>() : nullptr;
    gb.order = nullptr;
    gb.only_kept = only_kept;
    gb.t_group = tgrp2.as<double>();
    if (span > 1) CU(launch_assemble(n_batches, n, dp_lm, dp_me, tok, true, mb1.as<int>(), ctx->side));
    CU(cudaStreamWaitEvent(ctx->side, ev_table, 0));
    CU(launch_group_sims(gb, scr2.p, ctx->side));
    CU(cudaEventRecord(ev_after, ctx->side));
  }
  if (group_sims_fuse_reduce(ga)) {  // the kernel writes t_iter_before itself
    GroupSimArgs gr = ga;
    gr.t_iter = tb;
    gr.dp_sync = cm->model.dp_sync_seconds;
    CU(launch_group_sims(gr, scr.p, s, true));  // programmatic launch after the cost table
  } else {
    CU(launch_group_sims(ga, scr.p, s));
    CU(launch_t_iter_reduce(n_batches, dp_me, tgrp.as<double>(), cm->model.dp_sync_seconds, tb, s));
  }
  if (after_on_side) {
    CU(cudaStreamWaitEvent(s, ev_after, 0));
    CU(launch_t_iter_reduce(n_batches, dp_me, tgrp2.as<double>(), cm->model.dp_sync_seconds, ta, s,
                            only_kept, tb));
    if (ctx->warn_on)
      TRY(warn_stream(ctx, cm, plan, mode, ga, mb0.as<int>(), mb1.as<int>(), nullptr, s));
    return DTB_OK;  // `join` waits for the partition kernel and the exchange
  }
  CU(cudaStreamWaitEvent(s, ev_part, 0));  // the partition kernel's orders and kept flags
  if (span > 1) CU(launch_assemble(n_batches, n, dp_lm, dp_me, tok, true, mb1.as<int>(), s));
  if (mode->inter) {
    CU(inter.alloc(4ull * n_mb, s));
    ia.orders = inter.as<int>();
    DBuf redo, tab_fz;
    if (inter_tok) {
      CU(redo.alloc(static_cast<size_t>(ia.batch), s));
      CU(cudaMemsetAsync(redo.p, 0, static_cast<size_t>(ia.batch), s));
      ia.redo = redo.as<unsigned char>();
      CU(tab_fz.alloc(sizeof(double2) * tsize, s));
      CU(launch_table_fz(tab_eg.as<double4>(), tab_fz.as<double2>(), tsize, s));
      ia.table.fz = tab_fz.as<double2>();
      CU(launch_inter_tok(ia, s));
    } else if (inter_warp) {
      CU(launch_inter_warp(ia, s));
    } else {
      CU(launch_inter(ia, scr.p, inter_bytes, s));
    }
  }
  if (compose_needed) {
    CU(launch_compose(n_batches, n, dp_lm, dp_me, intra_out, mode->inter ? inter.as<int>() : nullptr,
                      order_out, s));
    CU(exchange(s, 0, nullptr));
  }
  ga.staged = true;
  ga.mbsum = span > 1 ? mb1.as<int>() : nullptr;
  ga.order = mode->inter ? inter.as<int>() : nullptr;
  ga.only_kept = only_kept;
  CU(launch_group_sims(ga, scr.p, s));
  CU(launch_t_iter_reduce(n_batches, dp_me, tgrp.as<double>(), cm->model.dp_sync_seconds, ta, s,
                          only_kept, tb));
  if (ctx->warn_on) {
    GroupSimArgs base = ga;
    base.only_kept = nullptr;
    TRY(warn_stream(ctx, cm, plan, mode, base, mb0.as<int>(), mb1.as<int>(),
                    mode->inter ? inter.as<int>() : nullptr, s));
  }
  return DTB_OK;  // `join` waits for the partition kernel and the exchange
}

// ------------------------------------------------------------ peer groups
namespace {
size_t replica_bytes(int64_t n_samples) {
  return (static_cast<size_t>(n_samples) * 2 + 255) / 256 * 256;
}
}  // namespace

// ------------------------------------------------------------ warning log
dtb_status dtb_warnings_enable(dtb_context* ctx, int32_t on) {
  if (ctx == nullptr) return fail(DTB_ERR_INVALID_ARGUMENT, "null context");
  ctx->warn_on = on != 0;
  ctx->warnings.clear();
  return DTB_OK;
}

int64_t dtb_warnings_count(const dtb_context* ctx) {
  return ctx == nullptr ? 0 : static_cast<int64_t>(ctx->warnings.size());
}

const char* dtb_warning_at(const dtb_context* ctx, int64_t i) {
  if (ctx == nullptr || i < 0 || i >= static_cast<int64_t>(ctx->warnings.size())) return nullptr;
  return ctx->warnings[static_cast<size_t>(i)].c_str();
}

dtb_status dtb_warnings_clear(dtb_context* ctx) {
  if (ctx == nullptr) return fail(DTB_ERR_INVALID_ARGUMENT, "null context");
  ctx->warnings.clear();
  return DTB_OK;
}

dtb_status dtb_peer_buffer_create(dtb_context* ctx, int64_t n_samples, uint16_t** replica,
                                  dtb_peer_handle* handle) {
  TRY(set_device(ctx));
  if (replica == nullptr || handle == nullptr || n_samples < 0)
    return fail(DTB_ERR_INVALID_ARGUMENT, "peer buffer: bad arguments");
  static_assert(sizeof(cudaIpcMemHandle_t) == sizeof(dtb_peer_handle), "IPC handle size");
  void* p = nullptr;
  const size_t bytes = replica_bytes(n_samples) + 4 * dtb::kMaxPeers;
  CU(cudaMalloc(&p, bytes));
  CU(cudaMemset(p, 0, bytes));  // flags start at epoch 0
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    CU(e);
  }
  std::memcpy(handle->bytes, &h, sizeof(h));
  *replica = static_cast<uint16_t*>(p);
  return DTB_OK;
}

dtb_status dtb_peer_buffer_destroy(dtb_context* ctx, uint16_t* replica) {
  TRY(set_device(ctx));
  if (replica) CU(cudaFree(replica));
  return DTB_OK;
}

dtb_status dtb_peer_group_open(dtb_context* ctx, int32_t rank, int32_t world, uint16_t* replica,
                               int64_t n_samples, const dtb_peer_handle* handles,
                               dtb_peer_group** out) {
  TRY(set_device(ctx));
  if (out == nullptr || handles == nullptr || replica == nullptr || world < 1 ||
      world > dtb::kMaxPeers || rank < 0 || rank >= world)
    return fail(DTB_ERR_INVALID_ARGUMENT, "peer group: rank %d of %d (at most %d ranks)", rank,
                world, dtb::kMaxPeers);
  auto* g = new dtb_peer_group;
  g->device = ctx->device;
  g->rank = rank;
  g->world = world;
  g->n_samples = n_samples;
  for (int p = 0; p < world; ++p) {
    void* ptr = replica;
    if (p != rank) {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handles[p].bytes, sizeof(h));
      const cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        dtb_peer_group_close(g);
        CU(e);
      }
      g->opened[p] = true;
    }
    g->replica[p] = static_cast<uint16_t*>(ptr);
    g->flags[p] = reinterpret_cast<unsigned*>(static_cast<char*>(ptr) + replica_bytes(n_samples));
  }
  cudaError_t e = cudaMalloc(&g->done, 2 * sizeof(unsigned));
  if (e == cudaSuccess) e = cudaMemset(g->done, 0, 2 * sizeof(unsigned));
  if (e != cudaSuccess) {
    dtb_peer_group_close(g);
    CU(e);
  }
  if (ctx->side == nullptr) CU(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
  *out = g;
  return DTB_OK;
}

dtb_status dtb_peer_group_close(dtb_peer_group* g) {
  if (g == nullptr) return DTB_OK;
  cudaSetDevice(g->device);
  for (int p = 0; p < g->world; ++p)
    if (g->opened[p]) cudaIpcCloseMemHandle(g->replica[p]);
  if (g->done) cudaFree(g->done);
  delete g;
  return DTB_OK;
}

dtb_status dtb_shard_range(int64_t n_batches, int32_t rank, int32_t world, int64_t* first,
                           int64_t* count) {
  if (world < 1 || rank < 0 || rank >= world || n_batches < 0 || !first || !count)
    return fail(DTB_ERR_INVALID_ARGUMENT, "shard range: rank %d of %d", rank, world);
  const int64_t base = n_batches / world, extra = n_batches % world;
  *first = rank * base + std::min<int64_t>(rank, extra);
  *count = base + (rank < extra ? 1 : 0);
  return DTB_OK;
}

dtb_status dtb_reorder_stream_shard_dev(dtb_context* ctx, const dtb_cost_model* cm,
                                        const dtb_plan* plan, const dtb_reorder_mode* mode,
                                        const dtb_samples* samples, int64_t n_batches,
                                        dtb_peer_group* group, double* load_before,
                                        double* load_after, double* t_iter_before,
                                        double* t_iter_after, uint8_t* greedy_kept,
                                        void* stream) {
  TRY(set_device(ctx));
  if (group == nullptr || group->device != ctx->device)
    return fail(DTB_ERR_INVALID_ARGUMENT, "peer group of another device");
  if (t_iter_before == nullptr || t_iter_after == nullptr)
    return fail(DTB_ERR_INVALID_ARGUMENT, "t_iter_before / t_iter_after are required");
  const dtb_reorder_mode def{1, 1, DTB_ASCENDING};
  const dtb_reorder_mode* md = mode ? mode : &def;
  TRY(stream_checks(cm, plan, md, samples->n, n_batches));
  if (samples->n > group->n_samples)
    return fail(DTB_ERR_INVALID_ARGUMENT, "stream of %lld samples, replicas hold %lld",
                static_cast<long long>(samples->n), static_cast<long long>(group->n_samples));
  int64_t first = 0, count = 0;
  TRY(dtb_shard_range(n_batches, group->rank, group->world, &first, &count));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long n = plan->global_batch;
  const int dp = plan->unit[DTB_BACKBONE].dp;
  const long long s0 = first * n, cnt = count * n;
  DBuf shard_order;
  CU(shard_order.alloc(4ull * std::max<long long>(cnt, 1), s));
  dtb::PeerBcast pb{};
  pb.count = cnt;
  pb.world = group->world;
  pb.rank = group->rank;
  pb.done = group->done;
  pb.epoch = group->done + 1;
  pb.flags_local = group->flags[group->rank];
  bool al = (reinterpret_cast<uintptr_t>(shard_order.p) & 15u) == 0;
  for (int p = 0; p < group->world; ++p) {
    pb.dst[p] = group->replica[p] + s0;
    pb.flags[p] = group->flags[p];
    al = al && (reinterpret_cast<uintptr_t>(pb.dst[p]) & 15u) == 0;
  }
  pb.aligned = al && n % 8 == 0 ? 1 : 0;
  pb.n = static_cast<int>(n);
  if (count == 0) {  // nothing to reorder; still take part in the barrier
    CU(launch_peer_broadcast(pb, s));
    return DTB_OK;
  }
  const int* ao = samples->audio_offsets ? samples->audio_offsets + s0 : nullptr;
  return run_stream(ctx, cm, plan, md, samples->image_offsets + s0, samples->image_tokens, ao,
                    samples->audio_tokens, count, shard_order.as<int>(),
                    load_before ? load_before + first * dp : nullptr,
                    load_after ? load_after + first * dp : nullptr, t_iter_before + first,
                    t_iter_after + first, greedy_kept ? greedy_kept + first : nullptr, s, &pb);
}

dtb_status dtb_reorder_stream_dev(dtb_context* ctx, const dtb_cost_model* cm,
                                  const dtb_plan* plan, const dtb_reorder_mode* mode,
                                  const dtb_samples* samples, int64_t n_batches,
                                  int32_t* output_order, double* load_before, double* load_after,
                                  double* t_iter_before, double* t_iter_after,
                                  uint8_t* greedy_kept, void* stream) {
  TRY(set_device(ctx));
  const dtb_reorder_mode def{1, 1, DTB_ASCENDING};
  const dtb_reorder_mode* md = mode ? mode : &def;
  TRY(stream_checks(cm, plan, md, samples->n, n_batches));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return run_stream(ctx, cm, plan, md, samples->image_offsets, samples->image_tokens,
                    samples->audio_offsets, samples->audio_tokens, n_batches, output_order,
                    load_before, load_after, t_iter_before, t_iter_after, greedy_kept, s);
}

dtb_status dtb_reorder_stream(dtb_context* ctx, const dtb_cost_model* cm, const dtb_plan* plan,
                              const dtb_reorder_mode* mode, const dtb_samples* samples,
                              int64_t n_batches, int32_t* output_order, double* load_before,
                              double* load_after, double* t_iter_before, double* t_iter_after,
                              uint8_t* greedy_kept) {
  TRY(set_device(ctx));
  const dtb_reorder_mode def{1, 1, DTB_ASCENDING};
  const dtb_reorder_mode* md = mode ? mode : &def;
  TRY(stream_checks(cm, plan, md, samples->n, n_batches));
  if (samples->image_offsets == nullptr)
    return fail(DTB_ERR_INVALID_ARGUMENT, "samples need image_offsets");
  cudaStream_t s = ctx->stream;
  TRY(reset_err(ctx));
  // Host buffers in, host buffers out, pipelined over chunks of global
  // batches (batches are independent): the host->device copy of chunk c+1
  // and the device->host copy of chunk c-1 overlap the kernels of chunk c
  // (copy_in / compute / copy_out streams ordered by events).  Device
  // buffers are full-size, so the CSR offsets stay absolute.
  if (ctx->copy_in == nullptr) {
    CU(cudaStreamCreateWithFlags(&ctx->copy_in, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&ctx->copy_out, cudaStreamNonBlocking));
  }
  const long long total = samples->n;
  const long long bs = plan->global_batch;
  const int dp = plan->unit[DTB_BACKBONE].dp;
  const bool audio = samples->audio_offsets != nullptr;
  const long long ni = samples->image_offsets[total];
  const long long na = audio ? samples->audio_offsets[total] : 0;
  DBuf io, it, ao, at, o, lb, la, tb, ta, kp;
  CU(io.alloc(4ull * (total + 1), s));
  CU(it.alloc(4ull * ni, s));
  if (audio) {
    CU(ao.alloc(4ull * (total + 1), s));
    CU(at.alloc(4ull * na, s));
  }
  CU(o.alloc(4ull * total, s));
  CU(lb.alloc(8ull * n_batches * dp, s));
  CU(la.alloc(8ull * n_batches * dp, s));
  CU(tb.alloc(8ull * n_batches, s));
  CU(ta.alloc(8ull * n_batches, s));
  CU(kp.alloc(n_batches, s));
  cudaEvent_t ready;
  CU(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  CU(cudaEventRecord(ready, s));  // allocations + error reset are ordered first
  CU(cudaStreamWaitEvent(ctx->copy_in, ready, 0));
  CU(cudaStreamWaitEvent(ctx->copy_out, ready, 0));
#ifndef DTB_E2E_CHUNKS
#define DTB_E2E_CHUNKS 8
#endif
  const long long chunk =
      std::max<long long>(16, (n_batches + DTB_E2E_CHUNKS - 1) / DTB_E2E_CHUNKS);
  const long long n_chunks = n_batches > 0 ? (n_batches + chunk - 1) / chunk : 0;
  std::vector<cudaEvent_t> in_done(n_chunks), run_done(n_chunks);
  dtb_status st = DTB_OK;
  auto h2d = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
    return bytes ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->copy_in)
                 : cudaSuccess;
  };
  auto d2h = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
    return (bytes && dst) ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->copy_out)
                          : cudaSuccess;
  };
  for (long long c = 0; c < n_chunks && st == DTB_OK; ++c) {
    const long long b0 = c * chunk, nb = std::min(chunk, n_batches - b0);
    const long long s0 = b0 * bs, s1 = (b0 + nb) * bs;
    cudaError_t e = cudaEventCreateWithFlags(&in_done[c], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&run_done[c], cudaEventDisableTiming);
    // inputs of the chunk: offsets [s0, s1] and their token ranges
    const long long i0 = samples->image_offsets[s0], i1 = samples->image_offsets[s1];
    if (e == cudaSuccess)
      e = h2d(io.as<int>() + s0, samples->image_offsets + s0, 4ull * (s1 - s0 + 1));
    if (e == cudaSuccess) e = h2d(it.as<int>() + i0, samples->image_tokens + i0, 4ull * (i1 - i0));
    if (audio && e == cudaSuccess) {
      const long long a0 = samples->audio_offsets[s0], a1 = samples->audio_offsets[s1];
      e = h2d(ao.as<int>() + s0, samples->audio_offsets + s0, 4ull * (s1 - s0 + 1));
      if (e == cudaSuccess) e = h2d(at.as<int>() + a0, samples->audio_tokens + a0, 4ull * (a1 - a0));
    }
    if (e == cudaSuccess) e = cudaEventRecord(in_done[c], ctx->copy_in);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, in_done[c], 0);
    if (e != cudaSuccess) {
      st = fail(DTB_ERR_CUDA, "%s", cudaGetErrorString(e));
      break;
    }
    st = run_stream(ctx, cm, plan, md, io.as<int>() + s0, it.as<int>(),
                    audio ? ao.as<int>() + s0 : nullptr, audio ? at.as<int>() : nullptr, nb,
                    o.as<int>() + s0, lb.as<double>() + b0 * dp, la.as<double>() + b0 * dp,
                    tb.as<double>() + b0, ta.as<double>() + b0, kp.as<unsigned char>() + b0, s);
    if (st != DTB_OK) break;
    e = cudaEventRecord(run_done[c], s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->copy_out, run_done[c], 0);
    if (e == cudaSuccess) e = d2h(output_order ? output_order + s0 : nullptr, o.as<int>() + s0,
                                  4ull * (s1 - s0));
    if (e == cudaSuccess)
      e = d2h(load_before ? load_before + b0 * dp : nullptr, lb.as<double>() + b0 * dp,
              8ull * nb * dp);
    if (e == cudaSuccess)
      e = d2h(load_after ? load_after + b0 * dp : nullptr, la.as<double>() + b0 * dp,
              8ull * nb * dp);
    if (e == cudaSuccess)
      e = d2h(t_iter_before ? t_iter_before + b0 : nullptr, tb.as<double>() + b0, 8ull * nb);
    if (e == cudaSuccess)
      e = d2h(t_iter_after ? t_iter_after + b0 : nullptr, ta.as<double>() + b0, 8ull * nb);
    if (e == cudaSuccess)
      e = d2h(greedy_kept ? greedy_kept + b0 : nullptr, kp.as<unsigned char>() + b0, nb);
    if (e != cudaSuccess) st = fail(DTB_ERR_CUDA, "%s", cudaGetErrorString(e));
  }
  // everything (copies included) completes before buffers are released
  cudaStreamSynchronize(ctx->copy_in);
  cudaStreamSynchronize(ctx->copy_out);
  cudaStreamSynchronize(s);
  for (long long c = 0; c < n_chunks; ++c) {
    if (in_done[c]) cudaEventDestroy(in_done[c]);
    if (run_done[c]) cudaEventDestroy(run_done[c]);
  }
  cudaEventDestroy(ready);
  if (st != DTB_OK) return st;
  return sync_and_check(ctx);
}

static dtb_status intra_stream(dtb_context* ctx, int64_t bs, int32_t dp_lm, int32_t sort_order,
                               const dtb_samples* samples, int64_t n_batches, int32_t* order_out,
                               double* load_before, double* load_after, uint8_t* greedy_kept,
                               unsigned long long* prof, void* stream) {
  TRY(set_device(ctx));
  if (dp_lm < 1) return fail(DTB_ERR_INTERNAL, "group count must be >= 1");
  if (bs < 1) return fail(DTB_ERR_INTERNAL, "cannot reorder an empty batch");
  if (samples->n != n_batches * bs)
    return fail(DTB_ERR_BATCH_SIZE_MISMATCH, "stream has %lld samples, expected %lld",
                static_cast<long long>(samples->n), static_cast<long long>(n_batches * bs));
  if (bs / dp_lm == 0) return fail(DTB_ERR_INTERNAL, "fewer samples than groups");
  if ((bs > fused_max_n() || dp_lm > fused_max_m()) && dp_lm > intra_generic_max_m())
    return fail(DTB_ERR_INVALID_ARGUMENT, "more than %d DP groups", intra_generic_max_m());
  FusedArgs fa{};
  fa.n = static_cast<int>(bs);
  fa.m = dp_lm;
  fa.order = sort_order;
  fa.intra = 1;
  fa.img_off = samples->image_offsets;
  fa.img_tok = samples->image_tokens;
  fa.aud_off = samples->audio_offsets;
  fa.aud_tok = samples->audio_tokens;
  fa.order_out = order_out;
  fa.load_before = load_before;
  fa.load_after = load_after;
  fa.kept = greedy_kept;
  DBuf wide;
  CU(wide.alloc(fused_wide_scratch_bytes(n_batches), static_cast<cudaStream_t>(stream)));
  fa.wide_scratch = wide.as<unsigned char>();
  DBuf tok16, wflag;
  const long long total = n_batches * bs;
  CU(tok16.alloc(2ull * total + 16, static_cast<cudaStream_t>(stream)));
  CU(wflag.alloc(4ull * n_batches, static_cast<cudaStream_t>(stream)));
  fa.tok16 = tok16.as<unsigned short>();
  fa.wide_flag = wflag.as<unsigned int>();
  fa.div_pg = FastDiv::make(static_cast<unsigned>(bs / dp_lm));
  fa.pg = static_cast<int>(bs / dp_lm);
  fa.dp_me = dp_lm;
  fa.prof = prof;
  fa.err = ctx->err;
  DBuf cscr;
  CU(launch_sort_partition(fa, n_batches, cscr, static_cast<cudaStream_t>(stream)));
  return DTB_OK;
}

dtb_status dtb_intra_stream_dev(dtb_context* ctx, int64_t bs, int32_t dp_lm, int32_t sort_order,
                                const dtb_samples* samples, int64_t n_batches, int32_t* order_out,
                                double* load_before, double* load_after, uint8_t* greedy_kept,
                                void* stream) {
  return intra_stream(ctx, bs, dp_lm, sort_order, samples, n_batches, order_out, load_before,
                      load_after, greedy_kept, nullptr, stream);
}

// Debug variant (not in the public header): per-batch phase timestamps
// (globaltimer ns) of the fused kernel, prof_dev[n_batches][64].
dtb_status dtb_debug_intra_stream_prof_dev(dtb_context* ctx, int64_t bs, int32_t dp_lm,
                                           int32_t sort_order, const dtb_samples* samples,
                                           int64_t n_batches, int32_t* order_out,
                                           unsigned long long* prof_dev, void* stream) {
  return intra_stream(ctx, bs, dp_lm, sort_order, samples, n_batches, order_out, nullptr,
                      nullptr, nullptr, prof_dev, stream);
}

dtb_status dtb_disaggregated_reorder(dtb_context* ctx, const dtb_cost_model* cm,
                                     const dtb_plan* plan, const dtb_reorder_mode* mode,
                                     const dtb_samples* batch, dtb_reorder_report* r) {
  return dtb_reorder_stream(ctx, cm, plan, mode, batch, 1, r->output_order,
                            r->group_load_before, r->group_load_after, &r->t_iter_before,
                            &r->t_iter_after, nullptr);
}

// ---------------------------------------------------------- orchestration
dtb_status dtb_predict_times(dtb_context* ctx, const dtb_cost_model* cm,
                             const dtb_workload_stats* stats, const dtb_plan* plans, int64_t n,
                             dtb_predicted_times* out) {
  TRY(set_device(ctx));
  if (n == 0) return DTB_OK;
  TRY(reset_err(ctx));
  DBuf dp, o;
  TRY(upload(dp, plans, n, ctx->stream));
  CU(o.alloc(sizeof(dtb_predicted_times) * n, ctx->stream));
  CU(launch_predict(cm->dev, *stats, dp.as<dtb_plan>(), n, o.as<dtb_predicted_times>(), ctx->err,
                    ctx->stream));
  TRY(download(out, o, n, ctx->stream));
  DevErr e;
  CU(cudaMemcpyAsync(&e, ctx->err, sizeof e, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  if (e.code == -1) {
    const long long idx = static_cast<long long>(e.ordered >> 8);
    const int code = static_cast<int>(e.ordered & 0xff);
    if (code == E_NO_MICROBATCH)
      return fail(DTB_ERR_INTERNAL, "plan yields no microbatches per iteration");
    // re-derive the unit from the plan's queries in reference order
    for (int u = 0; u < 3; ++u) {
      TRY(check_fwd_query(cm, u, plans[idx].unit[u].tp));
      TRY(check_bwd_query(cm, u, plans[idx].unit[u].tp));
    }
    return dev_status(e);
  }
  return dev_status(e);
}

dtb_status dtb_enumerate_parallelism(dtb_context* ctx, const dtb_cluster_spec* cluster,
                                     int64_t bs, int64_t* count, dtb_tuple* tuples,
                                     int64_t capacity) {
  TRY(set_device(ctx));
  if (bs < 1) return fail(DTB_ERR_INVALID_ARGUMENT, "global batch must be >= 1");
  DBuf scr, cnt, out;
  CU(scr.alloc(enumerate_scratch(bs), ctx->stream));
  CU(cnt.alloc(8, ctx->stream));
  if (tuples != nullptr && capacity > 0) CU(out.alloc(sizeof(dtb_tuple) * capacity, ctx->stream));
  CU(launch_enumerate(*cluster, bs, nullptr, 0, cnt.as<long long>(),
                      tuples && capacity > 0 ? out.as<dtb_tuple>() : nullptr, capacity, scr.p,
                      ctx->stream));
  long long c = 0;
  TRY(download(&c, cnt, 1, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  *count = c;
  if (tuples != nullptr && capacity > 0) {
    TRY(download(tuples, out, std::min<long long>(c, capacity), ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  }
  return DTB_OK;
}

static dtb_status orch_error(dtb_context* ctx, const dtb_cost_model* cm, const DevErr& e,
                             const dtb_tuple* dev_tuples) {
  if (e.code == 0) return DTB_OK;
  if (e.code != -1) return dev_status(e);
  const long long key = static_cast<long long>(e.ordered >> 8);
  const long long idx = key / 3;
  dtb_tuple t;
  CU(cudaMemcpy(&t, dev_tuples + idx, sizeof t, cudaMemcpyDeviceToHost));
  const int tps[3] = {t.tp_me, t.tp_lm, t.tp_mg};
  for (int u = 0; u < 3; ++u) {
    TRY(check_fwd_query(cm, u, tps[u]));
    TRY(check_bwd_query(cm, u, tps[u]));
  }
  return dev_status(e, tps);
}

dtb_status dtb_solve_subproblem(dtb_context* ctx, const dtb_cost_model* cm,
                                const dtb_workload_stats* stats, const dtb_tuple* tuples,
                                int64_t n, int64_t bs, int32_t vpp, dtb_candidate* out) {
  TRY(set_device(ctx));
  if (n == 0) return DTB_OK;
  TRY(reset_err(ctx));
  DBuf dt, o, bb;
  TRY(upload(dt, tuples, n, ctx->stream));
  CU(o.alloc(sizeof(dtb_candidate) * n, ctx->stream));
  const int grid = static_cast<int>(std::min<long long>((n + 127) / 128, 4096));
  CU(bb.alloc(sizeof(dtb_candidate) * grid, ctx->stream));
  OrchArgs a{};
  a.cm = cm->dev;
  a.stats = *stats;
  a.bs = bs;
  a.vpp = vpp;
  a.tuples = dt.as<dtb_tuple>();
  a.n = n;
  a.shard_index = 0;
  a.shard_count = 1;
  a.out = o.as<dtb_candidate>();
  a.block_best = bb.as<dtb_candidate>();
  a.err = ctx->err;
  DBuf lst;
  CU(lst.alloc(8ull * n + 16, ctx->stream));
  a.list = lst.as<long long>();
  a.list_count = reinterpret_cast<unsigned*>(a.list + n);
  CU(launch_orchestration(a, grid, ctx->stream));
  TRY(download(out, o, n, ctx->stream));
  DevErr e;
  CU(cudaMemcpyAsync(&e, ctx->err, sizeof e, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return orch_error(ctx, cm, e, dt.as<dtb_tuple>());
}

// Shared search driver: enumerate on device, solve the shard, reduce.
static dtb_status search(dtb_context* ctx, const dtb_cost_model* cm,
                         const dtb_workload_stats* stats, int64_t bs, int32_t vpp,
                         long long shard_index, long long shard_count, dtb_candidate* best_dev,
                         long long* evaluated_dev, dtb_candidate* table_dev, cudaStream_t s,
                         long long* n_tuples_out, DBuf& tuples) {
  DBuf scr, cnt;
  CU(scr.alloc(enumerate_scratch(bs), s));
  CU(cnt.alloc(8, s));
  CU(launch_enumerate(cm->cluster, bs, nullptr, 0, cnt.as<long long>(), nullptr, 0, scr.p, s));
  long long n = 0;
  CU(cudaMemcpyAsync(&n, cnt.p, 8, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  CU(tuples.alloc(sizeof(dtb_tuple) * (n > 0 ? n : 1), s));
  CU(launch_enumerate(cm->cluster, bs, nullptr, 0, cnt.as<long long>(), tuples.as<dtb_tuple>(),
                      n, scr.p, s));
  const long long mine = n > shard_index ? (n - shard_index + shard_count - 1) / shard_count : 0;
  int grid = static_cast<int>(std::min<long long>((mine + 127) / 128, 148 * 16));
  if (grid < 1) grid = 1;
  DBuf bb;
  CU(bb.alloc(sizeof(dtb_candidate) * grid, s));
  OrchArgs a{};
  a.cm = cm->dev;
  a.stats = *stats;
  a.bs = bs;
  a.vpp = vpp;
  a.tuples = tuples.as<dtb_tuple>();
  a.n = n;
  a.shard_index = shard_index;
  a.shard_count = shard_count;
  a.out = table_dev;
  a.block_best = bb.as<dtb_candidate>();
  a.err = ctx->err;
  DBuf lst;
  CU(lst.alloc(8ull * std::max<long long>(mine, 1) + 16, s));
  a.list = lst.as<long long>();
  a.list_count = reinterpret_cast<unsigned*>(a.list + std::max<long long>(mine, 1));
  CU(launch_orchestration(a, grid, s));
  CU(launch_best_reduce(bb.as<dtb_candidate>(), grid, best_dev, s));
  if (evaluated_dev)
    CU(cudaMemcpyAsync(evaluated_dev, &mine, 8, cudaMemcpyHostToDevice, s));
  if (n_tuples_out) *n_tuples_out = n;
  CU(cudaStreamSynchronize(s));  // `mine` and scratch lifetimes
  return DTB_OK;
}

dtb_status dtb_model_orchestration(dtb_context* ctx, const dtb_cost_model* cm,
                                   const dtb_workload_stats* stats, int64_t bs, int32_t vpp,
                                   dtb_orchestration_result* result, dtb_candidate* candidates,
                                   int64_t capacity) {
  TRY(set_device(ctx));
  const auto t0 = std::chrono::steady_clock::now();
  TRY(reset_err(ctx));
  DBuf best, table, tuples;
  CU(best.alloc(sizeof(dtb_candidate), ctx->stream));
  long long n = 0;
  // the table, when requested, needs the count first
  if (candidates != nullptr) {
    int64_t cnt = 0;
    TRY(dtb_enumerate_parallelism(ctx, &cm->cluster, bs, &cnt, nullptr, 0));
    CU(table.alloc(sizeof(dtb_candidate) * (cnt > 0 ? cnt : 1), ctx->stream));
  }
  TRY(search(ctx, cm, stats, bs, vpp, 0, 1, best.as<dtb_candidate>(), nullptr,
             candidates ? table.as<dtb_candidate>() : nullptr, ctx->stream, &n, tuples));
  DevErr e;
  CU(cudaMemcpy(&e, ctx->err, sizeof e, cudaMemcpyDeviceToHost));
  TRY(orch_error(ctx, cm, e, tuples.as<dtb_tuple>()));
  dtb_candidate b;
  CU(cudaMemcpy(&b, best.p, sizeof b, cudaMemcpyDeviceToHost));
  if (candidates != nullptr) {
    CU(cudaMemcpy(candidates, table.p, sizeof(dtb_candidate) * std::min<long long>(n, capacity),
                  cudaMemcpyDeviceToHost));
  }
  result->candidates_evaluated = n;
  result->solve_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (!b.feasible) return fail(DTB_ERR_INFEASIBLE, "no feasible plan for this model and cluster");
  result->best = b.plan;
  result->times = b.times;
  return DTB_OK;
}

dtb_status dtb_brute_force_oracle(dtb_context* ctx, const dtb_cost_model* cm,
                                  const dtb_workload_stats* stats, int64_t bs, int32_t vpp,
                                  int32_t gpu_cap, dtb_orchestration_result* result) {
  TRY(set_device(ctx));
  const int n_gpus = cm->cluster.total_gpus;
  if (n_gpus > gpu_cap)
    return fail(DTB_ERR_CAP_EXCEEDED, "exhaustive search capped at %d GPUs, got %d", gpu_cap,
                n_gpus);
  const auto t0 = std::chrono::steady_clock::now();
  TRY(reset_err(ctx));
  cudaStream_t s = ctx->stream;
  DBuf scr, cnt, tuples, ev, bb, best;
  CU(scr.alloc(enumerate_scratch(bs), s));
  CU(cnt.alloc(8, s));
  CU(launch_enumerate(cm->cluster, bs, nullptr, 0, cnt.as<long long>(), nullptr, 0, scr.p, s));
  long long n = 0;
  CU(cudaMemcpyAsync(&n, cnt.p, 8, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  CU(tuples.alloc(sizeof(dtb_tuple) * (n > 0 ? n : 1), s));
  CU(launch_enumerate(cm->cluster, bs, nullptr, 0, cnt.as<long long>(), tuples.as<dtb_tuple>(),
                      n, scr.p, s));
  const int grid = 148 * 16;
  CU(ev.alloc(8, s));
  CU(cudaMemsetAsync(ev.p, 0, 8, s));
  CU(bb.alloc(sizeof(dtb_candidate) * grid, s));
  const size_t bscr = brute_scratch(n);
  DBuf bs_scr;
  CU(bs_scr.alloc(bscr, s));
  // records of blocks that get no pairs must read as infeasible
  CU(cudaMemsetAsync(bb.p, 0, sizeof(dtb_candidate) * grid, s));
  CU(best.alloc(sizeof(dtb_candidate), s));
  OrchArgs a{};
  a.cm = cm->dev;
  a.stats = *stats;
  a.bs = bs;
  a.vpp = vpp;
  a.tuples = tuples.as<dtb_tuple>();
  a.n = n;
  a.shard_index = 0;
  a.shard_count = 1;
  a.block_best = bb.as<dtb_candidate>();
  a.err = ctx->err;
  CU(launch_brute(a, grid, reinterpret_cast<unsigned long long*>(ev.p), bs_scr.p, bscr, s));
  CU(launch_best_reduce(bb.as<dtb_candidate>(), grid, best.as<dtb_candidate>(), s));
  DevErr e;
  CU(cudaMemcpyAsync(&e, ctx->err, sizeof e, cudaMemcpyDeviceToHost, s));
  dtb_candidate b;
  unsigned long long evaluated = 0;
  CU(cudaMemcpyAsync(&b, best.p, sizeof b, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(&evaluated, ev.p, 8, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  TRY(orch_error(ctx, cm, e, tuples.as<dtb_tuple>()));
  result->candidates_evaluated = static_cast<int64_t>(evaluated);
  result->solve_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (!b.feasible) return fail(DTB_ERR_INFEASIBLE, "no feasible plan in the exhaustive search");
  result->best = b.plan;
  result->times = b.times;
  return DTB_OK;
}

dtb_status dtb_rigid_baseline(dtb_context* ctx, const dtb_cost_model* cm,
                              const dtb_workload_stats* stats, int64_t bs, int32_t vpp,
                              dtb_plan* plan) {
  TRY(set_device(ctx));
  TRY(reset_err(ctx));
  cudaStream_t s = ctx->stream;
  std::vector<long long> divs;
  for (long long d = 1; d * d <= bs; ++d)
    if (bs % d == 0) {
      divs.push_back(d);
      if (d != bs / d) divs.push_back(bs / d);
    }
  std::sort(divs.begin(), divs.end());
  const int nd = static_cast<int>(divs.size());
  DBuf dd, c, best;
  TRY(upload(dd, divs.data(), divs.size(), s));
  CU(c.alloc(sizeof(dtb_candidate) * (4 * nd > 0 ? 4 * nd : 1), s));
  CU(best.alloc(sizeof(dtb_candidate), s));
  CU(launch_rigid(cm->dev, *stats, bs, vpp, dd.as<long long>(), nd, c.as<dtb_candidate>(),
                  ctx->err, s));
  CU(launch_best_reduce(c.as<dtb_candidate>(), 4 * nd, best.as<dtb_candidate>(), s));
  DevErr e;
  dtb_candidate b;
  CU(cudaMemcpyAsync(&e, ctx->err, sizeof e, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(&b, best.p, sizeof b, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (e.code != 0) {
    if (e.code != -1) return dev_status(e);
    const long long x = static_cast<long long>(e.ordered >> 8);
    const int tp = std::array<int, 4>{1, 2, 4, 8}[x / nd];
    for (int u = 0; u < 3; ++u) {
      TRY(check_fwd_query(cm, u, tp));
      TRY(check_bwd_query(cm, u, tp));
    }
    const int tps[3] = {tp, tp, tp};
    return dev_status(e, tps);
  }
  if (!b.feasible) return fail(DTB_ERR_INFEASIBLE, "no feasible rigid configuration");
  *plan = b.plan;
  return DTB_OK;
}

dtb_status dtb_orchestration_shard_dev(dtb_context* ctx, const dtb_cost_model* cm,
                                       const dtb_workload_stats* stats, int64_t bs, int32_t vpp,
                                       int64_t shard_index, int64_t shard_count,
                                       dtb_candidate* best_dev, int64_t* evaluated_dev,
                                       void* stream) {
  TRY(set_device(ctx));
  if (shard_count < 1 || shard_index < 0 || shard_index >= shard_count)
    return fail(DTB_ERR_INVALID_ARGUMENT, "bad shard %lld of %lld", (long long)shard_index,
                (long long)shard_count);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  TRY(reset_err(ctx));
  CU(cudaStreamSynchronize(ctx->stream));
  DBuf tuples;
  long long n = 0;
  TRY(search(ctx, cm, stats, bs, vpp, shard_index, shard_count, best_dev,
             reinterpret_cast<long long*>(evaluated_dev), nullptr, s, &n, tuples));
  DevErr e;
  CU(cudaMemcpy(&e, ctx->err, sizeof e, cudaMemcpyDeviceToHost));
  return orch_error(ctx, cm, e, tuples.as<dtb_tuple>());
}

dtb_status dtb_best_reduce_dev(dtb_context* ctx, const dtb_candidate* records, int64_t n,
                               dtb_candidate* best_dev, void* stream) {
  TRY(set_device(ctx));
  CU(launch_best_reduce(records, n, best_dev, static_cast<cudaStream_t>(stream)));
  return DTB_OK;
}

}  // extern "C"

// ------------------------------------------------------------ trace ingest
namespace {

const char* trace_why(int reason) {
  switch (reason) {
    case JR_SYNTAX: return "syntax error while parsing value";
    case JR_NUMBER_OVERFLOW: return "number overflow";
    case JR_NOT_RECORD: return "record must be an object with text_tokens";
    case JR_TEXT_TYPE: return "text_tokens: type must be number";
    case JR_IMAGE_TYPE: return "image_subseqs: type must be an array of numbers";
    case JR_AUDIO_TYPE: return "audio_subseqs: type must be an array of numbers";
    case JR_NEG_TEXT: return "negative text token count";          // src/core.cpp:102
    case JR_NEG_SUBSEQ: return "negative subsequence token count"; // src/core.cpp:105
    case JR_NO_TOKENS: return "sample has no tokens";              // src/core.cpp:108
    case JR_OVER_CAP: return "sample exceeds the sequence length cap";  // src/core.cpp:110
    case JR_TOO_DEEP: return "nesting deeper than 1024 levels";
    case JR_INT32: return "token count or line length beyond the int32 CSR";
    default: return "unknown";
  }
}

dtb_status trace_capacity(const dtb_trace_csr* out, const dtb_trace_result* res) {
  if (res->n_samples > out->cap_samples || res->n_image > out->cap_image ||
      res->n_audio > out->cap_audio)
    return fail(DTB_ERR_INVALID_ARGUMENT,
                "CSR capacity too small: need %lld samples, %lld image, %lld audio subsequences",
                static_cast<long long>(res->n_samples), static_cast<long long>(res->n_image),
                static_cast<long long>(res->n_audio));
  if ((res->n_image > 0 && out->image_tokens == nullptr) ||
      (res->n_audio > 0 && out->audio_tokens == nullptr))
    return fail(DTB_ERR_INVALID_ARGUMENT, "null CSR token buffer");
  return DTB_OK;
}

// Parses the device byte buffer; on success leaves the CSR in device
// buffers `o` (allocated here when dev_out is null) and the sizes in res.
dtb_status ingest_impl(dtb_context* ctx, const unsigned char* b, long long len, long long cap,
                       const dtb_trace_csr* dev_out, dtb_trace_result* res, DBuf* own) {
  cudaStream_t s = ctx->stream;
  *res = dtb_trace_result{};
  DBuf scratch, nl, st, tx, ia, aa, cn, sc, bad;
  const size_t sb = ingest_lines_scratch(len);
  CU(scratch.alloc(sb, s));
  long long n_nl = 0;
  CU(launch_nl_count(b, len, scratch.p, sb, &n_nl, s));
  long long n_lines = n_nl;
  if (len > 0) {
    unsigned char last = 0;
    CU(cudaMemcpyAsync(&last, b + len - 1, 1, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if (last != '\n') ++n_lines;
  }
  res->n_lines = n_lines;
  CU(nl.alloc(8ull * (n_nl > 0 ? n_nl : 1), s));
  if (n_nl > 0) CU(launch_nl_write(b, len, scratch.p, nl.as<long long>(), s));
  const size_t nL = static_cast<size_t>(n_lines);
  CU(st.alloc(4 * nL, s));
  CU(tx.alloc(8 * nL, s));
  CU(ia.alloc(4 * nL, s));
  CU(aa.alloc(4 * nL, s));
  CU(cn.alloc(12 * (nL + 1), s));
  CU(sc.alloc(12 * (nL + 1), s));
  CU(bad.alloc(8, s));
  CU(cudaMemsetAsync(bad.p, 0xff, 8, s));
  IngestLines L{st.as<int>(), tx.as<long long>(), ia.as<int>(), aa.as<int>(), cn.as<int>(),
                sc.as<int>()};
  CU(launch_ingest_parse(b, len, nl.as<long long>(), n_nl, n_lines, cap, L,
                         bad.as<unsigned long long>(), scratch.p, sb, s));
  unsigned long long first_bad = 0;
  int tot[3] = {0, 0, 0};
  CU(cudaMemcpyAsync(&first_bad, bad.p, 8, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(tot, sc.as<int>() + 3 * nL, 12, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (first_bad != ~0ull) {
    int code = 0;
    CU(cudaMemcpyAsync(&code, st.as<int>() + first_bad, 4, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    const int status = code & 0xff, reason = (code >> 8) & 0xff;
    const int line = static_cast<int>(first_bad + 1);
    res->error_line = line;
    res->error_reason = reason;
    if (status == J_UNSUPPORTED)
      return fail(DTB_ERR_INVALID_ARGUMENT, "line %d: %s", line, trace_why(reason));
    const bool parse = status == J_PARSE;
    res->error_kind = parse ? DTB_TRACE_PARSE_ERROR : DTB_TRACE_INVARIANT_VIOLATION;
    return fail(DTB_ERR_TRACE, "%s at line %d: %s", parse ? "ParseError" : "InvariantViolation",
                line, trace_why(reason));
  }
  res->n_samples = tot[0];
  res->n_image = tot[1];
  res->n_audio = tot[2];
  if (dev_out == nullptr) return DTB_OK;
  if (own == nullptr) TRY(trace_capacity(dev_out, res));
  IngestOut o{};
  if (own != nullptr) {  // library-owned device CSR (host entry point)
    CU(own[0].alloc(4ull * tot[0], s));
    CU(own[1].alloc(4ull * (tot[0] + 1), s));
    CU(own[2].alloc(4ull * tot[1], s));
    CU(own[3].alloc(4ull * (tot[0] + 1), s));
    CU(own[4].alloc(4ull * tot[2], s));
    o = IngestOut{own[0].as<int>(), own[1].as<int>(), own[2].as<int>(), own[3].as<int>(),
                  own[4].as<int>()};
  } else {
    o = IngestOut{dev_out->text_tokens, dev_out->image_offsets, dev_out->image_tokens,
                  dev_out->audio_offsets, dev_out->audio_tokens};
  }
  CU(launch_ingest_write(b, len, nl.as<long long>(), n_nl, n_lines, L, o, s));
  return DTB_OK;
}

dtb_status trace_args(dtb_context* ctx, const char* bytes, int64_t len, int64_t cap,
                      const dtb_trace_csr* out, dtb_trace_result* res, bool* write) {
  TRY(set_device(ctx));
  if (res == nullptr || (bytes == nullptr && len > 0) || len < 0)
    return fail(DTB_ERR_INVALID_ARGUMENT, "null result / byte buffer");
  *write = out != nullptr && out->text_tokens != nullptr;
  if (*write && (out->image_offsets == nullptr || out->audio_offsets == nullptr))
    return fail(DTB_ERR_INVALID_ARGUMENT, "null CSR offsets");
  (void)cap;
  return DTB_OK;
}

}  // namespace

extern "C" {

dtb_status dtb_ingest_trace_dev(dtb_context* ctx, const char* bytes, int64_t len,
                                int64_t seq_len_cap, const dtb_trace_csr* out,
                                dtb_trace_result* res) {
  bool write = false;
  TRY(trace_args(ctx, bytes, len, seq_len_cap, out, res, &write));
  TRY(ingest_impl(ctx, reinterpret_cast<const unsigned char*>(bytes), len, seq_len_cap,
                  write ? out : nullptr, res, nullptr));
  CU(cudaStreamSynchronize(ctx->stream));
  return DTB_OK;
}

dtb_status dtb_ingest_trace(dtb_context* ctx, const char* bytes, int64_t len,
                            int64_t seq_len_cap, const dtb_trace_csr* out,
                            dtb_trace_result* res) {
  bool write = false;
  TRY(trace_args(ctx, bytes, len, seq_len_cap, out, res, &write));
  DBuf db;
  TRY(upload(db, reinterpret_cast<const unsigned char*>(bytes), static_cast<size_t>(len),
             ctx->stream));
  DBuf own[5];
  dtb_trace_csr dummy{};
  TRY(ingest_impl(ctx, db.as<unsigned char>(), len, seq_len_cap, write ? &dummy : nullptr, res,
                  own));
  if (!write) return DTB_OK;
  TRY(trace_capacity(out, res));
  TRY(download(out->text_tokens, own[0], static_cast<size_t>(res->n_samples), ctx->stream));
  TRY(download(out->image_offsets, own[1], static_cast<size_t>(res->n_samples + 1), ctx->stream));
  TRY(download(out->image_tokens, own[2], static_cast<size_t>(res->n_image), ctx->stream));
  TRY(download(out->audio_offsets, own[3], static_cast<size_t>(res->n_samples + 1), ctx->stream));
  TRY(download(out->audio_tokens, own[4], static_cast<size_t>(res->n_audio), ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return DTB_OK;
}

}  // extern "C"

// ---------------------------------------------------------- CUDA graphs
struct dtb_graph {
  int device = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};

dtb_status dtb_reorder_stream_graph_create(dtb_context* ctx, const dtb_cost_model* cm,
                                           const dtb_plan* plan, const dtb_reorder_mode* mode,
                                           const dtb_samples* samples, int64_t n_batches,
                                           dtb_peer_group* group, int32_t* output_order,
                                           double* load_before, double* load_after,
                                           double* t_iter_before, double* t_iter_after,
                                           uint8_t* greedy_kept, dtb_graph** out) {
  TRY(set_device(ctx));
  if (out == nullptr) return fail(DTB_ERR_INVALID_ARGUMENT, "null graph output");
  cudaStream_t cs = nullptr;
  CU(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  dtb_status st = DTB_OK;
  cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess) {
    st = group ? dtb_reorder_stream_shard_dev(ctx, cm, plan, mode, samples, n_batches, group,
                                              load_before, load_after, t_iter_before,
                                              t_iter_after, greedy_kept, cs)
               : dtb_reorder_stream_dev(ctx, cm, plan, mode, samples, n_batches, output_order,
                                        load_before, load_after, t_iter_before, t_iter_after,
                                        greedy_kept, cs);
    cudaGraph_t g = nullptr;
    const cudaError_t e2 = cudaStreamEndCapture(cs, &g);
    if (st == DTB_OK && e2 == cudaSuccess) {
      auto* gr = new dtb_graph;
      gr->device = ctx->device;
      gr->graph = g;
      e = cudaGraphInstantiate(&gr->exec, g, 0);
      if (e != cudaSuccess) {
        cudaGraphDestroy(g);
        delete gr;
      } else {
        *out = gr;
      }
    } else {
      if (g) cudaGraphDestroy(g);
      if (st == DTB_OK) e = e2;
    }
  }
  cudaStreamDestroy(cs);
  if (st != DTB_OK) return st;
  CU(e);
  return DTB_OK;
}

dtb_status dtb_graph_launch(dtb_graph* g, void* stream) {
  if (g == nullptr) return fail(DTB_ERR_INVALID_ARGUMENT, "null graph");
  CU(cudaSetDevice(g->device));
  CU(cudaGraphLaunch(g->exec, static_cast<cudaStream_t>(stream)));
  return DTB_OK;
}

dtb_status dtb_graph_destroy(dtb_graph* g) {
  if (g == nullptr) return DTB_OK;
  cudaSetDevice(g->device);
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  delete g;
  return DTB_OK;
}

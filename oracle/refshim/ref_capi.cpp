// ORACLE — test infrastructure only.  Never linked into or called by the
// product path (paper_2408_04275_b200/).  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load it.
//
// Exposes the UNMODIFIED reference planner (compiled from
// /root/reference/proj/core/src/*.cpp by oracle/Makefile into
// oracle/_ref/libmmplan_ref.so) behind the same C ABI as
// include/disttrain_b200.h, with the prefix `mmref_` instead of `dtb_`.
// Every function is a thin marshalling layer: CSR / POD -> mmplan types ->
// the reference call -> POD.  No algorithmic code lives here.
#include <algorithm>
#include <numeric>
#include <atomic>
#include <chrono>
#include <cstring>
#include <exception>
#include <memory>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "disttrain_b200.h"
#include "mmplan/core.hpp"
#include "mmplan/cost_model.hpp"
#include "mmplan/errors.hpp"
#include "mmplan/orchestrator.hpp"
#include "mmplan/pipeline_sim.hpp"
#include "mmplan/reorder.hpp"
#include "mmplan/simulate.hpp"
#include "mmplan/workload.hpp"

using namespace mmplan;

#define API(name) mmref_##name

namespace {

thread_local std::string g_err;
int g_threads = 1;

dtb_status fail(dtb_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

template <typename F>
dtb_status guarded(F&& f) {
  try {
    f();
    return DTB_OK;
  } catch (const InfeasibleError& e) {
    return fail(DTB_ERR_INFEASIBLE, e.what());
  } catch (const EmptyProfileError& e) {
    return fail(DTB_ERR_EMPTY_PROFILE, e.what());
  } catch (const ConfigError& e) {
    return fail(DTB_ERR_CONFIG, e.what());
  } catch (const KTooLargeError& e) {
    return fail(DTB_ERR_K_TOO_LARGE, e.what());
  } catch (const IndivisibleVppError& e) {
    return fail(DTB_ERR_INDIVISIBLE_VPP, e.what());
  } catch (const BatchSizeMismatchError& e) {
    return fail(DTB_ERR_BATCH_SIZE_MISMATCH, e.what());
  } catch (const CapExceededError& e) {
    return fail(DTB_ERR_CAP_EXCEEDED, e.what());
  } catch (const InternalError& e) {
    return fail(DTB_ERR_INTERNAL, e.what());
  } catch (const std::exception& e) {
    return fail(DTB_ERR_INTERNAL, e.what());
  }
}

ModuleKind kind_of(int32_t m) { return static_cast<ModuleKind>(m); }

ModelSpec to_model(const dtb_model_spec& m) {
  ModelSpec out;
  for (int u = 0; u < 3; ++u) {
    ModuleSpec& ms = out.module(kind_of(u));
    const dtb_module_spec& src = m.unit[u];
    ms.arch.layers = src.arch.layers;
    ms.arch.hidden = src.arch.hidden;
    ms.arch.ffn_hidden = src.arch.ffn_hidden;
    ms.arch.heads = src.arch.heads;
    ms.arch.groups = src.arch.groups;
    ms.mem.param_grad_bytes = src.mem.param_grad_bytes;
    ms.mem.optimizer_bytes = src.mem.optimizer_bytes;
    ms.mem.activation_bytes_per_mb = src.mem.activation_bytes_per_mb;
    ms.frozen = src.frozen != 0;
  }
  out.seq_len = m.seq_len;
  out.frozen_backward_factor = m.frozen_backward_factor;
  out.dp_sync_seconds = m.dp_sync_seconds;
  return out;
}

ClusterSpec to_cluster(const dtb_cluster_spec& c) {
  ClusterSpec out;
  out.total_gpus = c.total_gpus;
  out.gpus_per_node = c.gpus_per_node;
  out.peak_flops = c.peak_flops;
  out.gpu_mem_bytes = c.gpu_mem_bytes;
  out.intra_node_bw = c.intra_node_bw;
  out.inter_node_bw = c.inter_node_bw;
  return out;
}

Plan to_plan(const dtb_plan& p) {
  Plan out;
  for (int u = 0; u < 3; ++u) {
    out.unit(kind_of(u)) = {p.unit[u].tp, p.unit[u].dp, p.unit[u].pp};
  }
  out.global_batch = p.global_batch;
  out.vpp = p.vpp;
  return out;
}

dtb_plan from_plan(const Plan& p) {
  dtb_plan out{};
  for (int u = 0; u < 3; ++u) {
    const ParallelismChoice& pc = p.unit(kind_of(u));
    out.unit[u] = {pc.tp, pc.dp, pc.pp};
  }
  out.global_batch = p.global_batch;
  out.vpp = p.vpp;
  return out;
}

WorkloadStats to_stats(const dtb_workload_stats& s) {
  WorkloadStats out;
  out.seq_len = s.seq_len;
  out.mean_encoder_tokens = s.mean_encoder_tokens;
  out.mean_generator_tokens = s.mean_generator_tokens;
  return out;
}

ParallelismTuple to_tuple(const dtb_tuple& t) {
  ParallelismTuple out;
  out.tp_me = t.tp_me;
  out.dp_me = t.dp_me;
  out.tp_lm = t.tp_lm;
  out.dp_lm = t.dp_lm;
  out.tp_mg = t.tp_mg;
  out.dp_mg = t.dp_mg;
  return out;
}

dtb_tuple from_tuple(const ParallelismTuple& t) {
  return dtb_tuple{t.tp_me, t.dp_me, t.tp_lm, t.dp_lm, t.tp_mg, t.dp_mg};
}

std::vector<Sample> to_samples(const dtb_samples& s, int64_t begin,
                               int64_t count) {
  std::vector<Sample> out(static_cast<std::size_t>(count));
  for (int64_t i = 0; i < count; ++i) {
    const int64_t g = begin + i;
    Sample& smp = out[static_cast<std::size_t>(i)];
    smp.text_tokens = s.text_tokens ? s.text_tokens[g] : 0;
    for (int32_t k = s.image_offsets[g]; k < s.image_offsets[g + 1]; ++k) {
      smp.image_subseqs.push_back(s.image_tokens[k]);
    }
    if (s.audio_offsets != nullptr) {
      for (int32_t k = s.audio_offsets[g]; k < s.audio_offsets[g + 1]; ++k) {
        smp.audio_subseqs.push_back(s.audio_tokens[k]);
      }
    }
  }
  return out;
}

std::vector<Microbatch> to_microbatches(const dtb_microbatches& m,
                                        int64_t begin, int64_t count) {
  std::vector<Microbatch> out(static_cast<std::size_t>(count));
  for (int64_t i = 0; i < count; ++i) {
    Microbatch& mb = out[static_cast<std::size_t>(i)];
    mb.samples.resize(static_cast<std::size_t>(m.sample_count[begin + i]));
    mb.encoder_tokens = m.encoder_tokens[begin + i];
    mb.generator_tokens = m.generator_tokens[begin + i];
  }
  return out;
}

StageTimes to_times(const double* fwd, const double* bwd, int32_t l,
                    int32_t p) {
  StageTimes t = StageTimes::zeros(l, p);
  std::copy(fwd, fwd + static_cast<std::size_t>(l) * p, t.fwd.begin());
  std::copy(bwd, bwd + static_cast<std::size_t>(l) * p, t.bwd.begin());
  return t;
}

int32_t reason_code(const std::string& r) {
  if (r.empty()) return DTB_REASON_NONE;
  if (r == "dp does not divide the global batch")
    return DTB_REASON_DP_NOT_DIVIDING;
  if (r.rfind("activation memory of encoder", 0) == 0)
    return DTB_REASON_ACTIVATION_ENCODER;
  if (r.rfind("activation memory of backbone", 0) == 0)
    return DTB_REASON_ACTIVATION_BACKBONE;
  if (r.rfind("activation memory of generator", 0) == 0)
    return DTB_REASON_ACTIVATION_GENERATOR;
  if (r == "memory floor exceeds the cluster") return DTB_REASON_MEMORY_FLOOR;
  if (r == "no integer stage split is feasible")
    return DTB_REASON_NO_INTEGER_SPLIT;
  return -1;
}

dtb_candidate from_candidate(const CandidateResult& c) {
  dtb_candidate out{};
  out.tuple = from_tuple(c.tuple);
  out.feasible = c.feasible ? 1 : 0;
  out.reason = reason_code(c.infeasible_reason);
  out.plan = from_plan(c.plan);
  out.times = {c.times.t_warm, c.times.t_steady, c.times.t_iter};
  out.cont_x = c.cont_x;
  out.cont_y = c.cont_y;
  out.cont_z = c.cont_z;
  out.cont_t_iter = c.cont_t_iter;
  return out;
}

// Runs fn(i) for i in [0, n) on g_threads host threads (contiguous chunks).
template <typename F>
void parallel_for(int64_t n, F&& fn) {
  const int nt = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>(g_threads, n)));
  if (nt <= 1) {
    for (int64_t i = 0; i < n; ++i) fn(i);
    return;
  }
  std::vector<std::thread> pool;
  std::vector<std::exception_ptr> errs(nt);
  for (int t = 0; t < nt; ++t) {
    pool.emplace_back([&, t] {
      try {
        const int64_t lo = n * t / nt, hi = n * (t + 1) / nt;
        for (int64_t i = lo; i < hi; ++i) fn(i);
      } catch (...) {
        errs[t] = std::current_exception();
      }
    });
  }
  for (auto& th : pool) th.join();
  for (auto& e : errs) {
    if (e) std::rethrow_exception(e);
  }
}

}  // namespace

struct dtb_context {
  int device = -1;
  bool warn_on = false;
  std::vector<std::string> warnings;  // the reference CostModel's warning sink
};
struct dtb_cost_model {
  std::unique_ptr<CostModel> cm;
};

namespace {
// While the context's warning log is on, the call's CostModel appends to it
// (CostModel::set_warning_sink; the sink makes the model non-reentrant, so
// the batch fan-out runs on one thread meanwhile).
struct Sink {
  CostModel* cm = nullptr;
  int saved_threads = 0;
  Sink(dtb_context* ctx, const dtb_cost_model* h) {
    if (ctx != nullptr && ctx->warn_on) {
      cm = h->cm.get();
      cm->set_warning_sink(&ctx->warnings);
      saved_threads = g_threads;
      g_threads = 1;
    }
  }
  ~Sink() {
    if (cm != nullptr) {
      cm->set_warning_sink(nullptr);
      g_threads = saved_threads;
    }
  }
};
}  // namespace

extern "C" {

const char* API(last_error)(void) { return g_err.c_str(); }
int API(abi_version)(void) { return DTB_ABI_VERSION; }

// Host threads used by the batched / stream entry points (CPU baseline).
void API(set_threads)(int n) { g_threads = n < 1 ? 1 : n; }

dtb_status API(context_create)(int32_t device, dtb_context** out) {
  *out = new dtb_context{device};
  return DTB_OK;
}
dtb_status API(context_destroy)(dtb_context* ctx) {
  delete ctx;
  return DTB_OK;
}

dtb_status API(warnings_enable)(dtb_context* ctx, int32_t on) {
  ctx->warn_on = on != 0;
  ctx->warnings.clear();
  return DTB_OK;
}
int64_t API(warnings_count)(const dtb_context* ctx) {
  return static_cast<int64_t>(ctx->warnings.size());
}
const char* API(warning_at)(const dtb_context* ctx, int64_t i) {
  if (i < 0 || i >= static_cast<int64_t>(ctx->warnings.size())) return nullptr;
  return ctx->warnings[static_cast<std::size_t>(i)].c_str();
}
dtb_status API(warnings_clear)(dtb_context* ctx) {
  ctx->warnings.clear();
  return DTB_OK;
}

dtb_status API(cost_model_create)(dtb_context*, const dtb_model_spec* model,
                                  const dtb_cluster_spec* cluster,
                                  const dtb_costbook* book,
                                  dtb_cost_model** out) {
  return guarded([&] {
    CostBook cb;
    cb.analytic.efficiency = book->analytic_efficiency;
    cb.analytic.bwd_fwd_ratio = book->analytic_bwd_fwd_ratio;
    for (int64_t i = 0; i < book->n_rows; ++i) {
      const dtb_profile_row& r = book->rows[i];
      std::optional<double> bwd;
      if (r.has_bwd) bwd = r.bwd_s;
      cb.profile(kind_of(r.module)).add_row(r.tp, r.token_load, r.fwd_s, bwd);
    }
    auto* h = new dtb_cost_model;
    h->cm = std::make_unique<CostModel>(to_model(*model), to_cluster(*cluster),
                                        std::move(cb));
    *out = h;
  });
}
dtb_status API(cost_model_destroy)(dtb_cost_model* cm) {
  delete cm;
  return DTB_OK;
}

dtb_status API(cost_sizes)(dtb_context*, const dtb_samples* s, int64_t* out) {
  return guarded([&] {
    const auto samples = to_samples(*s, 0, s->n);
    for (int64_t i = 0; i < s->n; ++i) out[i] = samples[i].cost_size();
  });
}

dtb_status API(unit_times)(dtb_context* ctx, const dtb_cost_model* cm,
                           int32_t module, int32_t tp, int64_t n,
                           const double* loads, double* fwd, double* bwd) {
  const Sink sink(ctx, cm);
  return guarded([&] {
    for (int64_t i = 0; i < n; ++i) {
      if (fwd) fwd[i] = cm->cm->unit_forward_time(kind_of(module), tp, loads[i]);
      if (bwd) bwd[i] = cm->cm->unit_backward_time(kind_of(module), tp, loads[i]);
    }
  });
}

dtb_status API(memory_check)(dtb_context*, const dtb_cost_model* cm,
                             const dtb_plan* plan, dtb_memory_report* out) {
  return guarded([&] {
    const MemoryReport r =
        memory_check(to_plan(*plan), cm->cm->model(), cm->cm->cluster());
    for (int u = 0; u < 3; ++u) {
      out->bytes_per_gpu[u] = r.units[u].bytes_per_gpu;
      out->fits[u] = r.units[u].fits ? 1 : 0;
    }
    out->pass = r.pass ? 1 : 0;
    out->capacity_bytes = r.capacity_bytes;
  });
}

dtb_status API(build_stage_times)(dtb_context* ctx, const dtb_cost_model* cm,
                                  const dtb_plan* plan,
                                  const dtb_microbatches* mbs, double* fwd,
                                  double* bwd) {
  const Sink sink(ctx, cm);
  return guarded([&] {
    const auto v = to_microbatches(*mbs, 0, mbs->n);
    const StageTimes t = cm->cm->build_stage_times(to_plan(*plan), v);
    std::copy(t.fwd.begin(), t.fwd.end(), fwd);
    std::copy(t.bwd.begin(), t.bwd.end(), bwd);
  });
}

dtb_status API(microbatch_fwd_keys)(dtb_context* ctx, const dtb_cost_model* cm,
                                    const dtb_plan* plan,
                                    const dtb_microbatches* mbs, double* keys) {
  const Sink sink(ctx, cm);
  return guarded([&] {
    const auto v = to_microbatches(*mbs, 0, mbs->n);
    const auto k = microbatch_fwd_keys(to_plan(*plan), *cm->cm, v);
    std::copy(k.begin(), k.end(), keys);
  });
}

dtb_status API(compute_stats)(dtb_context*, const dtb_samples* s,
                              int64_t seq_len, dtb_workload_stats* out) {
  return guarded([&] {
    const WorkloadStats st = compute_stats(to_samples(*s, 0, s->n), seq_len);
    out->seq_len = st.seq_len;
    out->mean_encoder_tokens = st.mean_encoder_tokens;
    out->mean_generator_tokens = st.mean_generator_tokens;
  });
}

dtb_status API(intra_partition)(dtb_context*, const double* sizes, int64_t n,
                                int32_t m, int32_t order, int32_t equal_counts,
                                int32_t* flat_out, int64_t* offsets) {
  return guarded([&] {
    const IntraPartition part = intra_partition(
        std::span<const double>(sizes, static_cast<std::size_t>(n)), m,
        order == DTB_DESCENDING ? IntraSortOrder::Descending
                                : IntraSortOrder::Ascending,
        equal_counts != 0);
    int64_t pos = 0;
    offsets[0] = 0;
    for (std::size_t g = 0; g < part.groups.size(); ++g) {
      for (int idx : part.groups[g]) flat_out[pos++] = idx;
      offsets[g + 1] = pos;
    }
  });
}

dtb_status API(block_group_loads)(dtb_context*, const double* sizes,
                                  const int32_t* order, int64_t n, int32_t m,
                                  double* loads) {
  return guarded([&] {
    const auto v = block_group_loads(
        std::span<const double>(sizes, static_cast<std::size_t>(n)),
        std::span<const int>(order, static_cast<std::size_t>(n)), m);
    std::copy(v.begin(), v.end(), loads);
  });
}

dtb_status API(select_min)(dtb_context*, const double* keys, int64_t n_keys,
                           const int32_t* pending, int64_t n_pending, int32_t k,
                           int32_t* out) {
  return guarded([&] {
    const std::vector<int> pend(pending, pending + n_pending);
    const auto v = select_min(
        std::span<const double>(keys, static_cast<std::size_t>(n_keys)), pend,
        k);
    std::copy(v.begin(), v.end(), out);
  });
}

dtb_status API(select_closest)(dtb_context*, const double* keys,
                               int64_t n_keys, const int32_t* pending,
                               int64_t n_pending, int32_t k, double target,
                               int32_t* out) {
  return guarded([&] {
    const std::vector<int> pend(pending, pending + n_pending);
    const auto v = select_closest(
        std::span<const double>(keys, static_cast<std::size_t>(n_keys)), pend,
        k, target);
    std::copy(v.begin(), v.end(), out);
  });
}

dtb_status API(schedule)(dtb_context*, const double* fwd, const double* bwd,
                         int32_t l, int32_t p, int32_t vpp, int32_t* ev_device,
                         int32_t* ev_mb, int32_t* ev_stage, int32_t* ev_phase,
                         double* ev_start, double* ev_end,
                         double* iteration_time, double* device_busy) {
  return guarded([&] {
    const StageTimes t = to_times(fwd, bwd, l, p);
    const Timeline tl =
        vpp == 1 ? schedule_1f1b(t) : schedule_interleaved(t, vpp);
    for (std::size_t i = 0; i < tl.events.size(); ++i) {
      const TimelineEvent& e = tl.events[i];
      if (ev_device) ev_device[i] = e.device;
      if (ev_mb) ev_mb[i] = e.microbatch;
      if (ev_stage) ev_stage[i] = e.stage;
      if (ev_phase) ev_phase[i] = static_cast<int32_t>(e.phase);
      if (ev_start) ev_start[i] = e.start;
      if (ev_end) ev_end[i] = e.end;
    }
    if (iteration_time) *iteration_time = tl.iteration_time;
    if (device_busy) {
      std::copy(tl.device_busy.begin(), tl.device_busy.end(), device_busy);
    }
  });
}

dtb_status API(get_intervals)(dtb_context*, int64_t n_events,
                              const int32_t* ev_device, const int32_t* ev_mb,
                              const int32_t* ev_stage, const int32_t* ev_phase,
                              const double* ev_start, const double* ev_end,
                              int64_t* n_intervals, double* starts,
                              double* ends, int64_t* fill_offsets,
                              int32_t* fill_mb) {
  return guarded([&] {
    Timeline tl;
    for (int64_t i = 0; i < n_events; ++i) {
      tl.events.push_back({ev_device[i], ev_mb[i], ev_stage[i],
                           static_cast<Phase>(ev_phase[i]), ev_start[i],
                           ev_end[i]});
    }
    const IntervalSet set = get_intervals(tl);
    *n_intervals = static_cast<int64_t>(set.intervals.size());
    int64_t f = 0;
    fill_offsets[0] = 0;
    for (std::size_t i = 0; i < set.intervals.size(); ++i) {
      starts[i] = set.intervals[i].start;
      ends[i] = set.intervals[i].end;
      for (int mb : set.intervals[i].filled_by) fill_mb[f++] = mb;
      fill_offsets[i + 1] = f;
    }
  });
}

dtb_status API(interval_windows)(dtb_context*, const double* fwd,
                                 const double* bwd, int32_t l, int32_t p,
                                 double* volumes) {
  return guarded([&] {
    const auto v = interval_windows(to_times(fwd, bwd, l, p));
    std::copy(v.begin(), v.end(), volumes);
  });
}

dtb_status API(schedule_batch)(dtb_context*, int64_t batch, const double* fwd,
                               const double* bwd, int32_t l, int32_t p,
                               int32_t vpp, double* iteration_time,
                               double* device_busy) {
  return guarded([&] {
    const std::size_t cells = static_cast<std::size_t>(l) * p;
    parallel_for(batch, [&](int64_t b) {
      const StageTimes t = to_times(fwd + b * cells, bwd + b * cells, l, p);
      const Timeline tl =
          vpp == 1 ? schedule_1f1b(t) : schedule_interleaved(t, vpp);
      iteration_time[b] = tl.iteration_time;
      if (device_busy) {
        std::copy(tl.device_busy.begin(), tl.device_busy.end(),
                  device_busy + b * tl.device_busy.size());
      }
    });
  });
}

dtb_status API(exhaustive_order)(dtb_context*, const double* fwd, const double* bwd,
                                 int32_t l, int32_t p, int32_t vpp, double* best_time,
                                 int32_t* best_order, double* all_times) {
  return guarded([&] {
    if (l < 1 || l > 12) throw InternalError("exhaustive_order needs 1 <= l <= 12");
    const StageTimes t = to_times(fwd, bwd, l, p);
    // tests/test_reorder.cpp:55-59 (sim_time) + :226-232 (the permutation loop)
    std::vector<int> perm(l);
    std::iota(perm.begin(), perm.end(), 0);
    double best = 1e300;
    std::vector<int> arg = perm;
    int64_t k = 0;
    do {
      const StageTimes permuted = t.permuted(perm);
      const double it = vpp > 1 ? schedule_interleaved(permuted, vpp).iteration_time
                                : schedule_1f1b(permuted).iteration_time;
      if (all_times) all_times[k] = it;
      if (it < best) {
        best = it;
        arg = perm;
      }
      ++k;
    } while (std::next_permutation(perm.begin(), perm.end()));
    *best_time = best;
    std::copy(arg.begin(), arg.end(), best_order);
  });
}

dtb_status API(simulate_iteration)(dtb_context* ctx, const dtb_cost_model* cm,
                                   const dtb_plan* plan, int32_t n_groups,
                                   const int64_t* group_offsets,
                                   const dtb_microbatches* mbs, double* t_iter,
                                   double* group_times, int32_t* slowest_group,
                                   double* slowest_time, double* bubble) {
  const Sink sink(ctx, cm);
  return guarded([&] {
    std::vector<std::vector<Microbatch>> groups;
    for (int32_t g = 0; g < n_groups; ++g) {
      groups.push_back(to_microbatches(*mbs, group_offsets[g],
                                       group_offsets[g + 1] - group_offsets[g]));
    }
    const IterationResult r = simulate_iteration(to_plan(*plan), *cm->cm, groups);
    if (t_iter) *t_iter = r.t_iter;
    if (group_times) {
      std::copy(r.group_times.begin(), r.group_times.end(), group_times);
    }
    if (slowest_group) *slowest_group = r.slowest_group;
    if (slowest_time) *slowest_time = r.slowest_group_time;
    if (bubble) *bubble = r.mean_bubble_fraction;
  });
}

dtb_status API(inter_reorder)(dtb_context*, const double* fwd,
                              const double* bwd, int32_t l, int32_t p,
                              const double* keys, int32_t vpp,
                              int32_t* order_out) {
  return guarded([&] {
    const auto v = inter_reorder(
        to_times(fwd, bwd, l, p),
        std::span<const double>(keys, static_cast<std::size_t>(l)), vpp);
    std::copy(v.begin(), v.end(), order_out);
  });
}

dtb_status API(inter_reorder_batch)(dtb_context*, int64_t batch,
                                    const double* fwd, const double* bwd,
                                    int32_t l, int32_t p, const double* keys,
                                    int32_t vpp, int32_t* orders) {
  return guarded([&] {
    const std::size_t cells = static_cast<std::size_t>(l) * p;
    parallel_for(batch, [&](int64_t b) {
      const auto v = inter_reorder(
          to_times(fwd + b * cells, bwd + b * cells, l, p),
          std::span<const double>(keys + b * l, static_cast<std::size_t>(l)),
          vpp);
      std::copy(v.begin(), v.end(), orders + b * l);
    });
  });
}

static ReorderMode to_mode(const dtb_reorder_mode* m) {
  ReorderMode mode;
  if (m != nullptr) {
    mode.intra = m->intra != 0;
    mode.inter = m->inter != 0;
    mode.sort_order = m->sort_order == DTB_DESCENDING
                          ? IntraSortOrder::Descending
                          : IntraSortOrder::Ascending;
  }
  return mode;
}

dtb_status API(disaggregated_reorder)(dtb_context* ctx, const dtb_cost_model* cm,
                                      const dtb_plan* plan,
                                      const dtb_reorder_mode* mode,
                                      const dtb_samples* batch,
                                      dtb_reorder_report* report) {
  const Sink sink(ctx, cm);
  return guarded([&] {
    const auto samples = to_samples(*batch, 0, batch->n);
    const DisaggregatedResult r = disaggregated_reorder(
        samples, to_plan(*plan), *cm->cm, to_mode(mode));
    std::copy(r.report.output_order.begin(), r.report.output_order.end(),
              report->output_order);
    std::copy(r.report.group_load_before.begin(),
              r.report.group_load_before.end(), report->group_load_before);
    std::copy(r.report.group_load_after.begin(),
              r.report.group_load_after.end(), report->group_load_after);
    report->t_iter_before = r.report.t_iter_before;
    report->t_iter_after = r.report.t_iter_after;
  });
}

// Stream of independent global batches; with set_threads(n) the batches are
// fanned out over n host threads (each batch is one untouched reference
// call).  greedy_kept is derived from the report (loads_after differ from
// identity's only when the greedy split was kept).
struct mmref_stream {
  std::vector<std::vector<Sample>> batches;
};

dtb_status API(stream_prepare)(const dtb_samples* samples, int64_t n_batches,
                               mmref_stream** out) {
  return guarded([&] {
    auto* h = new mmref_stream;
    const int64_t bs = samples->n / n_batches;
    h->batches.resize(static_cast<std::size_t>(n_batches));
    for (int64_t b = 0; b < n_batches; ++b) {
      h->batches[b] = to_samples(*samples, b * bs, bs);
    }
    *out = h;
  });
}
dtb_status API(stream_destroy)(mmref_stream* h) {
  delete h;
  return DTB_OK;
}

dtb_status API(stream_run)(mmref_stream* h, const dtb_cost_model* cm,
                           const dtb_plan* plan, const dtb_reorder_mode* mode,
                           int64_t first_batch, int64_t n_batches,
                           int32_t* output_order, double* load_before,
                           double* load_after, double* t_before,
                           double* t_after) {
  return guarded([&] {
    const Plan pl = to_plan(*plan);
    const ReorderMode md = to_mode(mode);
    const int64_t bs = pl.global_batch;
    const int dp = pl.backbone.dp;
    parallel_for(n_batches, [&](int64_t i) {
      const int64_t b = first_batch + i;
      const DisaggregatedResult r =
          disaggregated_reorder(h->batches[b], pl, *cm->cm, md);
      if (output_order) {
        std::copy(r.report.output_order.begin(), r.report.output_order.end(),
                  output_order + i * bs);
      }
      if (load_before) {
        std::copy(r.report.group_load_before.begin(),
                  r.report.group_load_before.end(), load_before + i * dp);
      }
      if (load_after) {
        std::copy(r.report.group_load_after.begin(),
                  r.report.group_load_after.end(), load_after + i * dp);
      }
      if (t_before) t_before[i] = r.report.t_iter_before;
      if (t_after) t_after[i] = r.report.t_iter_after;
    });
  });
}

dtb_status API(reorder_stream)(dtb_context* ctx, const dtb_cost_model* cm,
                               const dtb_plan* plan,
                               const dtb_reorder_mode* mode,
                               const dtb_samples* samples, int64_t n_batches,
                               int32_t* output_order, double* load_before,
                               double* load_after, double* t_before,
                               double* t_after, uint8_t* greedy_kept) {
  const Sink sink(ctx, cm);
  mmref_stream* h = nullptr;
  dtb_status st = API(stream_prepare)(samples, n_batches, &h);
  if (st != DTB_OK) return st;
  st = API(stream_run)(h, cm, plan, mode, 0, n_batches, output_order,
                       load_before, load_after, t_before, t_after);
  delete h;
  if (st == DTB_OK && greedy_kept != nullptr) {
    (void)greedy_kept;  // not observable through the reference API
    return fail(DTB_ERR_INVALID_ARGUMENT,
                "greedy_kept is not exposed by the reference");
  }
  return st;
}

dtb_status API(predict_times)(dtb_context*, const dtb_cost_model* cm,
                              const dtb_workload_stats* stats,
                              const dtb_plan* plans, int64_t n,
                              dtb_predicted_times* out) {
  return guarded([&] {
    const WorkloadStats st = to_stats(*stats);
    for (int64_t i = 0; i < n; ++i) {
      const PredictedTimes t = predict_times(to_plan(plans[i]), *cm->cm, st);
      out[i] = {t.t_warm, t.t_steady, t.t_iter};
    }
  });
}

dtb_status API(enumerate_parallelism)(dtb_context*,
                                      const dtb_cluster_spec* cluster,
                                      int64_t bs, int64_t* count,
                                      dtb_tuple* tuples, int64_t capacity) {
  return guarded([&] {
    const auto v = enumerate_parallelism(to_cluster(*cluster), bs);
    *count = static_cast<int64_t>(v.size());
    if (tuples != nullptr) {
      const int64_t k = std::min<int64_t>(capacity, *count);
      for (int64_t i = 0; i < k; ++i) tuples[i] = from_tuple(v[i]);
    }
  });
}

dtb_status API(solve_subproblem)(dtb_context*, const dtb_cost_model* cm,
                                 const dtb_workload_stats* stats,
                                 const dtb_tuple* tuples, int64_t n,
                                 int64_t bs, int32_t vpp, dtb_candidate* out) {
  return guarded([&] {
    const WorkloadStats st = to_stats(*stats);
    parallel_for(n, [&](int64_t i) {
      out[i] = from_candidate(
          solve_subproblem(to_tuple(tuples[i]), *cm->cm, st, bs, vpp));
    });
  });
}

dtb_status API(model_orchestration)(dtb_context*, const dtb_cost_model* cm,
                                    const dtb_workload_stats* stats,
                                    int64_t bs, int32_t vpp,
                                    dtb_orchestration_result* result,
                                    dtb_candidate* candidates,
                                    int64_t capacity) {
  return guarded([&] {
    OrchestrationOptions opts;
    opts.vpp = vpp;
    opts.keep_candidates = candidates != nullptr;
    const OrchestrationResult r =
        model_orchestration(*cm->cm, to_stats(*stats), bs, opts);
    result->best = from_plan(r.best);
    result->times = {r.times.t_warm, r.times.t_steady, r.times.t_iter};
    result->candidates_evaluated =
        static_cast<int64_t>(r.candidates_evaluated);
    result->solve_seconds = r.solve_seconds;
    if (candidates != nullptr) {
      const int64_t k =
          std::min<int64_t>(capacity, static_cast<int64_t>(r.candidates.size()));
      for (int64_t i = 0; i < k; ++i) candidates[i] = from_candidate(r.candidates[i]);
    }
  });
}

dtb_status API(brute_force_oracle)(dtb_context*, const dtb_cost_model* cm,
                                   const dtb_workload_stats* stats, int64_t bs, int32_t vpp,
                                   int32_t gpu_cap, dtb_orchestration_result* result) {
  return guarded([&] {
    BruteForceOptions opts;
    opts.vpp = vpp;
    opts.gpu_cap = gpu_cap;
    const OrchestrationResult r = brute_force_oracle(*cm->cm, to_stats(*stats), bs, opts);
    result->best = from_plan(r.best);
    result->times = {r.times.t_warm, r.times.t_steady, r.times.t_iter};
    result->candidates_evaluated = static_cast<int64_t>(r.candidates_evaluated);
    result->solve_seconds = r.solve_seconds;
  });
}

dtb_status API(rigid_baseline)(dtb_context*, const dtb_cost_model* cm,
                               const dtb_workload_stats* stats, int64_t bs, int32_t vpp,
                               dtb_plan* plan) {
  return guarded([&] { *plan = from_plan(rigid_baseline(*cm->cm, to_stats(*stats), bs, vpp)); });
}

// Multi-threaded CPU baseline of model_orchestration: the reference's own
// enumerate_parallelism + solve_subproblem per tuple, fanned out over
// set_threads(n) host threads, folded with the reference's tie-break order
// (t_iter, total_gpus, tuple, pp triple).  Same result as the serial call.
dtb_status API(model_orchestration_mt)(dtb_context*, const dtb_cost_model* cm,
                                       const dtb_workload_stats* stats,
                                       int64_t bs, int32_t vpp,
                                       dtb_orchestration_result* result) {
  return guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    const WorkloadStats st = to_stats(*stats);
    const auto tuples = enumerate_parallelism(cm->cm->cluster(), bs);
    const int nt = std::max(1, g_threads);
    std::vector<CandidateResult> best(nt);
    std::vector<char> has(nt, 0);
    const auto better = [](const CandidateResult& a, const CandidateResult& b) {
      if (a.times.t_iter != b.times.t_iter) return a.times.t_iter < b.times.t_iter;
      const auto key = [](const CandidateResult& c) {
        return std::make_tuple(c.plan.total_gpus(), c.tuple, c.plan.encoder.pp,
                               c.plan.backbone.pp, c.plan.generator.pp);
      };
      return key(a) < key(b);
    };
    std::vector<std::thread> pool;
    const int64_t n = static_cast<int64_t>(tuples.size());
    for (int t = 0; t < nt; ++t) {
      pool.emplace_back([&, t] {
        for (int64_t i = t; i < n; i += nt) {
          CandidateResult c = solve_subproblem(tuples[i], *cm->cm, st, bs, vpp);
          if (!c.feasible) continue;
          if (!has[t] || better(c, best[t])) {
            best[t] = std::move(c);
            has[t] = 1;
          }
        }
      });
    }
    for (auto& th : pool) th.join();
    int w = -1;
    for (int t = 0; t < nt; ++t) {
      if (has[t] && (w < 0 || better(best[t], best[w]))) w = t;
    }
    if (w < 0) throw InfeasibleError("no feasible plan for this model and cluster");
    result->best = from_plan(best[w].plan);
    result->times = {best[w].times.t_warm, best[w].times.t_steady,
                     best[w].times.t_iter};
    result->candidates_evaluated = n;
    result->solve_seconds = std::chrono::duration<double>(
                                std::chrono::steady_clock::now() - t0)
                                .count();
  });
}

// ingest_trace (src/workload.cpp:115-153) over an istringstream of the
// bytes; CSR marshalling only.
dtb_status API(ingest_trace)(dtb_context*, const char* bytes, int64_t len, int64_t seq_len_cap,
                             const dtb_trace_csr* out, dtb_trace_result* res) {
  *res = dtb_trace_result{};
  std::string text(bytes ? bytes : "", static_cast<size_t>(len));
  {
    std::istringstream lines(text);
    std::string line;
    while (std::getline(lines, line)) ++res->n_lines;
  }
  std::vector<Sample> samples;
  try {
    std::istringstream in(text);
    samples = ingest_trace(in, seq_len_cap);
  } catch (const TraceError& e) {
    res->error_kind = e.kind() == "ParseError" ? DTB_TRACE_PARSE_ERROR
                                               : DTB_TRACE_INVARIANT_VIOLATION;
    res->error_line = e.line();
    return fail(DTB_ERR_TRACE, e.what());
  } catch (const std::exception& e) {
    return fail(DTB_ERR_INTERNAL, e.what());
  }
  int64_t ni = 0, na = 0;
  for (const Sample& smp : samples) {
    ni += static_cast<int64_t>(smp.image_subseqs.size());
    na += static_cast<int64_t>(smp.audio_subseqs.size());
  }
  res->n_samples = static_cast<int64_t>(samples.size());
  res->n_image = ni;
  res->n_audio = na;
  for (size_t k = 0; k < samples.size(); ++k) {
    const Sample& smp = samples[k];
    bool big = smp.text_tokens > 0x7fffffff;
    for (auto v : smp.image_subseqs) big |= v > 0x7fffffff;
    for (auto v : smp.audio_subseqs) big |= v > 0x7fffffff;
    if (big) {
      res->error_line = 0;
      return fail(DTB_ERR_INVALID_ARGUMENT, "token count beyond the int32 CSR");
    }
  }
  if (out == nullptr || out->text_tokens == nullptr) return DTB_OK;
  if (res->n_samples > out->cap_samples || ni > out->cap_image || na > out->cap_audio)
    return fail(DTB_ERR_INVALID_ARGUMENT, "CSR capacity too small");
  int64_t oi = 0, oa = 0;
  for (size_t k = 0; k < samples.size(); ++k) {
    const Sample& smp = samples[k];
    out->text_tokens[k] = static_cast<int32_t>(smp.text_tokens);
    out->image_offsets[k] = static_cast<int32_t>(oi);
    out->audio_offsets[k] = static_cast<int32_t>(oa);
    for (auto v : smp.image_subseqs) out->image_tokens[oi++] = static_cast<int32_t>(v);
    for (auto v : smp.audio_subseqs) out->audio_tokens[oa++] = static_cast<int32_t>(v);
  }
  out->image_offsets[samples.size()] = static_cast<int32_t>(oi);
  out->audio_offsets[samples.size()] = static_cast<int32_t>(oa);
  return DTB_OK;
}

}  // extern "C"

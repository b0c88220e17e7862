// mmplan:: drop-in shim over libdisttrain_b200.
//
// Defines the reference planner's hot-path entry points with their exact
// C++ signatures (proj/core/include/mmplan/reorder.hpp, pipeline_sim.hpp,
// simulate.hpp, orchestrator.hpp) and runs each one on the GPU through the
// C ABI (include/disttrain_b200.h): mmplan types are flattened to the ABI's
// POD/CSR layouts, the call is made, the result is rebuilt as the mmplan
// return type, and ABI statuses are rethrown as the reference's exception
// classes with the same message text (include/errors.hpp:23-86).
//
// Linking a consumer (the reference CLI, its tests) against this file and
// libdisttrain_b200.so instead of the reference's reorder.cpp /
// pipeline_sim.cpp / simulate.cpp / orchestrator.cpp moves those calls onto
// the B200; every other mmplan translation unit (core, cost_model, workload,
// validate, config, report) is used unchanged.  oracle/refcheck/Makefile
// builds the reference's own test binary this way (the reference's helper
// functions that stay on the host keep their reference implementations,
// renamed out of the way at compile time).
//
// Reading a CostBook's rows needs CostProfile's private table; the shim
// reaches it through an explicit instantiation (access checks do not apply
// there), since the reference exposes no accessor.
#include <algorithm>
#include <chrono>
#include <map>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
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

namespace {

using namespace mmplan;

// ---- CostProfile's row table (no public accessor in the reference)
using RowTable = std::map<int, std::vector<CostProfile::Point>>;
struct RowsTag {
  using type = RowTable CostProfile::*;
  friend type rows_member(RowsTag);
};
template <typename Tag, typename Tag::type M>
struct Expose {
  friend typename Tag::type rows_member(Tag) { return M; }
};
template struct Expose<RowsTag, &CostProfile::rows_>;

// ---- CostModel's warning sink (private member; same technique)
struct SinkTag {
  using type = std::vector<std::string>* CostModel::*;
  friend type sink_member(SinkTag);
};
template <typename Tag, typename Tag::type M>
struct ExposeSink {
  friend typename Tag::type sink_member(Tag) { return M; }
};
template struct ExposeSink<SinkTag, &CostModel::warnings_>;

// ---- one context per process (device 0, or DTB_SHIM_DEVICE)
dtb_context* ctx() {
  static dtb_context* c = [] {
    dtb_context* h = nullptr;
    const char* d = std::getenv("DTB_SHIM_DEVICE");
    if (dtb_context_create(d ? std::atoi(d) : 0, &h) != DTB_OK)
      throw std::runtime_error(std::string("dtb_context_create: ") + dtb_last_error());
    return h;
  }();
  return c;
}

[[noreturn]] void rethrow(dtb_status s) {
  const std::string msg = dtb_last_error();
  switch (s) {
    case DTB_ERR_INTERNAL: throw InternalError(msg);
    case DTB_ERR_K_TOO_LARGE: throw KTooLargeError(msg);
    case DTB_ERR_INDIVISIBLE_VPP: throw IndivisibleVppError(msg);
    case DTB_ERR_BATCH_SIZE_MISMATCH: throw BatchSizeMismatchError(msg);
    case DTB_ERR_CONFIG: throw ConfigError(msg);
    case DTB_ERR_EMPTY_PROFILE: throw EmptyProfileError(msg);
    case DTB_ERR_INFEASIBLE: throw InfeasibleError(msg);
    case DTB_ERR_CAP_EXCEEDED: throw CapExceededError(msg);
    default: throw std::runtime_error(msg);
  }
}
void check(dtb_status s) {
  if (s != DTB_OK) rethrow(s);
}

// ---- type conversions (the inverse of oracle/refshim/ref_capi.cpp)
dtb_model_spec to_c(const ModelSpec& m) {
  dtb_model_spec out{};
  for (int u = 0; u < 3; ++u) {
    const ModuleSpec& ms = m.module(static_cast<ModuleKind>(u));
    dtb_module_spec& d = out.unit[u];
    d.arch.layers = ms.arch.layers;
    d.arch.heads = ms.arch.heads;
    d.arch.groups = ms.arch.groups;
    d.arch.hidden = ms.arch.hidden;
    d.arch.ffn_hidden = ms.arch.ffn_hidden;
    d.mem.param_grad_bytes = ms.mem.param_grad_bytes;
    d.mem.optimizer_bytes = ms.mem.optimizer_bytes;
    d.mem.activation_bytes_per_mb = ms.mem.activation_bytes_per_mb;
    d.frozen = ms.frozen ? 1 : 0;
  }
  out.seq_len = m.seq_len;
  out.frozen_backward_factor = m.frozen_backward_factor;
  out.dp_sync_seconds = m.dp_sync_seconds;
  return out;
}

dtb_cluster_spec to_c(const ClusterSpec& c) {
  return dtb_cluster_spec{c.total_gpus, c.gpus_per_node, c.peak_flops,
                          c.gpu_mem_bytes, c.intra_node_bw, c.inter_node_bw};
}

dtb_plan to_c(const Plan& p) {
  dtb_plan out{};
  for (int u = 0; u < 3; ++u) {
    const ParallelismChoice& pc = p.unit(static_cast<ModuleKind>(u));
    out.unit[u] = {pc.tp, pc.dp, pc.pp};
  }
  out.vpp = p.vpp;
  out.global_batch = p.global_batch;
  return out;
}

Plan from_c(const dtb_plan& p) {
  Plan out;
  for (int u = 0; u < 3; ++u)
    out.unit(static_cast<ModuleKind>(u)) = {p.unit[u].tp, p.unit[u].dp, p.unit[u].pp};
  out.global_batch = p.global_batch;
  out.vpp = p.vpp;
  return out;
}

dtb_workload_stats to_c(const WorkloadStats& s) {
  return dtb_workload_stats{s.seq_len, s.mean_encoder_tokens, s.mean_generator_tokens};
}

dtb_tuple to_c(const ParallelismTuple& t) {
  return dtb_tuple{t.tp_me, t.dp_me, t.tp_lm, t.dp_lm, t.tp_mg, t.dp_mg};
}
ParallelismTuple from_c(const dtb_tuple& t) {
  ParallelismTuple out;
  out.tp_me = t.tp_me, out.dp_me = t.dp_me;
  out.tp_lm = t.tp_lm, out.dp_lm = t.dp_lm;
  out.tp_mg = t.tp_mg, out.dp_mg = t.dp_mg;
  return out;
}

PredictedTimes from_c(const dtb_predicted_times& t) {
  PredictedTimes out;
  out.t_warm = t.t_warm, out.t_steady = t.t_steady, out.t_iter = t.t_iter;
  return out;
}

CandidateResult from_c(const dtb_candidate& c) {
  CandidateResult out;
  out.tuple = from_c(c.tuple);
  out.feasible = c.feasible != 0;
  out.infeasible_reason = c.reason == DTB_REASON_NONE ? "" : dtb_infeasible_reason_text(c.reason);
  out.plan = c.feasible ? from_c(c.plan) : Plan{};
  out.times = from_c(c.times);
  out.cont_x = c.cont_x, out.cont_y = c.cont_y, out.cont_z = c.cont_z;
  out.cont_t_iter = c.cont_t_iter;
  return out;
}

// A device cost model for one CostModel (created per call: the reference's
// CostModel is a value type without identity).
struct CM {
  dtb_cost_model* h = nullptr;
  explicit CM(const CostModel& costs) {
    std::vector<dtb_profile_row> rows;
    for (int u = 0; u < 3; ++u) {
      const CostProfile& prof = costs.book().profile(static_cast<ModuleKind>(u));
      const RowTable& table = prof.*rows_member(RowsTag{});
      for (const auto& [tp, points] : table)
        for (const auto& pt : points)
          rows.push_back(dtb_profile_row{u, tp, pt.bwd_s.has_value() ? 1 : 0, 0, pt.token_load,
                                         pt.fwd_s, pt.bwd_s.value_or(0.0)});
    }
    const dtb_costbook book{rows.data(), static_cast<int64_t>(rows.size()),
                            costs.book().analytic.efficiency,
                            costs.book().analytic.bwd_fwd_ratio};
    const dtb_model_spec m = to_c(costs.model());
    const dtb_cluster_spec c = to_c(costs.cluster());
    check(dtb_cost_model_create(ctx(), &m, &c, &book, &h));
  }
  ~CM() { dtb_cost_model_destroy(h); }
  CM(const CM&) = delete;
  CM& operator=(const CM&) = delete;
};

// While a call runs, a sink attached to its CostModel receives what the
// device path logs (dtb_warnings_*): the reference's strings in the
// reference's query order (SURVEY.md §8(b) Warnings).
struct SinkBridge {
  std::vector<std::string>* sink;
  explicit SinkBridge(const CostModel& costs) : sink(costs.*sink_member(SinkTag{})) {
    if (sink != nullptr) dtb_warnings_enable(ctx(), 1);
  }
  ~SinkBridge() {
    if (sink == nullptr) return;
    const int64_t n = dtb_warnings_count(ctx());
    for (int64_t i = 0; i < n; ++i) sink->emplace_back(dtb_warning_at(ctx(), i));
    dtb_warnings_enable(ctx(), 0);
  }
  SinkBridge(const SinkBridge&) = delete;
  SinkBridge& operator=(const SinkBridge&) = delete;
};

struct CSR {
  std::vector<int32_t> text, io, it, ao, at;
  dtb_samples view{};
  explicit CSR(std::span<const Sample> batch) {
    io.push_back(0);
    ao.push_back(0);
    for (const Sample& s : batch) {
      text.push_back(static_cast<int32_t>(s.text_tokens));
      for (auto t : s.image_subseqs) it.push_back(static_cast<int32_t>(t));
      for (auto t : s.audio_subseqs) at.push_back(static_cast<int32_t>(t));
      io.push_back(static_cast<int32_t>(it.size()));
      ao.push_back(static_cast<int32_t>(at.size()));
    }
    if (it.empty()) it.push_back(0);
    if (at.empty()) at.push_back(0);
    view = dtb_samples{static_cast<int64_t>(batch.size()), text.data(), io.data(), it.data(),
                       ao.data(), at.data()};
  }
};

struct MBs {
  std::vector<int64_t> enc, gen;
  std::vector<int32_t> cnt;
  dtb_microbatches view{};
  void add(const Microbatch& mb) {
    enc.push_back(mb.encoder_tokens);
    gen.push_back(mb.generator_tokens);
    cnt.push_back(static_cast<int32_t>(mb.samples.size()));
  }
  void seal() {
    view = dtb_microbatches{static_cast<int64_t>(enc.size()), enc.data(), gen.data(), cnt.data()};
  }
};

Timeline schedule(const StageTimes& times, int vpp) {
  const int l = times.microbatches, p = times.stages;
  const std::size_t ne = static_cast<std::size_t>(2) * l * p;
  std::vector<int32_t> dev(ne), mb(ne), st(ne), ph(ne);
  std::vector<double> s(ne), e(ne), busy(static_cast<std::size_t>(std::max(1, p)));
  double it = 0.0;
  check(dtb_schedule(ctx(), times.fwd.data(), times.bwd.data(), l, p, vpp, dev.data(), mb.data(),
                     st.data(), ph.data(), s.data(), e.data(), &it, busy.data()));
  Timeline tl;
  tl.events.reserve(ne);
  for (std::size_t i = 0; i < ne; ++i)
    tl.events.push_back(TimelineEvent{dev[i], mb[i], st[i], static_cast<Phase>(ph[i]), s[i], e[i]});
  const int devices = vpp > 0 ? p / vpp : p;
  tl.device_count = devices;
  tl.microbatch_count = l;
  tl.stage_count = p;
  tl.iteration_time = it;
  tl.device_busy.assign(busy.begin(), busy.begin() + devices);
  return tl;
}

dtb_reorder_mode to_c(const ReorderMode& m) {
  return dtb_reorder_mode{m.intra ? 1 : 0, m.inter ? 1 : 0,
                          m.sort_order == IntraSortOrder::Descending ? DTB_DESCENDING
                                                                     : DTB_ASCENDING};
}

}  // namespace

namespace mmplan {

// ------------------------------------------------------------- reorder.hpp
IntraPartition intra_partition(std::span<const double> sizes, int m, IntraSortOrder order,
                               bool equal_counts) {
  std::vector<int32_t> flat(std::max<std::size_t>(sizes.size(), 1));
  std::vector<int64_t> offs(static_cast<std::size_t>(std::max(m, 0)) + 1);
  check(dtb_intra_partition(ctx(), sizes.data(), static_cast<int64_t>(sizes.size()), m,
                            order == IntraSortOrder::Descending ? DTB_DESCENDING : DTB_ASCENDING,
                            equal_counts ? 1 : 0, flat.data(), offs.data()));
  IntraPartition part;
  part.groups.resize(static_cast<std::size_t>(m));
  for (int g = 0; g < m; ++g)
    part.groups[g].assign(flat.begin() + offs[g], flat.begin() + offs[g + 1]);
  return part;
}

std::vector<int> intra_reorder_order(std::span<const double> sizes, int m, IntraSortOrder order) {
  return intra_partition(sizes, m, order, false).flat();
}

std::vector<Sample> intra_reorder(std::span<const Sample> batch, int m, IntraSortOrder order) {
  std::vector<double> sizes;
  sizes.reserve(batch.size());
  for (const Sample& s : batch) sizes.push_back(static_cast<double>(s.cost_size()));
  std::vector<Sample> out;
  for (int idx : intra_reorder_order(sizes, m, order)) out.push_back(batch[idx]);
  return out;
}

std::vector<double> block_group_loads(std::span<const double> sizes, std::span<const int> order,
                                      int m) {
  std::vector<double> loads(static_cast<std::size_t>(std::max(m, 1)));
  check(dtb_block_group_loads(ctx(), sizes.data(), order.data(),
                              static_cast<int64_t>(order.size()), m, loads.data()));
  loads.resize(static_cast<std::size_t>(std::max(m, 0)));
  return loads;
}

std::vector<int> select_min(std::span<const double> keys, const std::vector<int>& pending, int k) {
  std::vector<int32_t> out(static_cast<std::size_t>(std::max(k, 1)));
  check(dtb_select_min(ctx(), keys.data(), static_cast<int64_t>(keys.size()), pending.data(),
                       static_cast<int64_t>(pending.size()), k, out.data()));
  out.resize(static_cast<std::size_t>(std::max(k, 0)));
  return out;
}

std::vector<int> select_closest(std::span<const double> keys, const std::vector<int>& pending,
                                int k, double target) {
  std::vector<int32_t> out(static_cast<std::size_t>(std::max(k, 1)));
  check(dtb_select_closest(ctx(), keys.data(), static_cast<int64_t>(keys.size()), pending.data(),
                           static_cast<int64_t>(pending.size()), k, target, out.data()));
  out.resize(static_cast<std::size_t>(std::max(k, 0)));
  return out;
}

std::vector<int> inter_reorder(const StageTimes& times, std::span<const double> keys, int vpp) {
  const int l = times.microbatches;
  std::vector<int32_t> out(static_cast<std::size_t>(std::max(l, 1)));
  std::vector<double> k(keys.begin(), keys.end());
  if (k.empty()) k.push_back(0.0);
  std::vector<double> f = times.fwd, b = times.bwd;
  if (f.empty()) f.push_back(0.0), b.push_back(0.0);
  check(dtb_inter_reorder(ctx(), f.data(), b.data(), l, times.stages, k.data(), vpp, out.data()));
  out.resize(static_cast<std::size_t>(std::max(l, 0)));
  return out;
}

std::vector<double> microbatch_fwd_keys(const Plan& plan, const CostModel& costs,
                                        std::span<const Microbatch> microbatches) {
  const SinkBridge warnings(costs);
  MBs mbs;
  for (const Microbatch& mb : microbatches) mbs.add(mb);
  mbs.seal();
  CM cm(costs);
  const dtb_plan p = to_c(plan);
  std::vector<double> keys(std::max<std::size_t>(microbatches.size(), 1));
  check(dtb_microbatch_fwd_keys(ctx(), cm.h, &p, &mbs.view, keys.data()));
  keys.resize(microbatches.size());
  return keys;
}

DisaggregatedResult disaggregated_reorder(std::span<const Sample> batch, const Plan& plan,
                                          const CostModel& costs, const ReorderMode& mode) {
  const SinkBridge warnings(costs);
  CSR csr(batch);
  CM cm(costs);
  const dtb_plan p = to_c(plan);
  const dtb_reorder_mode md = to_c(mode);
  const int dp = std::max(plan.backbone.dp, 1);
  DisaggregatedResult r;
  r.report.output_order.assign(std::max<std::size_t>(batch.size(), 1), 0);
  r.report.group_load_before.assign(static_cast<std::size_t>(dp), 0.0);
  r.report.group_load_after.assign(static_cast<std::size_t>(dp), 0.0);
  dtb_reorder_report rep{r.report.output_order.data(), r.report.group_load_before.data(),
                         r.report.group_load_after.data(), 0.0, 0.0};
  check(dtb_disaggregated_reorder(ctx(), cm.h, &p, &md, &csr.view, &rep));
  r.report.output_order.resize(batch.size());
  r.report.t_iter_before = rep.t_iter_before;
  r.report.t_iter_after = rep.t_iter_after;
  // the reordered groups are the microbatches of the output order
  // (include/reorder.hpp: DisaggregatedResult)
  std::vector<Sample> staged;
  staged.reserve(batch.size());
  for (int idx : r.report.output_order) staged.push_back(batch[idx]);
  r.groups = assemble_microbatches(staged, plan);
  return r;
}

// -------------------------------------------------------- pipeline_sim.hpp
Timeline schedule_1f1b(const StageTimes& times) { return schedule(times, 1); }

Timeline schedule_interleaved(const StageTimes& times, int vpp) { return schedule(times, vpp); }

double iteration_time_1f1b(const StageTimes& times) {
  double it = 0.0;
  check(dtb_schedule(ctx(), times.fwd.data(), times.bwd.data(), times.microbatches, times.stages,
                     1, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, &it, nullptr));
  return it;
}

IntervalSet get_intervals(const Timeline& timeline) {
  const std::size_t ne = timeline.events.size();
  std::vector<int32_t> dev(ne + 1), mb(ne + 1), st(ne + 1), ph(ne + 1);
  std::vector<double> s(ne + 1), e(ne + 1);
  for (std::size_t i = 0; i < ne; ++i) {
    const TimelineEvent& ev = timeline.events[i];
    dev[i] = ev.device, mb[i] = ev.microbatch, st[i] = ev.stage;
    ph[i] = static_cast<int32_t>(ev.phase), s[i] = ev.start, e[i] = ev.end;
  }
  int64_t n = 0;
  std::vector<double> starts(ne + 1), ends(ne + 1);
  std::vector<int64_t> fo(ne + 2);
  std::vector<int32_t> fm(ne + 1);
  check(dtb_get_intervals(ctx(), static_cast<int64_t>(ne), dev.data(), mb.data(), st.data(),
                          ph.data(), s.data(), e.data(), &n, starts.data(), ends.data(), fo.data(),
                          fm.data()));
  IntervalSet set;
  for (int64_t i = 0; i < n; ++i) {
    Interval iv;
    iv.start = starts[i];
    iv.end = ends[i];
    iv.filled_by.assign(fm.begin() + fo[i], fm.begin() + fo[i + 1]);
    set.intervals.push_back(std::move(iv));
  }
  return set;
}

std::vector<double> interval_windows(const StageTimes& times) {
  std::vector<double> v(static_cast<std::size_t>(std::max(times.microbatches, 1)));
  check(dtb_interval_windows(ctx(), times.fwd.data(), times.bwd.data(), times.microbatches,
                             times.stages, v.data()));
  v.resize(static_cast<std::size_t>(std::max(times.microbatches, 0)));
  return v;
}

// ------------------------------------------------------------ simulate.hpp
IterationResult simulate_iteration(const Plan& plan, const CostModel& costs,
                                   const std::vector<std::vector<Microbatch>>& groups) {
  const SinkBridge warnings(costs);
  MBs mbs;
  std::vector<int64_t> offs{0};
  for (const auto& g : groups) {
    for (const Microbatch& mb : g) mbs.add(mb);
    offs.push_back(static_cast<int64_t>(mbs.enc.size()));
  }
  if (mbs.enc.empty()) mbs.enc.push_back(0), mbs.gen.push_back(0), mbs.cnt.push_back(0);
  mbs.seal();
  mbs.view.n = offs.back();
  CM cm(costs);
  const dtb_plan p = to_c(plan);
  IterationResult r;
  r.group_times.assign(std::max<std::size_t>(groups.size(), 1), 0.0);
  int32_t slowest = 0;
  check(dtb_simulate_iteration(ctx(), cm.h, &p, static_cast<int32_t>(groups.size()), offs.data(),
                               &mbs.view, &r.t_iter, r.group_times.data(), &slowest,
                               &r.slowest_group_time, &r.mean_bubble_fraction));
  r.group_times.resize(groups.size());
  r.slowest_group = slowest;
  return r;
}

// -------------------------------------------------------- orchestrator.hpp
PredictedTimes predict_times(const Plan& plan, const CostModel& costs, const WorkloadStats& stats) {
  CM cm(costs);
  const dtb_plan p = to_c(plan);
  const dtb_workload_stats s = to_c(stats);
  dtb_predicted_times t{};
  check(dtb_predict_times(ctx(), cm.h, &s, &p, 1, &t));
  return from_c(t);
}

std::vector<ParallelismTuple> enumerate_parallelism(const ClusterSpec& cluster,
                                                    std::int64_t global_batch) {
  const dtb_cluster_spec c = to_c(cluster);
  int64_t count = 0;
  check(dtb_enumerate_parallelism(ctx(), &c, global_batch, &count, nullptr, 0));
  std::vector<dtb_tuple> t(static_cast<std::size_t>(std::max<int64_t>(count, 1)));
  check(dtb_enumerate_parallelism(ctx(), &c, global_batch, &count, t.data(), count));
  std::vector<ParallelismTuple> out;
  out.reserve(static_cast<std::size_t>(count));
  for (int64_t i = 0; i < count; ++i) out.push_back(from_c(t[i]));
  return out;
}

CandidateResult solve_subproblem(const ParallelismTuple& tuple, const CostModel& costs,
                                 const WorkloadStats& stats, std::int64_t global_batch, int vpp) {
  CM cm(costs);
  const dtb_workload_stats s = to_c(stats);
  const dtb_tuple t = to_c(tuple);
  dtb_candidate c{};
  check(dtb_solve_subproblem(ctx(), cm.h, &s, &t, 1, global_batch, vpp, &c));
  return from_c(c);
}

OrchestrationResult model_orchestration(const CostModel& costs, const WorkloadStats& stats,
                                        std::int64_t global_batch,
                                        const OrchestrationOptions& options) {
  CM cm(costs);
  const dtb_workload_stats s = to_c(stats);
  std::vector<dtb_candidate> cands;
  if (options.keep_candidates) {
    const dtb_cluster_spec c = to_c(costs.cluster());
    int64_t count = 0;
    check(dtb_enumerate_parallelism(ctx(), &c, global_batch, &count, nullptr, 0));
    cands.resize(static_cast<std::size_t>(std::max<int64_t>(count, 1)));
  }
  dtb_orchestration_result res{};
  const auto t0 = std::chrono::steady_clock::now();
  check(dtb_model_orchestration(ctx(), cm.h, &s, global_batch, options.vpp, &res,
                                options.keep_candidates ? cands.data() : nullptr,
                                static_cast<int64_t>(cands.size())));
  OrchestrationResult r;
  r.best = from_c(res.best);
  r.times = from_c(res.times);
  r.candidates_evaluated = static_cast<std::size_t>(res.candidates_evaluated);
  r.solve_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (options.keep_candidates)
    for (int64_t i = 0; i < res.candidates_evaluated && i < static_cast<int64_t>(cands.size()); ++i)
      r.candidates.push_back(from_c(cands[i]));
  return r;
}

Plan rigid_baseline(const CostModel& costs, const WorkloadStats& stats, std::int64_t global_batch,
                    int vpp) {
  CM cm(costs);
  const dtb_workload_stats s = to_c(stats);
  dtb_plan p{};
  check(dtb_rigid_baseline(ctx(), cm.h, &s, global_batch, vpp, &p));
  return from_c(p);
}

OrchestrationResult brute_force_oracle(const CostModel& costs, const WorkloadStats& stats,
                                       std::int64_t global_batch,
                                       const BruteForceOptions& options) {
  CM cm(costs);
  const dtb_workload_stats s = to_c(stats);
  dtb_orchestration_result res{};
  check(dtb_brute_force_oracle(ctx(), cm.h, &s, global_batch, options.vpp, options.gpu_cap, &res));
  OrchestrationResult r;
  r.best = from_c(res.best);
  r.times = from_c(res.times);
  r.candidates_evaluated = static_cast<std::size_t>(res.candidates_evaluated);
  r.solve_seconds = res.solve_seconds;
  return r;
}

}  // namespace mmplan

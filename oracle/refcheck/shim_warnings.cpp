// TEST INFRASTRUCTURE (linked into oracle/_ref/refcheck only).
//
// The mmplan:: GPU shim forwards a CostModel's warning sink (SURVEY.md §8(b)
// "Warnings"): with a sink attached, the shim's disaggregated_reorder /
// simulate_iteration / microbatch_fwd_keys must append exactly the strings,
// in exactly the order, that the reference's own functions append — those
// are linked into the same binary as ref_* (oracle/refcheck/Makefile).
#include <doctest.h>

#include <random>
#include <string>
#include <vector>

#include "mmplan/cost_model.hpp"
#include "mmplan/reorder.hpp"
#include "mmplan/simulate.hpp"
#include "mmplan/workload.hpp"
#include "support/fixtures.hpp"

namespace mmplan {
DisaggregatedResult ref_disaggregated_reorder(std::span<const Sample> batch, const Plan& plan,
                                              const CostModel& costs, const ReorderMode& mode);
IterationResult ref_simulate_iteration(const Plan& plan, const CostModel& costs,
                                       const std::vector<std::vector<Microbatch>>& groups);
std::vector<double> ref_microbatch_fwd_keys(const Plan& plan, const CostModel& costs,
                                            std::span<const Microbatch> microbatches);
}  // namespace mmplan

using namespace mmplan;

namespace {

// Rows inside [600, 2500] token loads for encoder and backbone (means clamp
// on both sides), no generator rows (analytic fallback).
CostBook narrow_book() {
  CostBook book;
  book.analytic.efficiency = 0.5;
  for (int tp : kAllowedTp) {
    for (ModuleKind k : {ModuleKind::Encoder, ModuleKind::Backbone}) {
      book.profile(k).add_row(tp, 600.0, 0.01 * tp, 0.02 * tp);
      book.profile(k).add_row(tp, 2500.0, 0.05 * tp, 0.10 * tp);
    }
  }
  return book;
}

std::vector<Sample> random_batch(std::mt19937_64& rng, int n) {
  std::vector<Sample> batch;
  for (int i = 0; i < n; ++i) {
    std::vector<std::int64_t> imgs;
    const int k = static_cast<int>(rng() % 3);
    for (int j = 0; j < k; ++j) imgs.push_back(static_cast<std::int64_t>(rng() % 2400));
    batch.push_back(test::sample_with(100, imgs));
  }
  return batch;
}

}  // namespace

TEST_CASE("shim warning sink: disaggregated_reorder, simulate_iteration, fwd keys") {
  ModelSpec model = test::toy_model();
  model.seq_len = 4096;  // backbone load above its rows: warnings on every query
  CostModel costs(model, test::toy_cluster(64), narrow_book());
  std::mt19937_64 rng(7);
  for (int dp_me : {8, 2}) {
    Plan plan;
    plan.encoder = {1, dp_me, 1};
    plan.backbone = {1, 8, 2};
    plan.generator = {1, 4, 1};
    plan.global_batch = 256;
    const std::vector<Sample> batch = random_batch(rng, 256);
    for (bool inter : {false, true}) {
      ReorderMode mode;
      mode.inter = inter;
      std::vector<std::string> a, b;
      costs.set_warning_sink(&a);
      const DisaggregatedResult ra = disaggregated_reorder(batch, plan, costs, mode);
      costs.set_warning_sink(&b);
      const DisaggregatedResult rb = ref_disaggregated_reorder(batch, plan, costs, mode);
      costs.set_warning_sink(nullptr);
      CHECK(ra.report.output_order == rb.report.output_order);
      CHECK(!b.empty());
      CHECK(a == b);
    }
    const auto groups = assemble_microbatches(batch, plan);
    std::vector<std::string> a, b;
    costs.set_warning_sink(&a);
    simulate_iteration(plan, costs, groups);
    microbatch_fwd_keys(plan, costs, groups[0]);
    costs.set_warning_sink(&b);
    ref_simulate_iteration(plan, costs, groups);
    ref_microbatch_fwd_keys(plan, costs, groups[0]);
    costs.set_warning_sink(nullptr);
    CHECK(!b.empty());
    CHECK(a == b);
  }
}

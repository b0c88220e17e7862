/*
 * disttrain_b200.h — C-ABI drop-in boundary for the DistTrain (arXiv 2408.04275)
 * data-reordering and orchestration-search hot path, implemented with sm_100a
 * kernels (libdisttrain_b200.so).
 *
 * Every entry point replaces one function of the reference C++ planner
 * `mmplan` (read-only at /root/reference/proj/core).  The citation on each
 * declaration is the reference interface it stands in for
 * (`include/` = proj/core/include/mmplan/, `src/` = proj/core/src/).
 *
 * Conventions
 *  - Plain pointers and sizes only; no C++ or torch types cross the boundary.
 *  - Functions without a `_dev` suffix take HOST buffers (the call stages
 *    them through device memory and synchronises before returning).
 *    `_dev` functions take DEVICE pointers and a cudaStream_t passed as
 *    `void*`; they enqueue work and return without synchronising.
 *  - Every function returns a dtb_status.  Status codes map 1:1 onto the
 *    reference exception classes (include/errors.hpp:22-84); the message text
 *    of the last failure on the calling thread is `dtb_last_error()`.
 *  - Inputs are validated on the host before any launch, in the same order
 *    the reference validates them, so the same bad input raises the same
 *    error class with the same message.
 *  - The same ABI (with prefixes `mmref_` / `mmport_`) is exported by the
 *    test oracles under oracle/ so the parity tests can call all three
 *    implementations through one binding.
 */
#ifndef DISTTRAIN_B200_H
#define DISTTRAIN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DTB_ABI_VERSION 1

/* ---------------------------------------------------------------- status */

/* 1:1 with include/errors.hpp:23-86 (plus two ABI-level codes). */
typedef enum dtb_status {
  DTB_OK = 0,
  DTB_ERR_INTERNAL = 1,            /* InternalError        errors.hpp:56   */
  DTB_ERR_K_TOO_LARGE = 2,         /* KTooLargeError       errors.hpp:62   */
  DTB_ERR_INDIVISIBLE_VPP = 3,     /* IndivisibleVppError  errors.hpp:75   */
  DTB_ERR_BATCH_SIZE_MISMATCH = 4, /* BatchSizeMismatchError errors.hpp:81 */
  DTB_ERR_CONFIG = 5,              /* ConfigError          errors.hpp:23   */
  DTB_ERR_EMPTY_PROFILE = 6,       /* EmptyProfileError    errors.hpp:29   */
  DTB_ERR_INFEASIBLE = 7,          /* InfeasibleError      errors.hpp:50   */
  DTB_ERR_CAP_EXCEEDED = 8,        /* CapExceededError     errors.hpp:68   */
  DTB_ERR_TRACE = 9,               /* TraceError           errors.hpp:35   */
  DTB_ERR_INVALID_ARGUMENT = 100,  /* null pointer / ABI limit exceeded    */
  DTB_ERR_CUDA = 101               /* device failure (no reference analogue) */
} dtb_status;

/* Message of the last non-OK status returned on this thread. */
const char* dtb_last_error(void);
int dtb_abi_version(void);

/* ----------------------------------------------------------- domain PODs */

enum { DTB_ENCODER = 0, DTB_BACKBONE = 1, DTB_GENERATOR = 2 }; /* core.hpp:27 */
enum { DTB_ASCENDING = 0, DTB_DESCENDING = 1 };                 /* reorder.hpp:29 */
enum { DTB_FORWARD = 0, DTB_BACKWARD = 1 };                     /* core.hpp:195 */

/* ArchDesc (include/core.hpp:36-50). */
typedef struct dtb_arch {
  int32_t layers;
  int32_t heads;
  int32_t groups;
  int32_t reserved;
  int64_t hidden;
  int64_t ffn_hidden;
} dtb_arch;

/* ModuleMemory (include/core.hpp:57-61), bytes. */
typedef struct dtb_module_memory {
  double param_grad_bytes;
  double optimizer_bytes;
  double activation_bytes_per_mb;
} dtb_module_memory;

/* ModuleSpec (include/core.hpp:63-67). */
typedef struct dtb_module_spec {
  dtb_arch arch;
  dtb_module_memory mem;
  int32_t frozen;
  int32_t reserved;
} dtb_module_spec;

/* ModelSpec (include/core.hpp:69-88); unit[] indexed by DTB_ENCODER.. */
typedef struct dtb_model_spec {
  dtb_module_spec unit[3];
  int64_t seq_len;
  double frozen_backward_factor;
  double dp_sync_seconds;
} dtb_model_spec;

/* ClusterSpec (include/core.hpp:90-97). */
typedef struct dtb_cluster_spec {
  int32_t total_gpus;
  int32_t gpus_per_node;
  double peak_flops;
  double gpu_mem_bytes;
  double intra_node_bw;
  double inter_node_bw;
} dtb_cluster_spec;

/* One CostProfile::add_row call (include/cost_model.hpp:44-45).  Rows are
 * applied in array order with add_row semantics (sorted insert, last row
 * wins on a duplicate token load, src/cost_model.cpp:37-60). */
typedef struct dtb_profile_row {
  int32_t module;
  int32_t tp;
  int32_t has_bwd;
  int32_t reserved;
  double token_load;
  double fwd_s;
  double bwd_s;
} dtb_profile_row;

/* CostBook (include/cost_model.hpp:72-83). */
typedef struct dtb_costbook {
  const dtb_profile_row* rows;
  int64_t n_rows;
  double analytic_efficiency;    /* AnalyticCoeffs::efficiency, default 0.45 */
  double analytic_bwd_fwd_ratio; /* AnalyticCoeffs::bwd_fwd_ratio, default 2 */
} dtb_costbook;

/* ParallelismChoice (include/core.hpp:103-110). */
typedef struct dtb_parallelism {
  int32_t tp;
  int32_t dp;
  int32_t pp;
} dtb_parallelism;

/* Plan (include/core.hpp:115-150). */
typedef struct dtb_plan {
  dtb_parallelism unit[3];
  int32_t vpp;
  int64_t global_batch;
} dtb_plan;

/* WorkloadStats (include/cost_model.hpp:88-92). */
typedef struct dtb_workload_stats {
  int64_t seq_len;
  double mean_encoder_tokens;
  double mean_generator_tokens;
} dtb_workload_stats;

/* A span of Samples (include/core.hpp:155-170) in CSR form.  Sample i owns
 * image_tokens[image_offsets[i] .. image_offsets[i+1]) and likewise audio.
 * Offsets are absolute int32 indices (ABI limit: < 2^31 subsequences per
 * call); text_tokens may be NULL (the reorder path never reads it). */
typedef struct dtb_samples {
  int64_t n;
  const int32_t* text_tokens;
  const int32_t* image_offsets;
  const int32_t* image_tokens;
  const int32_t* audio_offsets;
  const int32_t* audio_tokens;
} dtb_samples;

/* A span of Microbatches (include/core.hpp:175-193) by their cached keys. */
typedef struct dtb_microbatches {
  int64_t n;
  const int64_t* encoder_tokens;
  const int64_t* generator_tokens;
  const int32_t* sample_count;
} dtb_microbatches;

/* ReorderMode (include/reorder.hpp:86-90). */
typedef struct dtb_reorder_mode {
  int32_t intra;
  int32_t inter;
  int32_t sort_order;
} dtb_reorder_mode;

/* ParallelismTuple (include/orchestrator.hpp:41-48). */
typedef struct dtb_tuple {
  int32_t tp_me, dp_me;
  int32_t tp_lm, dp_lm;
  int32_t tp_mg, dp_mg;
} dtb_tuple;

/* PredictedTimes (include/orchestrator.hpp:26-30). */
typedef struct dtb_predicted_times {
  double t_warm;
  double t_steady;
  double t_iter;
} dtb_predicted_times;

/* CandidateResult (include/orchestrator.hpp:57-67); the reason string is an
 * enum (text: dtb_infeasible_reason_text). */
enum {
  DTB_REASON_NONE = 0,
  DTB_REASON_DP_NOT_DIVIDING = 1,         /* src/orchestrator.cpp:72    */
  DTB_REASON_ACTIVATION_ENCODER = 2,      /* src/orchestrator.cpp:96-98 */
  DTB_REASON_ACTIVATION_BACKBONE = 3,
  DTB_REASON_ACTIVATION_GENERATOR = 4,
  DTB_REASON_MEMORY_FLOOR = 5,            /* src/orchestrator.cpp:108,172 */
  DTB_REASON_NO_INTEGER_SPLIT = 6         /* src/orchestrator.cpp:372   */
};
typedef struct dtb_candidate {
  dtb_tuple tuple;
  int32_t feasible;
  int32_t reason;
  dtb_plan plan;
  dtb_predicted_times times;
  double cont_x, cont_y, cont_z, cont_t_iter;
} dtb_candidate;
const char* dtb_infeasible_reason_text(int32_t reason);

/* OrchestrationResult (include/orchestrator.hpp:83-89). */
typedef struct dtb_orchestration_result {
  dtb_plan best;
  dtb_predicted_times times;
  int64_t candidates_evaluated;
  double solve_seconds;
} dtb_orchestration_result;

/* MemoryReport (include/cost_model.hpp:98-109). */
typedef struct dtb_memory_report {
  double bytes_per_gpu[3];
  int32_t fits[3];
  int32_t pass;
  double capacity_bytes;
} dtb_memory_report;

/* Per-call outputs of disaggregated_reorder (ReorderReport,
 * include/reorder.hpp:92-98) for one global batch; arrays caller-owned:
 * output_order[global_batch], group_load_before/after[backbone.dp]. */
typedef struct dtb_reorder_report {
  int32_t* output_order;
  double* group_load_before;
  double* group_load_after;
  double t_iter_before;
  double t_iter_after;
} dtb_reorder_report;

/* --------------------------------------------------------------- handles */

typedef struct dtb_context dtb_context;       /* device, stream, scratch */
typedef struct dtb_cost_model dtb_cost_model; /* CostModel (cost_model.hpp:152) */

dtb_status dtb_context_create(int32_t device, dtb_context** out);
dtb_status dtb_context_destroy(dtb_context* ctx);

/* Warning log — the reference's CostModel warning sink
 * (CostModel::set_warning_sink, include/cost_model.hpp:147,184; strings of
 * src/cost_model.cpp:84-95 and :248-251).  While enabled (enable also
 * clears), every successful call below appends, in the reference's query
 * order, the strings the reference's CostModel would append to its sink:
 *   "token load X below profile range; clamped",
 *   "token load X above profile range; clamped"   (X = std::to_string(load)),
 *   "module 'K' has no profile; using analytic estimate".
 * Covered: dtb_unit_times (per load: forward then backward query),
 * dtb_build_stage_times, dtb_microbatch_fwd_keys, dtb_simulate_iteration,
 * dtb_disaggregated_reorder and the stream calls (per batch, as
 * disaggregated_reorder; not inside CUDA graph captures).  Not covered: the
 * orchestration search's queries.  dtb_warning_at returns NULL out of range;
 * its pointer is valid until the log changes. */
dtb_status dtb_warnings_enable(dtb_context* ctx, int32_t on);
int64_t dtb_warnings_count(const dtb_context* ctx);
const char* dtb_warning_at(const dtb_context* ctx, int64_t i);
dtb_status dtb_warnings_clear(dtb_context* ctx);

/* CostModel(model, cluster, book) — include/cost_model.hpp:154. Applies
 * add_row to every row (ConfigError on a bad row, cost_model.cpp:39-48) and
 * uploads the flattened book to the device. */
dtb_status dtb_cost_model_create(dtb_context* ctx, const dtb_model_spec* model,
                                 const dtb_cluster_spec* cluster,
                                 const dtb_costbook* book,
                                 dtb_cost_model** out);
dtb_status dtb_cost_model_destroy(dtb_cost_model* cm);

/* ----------------------------------------------------- L1: cost model (a1-a7) */

/* Sample::cost_size for every sample (include/core.hpp:160-167,
 * src/core.cpp:90-95). out[n]. */
dtb_status dtb_cost_sizes(dtb_context* ctx, const dtb_samples* samples,
                          int64_t* out);

/* CostModel::unit_forward_time / unit_backward_time
 * (src/cost_model.cpp:255-278) at n token loads; either output may be NULL. */
dtb_status dtb_unit_times(dtb_context* ctx, const dtb_cost_model* cm,
                          int32_t module, int32_t tp, int64_t n,
                          const double* token_loads, double* fwd_out,
                          double* bwd_out);

/* memory_check (src/cost_model.cpp:167-189), one plan. */
dtb_status dtb_memory_check(dtb_context* ctx, const dtb_cost_model* cm,
                            const dtb_plan* plan, dtb_memory_report* out);

/* CostModel::build_stage_times (src/cost_model.cpp:334-362).
 * fwd/bwd: [mbs->n * virtual_stages] row-major. */
dtb_status dtb_build_stage_times(dtb_context* ctx, const dtb_cost_model* cm,
                                 const dtb_plan* plan,
                                 const dtb_microbatches* mbs, double* fwd,
                                 double* bwd);

/* microbatch_fwd_keys (src/reorder.cpp:300-317). keys[mbs->n]. */
dtb_status dtb_microbatch_fwd_keys(dtb_context* ctx, const dtb_cost_model* cm,
                                   const dtb_plan* plan,
                                   const dtb_microbatches* mbs, double* keys);

/* compute_stats (src/workload.cpp:206-220). */
dtb_status dtb_compute_stats(dtb_context* ctx, const dtb_samples* samples,
                             int64_t seq_len, dtb_workload_stats* out);

/* ------------------------------------------- L3: intra reorder (a10-a14) */

/* intra_partition (src/reorder.cpp:70-90) + IntraPartition::flat
 * (src/reorder.cpp:46-52).  flat_out[n]: group 0's members in assignment
 * order, then group 1's, ...; group_offsets_out[m+1] delimits the groups. */
dtb_status dtb_intra_partition(dtb_context* ctx, const double* sizes,
                               int64_t n, int32_t m, int32_t sort_order,
                               int32_t equal_counts, int32_t* flat_out,
                               int64_t* group_offsets_out);

/* block_group_loads (src/reorder.cpp:111-119). loads_out[m]. */
dtb_status dtb_block_group_loads(dtb_context* ctx, const double* sizes,
                                 const int32_t* order, int64_t n, int32_t m,
                                 double* loads_out);

/* select_min / select_closest (src/reorder.cpp:121-175). out[k]. */
dtb_status dtb_select_min(dtb_context* ctx, const double* keys, int64_t n_keys,
                          const int32_t* pending, int64_t n_pending, int32_t k,
                          int32_t* out);
dtb_status dtb_select_closest(dtb_context* ctx, const double* keys,
                              int64_t n_keys, const int32_t* pending,
                              int64_t n_pending, int32_t k, double target,
                              int32_t* out);

/* ---------------------------------------- L2: pipeline simulator (a15-a17) */

/* schedule_1f1b (vpp == 1) / schedule_interleaved (src/pipeline_sim.cpp:
 * 232-254).  fwd/bwd: [l*p].  Event arrays have 2*l*p entries, sorted as
 * Timeline::events (src/pipeline_sim.cpp:172-178); any event array may be
 * NULL.  device_busy[p/vpp] may be NULL. */
dtb_status dtb_schedule(dtb_context* ctx, const double* fwd, const double* bwd,
                        int32_t l, int32_t p, int32_t vpp, int32_t* ev_device,
                        int32_t* ev_microbatch, int32_t* ev_stage,
                        int32_t* ev_phase, double* ev_start, double* ev_end,
                        double* iteration_time, double* device_busy);

/* get_intervals (src/pipeline_sim.cpp:264-289) over an explicit event list
 * (any Timeline).  Outputs: n_intervals, starts/ends[n_intervals],
 * fill_offsets[n_intervals+1], fill_microbatch[fill_offsets[n]]; capacity of
 * every output array = n_events (+1 for offsets). */
dtb_status dtb_get_intervals(dtb_context* ctx, int64_t n_events,
                             const int32_t* ev_device,
                             const int32_t* ev_microbatch,
                             const int32_t* ev_stage, const int32_t* ev_phase,
                             const double* ev_start, const double* ev_end,
                             int64_t* n_intervals, double* starts,
                             double* ends, int64_t* fill_offsets,
                             int32_t* fill_microbatch);

/* interval_windows (src/pipeline_sim.cpp:291-298). volumes[l]. */
dtb_status dtb_interval_windows(dtb_context* ctx, const double* fwd,
                                const double* bwd, int32_t l, int32_t p,
                                double* volumes);

/* Batched makespans: iteration_time[b] of problem b (fwd/bwd [B*l*p]);
 * device_busy[B * p/vpp] may be NULL.  Same values as dtb_schedule. */
dtb_status dtb_schedule_batch(dtb_context* ctx, int64_t batch, const double* fwd,
                              const double* bwd, int32_t l, int32_t p,
                              int32_t vpp, double* iteration_time,
                              double* device_busy);
dtb_status dtb_schedule_batch_dev(dtb_context* ctx, int64_t batch,
                                  const double* fwd, const double* bwd,
                                  int32_t l, int32_t p, int32_t vpp,
                                  double* iteration_time, double* device_busy,
                                  void* stream);

/* Exhaustive ordering scorer — the reference's small-instance optimality
 * oracle for inter_reorder (tests/test_reorder.cpp:215-239 `sim_time` over
 * every std::next_permutation from the identity): the makespan
 * of StageTimes::permuted(order) (src/pipeline_sim.cpp:201-212) scheduled by
 * schedule_1f1b / schedule_interleaved for all l! orders, l <= 12.  Writes
 * the minimum makespan, the FIRST order (in next_permutation order) attaining
 * it, and, when all_times != NULL, every makespan in that order (l! doubles).
 * Same validation and errors as dtb_schedule. */
dtb_status dtb_exhaustive_order(dtb_context* ctx, const double* fwd, const double* bwd,
                                int32_t l, int32_t p, int32_t vpp, double* best_time,
                                int32_t* best_order, double* all_times);

/* simulate_iteration (src/simulate.cpp:23-48) over n_groups coupled groups;
 * group g owns microbatches [group_offsets[g], group_offsets[g+1]).
 * group_times[n_groups] may be NULL. */
dtb_status dtb_simulate_iteration(dtb_context* ctx, const dtb_cost_model* cm,
                                  const dtb_plan* plan, int32_t n_groups,
                                  const int64_t* group_offsets,
                                  const dtb_microbatches* mbs, double* t_iter,
                                  double* group_times, int32_t* slowest_group,
                                  double* slowest_group_time,
                                  double* mean_bubble_fraction);

/* ------------------------------------------- L3: inter reorder (a18-a19) */

/* inter_reorder (src/reorder.cpp:238-298). order_out[l]. */
dtb_status dtb_inter_reorder(dtb_context* ctx, const double* fwd,
                             const double* bwd, int32_t l, int32_t p,
                             const double* fwd_key, int32_t vpp,
                             int32_t* order_out);

/* Batched inter_reorder over independent problems (fwd/bwd [B*l*p],
 * keys [B*l], orders [B*l]). */
dtb_status dtb_inter_reorder_batch(dtb_context* ctx, int64_t batch,
                                   const double* fwd, const double* bwd,
                                   int32_t l, int32_t p, const double* fwd_key,
                                   int32_t vpp, int32_t* orders);
dtb_status dtb_inter_reorder_batch_dev(dtb_context* ctx, int64_t batch,
                                       const double* fwd, const double* bwd,
                                       int32_t l, int32_t p,
                                       const double* fwd_key, int32_t vpp,
                                       int32_t* orders, void* stream);

/* ------------------------------------- L3: disaggregated reorder (a20-a21) */

/* disaggregated_reorder (src/reorder.cpp:319-396) for ONE global batch of
 * batch->n samples.  The reordered microbatch groups of DisaggregatedResult
 * are assemble_microbatches(batch[output_order], plan). */
dtb_status dtb_disaggregated_reorder(dtb_context* ctx, const dtb_cost_model* cm,
                                     const dtb_plan* plan,
                                     const dtb_reorder_mode* mode,
                                     const dtb_samples* batch,
                                     dtb_reorder_report* report);

/* disaggregated_reorder over a stream of n_batches consecutive global
 * batches (samples->n == n_batches * plan->global_batch).  Outputs:
 * output_order[n] (batch-local indices), load_before/after[n_batches*dp_lm],
 * t_iter_before/after[n_batches]; greedy_kept[n_batches] (1 when the greedy
 * split won the fallback check, src/reorder.cpp:350-353) may be NULL.
 * Host variant pipelines host->device copies with compute. */
dtb_status dtb_reorder_stream(dtb_context* ctx, const dtb_cost_model* cm,
                              const dtb_plan* plan,
                              const dtb_reorder_mode* mode,
                              const dtb_samples* samples, int64_t n_batches,
                              int32_t* output_order, double* load_before,
                              double* load_after, double* t_iter_before,
                              double* t_iter_after, uint8_t* greedy_kept);
dtb_status dtb_reorder_stream_dev(dtb_context* ctx, const dtb_cost_model* cm,
                                  const dtb_plan* plan,
                                  const dtb_reorder_mode* mode,
                                  const dtb_samples* samples,
                                  int64_t n_batches, int32_t* output_order,
                                  double* load_before, double* load_after,
                                  double* t_iter_before, double* t_iter_after,
                                  uint8_t* greedy_kept, void* stream);

/* The intra stage of disaggregated_reorder alone (src/reorder.cpp:333-364)
 * over a stream: per global batch, cost -> stable sort -> equal-count greedy
 * over dp_lm groups -> keep-greedy-if-no-worse.  order_out[n] gets the
 * batch-local intra order; load_before/after[n_batches*dp_lm] and
 * greedy_kept[n_batches] may be NULL.  (The sort/partition kernel the
 * roofline is reported on.) */
dtb_status dtb_intra_stream_dev(dtb_context* ctx, int64_t global_batch,
                                int32_t dp_lm, int32_t sort_order,
                                const dtb_samples* samples, int64_t n_batches,
                                int32_t* order_out, double* load_before,
                                double* load_after, uint8_t* greedy_kept,
                                void* stream);

/* ------------------------------------------ L3: orchestration (a22-a29) */

/* predict_times (src/orchestrator.cpp:237-266) for n plans. */
dtb_status dtb_predict_times(dtb_context* ctx, const dtb_cost_model* cm,
                             const dtb_workload_stats* stats,
                             const dtb_plan* plans, int64_t n,
                             dtb_predicted_times* out);

/* enumerate_parallelism (src/orchestrator.cpp:268-301).  Writes the count;
 * with tuples != NULL also writes min(count, capacity) tuples in the
 * reference's sorted order. */
dtb_status dtb_enumerate_parallelism(dtb_context* ctx,
                                     const dtb_cluster_spec* cluster,
                                     int64_t global_batch, int64_t* count,
                                     dtb_tuple* tuples, int64_t capacity);

/* solve_subproblem (src/orchestrator.cpp:303-378) for n tuples. */
dtb_status dtb_solve_subproblem(dtb_context* ctx, const dtb_cost_model* cm,
                                const dtb_workload_stats* stats,
                                const dtb_tuple* tuples, int64_t n,
                                int64_t global_batch, int32_t vpp,
                                dtb_candidate* out);

/* model_orchestration (src/orchestrator.cpp:380-405).  With candidates !=
 * NULL the per-tuple table (OrchestrationOptions::keep_candidates) is
 * written in tuple order, up to `capacity` rows. */
dtb_status dtb_model_orchestration(dtb_context* ctx, const dtb_cost_model* cm,
                                   const dtb_workload_stats* stats,
                                   int64_t global_batch, int32_t vpp,
                                   dtb_orchestration_result* result,
                                   dtb_candidate* candidates,
                                   int64_t capacity);

/* brute_force_oracle (src/orchestrator.cpp:433-491): exhaustive integer
 * search over every tuple of enumerate_parallelism and every PP triple with
 * q_me*pp_me + q_lm*pp_lm + q_mg*pp_mg <= total_gpus, memory_check,
 * predict_times, BestTracker order; candidates_evaluated counts the
 * memory-feasible plans.  CapExceededError ("exhaustive search capped at
 * <cap> GPUs, got <n>") when total_gpus > gpu_cap (the reference's
 * BruteForceOptions default is 32; the GPU search accepts larger caps). */
dtb_status dtb_brute_force_oracle(dtb_context* ctx, const dtb_cost_model* cm,
                                  const dtb_workload_stats* stats, int64_t global_batch,
                                  int32_t vpp, int32_t gpu_cap,
                                  dtb_orchestration_result* result);

/* rigid_baseline (src/orchestrator.cpp:407-431): Megatron-style rigid
 * orchestration — encoder/generator share the backbone's TP and DP with one
 * pipeline stage each, the backbone takes every remaining GPU; the best by
 * predicted time (BestTracker order).  InfeasibleError "no feasible rigid
 * configuration". */
dtb_status dtb_rigid_baseline(dtb_context* ctx, const dtb_cost_model* cm,
                              const dtb_workload_stats* stats, int64_t global_batch,
                              int32_t vpp, dtb_plan* plan);

/* ------------------------------------------------------------ trace ingest
 * ingest_trace (src/workload.cpp:115-153): JSONL records
 * {"text_tokens": int, "image_subseqs": [int...], "audio_subseqs": [int...]}
 * one per line -> the sample CSR of dtb_samples.  Same line splitting
 * (std::getline), blank-line rule, JSON grammar (nlohmann 3.11.3, last
 * duplicate key wins), int64 conversion and Sample::valid checks as the
 * reference; a failure is DTB_ERR_TRACE with TraceError's kind() and line()
 * in dtb_trace_result; the message is "<kind> at line <n>: <why>".  ABI limits
 * (nesting deeper than 1024, token counts that do not fit int32, lines over
 * 2^31 bytes) are DTB_ERR_INVALID_ARGUMENT with the line. */
typedef struct dtb_trace_csr {
  int64_t cap_samples;     /* text_tokens holds cap_samples, the offsets cap_samples + 1 */
  int64_t cap_image;       /* image_tokens capacity */
  int64_t cap_audio;       /* audio_tokens capacity */
  int32_t* text_tokens;
  int32_t* image_offsets;
  int32_t* image_tokens;
  int32_t* audio_offsets;
  int32_t* audio_tokens;
} dtb_trace_csr;

enum { DTB_TRACE_NONE = 0, DTB_TRACE_PARSE_ERROR = 1, DTB_TRACE_INVARIANT_VIOLATION = 2 };

typedef struct dtb_trace_result {
  int64_t n_samples;       /* produced — or required, when a capacity is short */
  int64_t n_image;
  int64_t n_audio;
  int64_t n_lines;         /* getline lines, blank ones included */
  int32_t error_kind;      /* DTB_TRACE_*: TraceError::kind() */
  int32_t error_line;      /* TraceError::line(), 1-based */
  int32_t error_reason;    /* detail code (csrc/jsonl.cuh JReason) */
  int32_t reserved;
} dtb_trace_result;

/* Host bytes -> host CSR.  out == NULL (or out->text_tokens == NULL): sizes
 * only.  A short capacity returns DTB_ERR_INVALID_ARGUMENT with the required
 * sizes in res. */
dtb_status dtb_ingest_trace(dtb_context* ctx, const char* bytes, int64_t len,
                            int64_t seq_len_cap, const dtb_trace_csr* out,
                            dtb_trace_result* res);
/* Device bytes -> device CSR (all pointers device pointers; ctx stream). */
dtb_status dtb_ingest_trace_dev(dtb_context* ctx, const char* bytes, int64_t len,
                                int64_t seq_len_cap, const dtb_trace_csr* out,
                                dtb_trace_result* res);

/* One shard of the search for multi-GPU runs: evaluates the tuples whose
 * sorted index i satisfies i % shard_count == shard_index and writes the
 * shard's BestTracker winner (feasible == 0 when none) to *best_dev, a
 * DEVICE pointer; *evaluated_dev (device int64) gets the tuple count.
 * dtb_best_reduce_dev folds n such records (device array) into one with the
 * reference's tie-break (src/orchestrator.cpp:211-233). */
dtb_status dtb_orchestration_shard_dev(dtb_context* ctx,
                                       const dtb_cost_model* cm,
                                       const dtb_workload_stats* stats,
                                       int64_t global_batch, int32_t vpp,
                                       int64_t shard_index,
                                       int64_t shard_count,
                                       dtb_candidate* best_dev,
                                       int64_t* evaluated_dev, void* stream);
dtb_status dtb_best_reduce_dev(dtb_context* ctx, const dtb_candidate* records,
                               int64_t n, dtb_candidate* best_dev,
                               void* stream);

/* ------------------------------------- multi-GPU reorder stream (§8e) */

/* One process per GPU.  The reorder stream shards by global-batch range
 * (batches are independent; src/reorder.cpp:319-396 reads
 * one batch); the concatenated ordering is exchanged INSIDE the library over
 * NVLink: every rank owns a replica buffer of the whole ordering (u16
 * in-batch sample indices, global position = batch * global_batch + index),
 * opened by every peer over CUDA IPC, and the sharded call stores its shard
 * straight into every replica (peer stores) on a second stream that overlaps
 * the simulations, ending with a device-side flag barrier over the group.
 * Host transport of the 64-byte handles is the caller's (e.g.
 * torch.distributed all_gather_object); no NCCL on the data path. */
typedef struct dtb_peer_handle {
  unsigned char bytes[64]; /* cudaIpcMemHandle_t */
} dtb_peer_handle;
typedef struct dtb_peer_group dtb_peer_group;

/* Replica buffer for n_samples (device memory of ctx's GPU) and its handle. */
dtb_status dtb_peer_buffer_create(dtb_context* ctx, int64_t n_samples, uint16_t** replica,
                                  dtb_peer_handle* handle);
dtb_status dtb_peer_buffer_destroy(dtb_context* ctx, uint16_t* replica);
/* handles[world] in rank order (this rank's own handle included). */
dtb_status dtb_peer_group_open(dtb_context* ctx, int32_t rank, int32_t world,
                               uint16_t* replica, int64_t n_samples,
                               const dtb_peer_handle* handles, dtb_peer_group** out);
dtb_status dtb_peer_group_close(dtb_peer_group* group);
/* (first batch, batch count) of rank `rank` of `world` over n_batches:
 * contiguous ranges whose sizes differ by at most one (the first
 * n_batches % world ranks get one more). */
dtb_status dtb_shard_range(int64_t n_batches, int32_t rank, int32_t world, int64_t* first,
                           int64_t* count);
/* disaggregated_reorder over this rank's batch range of the stream
 * (`samples` = the WHOLE stream, device pointers; n_batches = the whole
 * stream's batch count).  Per-batch outputs are written at their global
 * batch positions of the (whole-stream-sized) device arrays
 * load_before/after[n_batches * dp_lm], t_iter_before/after[n_batches],
 * greedy_kept[n_batches] (any may be NULL except t_iter_before /
 * t_iter_after); the ordering goes to every replica of the group.  When the
 * call's work on `stream` completes, every rank's replica holds the whole
 * ordering of every rank that made the same call. */
dtb_status dtb_reorder_stream_shard_dev(dtb_context* ctx, const dtb_cost_model* cm,
                                        const dtb_plan* plan, const dtb_reorder_mode* mode,
                                        const dtb_samples* samples, int64_t n_batches,
                                        dtb_peer_group* group, double* load_before,
                                        double* load_after, double* t_iter_before,
                                        double* t_iter_after, uint8_t* greedy_kept,
                                        void* stream);

/* ------------------------------------------- CUDA graphs of a stream call */

/* The whole device pipeline of one reorder-stream call (cost pass,
 * partition, simulations, [inter reorder, composition], [peer exchange]) is
 * captured once into a CUDA graph for FIXED device pointers and replayed with
 * one launch: dtb_reorder_stream_dev when group == NULL (output_order
 * required), else dtb_reorder_stream_shard_dev (output_order ignored).  The
 * peer exchange's barrier counts calls on the device, so replays stay in
 * step across ranks. */
typedef struct dtb_graph dtb_graph;
dtb_status dtb_reorder_stream_graph_create(dtb_context* ctx, const dtb_cost_model* cm,
                                           const dtb_plan* plan, const dtb_reorder_mode* mode,
                                           const dtb_samples* samples, int64_t n_batches,
                                           dtb_peer_group* group, int32_t* output_order,
                                           double* load_before, double* load_after,
                                           double* t_iter_before, double* t_iter_after,
                                           uint8_t* greedy_kept, dtb_graph** out);
dtb_status dtb_graph_launch(dtb_graph* graph, void* stream);
dtb_status dtb_graph_destroy(dtb_graph* graph);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* DISTTRAIN_B200_H */

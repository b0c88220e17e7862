// Launcher declarations shared between the kernel translation units and the
// C-ABI layer (capi.cu).
#pragma once

#include <cstddef>
#include <cuda_runtime.h>

#include "dtb_internal.cuh"

namespace dtb {

// ---------------------------------------------------------------- intra
struct FusedArgs {
  int n;      // samples per global batch
  int m;      // backbone DP groups
  int order;  // DTB_ASCENDING / DTB_DESCENDING
  int intra;  // ReorderMode::intra
  const int* img_off;  // stream CSR (absolute offsets)
  const int* img_tok;
  const int* aud_off;  // may be null
  const int* aud_tok;
  int* order_out;       // [n_batches * n] batch-local intra order
  double* load_before;  // [n_batches * m] or null
  double* load_after;   // [n_batches * m] or null
  unsigned char* kept;  // [n_batches] or null
  // Per-position modality tokens of the intra order (see TokSrc): u16 for
  // batches whose greedy split was kept (identity batches reuse tok16), and
  // 32-bit input/staged copies for batches on the 32-bit path.  Any may be
  // null when no consumer needs them.
  unsigned short* tok16_staged;  // [n_batches * n]
  int* tok32_orig;               // [n_batches * n]
  int* tok32_staged;             // [n_batches * n]
  int pg;               // samples per backbone group (global_batch / dp_lm)
  int dp_me;
  unsigned char* wide_scratch;  // [n_batches * fused_wide_scratch_bytes(1)]
  unsigned long long* prof;     // optional [n_batches][64] phase timestamps (debug)
  // Output of the cost pass (launch_cost_stream): modality tokens per sample,
  // saturated to 0x7fff, and a per-batch flag set when any sample saturated
  // (that batch then takes the 32-bit path from the CSR).
  const unsigned short* tok16;
  unsigned int* wide_flag;  // set by the kernel for every batch it runs on the 32-bit path
  // Per-batch state from cost_stream_kernel (null: every batch takes the
  // sort path from tok16 / the 32-bit path from wide_flag) and its identity
  // block loads [n_batches * m].
  const unsigned* state;
  const unsigned* blk_ident;
  const unsigned* list;  // [1 + n]: batches to process (null: every batch, one CTA each)
  FastDiv div_pg;
  DevErr* err;
};

// Batch states written by cost_stream_kernel (read by intra_fused_kernel).
constexpr unsigned kBatchFast = 0;     // histogram path
constexpr unsigned kBatchDecided = 1;  // all outputs written (order stays the identity)
constexpr unsigned kBatchSort = 2;     // a token sum >= the histogram range: sort path
constexpr int kNarrowGroups = 128;    // groups of the partition kernel's shared-memory path
constexpr unsigned kBatchWide = 3;     // a token sum < 0 or > 0x7fff: 32-bit path

// Streaming cost pass (csrc/k_cost.cu) over chunks of 1024 samples, TMA-staged
// CSR: per-sample u16 tokens, identity order, identity block loads, and per
// batch (last chunk done) the keep decision when the averaging bound settles
// it.
struct CostArgs {
  int n, m, order, intra;
  long long n_batches;
  const int* img_off;
  const int* img_tok;
  const int* aud_off;  // may be null
  const int* aud_tok;
  int staged;  // 16-byte aligned CSR and n % 4 == 0: bulk copies
  unsigned short* tok16;   // [n_batches * n]
  int* order_out;          // [n_batches * n] batch-local identity
  unsigned short* tok16_staged;  // [n_batches * n] tokens in the kept order (small batches)
  unsigned* blk_ident;     // [n_batches * m]  zeroed
  unsigned* bstat;         // [n_batches * 4]  zeroed: zeros, sum of cost_size, flags, -
  unsigned* list;          // [1 + n_batches]: count (zeroed), batches left to the partition kernel
  unsigned* state;         // [n_batches]
  unsigned* wide_flag;     // [n_batches]
  int* tok32_orig;         // [n_batches * n]: 32-bit tokens of the batches routed to the wide path
  double* load_before;     // [n_batches * m] or null
  double* load_after;
  unsigned char* kept;     // [n_batches] or null
  FastDiv div_pg;
  FastDiv div_cpb;         // chunks per batch (set by launch_cost_stream)
  DevErr* err;             // a negative or >= 2^31 token sum (E_COST_RANGE)
};
size_t cost_scratch_bytes(long long n_batches, int m);  // blk_ident, bstat, list, state
cudaError_t launch_cost_stream(const CostArgs& a, cudaStream_t stream);

// Multi-GPU exchange (k_peer.cu): this rank's shard of the ordering (int32
// batch-local indices) stored as u16 into every rank's replica, then a flag
// barrier over the group.
constexpr int kMaxPeers = 8;
struct PeerBcast {
  const int* src;                   // [count] this rank's shard, batch-local indices
  long long count;
  unsigned short* dst[kMaxPeers];   // replica of rank p + the shard's stream offset
  unsigned* flags[kMaxPeers];       // flag array [world] of replica p
  const unsigned* flags_local;      // this rank's flag array
  unsigned* done;                   // CTA counter (zeroed by the launcher)
  unsigned* epoch;                  // this rank's call counter (device; graph-replay safe)
  int world, rank, aligned;         // aligned: src / dst 16-byte aligned
  // phase 0: every batch, then the flag barrier.  With the cost pass's
  // per-batch state: phase 1 sends the batches it decided (their order is
  // final before the partition kernel runs), phase 2 the rest, then the
  // barrier.  n: samples per global batch.
  const unsigned* state;
  int n, phase;
};
cudaError_t launch_peer_broadcast(const PeerBcast& a, cudaStream_t stream);

// Cost pass: tok16[i] = min(modality tokens of sample i, 0x7fff) for the
// whole stream, wide_flag[i / n] |= 1 on saturation or negative tokens.
// Modality tokens of position `pos` of global batch b, in the input order
// (staged == false) or the intra order (staged == true), written by the cost
// pass / fused kernel (FusedArgs).
struct TokSrc {
  const unsigned short* t16;         // input order (cost pass)
  const unsigned short* t16_staged;  // intra order where kept[b]
  const int* t32;                    // 32-bit path batches
  const int* t32_staged;
  const unsigned char* kept;
  const unsigned int* wide;
  int n;
  __device__ __forceinline__ long long get(long long b, int pos, bool staged) const {
    const long long x = b * n + pos;
    if (wide[b]) return staged ? t32_staged[x] : t32[x];
    return (staged && kept[b]) ? t16_staged[x] : t16[x];
  }
};

size_t fused_wide_scratch_bytes(long long n_batches);
size_t fused_smem_bytes();
int fused_max_n();
int fused_max_m();
cudaError_t launch_intra_fused(const FusedArgs& a, long long n_batches,
                               cudaStream_t stream, bool pdl = false);

size_t intra_generic_scratch(int n, int m);
int intra_generic_max_m();
cudaError_t launch_intra_generic(const double* sizes, int n, int m, int order,
                                 int equal_counts, void* scratch,
                                 size_t scratch_bytes, int* flat_out,
                                 long long* offsets_out, cudaStream_t stream);

cudaError_t launch_block_loads(const double* sizes, const int* order, int n,
                               int m, double* loads, cudaStream_t stream);  // order null: identity
// Generic route for global batches beyond the fused kernels (k_misc.cu).
cudaError_t launch_batch_tokens(const int* io, const int* it, const int* ao, const int* at,
                                long long first, int n, int* tok32, double* sizes, DevErr* err,
                                int bidx, cudaStream_t stream);
cudaError_t launch_generic_decide(const double* li, const double* lg, int m, int n, long long b,
                                  int intra, const int* flat, const int* tok32, int* order_out,
                                  int* tok32_staged, double* load_before, double* load_after,
                                  unsigned char* kept, unsigned* wide_flag, cudaStream_t stream);
cudaError_t launch_select(const double* keys, const int* pending, int np,
                          int k, int closest, double target, int* out,
                          cudaStream_t stream);
cudaError_t launch_cost_sizes(const int* img_off, const int* img_tok,
                              const int* aud_off, const int* aud_tok,
                              long long n, long long* out, cudaStream_t stream);
cudaError_t launch_compute_stats(const int* img_off, const int* img_tok,
                                 const int* aud_off, const int* aud_tok,
                                 long long n, double* out2, cudaStream_t stream);

// ------------------------------------------------------------- simulator
// Generic schedule of one problem (any vpp) with full event materialisation
// in op order: ev arrays [2*l*p]; busy [devices]; it [1].
cudaError_t launch_schedule_events(const double* fwd, const double* bwd, int l,
                                   int p, int vpp, int* ev_dev, int* ev_mb,
                                   int* ev_stage, int* ev_phase,
                                   double* ev_start, double* ev_end,
                                   double* busy, double* it, void* scratch,
                                   DevErr* err, cudaStream_t stream);
cudaError_t launch_sort_events(int n_events, int* dev, int* mb, int* stage,
                               int* phase, double* start, double* end,
                               void* scratch, size_t scratch_bytes,
                               cudaStream_t stream);
size_t sort_events_scratch(int n_events);
cudaError_t launch_get_intervals(long long n_events, const int* dev,
                                 const int* mb, const int* phase,
                                 const double* start, const double* end,
                                 long long* n_int, double* starts,
                                 double* ends, long long* fill_off,
                                 int* fill_mb, cudaStream_t stream);
cudaError_t launch_schedule_batch(long long batch, const double* fwd,
                                  const double* bwd, int l, int p, int vpp,
                                  double* it, double* busy, void* scratch,
                                  DevErr* err, cudaStream_t stream);
size_t schedule_batch_scratch(long long batch, int l, int p, int vpp);
// StageTimes::valid over explicit matrices (E_BAD_TIMES, a = 1 fwd / 2 bwd).
cudaError_t launch_check_times(const double* fwd, const double* bwd, long long cells,
                               DevErr* err, cudaStream_t stream);

// Stage-time rows for microbatches (build_stage_times), expanded to l x p.
cudaError_t launch_stage_times(const DevCM& cm, const dtb_plan& plan,
                               long long l, const long long* enc,
                               const long long* gen, const int* count,
                               double* fwd, double* bwd, DevErr* err,
                               cudaStream_t stream);
cudaError_t launch_fwd_keys(const DevCM& cm, const dtb_plan& plan, long long l,
                            const long long* enc, const long long* gen,
                            const int* count, double* keys, DevErr* err,
                            cudaStream_t stream);
cudaError_t launch_unit_times(const DevCM& cm, int kind, int tp, long long n,
                              const double* loads, double* fwd, double* bwd,
                              DevErr* err, cudaStream_t stream);

// Token-indexed cost table for the stream path: for every microbatch token
// sum s in [0, size), the build_stage_times entries of the encoder and
// generator units at load s / span, and microbatch_fwd_keys' key.  Each
// entry is computed once with exactly the reference's operation sequence,
// so a lookup is bit-identical to recomputing it.
struct CostTable {
  const double4* eg;   // (f, b) of the encoder unit, (f, b) of the generator
                       // unit: one 32-byte row per token sum (one 256-bit load)
  const double* key;   // forward key
  int size;            // sums >= size are evaluated directly
  int span;
  const double2* fz = nullptr;  // optional compact (encoder f, generator f) rows
};
constexpr int kCostTableMax = 1 << 20;
// compact forward rows of a cost table (the inter gather variant's reads)
cudaError_t launch_table_fz(const double4* eg, double2* fz, int size, cudaStream_t stream);
cudaError_t launch_cost_table(const DevCM& cm, const dtb_plan& plan, int span, int size,
                              double4* eg, double* key, DevErr* err, cudaStream_t stream);

// Makespans of coupled groups whose microbatches are given by token keys:
// group g of batch b covers microbatches [g*l, (g+1)*l) of batch b.
// t_group[b * groups + g] = iteration time; also device busy sums for the
// bubble fraction when busy != null ([b*groups+g][devices]).
struct GroupSimArgs {
  DevCM cm;
  dtb_plan plan;
  long long n_batches;
  int groups;        // coupled groups per batch
  int l;             // microbatches per group
  const long long* enc;  // [n_batches * groups * l] token sums (group-contiguous)
  const long long* gen;
  const int* count;      // sample counts (null = `span` for all)
  int span;
  // Stream form instead of enc/gen/count (encoder == generator tokens,
  // count == span): span == 1 reads microbatch (e, i) = position e*l + i of
  // `tok`; span > 1 reads assembled sums `mbsum` [n_batches][groups][l].
  bool stream;
  TokSrc tok;
  bool staged;           // read tok's intra order
  const int* mbsum;
  const int* order;      // optional [n_batches][groups][l] microbatch order
  CostTable table;       // optional (size 0 = evaluate directly)
  // optional [n_batches]: groups of batches whose flag is 0 are not
  // simulated (intra-only t_iter_after of a batch whose greedy split was
  // not kept is its t_iter_before: same microbatches, same operations)
  const unsigned char* only_kept;
  double* t_group;
  double* busy;
  DevErr* err;
  // optional [n_batches]: t_iter of each batch (max over its groups +
  // dp_sync, simulate.cpp:31-46) written by the simulation kernel itself when
  // group_sims_fuse_reduce(a) (one CTA per batch)
  double* t_iter;
  double dp_sync;
};
// Per-microbatch token sums in a's order (warning log), out[groups * l].
cudaError_t launch_mb_tokens(const GroupSimArgs& a, int* out, cudaStream_t stream);
__device__ __forceinline__ bool sim_skipped(const GroupSimArgs& a, long long gid) {
  return a.only_kept != nullptr && a.only_kept[gid / a.groups] == 0;
}
bool group_sims_fuse_reduce(const GroupSimArgs& a);
cudaError_t launch_group_sims(const GroupSimArgs& a, void* scratch,
                              cudaStream_t stream, bool pdl = false);
size_t group_sims_scratch(const GroupSimArgs& a);

// ------------------------------------------------- exhaustive orderings
int exhaustive_max_l();
int exhaustive_max_p();
size_t exhaustive_scratch(int n_blocks);
cudaError_t launch_exhaustive(const double* fwd, const double* bwd, int l, int p, int vpp,
                              double* all, double* best_t, int* best_order, void* scratch,
                              int n_blocks, DevErr* err, cudaStream_t stream);

// --------------------------------------------------------- inter reorder
struct InterArgs {
  long long batch;       // independent problems
  int l, p, vpp;
  const double* fwd;     // [batch * l * p] (explicit matrices), or null
  const double* bwd;
  const double* keys;    // [batch * l], or null (computed from tokens)
  // Disaggregated form: rows from per-microbatch token sums via the cost
  // model; problem = b*groups + e, microbatch i = staged position e*l + i
  // (span == 1, `tok`) or mbsum[b][e][i] (span > 1).
  DevCM cm;
  dtb_plan plan;
  bool stream;
  TokSrc tok;
  const int* mbsum;
  int groups;
  int span;
  CostTable table;       // optional (size 0 = evaluate directly)
  int* orders;           // [batch * l]
  DevErr* err;
  unsigned char* redo;   // inter_tok: zeroed flag per problem (gather pass), or null
  bool redo_only;        // inter_tok shared-memory pass over flagged problems only
};
cudaError_t launch_inter(const InterArgs& a, void* scratch, size_t bytes,
                         cudaStream_t stream);
// Shared-memory kernel for the stream token form (vpp == 1, compiled stage
// layouts); cudaErrorNotSupported when it does not apply.
cudaError_t launch_inter_tok(const InterArgs& a, cudaStream_t stream);
bool inter_tok_applies(const InterArgs& a);
// Warp per problem, problem resident in shared memory (k_inter3.cu): stream
// token form, vpp == 1, any stage count, l up to the shared-memory limit.
bool inter_warp_applies(const InterArgs& a);
cudaError_t launch_inter_warp(const InterArgs& a, cudaStream_t stream);
size_t inter_scratch(const InterArgs& a);

// --------------------------------------------------------- orchestration
struct OrchArgs {
  DevCM cm;
  dtb_workload_stats stats;
  long long bs;
  int vpp;
  const dtb_tuple* tuples;
  long long n;
  long long shard_index, shard_count;  // evaluate i % count == index
  dtb_candidate* out;                  // per-tuple results or null
  dtb_candidate* block_best;           // [grid] winners
  DevErr* err;
  // optional compaction (launch_orchestration): list [n] of the tuples that
  // pass tuple_costs, list_count (device) their number
  long long* list;
  unsigned* list_count;
};
cudaError_t launch_enumerate(const dtb_cluster_spec& c, long long bs,
                             const long long* divs, int n_divs,
                             long long* count, dtb_tuple* out,
                             long long capacity, void* scratch,
                             cudaStream_t stream);
cudaError_t launch_orchestration(const OrchArgs& a, int grid,
                                 cudaStream_t stream);
size_t brute_scratch(long long n_tuples);
// block_best must hold max_grid records; the launcher synchronises `stream`
// once (pair count).
cudaError_t launch_brute(const OrchArgs& a, int max_grid, unsigned long long* evaluated,
                         void* scratch, size_t bytes, cudaStream_t stream);
cudaError_t launch_rigid(const DevCM& cm, const dtb_workload_stats& stats, long long bs, int vpp,
                         const long long* divs, int n_divs, dtb_candidate* out, DevErr* err,
                         cudaStream_t stream);
cudaError_t launch_best_reduce(const dtb_candidate* in, long long n,
                               dtb_candidate* out, cudaStream_t stream);
cudaError_t launch_predict(const DevCM& cm, const dtb_workload_stats& stats,
                           const dtb_plan* plans, long long n,
                           dtb_predicted_times* out, DevErr* err,
                           cudaStream_t stream);
cudaError_t launch_memory_check(const DevCM& cm, const dtb_plan& plan,
                                dtb_memory_report* out, cudaStream_t stream);

// ------------------------------------------------ disaggregated glue
// Microbatch token sums of assembled coupled groups (assemble_microbatches,
// src/workload.cpp:179-204) from per-position tokens, [n_batches][dp_me][pg].
cudaError_t launch_assemble(long long n_batches, int n, int dp_lm, int dp_me, TokSrc tok,
                            bool staged, int* mbsum_out, cudaStream_t stream);
// output_order composition (src/reorder.cpp:370-391).
cudaError_t launch_compose(long long n_batches, int n, int dp_lm, int dp_me,
                           const int* intra, const int* inter, int* out,
                           cudaStream_t stream);
cudaError_t launch_t_iter_reduce(long long n_batches, int groups,
                                 const double* t_group, double dp_sync,
                                 double* t_iter, cudaStream_t stream,
                                 const unsigned char* only_kept = nullptr,
                                 const double* t_same = nullptr);

// ---------------------------------------------------------------- ingest
// Trace JSONL -> sample CSR (csrc/k_ingest.cu, parser csrc/jsonl.cuh).
struct IngestLines {     // per line, n_lines (+1 for counts / scan)
  int* status;           // JStatus | JReason << 8
  long long* text;
  int* img_at;
  int* aud_at;
  int* counts;           // (sample, image, audio) per line, 3 ints, n_lines + 1
  int* scan;             // exclusive scan of counts, 3 ints, n_lines + 1
};
struct IngestOut {
  int* text_tokens;
  int* image_offsets;
  int* image_tokens;
  int* audio_offsets;
  int* audio_tokens;
};
size_t ingest_lines_scratch(long long len);
// newline count (synchronises the stream), then positions in byte order;
// the write reuses the count's scratch
cudaError_t launch_nl_count(const unsigned char* bytes, long long len, void* scratch,
                            size_t scratch_bytes, long long* n_nl, cudaStream_t stream);
cudaError_t launch_nl_write(const unsigned char* bytes, long long len, void* scratch,
                            long long* nl, cudaStream_t stream);
cudaError_t launch_ingest_parse(const unsigned char* bytes, long long len, const long long* nl,
                                long long n_nl, long long n_lines, long long seq_len_cap,
                                const IngestLines& lines, unsigned long long* first_bad,
                                void* scratch, size_t scratch_bytes, cudaStream_t stream);
cudaError_t launch_ingest_write(const unsigned char* bytes, long long len, const long long* nl,
                                long long n_nl, long long n_lines, const IngestLines& lines,
                                const IngestOut& out, cudaStream_t stream);

}  // namespace dtb

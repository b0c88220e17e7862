// Pipeline simulator kernels: schedules with events, intervals, batched
// makespans, cost-model stage times, and per-coupled-group iteration sims
// (reference: src/pipeline_sim.cpp, src/simulate.cpp, src/cost_model.cpp).
#include <cub/cub.cuh>

#include <algorithm>

#include "kernels.cuh"
#include "pdl.cuh"
#include "sched.cuh"

#ifndef DTB_SIM_EXPERIMENT
#define DTB_SIM_EXPERIMENT 0
#endif

namespace dtb {

// StageTimes::valid (pipeline_sim.cpp:214-230): 0 ok, 1 negative/NaN fwd,
// 2 negative/NaN bwd.
__device__ __forceinline__ int check_times(const double* f, const double* b,
                                           int cells) {
  for (int i = 0; i < cells; ++i)
    if (!(f[i] >= 0.0)) return 1;
  for (int i = 0; i < cells; ++i)
    if (!(b[i] >= 0.0)) return 2;
  return 0;
}

// Whole-array validation: the forward matrix is checked before the backward
// one, as in the reference, so a fwd failure anywhere wins.
__global__ void check_times_kernel(const double* f, const double* b, long long cells,
                                   int* flags) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < cells;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (!(f[i] >= 0.0)) atomicOr(flags, 1);
    if (!(b[i] >= 0.0)) atomicOr(flags, 2);
  }
}

__global__ void check_times_finish(const int* flags, DevErr* err) {
  if (*flags & 1) dev_fail(err, E_BAD_TIMES, 1);
  else if (*flags & 2) dev_fail(err, E_BAD_TIMES, 2);
}

cudaError_t launch_check_times(const double* fwd, const double* bwd, long long cells,
                               DevErr* err, cudaStream_t stream) {
  int* flags = &err->pad;  // scratch word inside the error record
  cudaMemsetAsync(flags, 0, sizeof(int), stream);
  if (cells > 0) {
    long long blocks = (cells + 255) / 256;
    if (blocks > 1024) blocks = 1024;
    check_times_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(fwd, bwd, cells, flags);
  }
  check_times_finish<<<1, 1, 0, stream>>>(flags, err);
  return cudaGetLastError();
}

// ------------------------------------------------------------ one problem
__global__ void schedule_events_kernel(const double* __restrict__ fwd,
                                       const double* __restrict__ bwd, int l,
                                       int p, int vpp, int* ev_dev, int* ev_mb,
                                       int* ev_stage, int* ev_phase,
                                       double* ev_start, double* ev_end,
                                       double* busy, double* it,
                                       double* f_end, double* b_end, int* next,
                                       double* avail, DevErr* err) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int bad = check_times(fwd, bwd, l * p);
  if (bad) {
    dev_fail(err, E_BAD_TIMES, bad);
    return;
  }
  const int devices = p / vpp;
  const int per = 2 * l * vpp;
  for (int d = 0; d < devices; ++d) busy[d] = 0.0;
  double iter = 0.0;
  int* count = reinterpret_cast<int*>(avail + devices);  // per-device emit cursor
  for (int d = 0; d < devices; ++d) count[d] = 0;
  auto dur = [&](int mb, int s, int ph) {
    return ph == DTB_FORWARD ? fwd[mb * p + s] : bwd[mb * p + s];
  };
  auto visit = [&](int d, Op op, double start, double end) {
    const int e = d * per + count[d]++;
    ev_dev[e] = d;
    ev_mb[e] = op.mb;
    ev_stage[e] = op.stage;
    ev_phase[e] = op.phase;
    ev_start[e] = start;
    ev_end[e] = end;
    busy[d] += dur(op.mb, op.stage, op.phase);
    iter = smax(iter, end);
  };
  const int e = dataflow_schedule(l, p, vpp, dur, f_end, b_end, next, avail, visit);
  if (e) dev_fail(err, e);
  *it = iter;
}

cudaError_t launch_schedule_events(const double* fwd, const double* bwd, int l,
                                   int p, int vpp, int* ev_dev, int* ev_mb,
                                   int* ev_stage, int* ev_phase,
                                   double* ev_start, double* ev_end,
                                   double* busy, double* it, void* scratch,
                                   DevErr* err, cudaStream_t stream) {
  char* s = static_cast<char*>(scratch);
  double* f_end = reinterpret_cast<double*>(s);
  double* b_end = f_end + static_cast<size_t>(l) * p;
  double* avail = b_end + static_cast<size_t>(l) * p;
  int* next = reinterpret_cast<int*>(avail + 2 * p + 2);
  schedule_events_kernel<<<1, 32, 0, stream>>>(fwd, bwd, l, p, vpp, ev_dev,
                                               ev_mb, ev_stage, ev_phase,
                                               ev_start, ev_end, busy, it,
                                               f_end, b_end, next, avail, err);
  return cudaGetLastError();
}

// Timeline::events order (pipeline_sim.cpp:172-178): (start, device,
// microbatch, stage); phase last for a total order.
__device__ __forceinline__ unsigned long long ord_time(double x) {
  if (x == 0.0) x = 0.0;
  const unsigned long long b = __double_as_longlong(x);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void event_keys_kernel(int n, const int* dev, const int* mb,
                                  const int* stage, const int* phase,
                                  const double* start,
                                  unsigned long long* k_secondary,
                                  unsigned long long* k_start, int* idx) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  k_secondary[i] = (static_cast<unsigned long long>(dev[i]) << 48) |
                   (static_cast<unsigned long long>(mb[i]) << 24) |
                   (static_cast<unsigned long long>(stage[i]) << 1) |
                   static_cast<unsigned long long>(phase[i]);
  k_start[i] = ord_time(start[i]);
  idx[i] = i;
}

__global__ void gather_events_kernel(int n, const int* perm, const int* dev,
                                     const int* mb, const int* stage,
                                     const int* phase, const double* start,
                                     const double* end, int* o_dev, int* o_mb,
                                     int* o_stage, int* o_phase,
                                     double* o_start, double* o_end) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int j = perm[i];
  o_dev[i] = dev[j];
  o_mb[i] = mb[j];
  o_stage[i] = stage[j];
  o_phase[i] = phase[j];
  o_start[i] = start[j];
  o_end[i] = end[j];
}

size_t sort_events_scratch(int n) {
  size_t t1 = 0, t2 = 0;
  cub::DoubleBuffer<unsigned long long> dk(nullptr, nullptr);
  cub::DoubleBuffer<int> dv(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, t1, dk, dv, n, 0, 64);
  t2 = t1;
  return static_cast<size_t>(n) * (8 * 4 + 4 * 2 + 4 * 4 + 8 * 2) + t2 + 4096;
}

// Sorts the event arrays in place into Timeline order: a stable radix sort
// by the secondary key, then a stable radix sort by start time.
cudaError_t launch_sort_events(int n, int* dev, int* mb, int* stage,
                               int* phase, double* start, double* end,
                               void* scratch, size_t bytes,
                               cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  char* p = static_cast<char*>(scratch);
  auto take = [&](size_t b) {
    char* r = p;
    p += (b + 255) & ~size_t(255);
    return r;
  };
  auto* ks = reinterpret_cast<unsigned long long*>(take(8ull * n));
  auto* ks2 = reinterpret_cast<unsigned long long*>(take(8ull * n));
  auto* kt = reinterpret_cast<unsigned long long*>(take(8ull * n));
  auto* kt2 = reinterpret_cast<unsigned long long*>(take(8ull * n));
  int* idx = reinterpret_cast<int*>(take(4ull * n));
  int* idx2 = reinterpret_cast<int*>(take(4ull * n));
  int* o_dev = reinterpret_cast<int*>(take(4ull * n));
  int* o_mb = reinterpret_cast<int*>(take(4ull * n));
  int* o_stage = reinterpret_cast<int*>(take(4ull * n));
  int* o_phase = reinterpret_cast<int*>(take(4ull * n));
  double* o_start = reinterpret_cast<double*>(take(8ull * n));
  double* o_end = reinterpret_cast<double*>(take(8ull * n));
  const size_t used = static_cast<size_t>(p - static_cast<char*>(scratch));
  size_t temp = bytes - used;
  const int grid = (n + 255) / 256;
  event_keys_kernel<<<grid, 256, 0, stream>>>(n, dev, mb, stage, phase, start,
                                              ks, kt, idx);
  // 1) by secondary key (carry the start key along as a second pass input)
  cub::DoubleBuffer<unsigned long long> dk(ks, ks2);
  cub::DoubleBuffer<int> dv(idx, idx2);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(p, temp, dk, dv, n, 0, 64, stream);
  if (e != cudaSuccess) return e;
  // gather start keys into the secondary order, then sort stably by start
  int* perm = dv.Current();
  int* spare = dv.Alternate();
  gather_events_kernel<<<grid, 256, 0, stream>>>(n, perm, dev, mb, stage, phase,
                                                 start, end, o_dev, o_mb, o_stage,
                                                 o_phase, o_start, o_end);
  event_keys_kernel<<<grid, 256, 0, stream>>>(n, o_dev, o_mb, o_stage, o_phase,
                                              o_start, ks, kt, spare);
  cub::DoubleBuffer<unsigned long long> dk2(kt, kt2);
  cub::DoubleBuffer<int> dv2(spare, perm);
  e = cub::DeviceRadixSort::SortPairs(p, temp, dk2, dv2, n, 0, 64, stream);
  if (e != cudaSuccess) return e;
  gather_events_kernel<<<grid, 256, 0, stream>>>(n, dv2.Current(), o_dev, o_mb,
                                                 o_stage, o_phase, o_start, o_end,
                                                 dev, mb, stage, phase, start, end);
  return cudaGetLastError();
}

// get_intervals (pipeline_sim.cpp:264-289) over a sorted event list.
__global__ void get_intervals_kernel(long long n, const int* dev, const int* mb,
                                     const int* phase, const double* start,
                                     const double* end, long long* n_int,
                                     double* starts, double* ends,
                                     long long* fill_off, int* fill_mb) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  // first device-0 forward and whether any device-0 backward exists
  long long f_first = -1;
  bool any_b = false;
  for (long long i = 0; i < n; ++i) {
    if (dev[i] != 0) continue;
    if (phase[i] == DTB_FORWARD) {
      if (f_first < 0) f_first = i;
    } else {
      any_b = true;
    }
  }
  fill_off[0] = 0;
  if (f_first < 0 || !any_b) {
    *n_int = 0;
    return;
  }
  double anchor = end[f_first];
  long long fill = 0;  // cursor over device-0 forwards in event order
  auto next_fwd = [&](long long from) {
    while (from < n && !(dev[from] == 0 && phase[from] == DTB_FORWARD)) ++from;
    return from;
  };
  fill = next_fwd(0);
  long long k = 0, filled = 0;
  for (long long i = 0; i < n; ++i) {
    if (dev[i] != 0 || phase[i] != DTB_BACKWARD) continue;
    const double s = anchor, e = start[i];
    while (fill < n && start[fill] < s) fill = next_fwd(fill + 1);
    while (fill < n && start[fill] < e) {
      fill_mb[filled++] = mb[fill];
      fill = next_fwd(fill + 1);
    }
    starts[k] = s;
    ends[k] = e;
    ++k;
    fill_off[k] = filled;
    anchor = end[i];
  }
  *n_int = k;
}

cudaError_t launch_get_intervals(long long n, const int* dev, const int* mb,
                                 const int* phase, const double* start,
                                 const double* end, long long* n_int,
                                 double* starts, double* ends,
                                 long long* fill_off, int* fill_mb,
                                 cudaStream_t stream) {
  get_intervals_kernel<<<1, 32, 0, stream>>>(n, dev, mb, phase, start, end,
                                             n_int, starts, ends, fill_off,
                                             fill_mb);
  return cudaGetLastError();
}

// --------------------------------------------------------- batched makespans
__global__ void schedule_batch_kernel(long long batch, const double* __restrict__ fwd,
                                      const double* __restrict__ bwd, int l, int p,
                                      int vpp, double* __restrict__ it,
                                      double* __restrict__ busy_out,
                                      double* scratch, DevErr* err) {
  const long long b = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  const size_t cells = static_cast<size_t>(l) * p;
  const double* f = fwd + b * cells;
  const double* bw = bwd + b * cells;
  const int bad = check_times(f, bw, static_cast<int>(cells));
  if (bad) {
    dev_fail(err, E_BAD_TIMES, bad);
    return;
  }
  const int devices = p / vpp;
  // per-thread scratch: 2*p (+ cells*2 for the dataflow path) doubles
  const size_t per = vpp == 1 ? static_cast<size_t>(3 * p + devices)
                              : static_cast<size_t>(2 * cells + 2 * devices + devices);
  double* s = scratch + b * per;
  double* busy = vpp == 1 ? s + 3 * p : s + 2 * cells + 2 * devices;
  for (int d = 0; d < devices; ++d) busy[d] = 0.0;
  double iter = 0.0;
  auto dur = [&](int mb, int st, int ph) {
    return ph == DTB_FORWARD ? f[mb * p + st] : bw[mb * p + st];
  };
  auto visit = [&](int d, Op op, double start, double end) {
    busy[d] += dur(op.mb, op.stage, op.phase);
    iter = smax(iter, end);
  };
  if (vpp == 1) {
    tick_1f1b(l, p, dur, s, s + p, s + 2 * p, visit);
  } else {
    const int e = dataflow_schedule(l, p, vpp, dur, s, s + cells,
                                    reinterpret_cast<int*>(s + 2 * cells + devices),
                                    s + 2 * cells, visit);
    if (e) dev_fail(err, e);
  }
  it[b] = iter;
  if (busy_out != nullptr)
    for (int d = 0; d < devices; ++d) busy_out[b * devices + d] = busy[d];
}

size_t schedule_batch_scratch(long long batch, int l, int p, int vpp) {
  const size_t cells = static_cast<size_t>(l) * p;
  const int devices = p / vpp;
  const size_t per = vpp == 1 ? static_cast<size_t>(3 * p + devices)
                              : 2 * cells + 3 * static_cast<size_t>(devices);
  return batch * per * sizeof(double) + 256;
}

cudaError_t launch_schedule_batch(long long batch, const double* fwd,
                                  const double* bwd, int l, int p, int vpp,
                                  double* it, double* busy, void* scratch,
                                  DevErr* err, cudaStream_t stream) {
  const int T = 128;
  const long long grid = (batch + T - 1) / T;
  schedule_batch_kernel<<<static_cast<unsigned>(grid), T, 0, stream>>>(
      batch, fwd, bwd, l, p, vpp, it, busy, static_cast<double*>(scratch), err);
  return cudaGetLastError();
}

// ------------------------------------------------------- cost-model kernels
__global__ void stage_times_kernel(DevCM cm, dtb_plan plan, long long l,
                                   const long long* enc, const long long* gen,
                                   const int* count, double* fwd, double* bwd,
                                   DevErr* err) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= l) return;
  StageRow row;
  const int e = dev_stage_row(cm, plan, mb_mean(enc[i], count[i]),
                              mb_mean(gen[i], count[i]), &row);
  if (e) {
    dev_fail(err, e, e == E_EMPTY_TP || e == E_TP_NOT_ALLOWED ? 0 : 0);
    return;
  }
  const int p = plan_stages(plan);
  for (int s = 0; s < p; ++s) {
    const int u = stage_unit(plan, s);
    fwd[i * p + s] = row.f[u];
    bwd[i * p + s] = row.b[u];
  }
}

cudaError_t launch_stage_times(const DevCM& cm, const dtb_plan& plan,
                               long long l, const long long* enc,
                               const long long* gen, const int* count,
                               double* fwd, double* bwd, DevErr* err,
                               cudaStream_t stream) {
  if (l == 0) return cudaSuccess;
  const long long grid = (l + 127) / 128;
  stage_times_kernel<<<static_cast<unsigned>(grid), 128, 0, stream>>>(
      cm, plan, l, enc, gen, count, fwd, bwd, err);
  return cudaGetLastError();
}

__global__ void fwd_keys_kernel(DevCM cm, dtb_plan plan, long long l,
                                const long long* enc, const long long* gen,
                                const int* count, double* keys, DevErr* err) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= l) return;
  const int e = dev_fwd_key(cm, plan, mb_mean(enc[i], count[i]),
                            mb_mean(gen[i], count[i]), &keys[i]);
  if (e) dev_fail(err, e);
}

cudaError_t launch_fwd_keys(const DevCM& cm, const dtb_plan& plan, long long l,
                            const long long* enc, const long long* gen,
                            const int* count, double* keys, DevErr* err,
                            cudaStream_t stream) {
  if (l == 0) return cudaSuccess;
  fwd_keys_kernel<<<static_cast<unsigned>((l + 127) / 128), 128, 0, stream>>>(
      cm, plan, l, enc, gen, count, keys, err);
  return cudaGetLastError();
}

__global__ void unit_times_kernel(DevCM cm, int kind, int tp, long long n,
                                  const double* loads, double* fwd, double* bwd,
                                  DevErr* err) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  int e = 0;
  if (fwd) e = dev_unit_fwd(cm, kind, tp, loads[i], &fwd[i]);
  if (!e && bwd) e = dev_unit_bwd(cm, kind, tp, loads[i], &bwd[i]);
  if (e) dev_fail(err, e, tp, kind);
}

cudaError_t launch_unit_times(const DevCM& cm, int kind, int tp, long long n,
                              const double* loads, double* fwd, double* bwd,
                              DevErr* err, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  unit_times_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, stream>>>(
      cm, kind, tp, n, loads, fwd, bwd, err);
  return cudaGetLastError();
}

// ------------------------------------------------- coupled-group iteration
// Microbatch token keys of coupled group `gid`, position i (after the
// group's optional reorder): stream form (positions of TokSrc when span == 1,
// assembled sums otherwise; enc == gen, count == span) or group-contiguous
// int64 enc/gen/count arrays.
__device__ __forceinline__ long long stream_tok(const GroupSimArgs& a, long long b, int grp,
                                                int src_i) {
  if (a.span == 1) return a.tok.get(b, grp * a.l + src_i, a.staged);
  return a.mbsum[(b * a.groups + grp) * static_cast<long long>(a.l) + src_i];
}

struct GroupTok {
  const GroupSimArgs* a;
  long long gid;
  __device__ __forceinline__ void operator()(int i, long long* e, long long* g, int* c) const {
    const int l = a->l;
    const int src_i = a->order ? a->order[gid * l + i] : i;
    if (a->stream) {
      const long long b = gid / a->groups;
      const int grp = static_cast<int>(gid % a->groups);
      const long long v = stream_tok(*a, b, grp, src_i);
      *e = v;
      *g = v;
      *c = a->span;
    } else {
      const long long src = gid * l + src_i;
      *e = a->enc[src];
      *g = a->gen ? a->gen[src] : a->enc[src];
      *c = a->count ? a->count[src] : a->span;
    }
  }
};

// Fast path: plain 1F1B with P stages known at compile time.  Tick state
// lives in registers; build_stage_times entries are evaluated on demand —
// backbone entries are constants (their load is always seq_len) and every
// encoder/generator cell needs its value exactly once, so no row cache.
template <int P, bool STREAM>
__global__ void __launch_bounds__(128)
group_sims_fast(GroupSimArgs a) {
  const long long gid = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (gid >= a.n_batches * a.groups || sim_skipped(a, gid)) return;
  const int l = a.l;
  // token access: stream layout [b][i][e] or group-contiguous arrays
  const long long bidx = gid / a.groups;
  const int grp = static_cast<int>(gid - bidx * a.groups);
  const long long* encp = STREAM ? nullptr : a.enc + gid * l;
  const long long* genp = STREAM ? nullptr : (a.gen ? a.gen + gid * l : encp);
  const int* cntp = STREAM ? nullptr : (a.count ? a.count + gid * l : nullptr);
  const int* ord = a.order ? a.order + gid * l : nullptr;
  UnitEval ue, ub, ug;
  ue.init(a.cm, a.plan, DTB_ENCODER);
  ub.init(a.cm, a.plan, DTB_BACKBONE);
  ug.init(a.cm, a.plan, DTB_GENERATOR);
  double fB, bB;
  ub.eval(a.cm.seq_len, &fB, &bB);  // backbone load is always seq_len
  int unit[P];
#pragma unroll
  for (int s = 0; s < P; ++s) unit[s] = stage_unit(a.plan, s);
  // shift register of the live microbatch rows: slot k holds microbatch
  // i - k while ticks 2i, 2i+1 run (every index below is a constant)
  double rfE[P + 1], rbE[P + 1], rfG[P + 1], rbG[P + 1];
  double avail[P], prev[P], cur[P], busy[P];
#pragma unroll
  for (int s = 0; s < P; ++s) avail[s] = prev[s] = cur[s] = busy[s] = 0.0;
#pragma unroll
  for (int k = 0; k <= P; ++k) rfE[k] = rbE[k] = rfG[k] = rbG[k] = 0.0;
  double iter = 0.0;
  int fault = 0;
  auto cell = [&](int s, int mb, bool fwd, int k) {
    if (mb < 0 || mb >= l) return;
    const int u = unit[s];
    const double x = u == DTB_BACKBONE ? (fwd ? fB : bB)
                     : u == DTB_ENCODER ? (fwd ? rfE[k] : rbE[k])
                                        : (fwd ? rfG[k] : rbG[k]);
    const double dep = fwd ? (s > 0 ? prev[s - 1] : 0.0) : (s + 1 < P ? prev[s + 1] : prev[s]);
    const double start = smax(avail[s], dep);
    const double end = start + x;
    avail[s] = end;
    cur[s] = end;
    busy[s] += x;
    iter = smax(iter, end);
  };
  for (int i = 0; i < l + P - 1; ++i) {
#pragma unroll
    for (int k = P; k > 0; --k) {
      rfE[k] = rfE[k - 1];
      rbE[k] = rbE[k - 1];
      rfG[k] = rfG[k - 1];
      rbG[k] = rbG[k - 1];
    }
    if (i < l) {
      const int src = ord ? ord[i] : i;
      long long te, tg;
      int c;
      if (STREAM) {
        te = tg = stream_tok(a, bidx, grp, src);
        c = a.span;
      } else {
        te = encp[src];
        tg = genp[src];
        c = cntp ? cntp[src] : a.span;
      }
      if (te < 0 || tg < 0) fault = E_NEG_LOAD;
      if (STREAM && te >= 0 && te < a.table.size) {
        const double4 r = ld_row(a.table.eg + te);
        rfE[0] = r.x;
        rbE[0] = r.y;
        rfG[0] = r.z;
        rbG[0] = r.w;
      } else {
        ue.eval(mb_mean_fast(te, c), &rfE[0], &rbE[0]);
        ug.eval(mb_mean_fast(tg, c), &rfG[0], &rbG[0]);
      }
    }
    // even tick 2i: F(i - s/2, s) on even s, B(i - P + (s+1)/2, s) on odd s
#pragma unroll
    for (int s = 0; s < P; ++s) {
      if ((s & 1) == 0) cell(s, i - s / 2, true, s / 2);
      else cell(s, i - P + (s + 1) / 2, false, P - (s + 1) / 2);
    }
#pragma unroll
    for (int s = 0; s < P; ++s) prev[s] = cur[s];
    // odd tick 2i+1: F(i - (s-1)/2, s) on odd s, B(i - P + 1 + s/2, s) on even s
#pragma unroll
    for (int s = 0; s < P; ++s) {
      if (s & 1) cell(s, i - (s - 1) / 2, true, (s - 1) / 2);
      else cell(s, i - P + 1 + s / 2, false, P - 1 - s / 2);
    }
#pragma unroll
    for (int s = 0; s < P; ++s) prev[s] = cur[s];
  }
  if (a.busy) {
    double bub = 0.0;
    if (iter > 0.0) {
      double idle = 0.0;
#pragma unroll
      for (int s = 0; s < P; ++s) idle += iter - busy[s];
      bub = idle / (P * iter);
    }
    a.busy[gid] = bub;
  }
  if (fault) dev_fail(a.err, fault);
  a.t_group[gid] = iter;
}

// ---------------------------------------------------- tiled stream sims
// The disaggregated stream path's simulations (simulate_iteration,
// src/simulate.cpp:23-48, over plain 1F1B, src/pipeline_sim.cpp:36-52 and
// :108-183), one thread per coupled group, no shared memory, no barriers.
//
// The stage -> unit layout (PE encoder | PB backbone | PG generator stages)
// is a template parameter, so every cell's duration is a register chosen at
// compile time: backbone cells are constants (their load is always seq_len),
// encoder/generator cells come from the token-indexed cost table through
// short delay lines (forward of stage s runs microbatch i - s/2 at iteration
// i, backward runs i - P + 1 + s/2; only the delays actually read survive).
// Microbatches are processed in chunks of kSimChunk: the chunk's cost-table
// lookups are all in flight together and its token sums are prefetched one
// chunk ahead, so a group pays one memory latency per chunk, not per
// microbatch.
//
// Exactness: every cell is start = max(avail, dep), end = start + x with the
// reference's operands.  All durations are >= 0 and never NaN (profile times
// are validated strictly positive, src/cost_model.cpp:37-47; analytic and
// comm terms are non-negative), so the per-device end times are
// non-decreasing and the iteration time (max over all events) == max over
// the devices' last ends.  max is smax (std::max's compare + select: one
// DSETP and two FSEL) — fmax lowers to DSETP.MAX + SEL + FSEL + a NaN-quieting
// LOP3 and extra moves on sm_100.
constexpr int kSimT = 128;
constexpr int kSimChunk = 4;


struct Dur4 {
  double ef, eb, gf, gb;
};

// Cold path: token sums beyond the cost table (32-bit batches only).
__device__ __noinline__ Dur4 sim_eval_direct(const GroupSimArgs* a, long long te) {
  UnitEval ue, ug;
  ue.init(a->cm, a->plan, DTB_ENCODER);
  ug.init(a->cm, a->plan, DTB_GENERATOR);
  const double x = mb_mean_fast(te, a->span);
  Dur4 r;
  ue.eval(x, &r.ef, &r.eb);
  ug.eval(x, &r.gf, &r.gb);
  return r;
}

// DIRECT: token sums may fall outside the cost table (32-bit batches,
// negative sums): evaluate build_stage_times per microbatch instead.
template <int PE, int PB, int PG, bool BUSY, bool DIRECT>
__device__ __forceinline__ void sim_group(const GroupSimArgs& a, long long gid) {
  constexpr int P = PE + PB + PG;
  constexpr int C = kSimChunk;
  const int l = a.l;
  // this group's token source: position e*l + i of batch b (span == 1) or
  // the assembled sums [gid][i] (span > 1); optional inter order
  const long long b = gid / a.groups;
  const int grp = static_cast<int>(gid - b * a.groups);
  const int* ord = a.order ? a.order + gid * l : nullptr;
  const unsigned short* t16 = nullptr;
  const int* t32 = nullptr;
  if (a.span == 1) {
    const long long x0 = b * a.tok.n + static_cast<long long>(grp) * l;
    if (a.tok.wide[b]) t32 = (a.staged ? a.tok.t32_staged : a.tok.t32) + x0;
    else t16 = (a.staged && a.tok.kept[b] ? a.tok.t16_staged : a.tok.t16) + x0;
  } else {
    t32 = a.mbsum + gid * l;
  }
  auto token = [&](int i) -> int {
    const int src = ord ? __ldg(ord + i) : i;
    return t16 ? static_cast<int>(__ldg(t16 + src)) : __ldg(t32 + src);
  };

  UnitEval ub;
  ub.init(a.cm, a.plan, DTB_BACKBONE);
  double fB, bB;
  ub.eval(a.cm.seq_len, &fB, &bB);  // backbone load is always seq_len

  // delay lines (index = delay in iterations)
  double eF[P], eB[P], gF[P], gB[P];
  double av[P], busy[P];
#pragma unroll
  for (int s = 0; s < P; ++s) {
    eF[s] = eB[s] = gF[s] = gB[s] = 0.0;
    av[s] = busy[s] = 0.0;
  }
  int fault = 0;
  auto dur = [&](int s, bool fwd, int d) -> double {
    return s < PE ? (fwd ? eF[d] : eB[d])
                  : s < PE + PB ? (fwd ? fB : bB) : (fwd ? gF[d] : gB[d]);
  };
  auto tick_iter = [&](int i, bool check) {
    double pv[P];
#pragma unroll
    for (int s = 0; s < P; ++s) pv[s] = av[s];
    // even tick 2i: F(i - s/2, s) on even s, B(i - P + (s+1)/2, s) on odd s
#pragma unroll
    for (int s = 0; s < P; ++s) {
      const bool fwd = (s & 1) == 0;
      const int d = fwd ? s / 2 : P - (s + 1) / 2;
      const int mb = i - d;
      if (!check || (mb >= 0 && mb < l)) {
        const double x = dur(s, fwd, d);
        const double dep = fwd ? (s > 0 ? pv[s - 1] : 0.0) : (s + 1 < P ? pv[s + 1] : pv[s]);
        const double start = (s == 0 && fwd) || (s == P - 1 && !fwd) ? av[s] : smax(av[s], dep);
        av[s] = start + x;
        if (BUSY) busy[s] += x;
      }
    }
#pragma unroll
    for (int s = 0; s < P; ++s) pv[s] = av[s];
    // odd tick 2i+1: F(i - (s-1)/2, s) on odd s, B(i - P + 1 + s/2, s) on even s
#pragma unroll
    for (int s = 0; s < P; ++s) {
      const bool fwd = (s & 1) == 1;
      const int d = fwd ? (s - 1) / 2 : P - 1 - s / 2;
      const int mb = i - d;
      if (!check || (mb >= 0 && mb < l)) {
        const double x = dur(s, fwd, d);
        const double dep = fwd ? pv[s - 1] : (s + 1 < P ? pv[s + 1] : pv[s]);
        const double start = (s == P - 1 && !fwd) ? av[s] : smax(av[s], dep);
        av[s] = start + x;
        if (BUSY) busy[s] += x;
      }
    }
  };
  auto shift = [&]() {
#pragma unroll
    for (int k = P - 1; k > 0; --k) {
      eF[k] = eF[k - 1];
      eB[k] = eB[k - 1];
      gF[k] = gF[k - 1];
      gB[k] = gB[k - 1];
    }
  };

  if (DIRECT) {
    for (int i = 0; i < l; ++i) {
      shift();
      const int te = token(i);
      if (te < 0) fault = E_NEG_LOAD;
      const Dur4 r = sim_eval_direct(&a, te);
      eF[0] = r.ef;
      eB[0] = r.eb;
      gF[0] = r.gf;
      gB[0] = r.gb;
      tick_iter(i, i < P - 1);
    }
    for (int i = l; i < l + P - 1; ++i) {
      shift();
      tick_iter(i, true);
    }
  } else {
    // Chunks of P microbatches, two row rings (rA, rB) used alternately:
    // iteration j of a chunk reads delay d from cur[j - d] or, across the
    // chunk boundary, prev[j - d + P] — every index is a compile-time
    // constant, so the delay lines cost no register moves.  A chunk's
    // cost-table rows are all in flight before its first tick; its token
    // sums were loaded two chunks ahead (vector loads when possible).
    const bool vec = ord == nullptr && (P % 4) == 0 && (l % 4) == 0;
    // token sums of a chunk are fetched raw (vector registers) and unpacked
    // only when the chunk's rows are addressed one chunk later, so the load
    // latency is covered by a chunk of ticks
    constexpr int NV = P / 4 > 0 ? P / 4 : 1;
    uint2 rv16[NV];
    int4 rv32[NV];
    int tk[P] = {}, tk_next[P] = {};
    auto fetch = [&](int i0) {
      if (i0 >= l) return;
#if DTB_SIM_EXPERIMENT == 2
#pragma unroll
      for (int j = 0; j < P; ++j) tk_next[j] = (i0 + j) & 1023;
      return;
#endif
      if (vec) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          if (t16) rv16[v] = __ldg(reinterpret_cast<const uint2*>(t16 + i0 + 4 * v));
          else rv32[v] = __ldg(reinterpret_cast<const int4*>(t32 + i0 + 4 * v));
        }
      } else {
#pragma unroll
        for (int j = 0; j < P; ++j) tk_next[j] = i0 + j < l ? token(i0 + j) : 0;
      }
    };
    auto promote = [&]() {
#if DTB_SIM_EXPERIMENT != 2
      if (vec) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          if (t16) {
            tk[4 * v] = rv16[v].x & 0xffff;
            tk[4 * v + 1] = rv16[v].x >> 16;
            tk[4 * v + 2] = rv16[v].y & 0xffff;
            tk[4 * v + 3] = rv16[v].y >> 16;
          } else {
            tk[4 * v] = rv32[v].x;
            tk[4 * v + 1] = rv32[v].y;
            tk[4 * v + 2] = rv32[v].z;
            tk[4 * v + 3] = rv32[v].w;
          }
        }
        return;
      }
#endif
#pragma unroll
      for (int j = 0; j < P; ++j) tk[j] = tk_next[j];
    };
    auto tick_ring = [&](int i, bool check, const double4* cur, const double4* prev, int j) {
      // j is a compile-time constant at every call site (fully unrolled)
      double pv[P];
#pragma unroll
      for (int s = 0; s < P; ++s) pv[s] = av[s];
      auto row = [&](int d) -> const double4& { return j - d >= 0 ? cur[j - d] : prev[j - d + P]; };
      auto du = [&](int s, bool fwd, int d) -> double {
        return s < PE ? (fwd ? row(d).x : row(d).y)
                      : s < PE + PB ? (fwd ? fB : bB) : (fwd ? row(d).z : row(d).w);
      };
#pragma unroll
      for (int s = 0; s < P; ++s) {
        const bool fwd = (s & 1) == 0;
        const int d = fwd ? s / 2 : P - (s + 1) / 2;
        const int mb = i - d;
        if (!check || (mb >= 0 && mb < l)) {
          const double x = du(s, fwd, d);
          const double dep = fwd ? (s > 0 ? pv[s - 1] : 0.0) : (s + 1 < P ? pv[s + 1] : pv[s]);
          const double start = (s == 0 && fwd) || (s == P - 1 && !fwd) ? av[s] : smax(av[s], dep);
          av[s] = start + x;
          if (BUSY) busy[s] += x;
        }
      }
#pragma unroll
      for (int s = 0; s < P; ++s) pv[s] = av[s];
#pragma unroll
      for (int s = 0; s < P; ++s) {
        const bool fwd = (s & 1) == 1;
        const int d = fwd ? (s - 1) / 2 : P - 1 - s / 2;
        const int mb = i - d;
        if (!check || (mb >= 0 && mb < l)) {
          const double x = du(s, fwd, d);
          const double dep = fwd ? pv[s - 1] : (s + 1 < P ? pv[s + 1] : pv[s]);
          const double start = (s == P - 1 && !fwd) ? av[s] : smax(av[s], dep);
          av[s] = start + x;
          if (BUSY) busy[s] += x;
        }
      }
    };
    // rows of chunk c + 1 are loaded (nxt) while chunk c ticks; at the chunk
    // boundary they become `cur`
    auto run_chunk = [&](int i0, double4* cur, const double4* prev) {
#pragma unroll
      for (int j = 0; j < P; ++j) {
        const int i = i0 + j;
        if (i >= l + P - 1) break;
        if (i < P - 1 || i >= l) tick_ring(i, true, cur, prev, j);
        else tick_ring(i, false, cur, prev, j);
      }
    };
    double4 rA[P], rB[P], nxt[P];
#pragma unroll
    for (int j = 0; j < P; ++j) rA[j] = rB[j] = make_double4(0.0, 0.0, 0.0, 0.0);
    auto load_rows = [&](int i0) {
      promote();
      fetch(i0 + P);
#pragma unroll
      for (int j = 0; j < P; ++j)
        if (i0 + j < l) {
#if DTB_SIM_EXPERIMENT == 1
          const double x = static_cast<double>(tk[j]);
          nxt[j] = make_double4(x, x + 1.0, x + 2.0, x + 3.0);
#else
          nxt[j] = ld_row(a.table.eg + tk[j]);
#endif
        }
    };
    fetch(0);
    load_rows(0);
    for (int i0 = 0; i0 < l + P - 1; i0 += 2 * P) {
#pragma unroll
      for (int j = 0; j < P; ++j) rA[j] = nxt[j];
      load_rows(i0 + P);
      run_chunk(i0, rA, rB);
#pragma unroll
      for (int j = 0; j < P; ++j) rB[j] = nxt[j];
      load_rows(i0 + 2 * P);
      run_chunk(i0 + P, rB, rA);
    }
  }
  double iter = 0.0;
#pragma unroll
  for (int s = 0; s < P; ++s) iter = smax(iter, av[s]);
  if (a.busy) {
    double bub = 0.0;
    if (iter > 0.0) {
      double idle = 0.0;
#pragma unroll
      for (int s = 0; s < P; ++s) idle += iter - busy[s];
      bub = idle / (P * iter);
    }
    a.busy[gid] = bub;
  }
  if (fault) dev_fail(a.err, fault);
  a.t_group[gid] = iter;
}

template <int PE, int PB, int PG, bool BUSY>
__device__ __noinline__ void sim_group_direct(const GroupSimArgs* a, long long gid) {
  sim_group<PE, PB, PG, BUSY, true>(*a, gid);
}

template <int PE, int PB, int PG, bool BUSY>
__global__ void __launch_bounds__(kSimT, 4)
group_sims_tiled(const __grid_constant__ GroupSimArgs a) {
  pdl_wait();  // tokens, flags, cost table of the preceding kernels
  const long long gid = blockIdx.x * static_cast<long long>(kSimT) + threadIdx.x;
  const bool live = gid < a.n_batches * a.groups && !sim_skipped(a, gid);
  if (live) {
    // u16 token sums are < 0x8000 <= table.size; assembled sums of u16
    // batches are < span * 0x8000 — inside the table unless it was capped
    const long long b = gid / a.groups;
    const bool direct = a.tok.wide[b] ||
                        (a.span > 1 && static_cast<long long>(a.span) * 0x8000 > a.table.size);
    if (direct) sim_group_direct<PE, PB, PG, BUSY>(&a, gid);
    else sim_group<PE, PB, PG, BUSY, false>(a, gid);
  }
  if (a.t_iter == nullptr) return;
  // fused t_iter_reduce (groups == kSimT: this CTA is batch blockIdx.x):
  // slowest group (max is exact in any order for these non-negative,
  // non-NaN makespans) + dp_sync
  __syncthreads();
  if (threadIdx.x < 32) {
    const long long b = blockIdx.x;
    double worst = 0.0;
    for (int g = threadIdx.x; g < kSimT; g += 32) {
      const double t = a.t_group[b * kSimT + g];
      if (t > worst) worst = t;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double y = __shfl_xor_sync(0xffffffffu, worst, o);
      if (y > worst) worst = y;
    }
    if (threadIdx.x == 0) a.t_iter[b] = worst + a.dp_sync;
  }
}

using TiledFn = void (*)(GroupSimArgs);
template <bool BUSY>
static TiledFn tiled_for(int pe, int pb, int pg) {
#define DTB_TILED(E, B, G) \
  if (pe == E && pb == B && pg == G) return group_sims_tiled<E, B, G, BUSY>;
  DTB_TILED(1, 1, 1)
  DTB_TILED(1, 2, 1)
  DTB_TILED(2, 1, 1)
  DTB_TILED(1, 1, 2)
  DTB_TILED(1, 3, 1)
  DTB_TILED(1, 4, 1)
  DTB_TILED(2, 2, 1)
  DTB_TILED(1, 2, 2)
  DTB_TILED(2, 2, 2)
  DTB_TILED(1, 6, 1)
#undef DTB_TILED
  return nullptr;
}

// General path (any stage count, interleaved schedules): rows of
// build_stage_times materialised per group in scratch.
// Doubles of scratch per group: end-time matrices (interleaved) or three
// p-vectors (1F1B tick program), the l x 6 rows, avail/busy/next.
__host__ __device__ inline long long sim_scratch_per(int l, int p, int vpp) {
  const int devices = p / vpp;
  return (vpp == 1 ? 3LL * p : 2LL * l * p) + 6LL * l + 3 * devices;
}
__global__ void group_sims_kernel(GroupSimArgs a, double* scratch) {
  const long long gid = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long total = a.n_batches * a.groups;
  if (gid >= total || sim_skipped(a, gid)) return;
  const GroupTok tok{&a, gid};
  const int l = a.l;
  const int p = plan_stages(a.plan);
  const int vpp = a.plan.vpp;
  const int devices = p / vpp;
  // vpp == 1 (tick program) keeps only three p-vectors of end times
  const bool tick = vpp == 1;
  double* s = scratch + gid * sim_scratch_per(l, p, vpp);
  double* f_end = s;
  double* b_end = s + static_cast<size_t>(l) * p;
  double* rows = tick ? s + 3LL * p : b_end + static_cast<size_t>(l) * p;  // [l][6]
  double* avail = rows + 6 * static_cast<size_t>(l);
  double* busy = avail + devices;
  int* next = reinterpret_cast<int*>(busy + devices);
  int fault = 0;
  for (int i = 0; i < l; ++i) {
    long long e, g;
    int c;
    tok(i, &e, &g, &c);
    StageRow r;
    const int code = dev_stage_row(a.cm, a.plan, mb_mean(e, c), mb_mean(g, c), &r);
    if (code) fault = code;
    for (int u = 0; u < 3; ++u) {
      rows[i * 6 + u] = r.f[u];
      rows[i * 6 + 3 + u] = r.b[u];
    }
  }
  for (int d = 0; d < devices; ++d) busy[d] = 0.0;
  double iter = 0.0;
  auto dur = [&](int mb, int st, int ph) {
    return rows[mb * 6 + (ph == DTB_FORWARD ? 0 : 3) + stage_unit(a.plan, st)];
  };
  // busy accumulates the durations themselves (pipeline_sim.cpp:157)
  auto visit = [&](int d, Op op, double start, double end) {
    busy[d] += dur(op.mb, op.stage, op.phase);
    iter = smax(iter, end);
  };
  if (tick) {
    tick_1f1b(l, p, dur, f_end, f_end + p, f_end + 2 * p, visit);
  } else {
    const int e = dataflow_schedule(l, p, vpp, dur, f_end, b_end, next, avail, visit);
    if (e) fault = e;
  }
  double bub = 0.0;
  if (iter > 0.0 && devices > 0) {
    double idle = 0.0;
    for (int d = 0; d < devices; ++d) idle += iter - busy[d];
    bub = idle / (devices * iter);
  }
  if (a.busy) a.busy[gid] = bub;
  if (fault) dev_fail(a.err, fault);
  a.t_group[gid] = iter;
}

// General 1F1B path for many stages (p > 8, vpp 1): one warp per group.
// Every op of tick t depends only on ops of tick t-1 (tick_1f1b), so the
// stages of a tick are independent: lanes own stages s = lane + 32k and the
// tick state (prev, cur, avail, busy) lives in shared memory, exchanged with
// __syncwarp between ticks.  Per-stage op order and every FP operation are
// tick_1f1b's; the bubble sum runs over devices in order on lane 0.  Rows
// of build_stage_times are materialised per group in scratch by all lanes.
constexpr int kWarpSimWarps = 4;
__global__ void __launch_bounds__(32 * kWarpSimWarps)
group_sims_warp(GroupSimArgs a, double* scratch) {
  extern __shared__ double wsh[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long gid = blockIdx.x * static_cast<long long>(kWarpSimWarps) + warp;
  if (gid >= a.n_batches * a.groups || sim_skipped(a, gid)) return;  // uniform per warp
  const GroupTok tok{&a, gid};
  const int l = a.l;
  const int p = plan_stages(a.plan);
  double* rows = scratch + gid * sim_scratch_per(l, p, 1);
  double* prev = wsh + static_cast<size_t>(warp) * 4 * p;
  double* cur = prev + p;
  double* avail = cur + p;
  double* busy = avail + p;
  int fault = 0, fault_i = -1;
  for (int i = lane; i < l; i += 32) {
    long long e, g;
    int c;
    tok(i, &e, &g, &c);
    StageRow r;
    const int code = dev_stage_row(a.cm, a.plan, mb_mean(e, c), mb_mean(g, c), &r);
    if (code) {
      fault = code;
      fault_i = i;
    }
    for (int u = 0; u < 3; ++u) {
      rows[i * 6 + u] = r.f[u];
      rows[i * 6 + 3 + u] = r.b[u];
    }
  }
  for (int off = 16; off > 0; off >>= 1) {  // last failing row wins, as in i order
    const int oi = __shfl_down_sync(0xffffffffu, fault_i, off);
    const int oc = __shfl_down_sync(0xffffffffu, fault, off);
    if (oi > fault_i) {
      fault_i = oi;
      fault = oc;
    }
  }
  for (int s = lane; s < p; s += 32) {
    prev[s] = 0.0;
    cur[s] = 0.0;
    avail[s] = 0.0;
    busy[s] = 0.0;
  }
  __syncwarp();
  auto dur = [&](int mb, int st, int ph) {
    return rows[mb * 6 + (ph == DTB_FORWARD ? 0 : 3) + stage_unit(a.plan, st)];
  };
  double iter = 0.0;
  const int last_tick = 2 * l + 2 * p - 3;
  for (int t = 0; t <= last_tick; ++t) {
    for (int s = lane; s < p; s += 32) {
      const int q0 = t - s;
      if (q0 < 0) continue;
      if ((q0 & 1) == 0) {
        const int i = q0 >> 1;
        if (i >= l) continue;
        const double dep = s > 0 ? prev[s - 1] : 0.0;
        const double start = smax(avail[s], dep);
        const double d = dur(i, s, DTB_FORWARD);
        const double end = start + d;
        avail[s] = end;
        cur[s] = end;
        busy[s] += d;
        iter = smax(iter, end);
      } else {
        const int q = t - 2 * p + 1 + s;
        if (q < 0 || (q & 1)) continue;
        const int j = q >> 1;
        if (j >= l) continue;
        const double dep = s + 1 < p ? prev[s + 1] : prev[s];
        const double start = smax(avail[s], dep);
        const double d = dur(j, s, DTB_BACKWARD);
        const double end = start + d;
        avail[s] = end;
        cur[s] = end;
        busy[s] += d;
        iter = smax(iter, end);
      }
    }
    __syncwarp();
    for (int s = lane; s < p; s += 32) prev[s] = cur[s];
    __syncwarp();
  }
  for (int off = 16; off > 0; off >>= 1) iter = smax(iter, __shfl_xor_sync(0xffffffffu, iter, off));
  if (lane != 0) return;
  double bub = 0.0;
  if (iter > 0.0 && p > 0) {
    double idle = 0.0;
    for (int d = 0; d < p; ++d) idle += iter - busy[d];
    bub = idle / (p * iter);
  }
  if (a.busy) a.busy[gid] = bub;
  if (fault) dev_fail(a.err, fault);
  a.t_group[gid] = iter;
}

// Register form of group_sims_warp for p <= 32K stages: lane-owned stage
// state (avail, busy) in registers; since a stage's "cur" end time always
// equals its avail, the neighbours' previous-tick values are exchanged through
// a double-buffered shared row (one __syncwarp per tick), and the next tick's
// durations are loaded before this tick's dependency chain.
// 64 registers (8 blocks per SM) hold K <= 3 stages per lane without spills
// (tuned on p = 79); K = 4 (97..128 stages) needs more and gets 6 blocks.
template <int K>
__global__ void __launch_bounds__(32 * kWarpSimWarps, K <= 3 ? 8 : 6)
group_sims_warp_reg(GroupSimArgs a, double* scratch) {
  extern __shared__ double wsh[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long gid = blockIdx.x * static_cast<long long>(kWarpSimWarps) + warp;
  if (gid >= a.n_batches * a.groups || sim_skipped(a, gid)) return;  // uniform per warp
  const GroupTok tok{&a, gid};
  const int l = a.l;
  const int p = plan_stages(a.plan);
  double* rows = scratch + gid * sim_scratch_per(l, p, 1);
  double* buf = wsh + static_cast<size_t>(warp) * 2 * p;
  int fault = 0, fault_i = -1;
  for (int i = lane; i < l; i += 32) {
    long long e, g;
    int c;
    tok(i, &e, &g, &c);
    StageRow r;
    const int code = dev_stage_row(a.cm, a.plan, mb_mean(e, c), mb_mean(g, c), &r);
    if (code) {
      fault = code;
      fault_i = i;
    }
    for (int u = 0; u < 3; ++u) {
      rows[i * 6 + u] = r.f[u];
      rows[i * 6 + 3 + u] = r.b[u];
    }
  }
  for (int off = 16; off > 0; off >>= 1) {  // last failing row wins, as in i order
    const int oi = __shfl_down_sync(0xffffffffu, fault_i, off);
    const int oc = __shfl_down_sync(0xffffffffu, fault, off);
    if (oi > fault_i) {
      fault_i = oi;
      fault = oc;
    }
  }
  for (int s = lane; s < 2 * p; s += 32) buf[s] = 0.0;
  double avail[K], busy[K], nd[K], nd2[K];
  int unit[K], nk[K], nk2[K];  // op kind at ticks t+1 / t+2 (0 none, 1 F, 2 B)
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int st = lane + 32 * k;
    avail[k] = 0.0;
    busy[k] = 0.0;
    unit[k] = st < p ? stage_unit(a.plan, st) : 0;
  }
  __syncwarp();  // rows and buf visible to the warp
  auto fetch = [&](int t, double (&nd)[K], int (&nk)[K]) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int st = lane + 32 * k;
      nk[k] = 0;
      nd[k] = 0.0;
      if (st >= p) continue;
      const int q0 = t - st;
      if (q0 < 0) continue;
      if ((q0 & 1) == 0) {
        const int i = q0 >> 1;
        if (i >= l) continue;
        nk[k] = 1;
        nd[k] = rows[i * 6 + unit[k]];
      } else {
        const int q = t - 2 * p + 1 + st;
        if (q < 0 || (q & 1)) continue;
        const int j = q >> 1;
        if (j >= l) continue;
        nk[k] = 2;
        nd[k] = rows[j * 6 + 3 + unit[k]];
      }
    }
  };
  double iter = 0.0;
  const int last_tick = 2 * l + 2 * p - 3;
  fetch(0, nd, nk);
  fetch(1, nd2, nk2);
  for (int t = 0; t <= last_tick; ++t) {
    double d[K];
    int kind[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      d[k] = nd[k];
      kind[k] = nk[k];
      nd[k] = nd2[k];
      nk[k] = nk2[k];
    }
    fetch(t + 2, nd2, nk2);  // two ticks ahead (beyond last_tick: no ops)
    const double* prev = buf + (t & 1) * p;
    double* cur = buf + ((t + 1) & 1) * p;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int st = lane + 32 * k;
      if (st >= p) continue;
      if (kind[k] != 0) {
        const double dep = kind[k] == 1 ? (st > 0 ? prev[st - 1] : 0.0)
                                        : (st + 1 < p ? prev[st + 1] : prev[st]);
        const double start = smax(avail[k], dep);
        const double end = start + d[k];
        avail[k] = end;
        busy[k] += d[k];
        iter = smax(iter, end);
      }
      cur[st] = avail[k];
    }
    __syncwarp();
  }
  for (int off = 16; off > 0; off >>= 1) iter = smax(iter, __shfl_xor_sync(0xffffffffu, iter, off));
  // busy per stage to shared (buf is free now) for the in-order bubble sum
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int st = lane + 32 * k;
    if (st < p) buf[st] = busy[k];
  }
  __syncwarp();
  if (lane != 0) return;
  double bub = 0.0;
  if (iter > 0.0 && p > 0) {
    double idle = 0.0;
    for (int dd = 0; dd < p; ++dd) idle += iter - buf[dd];
    bub = idle / (p * iter);
  }
  if (a.busy) a.busy[gid] = bub;
  if (fault) dev_fail(a.err, fault);
  a.t_group[gid] = iter;
}

static bool fast_sims(const GroupSimArgs& a) {
  const int p = plan_stages(a.plan);
  return a.plan.vpp == 1 && p >= 2 && p <= 8;
}

size_t group_sims_scratch(const GroupSimArgs& a) {
  if (fast_sims(a)) return 256;
  const long long per = sim_scratch_per(a.l, plan_stages(a.plan), a.plan.vpp);
  return static_cast<size_t>(a.n_batches * a.groups * per) * sizeof(double) + 256;
}

bool group_sims_fuse_reduce(const GroupSimArgs& a) {
  return a.stream && a.plan.vpp == 1 && a.groups == kSimT && a.only_kept == nullptr &&
         tiled_for<false>(a.plan.unit[0].pp, a.plan.unit[1].pp, a.plan.unit[2].pp) != nullptr;
}

cudaError_t launch_group_sims(const GroupSimArgs& a, void* scratch,
                              cudaStream_t stream, bool pdl) {
  const long long total = a.n_batches * a.groups;
  if (total == 0) return cudaSuccess;
  const int T = 128;
  const unsigned grid = static_cast<unsigned>((total + T - 1) / T);
  if (a.stream && a.plan.vpp == 1) {
    const TiledFn fn = a.busy ? tiled_for<true>(a.plan.unit[0].pp, a.plan.unit[1].pp,
                                                a.plan.unit[2].pp)
                              : tiled_for<false>(a.plan.unit[0].pp, a.plan.unit[1].pp,
                                                 a.plan.unit[2].pp);
    if (fn != nullptr) {
#ifndef DTB_SIM_CARVEOUT
#define DTB_SIM_CARVEOUT 0
#endif
      // no shared memory: all of the unified L1 caches cost-table rows (the
      // rows a stream touches, token sums <= seq_len, are ~260 KB)
      cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, DTB_SIM_CARVEOUT);
      const unsigned g = static_cast<unsigned>((total + kSimT - 1) / kSimT);
      if (pdl) return launch_pdl(fn, dim3(g), dim3(kSimT), 0, stream, a);
      fn<<<g, kSimT, 0, stream>>>(a);
      return cudaGetLastError();
    }
  }
  if (fast_sims(a)) {
    switch (plan_stages(a.plan)) {
      case 2: a.stream ? group_sims_fast<2, true><<<grid, T, 0, stream>>>(a) : group_sims_fast<2, false><<<grid, T, 0, stream>>>(a); break;
      case 3: a.stream ? group_sims_fast<3, true><<<grid, T, 0, stream>>>(a) : group_sims_fast<3, false><<<grid, T, 0, stream>>>(a); break;
      case 4: a.stream ? group_sims_fast<4, true><<<grid, T, 0, stream>>>(a) : group_sims_fast<4, false><<<grid, T, 0, stream>>>(a); break;
      case 5: a.stream ? group_sims_fast<5, true><<<grid, T, 0, stream>>>(a) : group_sims_fast<5, false><<<grid, T, 0, stream>>>(a); break;
      case 6: a.stream ? group_sims_fast<6, true><<<grid, T, 0, stream>>>(a) : group_sims_fast<6, false><<<grid, T, 0, stream>>>(a); break;
      case 7: a.stream ? group_sims_fast<7, true><<<grid, T, 0, stream>>>(a) : group_sims_fast<7, false><<<grid, T, 0, stream>>>(a); break;
      default: a.stream ? group_sims_fast<8, true><<<grid, T, 0, stream>>>(a) : group_sims_fast<8, false><<<grid, T, 0, stream>>>(a); break;
    }
  } else if (a.plan.vpp == 1 && plan_stages(a.plan) > 8 && plan_stages(a.plan) <= 128) {
    const int p = plan_stages(a.plan);
    const size_t smem = kWarpSimWarps * 2 * sizeof(double) * p;
    const unsigned g = static_cast<unsigned>((total + kWarpSimWarps - 1) / kWarpSimWarps);
    double* sc = static_cast<double*>(scratch);
    if (p <= 64)
      group_sims_warp_reg<2><<<g, 32 * kWarpSimWarps, smem, stream>>>(a, sc);
    else if (p <= 96)
      group_sims_warp_reg<3><<<g, 32 * kWarpSimWarps, smem, stream>>>(a, sc);
    else
      group_sims_warp_reg<4><<<g, 32 * kWarpSimWarps, smem, stream>>>(a, sc);
  } else if (a.plan.vpp == 1 && plan_stages(a.plan) > 8 &&
             kWarpSimWarps * 4 * sizeof(double) * plan_stages(a.plan) <= 200 * 1024) {
    const size_t smem = kWarpSimWarps * 4 * sizeof(double) * plan_stages(a.plan);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(group_sims_warp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
    const unsigned g = static_cast<unsigned>((total + kWarpSimWarps - 1) / kWarpSimWarps);
    group_sims_warp<<<g, 32 * kWarpSimWarps, smem, stream>>>(a, static_cast<double*>(scratch));
  } else {
    group_sims_kernel<<<grid, T, 0, stream>>>(a, static_cast<double*>(scratch));
  }
  return cudaGetLastError();
}

// Per-microbatch token sums of a stream's groups as a simulation reads them
// (warning log only): out[gid * l + i] = the token sum of microbatch i of
// coupled group gid in a's order (input / intra / inter, assembled sums when
// span > 1).  Thread per (group, microbatch).
__global__ void mb_tokens_kernel(const __grid_constant__ GroupSimArgs a, int* out) {
  const long long total = a.n_batches * a.groups * static_cast<long long>(a.l);
  for (long long x = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long gid = x / a.l;
    const int i = static_cast<int>(x - gid * a.l);
    const long long b = gid / a.groups;
    const int grp = static_cast<int>(gid - b * a.groups);
    const int src = a.order ? a.order[gid * a.l + i] : i;
    int t;
    if (a.span == 1) {
      const long long x0 = b * a.tok.n + static_cast<long long>(grp) * a.l + src;
      if (a.tok.wide[b]) t = (a.staged ? a.tok.t32_staged : a.tok.t32)[x0];
      else t = (a.staged && a.tok.kept[b] ? a.tok.t16_staged : a.tok.t16)[x0];
    } else {
      t = a.mbsum[gid * a.l + src];
    }
    out[x] = t;
  }
}

cudaError_t launch_mb_tokens(const GroupSimArgs& a, int* out, cudaStream_t stream) {
  const long long total = a.n_batches * a.groups * static_cast<long long>(a.l);
  if (total == 0) return cudaSuccess;
  const unsigned grid = static_cast<unsigned>(std::min<long long>((total + 255) / 256, 148 * 16));
  mb_tokens_kernel<<<grid, 256, 0, stream>>>(a, out);
  return cudaGetLastError();
}

// Token-indexed cost table (see CostTable): thread per token sum s.
__global__ void cost_table_kernel(DevCM cm, dtb_plan plan, int span, int size, double4* eg,
                                  double* key, DevErr* err) {
  // the table reads only the cost model, but the kernels after it rely on
  // everything before it being complete (PDL waits chain one kernel back)
  pdl_wait();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= size) return;
  UnitEval ue, ug;
  ue.init(cm, plan, DTB_ENCODER);
  ug.init(cm, plan, DTB_GENERATOR);
  const double x = mb_mean_fast(s, span);
  double4 r;
  ue.eval(x, &r.x, &r.y);
  ug.eval(x, &r.z, &r.w);
  eg[s] = r;
  const int e = dev_fwd_key(cm, plan, x, x, &key[s]);
  if (e) dev_fail(err, e);
}

cudaError_t launch_cost_table(const DevCM& cm, const dtb_plan& plan, int span, int size,
                              double4* eg, double* key, DevErr* err, cudaStream_t stream) {
  if (size <= 0) return cudaSuccess;
  cudaError_t e = launch_pdl(cost_table_kernel, dim3((size + 255) / 256), dim3(256), 0, stream, cm,
                             plan, span, size, eg, key, err);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// simulate_iteration's fold over groups (simulate.cpp:31-46): slowest group
// by strict '>' in group order, t_iter = slowest + dp_sync.  bubble (in/out)
// holds per-group fractions; the mean is a sequential sum in group order.
// One warp per batch: max over its groups (max is exact in any order for
// these non-negative, non-NaN makespans), then + dp_sync.
__global__ void t_iter_reduce_kernel(long long n_batches, int groups,
                                     const double* t_group, double dp_sync,
                                     double* t_iter, const unsigned char* only_kept,
                                     const double* t_same) {
  const long long b = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (b >= n_batches) return;
  if (only_kept != nullptr && only_kept[b] == 0) {  // not simulated: same as t_same
    if (lane == 0) t_iter[b] = t_same[b];
    return;
  }
  double worst = 0.0;
  for (int g = lane; g < groups; g += 32) {
    const double t = t_group[b * groups + g];
    if (t > worst) worst = t;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double y = __shfl_xor_sync(0xffffffffu, worst, o);
    if (y > worst) worst = y;
  }
  if (lane == 0) t_iter[b] = worst + dp_sync;
}

cudaError_t launch_t_iter_reduce(long long n_batches, int groups,
                                 const double* t_group, double dp_sync,
                                 double* t_iter, cudaStream_t stream,
                                 const unsigned char* only_kept, const double* t_same) {
  if (n_batches == 0) return cudaSuccess;
  t_iter_reduce_kernel<<<static_cast<unsigned>((n_batches * 32 + 255) / 256), 256, 0,
                         stream>>>(n_batches, groups, t_group, dp_sync, t_iter, only_kept,
                                   t_same);
  return cudaGetLastError();
}

}  // namespace dtb

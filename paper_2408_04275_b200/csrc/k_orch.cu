// Orchestration search (Alg. 1; reference src/orchestrator.cpp:30-405).
//
//  enumerate: the sorted (TP, DP) tuple list is generated in place: one
//  thread per (tp_me, dp_me, tp_lm, dp_lm, tp_mg) prefix counts its valid
//  dp_mg, a scan gives offsets, and each prefix writes its tuples — the loop
//  nesting equals the reference's sort key, so the output is already in
//  std::sort order (orchestrator.cpp:268-301).
//  solve: one thread per tuple runs tuple_costs, the 400-iteration
//  continuous solve, PP rounding with memory_check + predict_times, and its
//  own BestTracker; a block then a grid lexicographic min over
//  (t_iter, total_gpus, tuple, pp triple) picks the plan
//  (orchestrator.cpp:211-233).  All arithmetic mirrors the reference op by
//  op (compiled with -fmad=false), so t_iter and the plan are bit-exact.
#include <algorithm>
#include <vector>

#include <cub/cub.cuh>

#include "kernels.cuh"

namespace dtb {

__constant__ int kTpc[4] = {1, 2, 4, 8};

// ------------------------------------------------------------ enumeration
__global__ void divisors_kernel(long long bs, long long* out, int* n_out) {
  if (threadIdx.x || blockIdx.x) return;
  int k = 0;
  for (long long d = 1; d * d <= bs; ++d) {
    if (bs % d == 0) {
      out[k++] = d;
      if (d != bs / d) out[k++] = bs / d;
    }
  }
  for (int i = 1; i < k; ++i)
    for (int j = i; j > 0 && out[j - 1] > out[j]; --j) {
      const long long t = out[j];
      out[j] = out[j - 1];
      out[j - 1] = t;
    }
  *n_out = k;
}

struct EnumCtx {
  const long long* divs;
  int D;
  int n;  // total GPUs
};

// prefix index -> (a, j, bb, i, cc) = (tp_me idx, dp_me idx, tp_lm idx,
// dp_lm idx, tp_mg idx), in sorted-key order.
__device__ __forceinline__ void decode_prefix(long long x, int D, int* a, int* j,
                                              int* bb, int* i, int* cc) {
  *cc = static_cast<int>(x % 4); x /= 4;
  *i = static_cast<int>(x % D); x /= D;
  *bb = static_cast<int>(x % 4); x /= 4;
  *j = static_cast<int>(x % D); x /= D;
  *a = static_cast<int>(x);
}

template <bool WRITE>
__global__ void enum_kernel(EnumCtx c, long long n_prefix, long long* counts,
                            const long long* offsets, dtb_tuple* out,
                            long long capacity) {
  const long long x = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (x >= n_prefix) return;
  int a, j, bb, i, cc;
  decode_prefix(x, c.D, &a, &j, &bb, &i, &cc);
  const long long dp_me = c.divs[j], dp_lm = c.divs[i];
  const int tp_me = kTpc[a], tp_lm = kTpc[bb], tp_mg = kTpc[cc];
  long long cnt = 0;
  long long pos = WRITE ? offsets[x] : 0;
  // reference loop guards (orchestrator.cpp:276-293)
  if (dp_lm % dp_me == 0 && tp_lm * dp_lm <= c.n && tp_me * dp_me <= c.n) {
    for (int q = 0; q < c.D && c.divs[q] <= dp_lm; ++q) {
      const long long dp_mg = c.divs[q];
      if (dp_lm % dp_mg) continue;
      if (tp_me * dp_me + tp_lm * dp_lm + tp_mg * dp_mg > c.n) continue;
      if (WRITE) {
        if (pos < capacity)
          out[pos] = dtb_tuple{tp_me, static_cast<int>(dp_me), tp_lm,
                               static_cast<int>(dp_lm), tp_mg, static_cast<int>(dp_mg)};
        ++pos;
      } else {
        ++cnt;
      }
    }
  }
  if (!WRITE) counts[x] = cnt;
}

cudaError_t launch_enumerate(const dtb_cluster_spec& c, long long bs,
                             const long long* /*unused*/, int /*unused*/,
                             long long* count_dev, dtb_tuple* out,
                             long long capacity, void* scratch,
                             cudaStream_t stream) {
  // scratch: divs[4096] | n_divs | counts[] | offsets[] | cub temp.  The
  // ascending divisors of the global batch (orchestrator.cpp:30-40) are
  // formed on the host — a single-thread device kernel plus a readback cost
  // ~50 us per search.
  char* p = static_cast<char*>(scratch);
  long long* divs = reinterpret_cast<long long*>(p);
  std::vector<long long> hd;
  for (long long d = 1; d * d <= bs; ++d)
    if (bs % d == 0) {
      hd.push_back(d);
      if (d != bs / d) hd.push_back(bs / d);
    }
  std::sort(hd.begin(), hd.end());
  const int D = static_cast<int>(hd.size());
  if (D > 4096) return cudaErrorInvalidValue;
  // pageable source: the copy is staged before this call returns
  cudaError_t e = cudaMemcpyAsync(divs, hd.data(), sizeof(long long) * D,
                                  cudaMemcpyHostToDevice, stream);
  if (e != cudaSuccess) return e;
  const long long n_prefix = 16LL * D * D * 4;
  long long* counts = reinterpret_cast<long long*>(p + 4096 * 8 + 256);
  long long* offsets = counts + n_prefix + 1;
  void* temp = offsets + n_prefix + 1;
  EnumCtx ctx{divs, D, c.total_gpus};
  const int T = 256;
  const unsigned grid = static_cast<unsigned>((n_prefix + T - 1) / T);
  enum_kernel<false><<<grid, T, 0, stream>>>(ctx, n_prefix, counts, nullptr, nullptr, 0);
  size_t temp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, counts, offsets, n_prefix + 1, stream);
  cudaMemsetAsync(counts + n_prefix, 0, sizeof(long long), stream);
  e = cub::DeviceScan::ExclusiveSum(temp, temp_bytes, counts, offsets, n_prefix + 1, stream);
  if (e != cudaSuccess) return e;
  cudaMemcpyAsync(count_dev, offsets + n_prefix, sizeof(long long), cudaMemcpyDeviceToDevice,
                  stream);
  if (out != nullptr)
    enum_kernel<true><<<grid, T, 0, stream>>>(ctx, n_prefix, nullptr, offsets, out, capacity);
  return cudaGetLastError();
}

size_t enumerate_scratch(long long bs) {
  long long D = 0;
  for (long long d = 1; d * d <= bs; ++d)
    if (bs % d == 0) D += (d != bs / d) ? 2 : 1;
  const long long n_prefix = 16LL * D * D * 4;
  size_t temp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, static_cast<long long*>(nullptr),
                                static_cast<long long*>(nullptr), n_prefix + 1);
  return 4096 * 8 + 256 + 2 * (n_prefix + 1) * 8 + temp_bytes + 1024;
}

// -------------------------------------------------------------- device model
__device__ __forceinline__ double stats_load(const DevCM& cm, int u,
                                             const dtb_workload_stats& s) {
  return u == DTB_ENCODER ? s.mean_encoder_tokens
         : u == DTB_GENERATOR ? s.mean_generator_tokens
                              : cm.seq_len;
}

__device__ __forceinline__ int fwdbwd(const DevCM& cm, int u, int tp, double load,
                                      double* out) {
  double f, b;
  int e = dev_unit_fwd(cm, u, tp, load, &f);
  if (e) return e;
  e = dev_unit_bwd(cm, u, tp, load, &b);
  if (e) return e;
  *out = f + b;
  return 0;
}

// predict_times (orchestrator.cpp:237-266).
__device__ int dev_predict(const DevCM& cm, const dtb_plan& plan,
                           const dtb_workload_stats& stats,
                           dtb_predicted_times* out) {
  const long long mbs = plan.global_batch / plan.unit[DTB_BACKBONE].dp;
  if (mbs < 1) return E_NO_MICROBATCH;
  double warm = 0.0, stage_max = 0.0;
  for (int u = 0; u < 3; ++u) {
    const dtb_parallelism& pc = plan.unit[u];
    const double coupling =
        u == DTB_BACKBONE ? 1.0 : static_cast<double>(plan.unit[DTB_BACKBONE].dp) / pc.dp;
    const double load = stats_load(cm, u, stats);
    double cfb;
    const int e = fwdbwd(cm, u, pc.tp, load, &cfb);
    if (e) return e;
    const double comm = dev_comm(cm, plan, u, load);
    warm += coupling * cfb / plan.vpp + pc.pp * 2.0 * comm;
    stage_max = smax(stage_max, coupling * cfb / pc.pp + plan.vpp * 2.0 * comm);
  }
  out->t_warm = warm;
  out->t_steady = stage_max * static_cast<double>(mbs - 1);
  out->t_iter = out->t_warm + out->t_steady + cm.dp_sync;
  return 0;
}

// memory_check (cost_model.cpp:167-189).
__device__ __forceinline__ bool dev_memory_pass(const DevCM& cm, const dtb_plan& plan,
                                                double* bytes_out) {
  const double dp_lm = static_cast<double>(plan.unit[DTB_BACKBONE].dp);
  bool pass = true;
  for (int u = 0; u < 3; ++u) {
    const dtb_parallelism& pc = plan.unit[u];
    const double gpus = static_cast<double>(pc.tp * pc.dp * pc.pp);
    const double bytes = (static_cast<double>(pc.dp) * cm.mem_pg[u] + cm.mem_opt[u] +
                          dp_lm * cm.mem_act[u] * pc.pp) /
                         gpus;
    if (bytes_out) bytes_out[u] = bytes;
    pass = pass && bytes <= cm.cluster.gpu_mem_bytes;
  }
  return pass;
}

__device__ __forceinline__ int plan_gpus(const dtb_plan& p) {
  return p.unit[0].tp * p.unit[0].dp * p.unit[0].pp +
         p.unit[1].tp * p.unit[1].dp * p.unit[1].pp +
         p.unit[2].tp * p.unit[2].dp * p.unit[2].pp;
}

// BestTracker order (orchestrator.cpp:219-227): true when a beats b.
__device__ __forceinline__ bool cand_better(const dtb_candidate& a,
                                            const dtb_candidate& b) {
  if (!a.feasible) return false;
  if (!b.feasible) return true;
  if (a.times.t_iter != b.times.t_iter) return a.times.t_iter < b.times.t_iter;
  const int ga = plan_gpus(a.plan), gb = plan_gpus(b.plan);
  if (ga != gb) return ga < gb;
  const int* ta = &a.tuple.tp_me;
  const int* tb = &b.tuple.tp_me;
  for (int i = 0; i < 6; ++i)
    if (ta[i] != tb[i]) return ta[i] < tb[i];
  for (int u = 0; u < 3; ++u)
    if (a.plan.unit[u].pp != b.plan.unit[u].pp) return a.plan.unit[u].pp < b.plan.unit[u].pp;
  return false;
}

__device__ __forceinline__ dtb_plan plan_from(const dtb_tuple& t, int pe, int pl,
                                              int pg, long long bs, int vpp) {
  dtb_plan p;
  p.unit[0] = {t.tp_me, t.dp_me, pe};
  p.unit[1] = {t.tp_lm, t.dp_lm, pl};
  p.unit[2] = {t.tp_mg, t.dp_mg, pg};
  p.vpp = vpp;
  p.global_batch = bs;
  return p;
}

struct Cont {
  double a[3], b[3], c[3], floor[3], w0, steady_mult, dp_sync;
};

__device__ __forceinline__ double gpus_at(const Cont& k, double bound, double* g) {
  double sum = 0.0;
#pragma unroll
  for (int u = 0; u < 3; ++u) {
    const double need = bound > k.c[u] ? k.b[u] / (bound - k.c[u]) : __longlong_as_double(0x7ff0000000000000ll);
    g[u] = smax(k.floor[u], need);
    sum += g[u];
  }
  return sum;
}

__device__ __forceinline__ double objective(const Cont& k, double bound, double* g) {
  gpus_at(k, bound, g);
  double warm_comm = 0.0, stage_max = 0.0;
#pragma unroll
  for (int u = 0; u < 3; ++u) {
    warm_comm += k.a[u] * g[u];
    stage_max = smax(stage_max, k.b[u] / g[u] + k.c[u]);
  }
  return k.w0 + warm_comm + stage_max * k.steady_mult + k.dp_sync;
}

// solve_subproblem (orchestrator.cpp:303-378) incl. tuple_costs (:65-113)
// and solve_continuous (:130-209).  Returns an E_* code; fills `out`.
// screen_only: stop after tuple_costs; a tuple that passes its early
// infeasibility exits is marked reason = kNeedsSolve (the caller solves it
// in a second, compacted pass).
constexpr int kNeedsSolve = -1;
__device__ int dev_solve(const DevCM& cm, const dtb_workload_stats& stats,
                         const dtb_tuple& t, long long bs, int vpp, int* fail_unit,
                         dtb_candidate* out, bool screen_only = false) {
  dtb_candidate& r = *out;
  r.tuple = t;
  r.feasible = 0;
  r.reason = DTB_REASON_NONE;
  for (int u = 0; u < 3; ++u) r.plan.unit[u] = {1, 1, 1};
  r.plan.vpp = 1;
  r.plan.global_batch = 1;
  r.times = {0.0, 0.0, 0.0};
  r.cont_x = r.cont_y = r.cont_z = r.cont_t_iter = 0.0;
  // ---- tuple_costs
  if (bs % t.dp_lm != 0) {
    r.reason = DTB_REASON_DP_NOT_DIVIDING;
    return 0;
  }
  const long long microbatches = bs / t.dp_lm;
  const dtb_plan probe = plan_from(t, 1, 1, 1, bs, 1);
  const int tps[3] = {t.tp_me, t.tp_lm, t.tp_mg};
  const int dps[3] = {t.dp_me, t.dp_lm, t.dp_mg};
  double coupling[3], cfb[3], comm[3], floor_g[3];
  int q[3];
  for (int u = 0; u < 3; ++u) {
    coupling[u] = static_cast<double>(t.dp_lm) / dps[u];
    const double load = stats_load(cm, u, stats);
    const int e = fwdbwd(cm, u, tps[u], load, &cfb[u]);
    if (e) {
      *fail_unit = u;
      return e;
    }
    comm[u] = dev_comm(cm, probe, u, load);
    q[u] = tps[u] * dps[u];
    const double act_const = static_cast<double>(t.dp_lm) * cm.mem_act[u] / q[u];
    const double headroom = cm.cluster.gpu_mem_bytes - act_const;
    if (headroom <= 0.0) {
      r.reason = DTB_REASON_ACTIVATION_ENCODER + u;
      return 0;
    }
    const double mem_floor = (dps[u] * cm.mem_pg[u] + cm.mem_opt[u]) / headroom;
    floor_g[u] = smax(static_cast<double>(q[u]), mem_floor);
  }
  double floor_sum = 0.0;
  for (int u = 0; u < 3; ++u) floor_sum += floor_g[u];
  if (floor_sum > cm.cluster.total_gpus) {
    r.reason = DTB_REASON_MEMORY_FLOOR;
    return 0;
  }
  if (screen_only) {
    r.reason = kNeedsSolve;
    return 0;
  }
  // ---- solve_continuous
  Cont k;
  k.w0 = 0.0;
  for (int u = 0; u < 3; ++u) {
    k.b[u] = coupling[u] * cfb[u] * q[u];
    k.c[u] = 2.0 * vpp * comm[u];
    k.a[u] = 2.0 * comm[u] / q[u];
    k.w0 += coupling[u] * cfb[u];
    k.floor[u] = floor_g[u];
  }
  k.w0 /= vpp;
  k.steady_mult = static_cast<double>(microbatches - 1);
  k.dp_sync = cm.dp_sync;
  const double total = static_cast<double>(cm.cluster.total_gpus);
  double hi = 0.0, cmax = 0.0;
  for (int u = 0; u < 3; ++u) {
    hi = smax(hi, k.b[u] / k.floor[u] + k.c[u]);
    cmax = smax(cmax, k.c[u]);
  }
  double lo = cmax + 1e-300;
  double g[3];
  if (gpus_at(k, hi, g) > total) {
    r.reason = DTB_REASON_MEMORY_FLOOR;
    return 0;
  }
  double bad = lo, good = hi;
#pragma unroll 4
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (bad + good);
    if (gpus_at(k, mid, g) <= total) good = mid;
    else bad = mid;
  }
  lo = good;
  double t_lo = lo, t_hi = hi;
#pragma unroll 2
  for (int it = 0; it < 200; ++it) {
    const double m1 = t_lo + (t_hi - t_lo) / 3.0;
    const double m2 = t_hi - (t_hi - t_lo) / 3.0;
    if (objective(k, m1, g) <= objective(k, m2, g)) t_hi = m2;
    else t_lo = m1;
  }
  double gpus[3];
  const double t_cont = objective(k, 0.5 * (t_lo + t_hi), gpus);
  r.cont_x = gpus[0];
  r.cont_y = gpus[1];
  r.cont_z = gpus[2];
  r.cont_t_iter = t_cont;
  // ---- rounding neighbourhood
  const int n = cm.cluster.total_gpus;
  const int q_sum = q[0] + q[1] + q[2];
  int cands[3][6], nc[3];
  for (int u = 0; u < 3; ++u) {
    const double cont_pp = gpus[u] / q[u];
    const int pp_max = (n - (q_sum - q[u])) / q[u];
    const int fl = static_cast<int>(floor(cont_pp)), ce = static_cast<int>(ceil(cont_pp));
    const int raw[6] = {fl - 1, fl, ce, ce + 1, 1, pp_max};
    int c = 0;
    for (int x = 0; x < 6; ++x) {
      const int v = raw[x];
      if (v < 1 || v > pp_max) continue;
      // insert sorted, unique (std::set)
      int pos = 0;
      while (pos < c && cands[u][pos] < v) ++pos;
      if (pos < c && cands[u][pos] == v) continue;
      for (int y = c; y > pos; --y) cands[u][y] = cands[u][y - 1];
      cands[u][pos] = v;
      ++c;
    }
    nc[u] = c;
  }
  dtb_candidate best;
  best.feasible = 0;
  for (int x = 0; x < nc[0]; ++x)
    for (int y = 0; y < nc[1]; ++y)
      for (int z = 0; z < nc[2]; ++z) {
        const long gsum = static_cast<long>(q[0]) * cands[0][x] +
                          static_cast<long>(q[1]) * cands[1][y] +
                          static_cast<long>(q[2]) * cands[2][z];
        if (gsum > n) continue;
        dtb_candidate c;
        c.tuple = t;
        c.feasible = 1;
        c.reason = DTB_REASON_NONE;
        c.plan = plan_from(t, cands[0][x], cands[1][y], cands[2][z], bs, vpp);
        if (vpp > 1 && microbatches % (cands[0][x] + cands[1][y] + cands[2][z]) != 0) continue;
        if (!dev_memory_pass(cm, c.plan, nullptr)) continue;
        const int e = dev_predict(cm, c.plan, stats, &c.times);
        if (e) return e;
        if (cand_better(c, best)) best = c;
      }
  if (!best.feasible) {
    r.reason = DTB_REASON_NO_INTEGER_SPLIT;
    return 0;
  }
  r.feasible = 1;
  r.plan = best.plan;
  r.times = best.times;
  return 0;
}

constexpr int kOrchT = 128;

// Pass 1: tuple_costs of every tuple of the shard.  About a third of the
// tuples stop there (dp does not divide, activation memory, memory floor);
// their records are final.  The others are appended to a compact list
// (warp-aggregated) so the continuous solve runs on full warps.  The order
// of the list does not matter: the winner is a total-order minimum and
// records / errors are keyed by tuple index.
__global__ void __launch_bounds__(kOrchT)
orch_screen_kernel(OrchArgs a) {
  const long long stride = static_cast<long long>(gridDim.x) * kOrchT;
  const long long mine = a.n > a.shard_index
                             ? (a.n - a.shard_index + a.shard_count - 1) / a.shard_count
                             : 0;
  for (long long x0 = blockIdx.x * static_cast<long long>(kOrchT); x0 < mine; x0 += stride) {
    const long long x = x0 + threadIdx.x;
    const long long idx = a.shard_index + x * a.shard_count;
    bool survive = false;
    if (x < mine) {
      dtb_candidate c;
      int unit = 0;
      const int e = dev_solve(a.cm, a.stats, a.tuples[idx], a.bs, a.vpp, &unit, &c, true);
      if (e) {
        dev_fail_ordered(a.err, static_cast<unsigned long long>(idx * 3 + unit), e);
      } else if (c.reason == kNeedsSolve) {
        survive = true;
      } else if (a.out) {
        a.out[idx] = c;
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, survive);
    unsigned base = 0;
    if ((threadIdx.x & 31) == 0 && m) base = atomicAdd(a.list_count, static_cast<unsigned>(__popc(m)));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (survive) a.list[base + __popc(m & ((1u << (threadIdx.x & 31)) - 1u))] = idx;
  }
}

__global__ void __launch_bounds__(kOrchT)
orch_kernel(OrchArgs a) {
  __shared__ dtb_candidate s_best[kOrchT];
  const long long stride = static_cast<long long>(gridDim.x) * kOrchT;
  dtb_candidate mine;
  mine.feasible = 0;
  const long long listed = a.list ? static_cast<long long>(*a.list_count) : 0;
  for (long long x = blockIdx.x * static_cast<long long>(kOrchT) + threadIdx.x;; x += stride) {
    long long idx;
    if (a.list) {
      if (x >= listed) break;
      idx = a.list[x];
    } else {
      idx = a.shard_index + x * a.shard_count;
      if (idx >= a.n) break;
    }
    dtb_candidate c;
    int unit = 0;
    const int e = dev_solve(a.cm, a.stats, a.tuples[idx], a.bs, a.vpp, &unit, &c);
    if (e) {
      // first failing (tuple, unit) in the reference's evaluation order
      dev_fail_ordered(a.err, static_cast<unsigned long long>(idx * 3 + unit), e);
      continue;
    }
    if (a.out) a.out[idx] = c;
    if (cand_better(c, mine)) mine = c;
  }
  s_best[threadIdx.x] = mine;
  __syncthreads();
  for (int w = kOrchT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w && cand_better(s_best[threadIdx.x + w], s_best[threadIdx.x]))
      s_best[threadIdx.x] = s_best[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) a.block_best[blockIdx.x] = s_best[0];
}

cudaError_t launch_orchestration(const OrchArgs& a, int grid, cudaStream_t stream) {
  if (a.list != nullptr) {
    cudaError_t e = cudaMemsetAsync(a.list_count, 0, sizeof(unsigned), stream);
    if (e != cudaSuccess) return e;
    orch_screen_kernel<<<grid, kOrchT, 0, stream>>>(a);
  }
  orch_kernel<<<grid, kOrchT, 0, stream>>>(a);
  return cudaGetLastError();
}

// brute_force_oracle (orchestrator.cpp:433-491).  The work per tuple grows
// like (n / q)^3, so tuples are split into (tuple, pp_me, pp_lm) PAIRS — a
// count pass and a scan give each tuple its pair range — and one thread per
// pair walks pp_mg; memory_check, predict_times and a private BestTracker,
// then the same block/grid lexicographic reduction (a total order: the
// split does not change the winner).
__device__ __forceinline__ long long brute_pairs_of(const dtb_tuple& t, int n) {
  const int q_me = t.tp_me * t.dp_me, q_lm = t.tp_lm * t.dp_lm, q_mg = t.tp_mg * t.dp_mg;
  long long c = 0;
  for (int pe = 1; q_me * pe + q_lm + q_mg <= n; ++pe) c += (n - q_me * pe - q_mg) / q_lm;
  return c;
}

__global__ void brute_count_kernel(const dtb_tuple* tuples, long long n_tuples, int n,
                                   long long* counts) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i < n_tuples) counts[i] = brute_pairs_of(tuples[i], n);
}

__global__ void __launch_bounds__(kOrchT)
brute_kernel(OrchArgs a, const long long* offsets, long long total,
             unsigned long long* evaluated) {
  __shared__ dtb_candidate s_best[kOrchT];
  const long long stride = static_cast<long long>(gridDim.x) * kOrchT;
  const int n = a.cm.cluster.total_gpus;
  dtb_candidate mine;
  mine.feasible = 0;
  unsigned long long count = 0;
  for (long long x = blockIdx.x * static_cast<long long>(kOrchT) + threadIdx.x; x < total;
       x += stride) {
    // tuple: last offset <= x
    long long lo = 0, hi = a.n - 1;
    while (lo < hi) {
      const long long mid = (lo + hi + 1) >> 1;
      if (offsets[mid] <= x) lo = mid;
      else hi = mid - 1;
    }
    const long long idx = lo;
    const dtb_tuple t = a.tuples[idx];
    const int q_me = t.tp_me * t.dp_me, q_lm = t.tp_lm * t.dp_lm, q_mg = t.tp_mg * t.dp_mg;
    long long r = x - offsets[idx];
    int pe = 1;
    for (;; ++pe) {
      const long long c = (n - q_me * pe - q_mg) / q_lm;
      if (r < c) break;
      r -= c;
    }
    const int pl = static_cast<int>(r) + 1;
    const long long mbs = a.bs / t.dp_lm;
    for (int pg = 1; q_me * pe + q_lm * pl + q_mg * pg <= n; ++pg) {
      if (a.vpp > 1 && mbs % (pe + pl + pg) != 0) continue;
      dtb_candidate c;
      c.tuple = t;
      c.feasible = 1;
      c.reason = DTB_REASON_NONE;
      c.plan = plan_from(t, pe, pl, pg, a.bs, a.vpp);
      if (!dev_memory_pass(a.cm, c.plan, nullptr)) continue;
      const int e = dev_predict(a.cm, c.plan, a.stats, &c.times);
      if (e) {
        dev_fail_ordered(a.err, static_cast<unsigned long long>(idx * 3), e);
        break;
      }
      ++count;
      if (cand_better(c, mine)) mine = c;
    }
  }
  atomicAdd(evaluated, count);
  s_best[threadIdx.x] = mine;
  __syncthreads();
  for (int w = kOrchT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w && cand_better(s_best[threadIdx.x + w], s_best[threadIdx.x]))
      s_best[threadIdx.x] = s_best[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) a.block_best[blockIdx.x] = s_best[0];
}

size_t brute_scratch(long long n_tuples) {
  size_t temp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, temp, static_cast<long long*>(nullptr),
                                static_cast<long long*>(nullptr), static_cast<int>(n_tuples));
  return 16 * static_cast<size_t>(n_tuples) + temp + 512;
}

// Counts, scans and returns (via *total_out, host) the pair count; then the
// search.  scratch: brute_scratch(n) bytes.
cudaError_t launch_brute(const OrchArgs& a, int max_grid, unsigned long long* evaluated,
                         void* scratch, size_t bytes, cudaStream_t stream) {
  auto* counts = static_cast<long long*>(scratch);
  auto* offsets = counts + a.n;
  char* temp = reinterpret_cast<char*>(offsets + a.n + 1);
  size_t temp_bytes = bytes - 16 * static_cast<size_t>(a.n) - 16;
  const int n = a.cm.cluster.total_gpus;
  if (a.n == 0) return cudaSuccess;
  brute_count_kernel<<<static_cast<unsigned>((a.n + 127) / 128), 128, 0, stream>>>(a.tuples, a.n,
                                                                                    n, counts);
  cudaError_t e = cub::DeviceScan::ExclusiveSum(temp, temp_bytes, counts, offsets,
                                                static_cast<int>(a.n), stream);
  if (e != cudaSuccess) return e;
  long long last_off = 0, last_cnt = 0;
  cudaMemcpyAsync(&last_off, offsets + a.n - 1, 8, cudaMemcpyDeviceToHost, stream);
  cudaMemcpyAsync(&last_cnt, counts + a.n - 1, 8, cudaMemcpyDeviceToHost, stream);
  e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return e;
  const long long total = last_off + last_cnt;
  long long grid = (total + kOrchT - 1) / kOrchT;
  if (grid > max_grid) grid = max_grid;
  if (grid < 1) grid = 1;
  brute_kernel<<<static_cast<unsigned>(grid), kOrchT, 0, stream>>>(a, offsets, total, evaluated);
  return cudaGetLastError();
}

// rigid_baseline (orchestrator.cpp:407-431): one thread per (tp, dp divisor);
// validate_plan reduces to memory_check for these plans (every other rule
// holds by construction).  Writes one candidate per pair (feasible = 0 when
// skipped) for the BestTracker reduction.
__global__ void rigid_kernel(DevCM cm, dtb_workload_stats stats, long long bs, int vpp,
                             const long long* divs, int n_divs, dtb_candidate* out,
                             DevErr* err) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= 4 * n_divs) return;
  const int tp = kTpc[x / n_divs];
  const long long dp = divs[x % n_divs];
  dtb_candidate c;
  c.feasible = 0;
  c.reason = DTB_REASON_NONE;
  const long q = static_cast<long>(tp) * dp;
  const int pl = static_cast<int>((cm.cluster.total_gpus - 2 * q) / q);
  if (pl >= 1) {
    const dtb_tuple t = {tp, static_cast<int>(dp), tp, static_cast<int>(dp), tp,
                         static_cast<int>(dp)};
    c.tuple = t;
    c.plan = plan_from(t, 1, pl, 1, bs, vpp);
    const bool vpp_ok = vpp == 1 || (bs / dp) % (pl + 2) == 0;
    if (vpp_ok && dev_memory_pass(cm, c.plan, nullptr)) {
      const int e = dev_predict(cm, c.plan, stats, &c.times);
      if (e) dev_fail_ordered(err, static_cast<unsigned long long>(x), e);
      else c.feasible = 1;
    }
  }
  out[x] = c;
}

cudaError_t launch_rigid(const DevCM& cm, const dtb_workload_stats& stats, long long bs, int vpp,
                         const long long* divs, int n_divs, dtb_candidate* out, DevErr* err,
                         cudaStream_t stream) {
  if (n_divs < 1) return cudaSuccess;
  rigid_kernel<<<(4 * n_divs + 127) / 128, 128, 0, stream>>>(cm, stats, bs, vpp, divs, n_divs,
                                                             out, err);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(kOrchT)
best_reduce_kernel(const dtb_candidate* in, long long n, dtb_candidate* out) {
  __shared__ dtb_candidate s_best[kOrchT];
  dtb_candidate mine;
  mine.feasible = 0;
  for (long long i = threadIdx.x; i < n; i += kOrchT)
    if (cand_better(in[i], mine)) mine = in[i];
  s_best[threadIdx.x] = mine;
  __syncthreads();
  for (int w = kOrchT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w && cand_better(s_best[threadIdx.x + w], s_best[threadIdx.x]))
      s_best[threadIdx.x] = s_best[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s_best[0];
}

cudaError_t launch_best_reduce(const dtb_candidate* in, long long n, dtb_candidate* out,
                               cudaStream_t stream) {
  best_reduce_kernel<<<1, kOrchT, 0, stream>>>(in, n, out);
  return cudaGetLastError();
}

__global__ void predict_kernel(DevCM cm, dtb_workload_stats stats, const dtb_plan* plans,
                               long long n, dtb_predicted_times* out, DevErr* err) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const int e = dev_predict(cm, plans[i], stats, &out[i]);
  if (e) dev_fail_ordered(err, static_cast<unsigned long long>(i), e);
}

cudaError_t launch_predict(const DevCM& cm, const dtb_workload_stats& stats,
                           const dtb_plan* plans, long long n, dtb_predicted_times* out,
                           DevErr* err, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  predict_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, stream>>>(cm, stats, plans,
                                                                           n, out, err);
  return cudaGetLastError();
}

__global__ void memory_check_kernel(DevCM cm, dtb_plan plan, dtb_memory_report* out) {
  if (threadIdx.x || blockIdx.x) return;
  double bytes[3];
  const bool pass = dev_memory_pass(cm, plan, bytes);
  for (int u = 0; u < 3; ++u) {
    out->bytes_per_gpu[u] = bytes[u];
    out->fits[u] = bytes[u] <= cm.cluster.gpu_mem_bytes;
  }
  out->pass = pass;
  out->capacity_bytes = cm.cluster.gpu_mem_bytes;
}

cudaError_t launch_memory_check(const DevCM& cm, const dtb_plan& plan, dtb_memory_report* out,
                                cudaStream_t stream) {
  memory_check_kernel<<<1, 32, 0, stream>>>(cm, plan, out);
  return cudaGetLastError();
}

}  // namespace dtb

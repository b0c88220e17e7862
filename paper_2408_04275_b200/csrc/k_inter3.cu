// inter_reorder (Alg. 3, src/reorder.cpp:238-298) for pipelines the
// compiled layouts of k_inter2.cu do not cover — many stages (p > 8, e.g. the
// 79-stage plan model_orchestration picks for BASELINE config 5) or long
// sequences (l > 255) — in the disaggregated token form, vpp == 1.
//
// One WARP per problem, the whole problem resident in shared memory: the
// microbatch rows of build_stage_times (6 doubles: f and b per unit) and
// keys, the placed order, the pending rows as a compacted ascending list, and
// the 1F1B tick state.  The algorithm is inter_one's (k_inter.cu): cells at
// ticks < 2 * placed depend on placed rows only and are committed once; each
// step evaluates only the speculative ticks up to B(step - 1, 0) with the
// candidate rows (placed | pending mean | reserved tail, src/reorder.cpp:
// 182-225).  Work is spread over the lanes:
//   * tick program: lanes own stages s = lane + 32 k (all stages of a tick
//     are independent; one __syncwarp exchange per tick);
//   * pending means: every stage of a unit carries the unit's value, so a
//     step needs 6 means (3 units x f / b), each a SEQUENTIAL sum over the
//     pending rows in ascending index order (src/reorder.cpp:191-201) — lanes
//     0..5 compute one each;
//   * select_closest / select_min picks: a warp argmin under the reference's
//     comparator (a total order: |residual - key|, over-target last, index).
// Bit-identical to the reference: same operations in the same order per
// value.
#include "kernels.cuh"

namespace dtb {

constexpr int kIW = 32;

struct InterWarpLayout {
  int l, p, devices;
  size_t off_rows, off_keys, off_state, off_ret, off_rear, off_plist, bytes;
  __host__ __device__ static InterWarpLayout make(int l, int p) {
    InterWarpLayout L{};
    L.l = l;
    L.p = p;
    L.devices = p;
    size_t o = 0;
    L.off_rows = o;
    o += 48ull * l;  // rows [l][6] doubles
    L.off_keys = o;
    o += 8ull * l;
    L.off_state = o;
    o += 8ull * (6 * p + 8);  // av pv cv | s_av s_pv s_cv | means[6] | scalars
    L.off_ret = o;
    o += 4ull * l;
    L.off_rear = o;
    o += 4ull * l;
    L.off_plist = o;
    o += 2ull * l + 16;
    L.bytes = (o + 15) & ~size_t(15);
    return L;
  }
};

size_t inter_warp_smem(int l, int p) { return InterWarpLayout::make(l, p).bytes; }

// (a better than b) for select_closest at `residual`
__device__ __forceinline__ bool closest_better(double ka, int ia, double kb, int ib,
                                               double residual) {
  const double da = fabs(residual - ka), db = fabs(residual - kb);
  if (da != db) return da < db;
  const bool ua = ka <= residual, ub = kb <= residual;
  if (ua != ub) return ua;
  return ia < ib;
}

__global__ void __launch_bounds__(kIW)
inter_warp_kernel(const __grid_constant__ InterArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  const long long prob = blockIdx.x;
  if (prob >= a.batch) return;
  const int l = a.l, p = a.p, lane = threadIdx.x;
  const InterWarpLayout L = InterWarpLayout::make(l, p);
  double* rows = reinterpret_cast<double*>(sm + L.off_rows);
  double* keys = reinterpret_cast<double*>(sm + L.off_keys);
  double* st = reinterpret_cast<double*>(sm + L.off_state);
  double* av = st;
  double* pv = av + p;
  double* cv = pv + p;
  double* s_av = cv + p;
  double* s_pv = s_av + p;
  double* s_cv = s_pv + p;
  double* mean = s_cv + p;  // [6]: f(unit 0..2), b(unit 0..2)
  int* ret = reinterpret_cast<int*>(sm + L.off_ret);
  int* rear = reinterpret_cast<int*>(sm + L.off_rear);
  unsigned short* plist = reinterpret_cast<unsigned short*>(sm + L.off_plist);
  int* out = a.orders + prob * l;
  const int devices = p;  // vpp == 1

  // ---- rows and keys (build_stage_times / microbatch_fwd_keys per microbatch)
  const long long bb = prob / a.groups;
  const int grp = static_cast<int>(prob % a.groups);
  int e = 0;
  for (int i = lane; i < l; i += kIW) {
    const long long v = a.span == 1 ? a.tok.get(bb, grp * l + i, true)
                                    : a.mbsum[(bb * a.groups + grp) * static_cast<long long>(l) + i];
    const double me = mb_mean(v, a.span);
    StageRow r;
    int ei = dev_stage_row(a.cm, a.plan, me, me, &r);
    if (!ei) ei = dev_fwd_key(a.cm, a.plan, me, me, &keys[i]);
    for (int u = 0; u < 3; ++u) {
      rows[i * 6 + u] = r.f[u];
      rows[i * 6 + 3 + u] = r.b[u];
    }
    if (ei && !e) e = ei;
    out[i] = i;
  }
  e = __reduce_max_sync(0xffffffffu, e);
  if (e) {
    if (lane == 0) dev_fail(a.err, e);
    return;
  }
  if (l <= 1 || devices == 1) return;  // identity (src/reorder.cpp:246-253)
  for (int i = lane; i < l; i += kIW) plist[i] = static_cast<unsigned short>(i);
  __syncwarp();
  int npend = l, nret = 0;
  // remove entry k of the pending list (ascending order kept)
  auto remove_at = [&](int k) {
    for (int base = k; base < npend - 1; base += kIW) {
      const int q = base + lane;
      const unsigned short nx = q < npend - 1 ? plist[q + 1] : 0;
      __syncwarp();
      if (q < npend - 1) plist[q] = nx;
      __syncwarp();
    }
    --npend;
  };
  // select_min over pending: smallest (key, index); returns the list slot
  auto argmin_key = [&]() -> int {
    int bk = -1;
    double bv = 0.0;
    int bi = 0x7fffffff;
    for (int q = lane; q < npend; q += kIW) {
      const int idx = plist[q];
      const double k = keys[idx];
      if (bk < 0 || k < bv || (k == bv && idx < bi)) bk = q, bv = k, bi = idx;
    }
    for (int o = 16; o > 0; o >>= 1) {
      const int ok = __shfl_xor_sync(0xffffffffu, bk, o);
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ok >= 0 && (bk < 0 || ov < bv || (ov == bv && oi < bi))) bk = ok, bv = ov, bi = oi;
    }
    return bk;
  };
  auto argmin_closest = [&](double residual) -> int {
    int bk = -1;
    double bv = 0.0;
    int bi = 0x7fffffff;
    for (int q = lane; q < npend; q += kIW) {
      const int idx = plist[q];
      const double k = keys[idx];
      if (bk < 0 || closest_better(k, idx, bv, bi, residual)) bk = q, bv = k, bi = idx;
    }
    for (int o = 16; o > 0; o >>= 1) {
      const int ok = __shfl_xor_sync(0xffffffffu, bk, o);
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ok >= 0 && (bk < 0 || closest_better(ov, oi, bv, bi, residual))) bk = ok, bv = ov, bi = oi;
    }
    return bk;
  };
  {
    const int k = argmin_key();
    if (lane == 0) ret[0] = plist[k];
    nret = 1;
    remove_at(k);
  }
  const int tail_n = min(devices - 1, npend);
  for (int t = 0; t < tail_n; ++t) {
    const int k = argmin_key();
    if (lane == 0) rear[t] = plist[k];
    remove_at(k);
  }
  __syncwarp();
  if (npend > 0) {  // the reference validates every candidate matrix (pipeline_sim.cpp:214-230)
    int bad = 0;
    for (int q = lane; q < 6 * l; q += kIW) bad |= !(rows[q] >= 0.0);
    if (__any_sync(0xffffffffu, bad)) {
      if (lane == 0) dev_fail(a.err, E_BAD_TIMES);
      return;
    }
  }
  // unit of each stage (compile-free: boundaries)
  const int e_end = a.plan.unit[0].pp, b_end = e_end + a.plan.unit[1].pp;
  auto unit_of = [&](int s) { return s < e_end ? 0 : s < b_end ? 1 : 2; };
  for (int s = lane; s < p; s += kIW) av[s] = pv[s] = cv[s] = 0.0;
  __syncwarp();
  int np = nret, Tc = 0;
  double f00_end = 0.0, last_b0_end = 0.0;
  // one tick range [t0, t1] on (A, P, Cc); dur(i, s, ph); lane 0 sees stage 0
  auto run_ticks = [&](int t0, int t1, double* A, double* P, double* Cc, auto&& dur,
                       auto&& visit0) {
    for (int t = t0; t <= t1; ++t) {
      for (int s = lane; s < p; s += kIW) {
        const int aa = t - s;
        if (aa < 0) continue;
        if ((aa & 1) == 0) {
          const int i = aa >> 1;
          if (i >= l) continue;
          const double dep = s > 0 ? P[s - 1] : 0.0;
          const double start = smax(A[s], dep);
          const double end = start + dur(i, s, DTB_FORWARD);
          A[s] = end;
          Cc[s] = end;
          if (s == 0) visit0(i, DTB_FORWARD, start, end);
        } else {
          const int q = t - 2 * p + 1 + s;
          if (q < 0) continue;
          const int j = q >> 1;
          if (j >= l) continue;
          const double dep = s + 1 < p ? P[s + 1] : P[s];
          const double start = smax(A[s], dep);
          const double end = start + dur(j, s, DTB_BACKWARD);
          A[s] = end;
          Cc[s] = end;
          if (s == 0) visit0(j, DTB_BACKWARD, start, end);
        }
      }
      __syncwarp();
      for (int s = lane; s < p; s += kIW) P[s] = Cc[s];
      __syncwarp();
    }
  };
  auto placed_dur = [&](int r, int s, int ph) -> double {
    return rows[ret[r] * 6 + (ph == DTB_FORWARD ? 0 : 3) + unit_of(s)];
  };
  int step = 1;
  while (npend > 0) {
    const int wi = step - 1;
    const int t_target = 2 * wi + 2 * p - 1;  // tick of B(wi, 0)
    // pending means of this step: lanes 0..5, sequential in index order
    if (lane < 6) {
      double acc = 0.0;
      for (int q = 0; q < npend; ++q) acc += rows[plist[q] * 6 + lane];
      mean[lane] = acc / static_cast<double>(npend);
    }
    for (int s = lane; s < p; s += kIW) s_av[s] = av[s], s_pv[s] = pv[s], s_cv[s] = cv[s];
    __syncwarp();
    double sf00 = f00_end, sb0 = last_b0_end, b_start = 0.0;
    auto cand = [&](int r, int s, int ph) -> double {
      const int c = (ph == DTB_FORWARD ? 0 : 3) + unit_of(s);
      if (r < np) return rows[ret[r] * 6 + c];
      if (r < np + npend) return mean[c];
      return rows[rear[r - np - npend] * 6 + c];
    };
    auto spec_visit = [&](int i, int ph, double start, double end) {
      if (ph == DTB_FORWARD) {
        if (i == 0) sf00 = end;
      } else if (i == wi) {
        b_start = start;
      } else if (i < wi) {
        sb0 = end;
      }
    };
    run_ticks(Tc, t_target, s_av, s_pv, s_cv, cand, spec_visit);
    // stage 0 lives on lane 0: broadcast its observations
    sf00 = __shfl_sync(0xffffffffu, sf00, 0);
    sb0 = __shfl_sync(0xffffffffu, sb0, 0);
    b_start = __shfl_sync(0xffffffffu, b_start, 0);
    const double anchor = wi == 0 ? sf00 : sb0;
    const double target = 0.0 + (b_start - anchor);
    const int take = step == 1 ? min(devices - 1, npend) : 1;
    double residual = target;
    for (int t = 0; t < take; ++t) {
      const int k = argmin_closest(residual);
      const int pick = plist[k];
      residual -= keys[pick];
      if (lane == 0) ret[nret] = pick;
      ++nret;
      remove_at(k);
    }
    __syncwarp();
    const int Tc_new = 2 * nret;
    np = nret;
    if (Tc_new > Tc) {
      auto commit_visit = [&](int i, int ph, double start, double end) {
        if (ph == DTB_FORWARD) {
          if (i == 0) f00_end = end;
        } else {
          last_b0_end = end;
        }
      };
      run_ticks(Tc, Tc_new - 1, av, pv, cv, placed_dur, commit_visit);
      f00_end = __shfl_sync(0xffffffffu, f00_end, 0);
      last_b0_end = __shfl_sync(0xffffffffu, last_b0_end, 0);
      Tc = Tc_new;
    }
    ++step;
  }
  __syncwarp();
  for (int t = lane; t < tail_n; t += kIW) ret[nret + t] = rear[t];
  __syncwarp();
  for (int i = lane; i < l; i += kIW) out[i] = ret[i];
}

bool inter_warp_applies(const InterArgs& a) {
  if (!a.stream || a.fwd != nullptr || a.vpp != 1 || a.l < 1 || a.l > 65535) return false;
  int dev = 0, max_smem = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return inter_warp_smem(a.l, a.p) <= static_cast<size_t>(max_smem);
}

cudaError_t launch_inter_warp(const InterArgs& a, cudaStream_t stream) {
  const size_t bytes = inter_warp_smem(a.l, a.p);
  cudaError_t e = cudaFuncSetAttribute(inter_warp_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(bytes));
  if (e != cudaSuccess) return e;
  if (a.batch <= 0) return cudaSuccess;
  inter_warp_kernel<<<static_cast<unsigned>(a.batch), kIW, bytes, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace dtb

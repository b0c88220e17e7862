#include <climits>
// Small kernels of the path: per-sample costs, workload stats,
// block_group_loads, select_min/select_closest, microbatch assembly and
// output-order composition.
#include "kernels.cuh"

namespace dtb {

__device__ __forceinline__ long long modality(const int* io, const int* it, const int* ao,
                                              const int* at, long long i) {
  long long t = 0;
  for (int q = io[i]; q < io[i + 1]; ++q) t += it[q];
  if (ao != nullptr)
    for (int q = ao[i]; q < ao[i + 1]; ++q) t += at[q];
  return t;
}

// Sample::cost_size (core.hpp:160-167): encoder + generator tokens.
__global__ void cost_sizes_kernel(const int* io, const int* it, const int* ao, const int* at,
                                  long long n, long long* out) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const long long t = modality(io, it, ao, at, i);
  out[i] = t + t;
}

cudaError_t launch_cost_sizes(const int* io, const int* it, const int* ao, const int* at,
                              long long n, long long* out, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  cost_sizes_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(io, it, ao, at,
                                                                              n, out);
  return cudaGetLastError();
}

// compute_stats (workload.cpp:206-220).  The reference sums integer token
// counts as doubles sequentially; every partial sum is an integer < 2^53, so
// the exact int64 total converts to the same double.
__global__ void stats_kernel(const int* io, const int* it, const int* ao, const int* at,
                             long long n, unsigned long long* acc) {
  long long local = 0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    local += modality(io, it, ao, at, i);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(kFull, local, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(acc, static_cast<unsigned long long>(local));
}

__global__ void stats_finish_kernel(const unsigned long long* acc, long long n, double* out2) {
  const double enc = static_cast<double>(static_cast<long long>(*acc));
  out2[0] = n ? enc / static_cast<double>(n) : 0.0;
  out2[1] = out2[0];
}

cudaError_t launch_compute_stats(const int* io, const int* it, const int* ao, const int* at,
                                 long long n, double* out2, cudaStream_t stream) {
  auto* acc = reinterpret_cast<unsigned long long*>(out2 + 2);
  cudaMemsetAsync(acc, 0, sizeof(unsigned long long), stream);
  if (n > 0) {
    long long blocks = (n + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    stats_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(io, it, ao, at, n, acc);
  }
  stats_finish_kernel<<<1, 1, 0, stream>>>(acc, n, out2);
  return cudaGetLastError();
}

// block_group_loads (reorder.cpp:111-119): block g sums its positions in
// position order (sequential, as the reference), last block takes the rest.
__global__ void block_loads_kernel(const double* sizes, const int* order, int n, int m,
                                   double* loads) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= m) return;
  const int per = n / m;
  const int lo = g * per;
  const int hi = g == m - 1 ? n : lo + per;
  double acc = 0.0;
  for (int pos = lo; pos < hi; ++pos) acc += sizes[order ? order[pos] : pos];
  loads[g] = acc;
}

cudaError_t launch_block_loads(const double* sizes, const int* order, int n, int m,
                               double* loads, cudaStream_t stream) {
  block_loads_kernel<<<(m + 127) / 128, 128, 0, stream>>>(sizes, order, n, m, loads);
  return cudaGetLastError();
}

// ---- one global batch beyond the fused kernels' limits (n > 16,384 or
// more than 512 groups): per-sample cost_size (include/core.hpp:160-167) as
// int64 -> double sizes and 32-bit tokens for the simulations; a
// modality-token sum beyond int32 is reported (E_COST_RANGE).
__global__ void batch_tokens_kernel(const int* io, const int* it, const int* ao, const int* at,
                                    long long first, int n, int* tok32, double* sizes,
                                    DevErr* err, int bidx) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long s = first + i;
  long long t = 0;
  for (int x = io[s]; x < io[s + 1]; ++x) t += it[x];
  if (ao != nullptr)
    for (int x = ao[s]; x < ao[s + 1]; ++x) t += at[x];
  sizes[i] = static_cast<double>(t + t);
  if (t < INT_MIN || t > INT_MAX) dev_fail(err, E_COST_RANGE, bidx);
  if (tok32 != nullptr) tok32[s] = static_cast<int>(t);
}

// The keep decision of disaggregated_reorder (src/reorder.cpp:340-354) for
// one batch of the generic route and its outputs: loads, kept, the intra
// order (greedy flat order if kept, else identity) and the staged tokens.
__global__ void __launch_bounds__(1024)
generic_decide_kernel(const double* li, const double* lg, int m, int n, long long b, int intra,
                      const int* flat, const int* tok32, int* order_out, int* tok32_staged,
                      double* load_before, double* load_after, unsigned char* kept,
                      unsigned* wide_flag) {
  __shared__ double red[2][32];
  double mi = 0.0, mg = 0.0;
  for (int g = threadIdx.x; g < m; g += blockDim.x) {
    mi = fmax(mi, li[g]);
    mg = fmax(mg, lg[g]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mi = fmax(mi, __shfl_xor_sync(0xffffffffu, mi, o));
    mg = fmax(mg, __shfl_xor_sync(0xffffffffu, mg, o));
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = mi;
    red[1][threadIdx.x >> 5] = mg;
  }
  __syncthreads();
  mi = red[0][0];
  mg = red[1][0];
  for (unsigned w = 1; w < blockDim.x / 32; ++w) {
    mi = fmax(mi, red[0][w]);
    mg = fmax(mg, red[1][w]);
  }
  // sizes are non-negative integers here (loads exact), so max is exact
  const bool keep = intra && mg <= mi;
  const long long first = b * n;
  for (int g = threadIdx.x; g < m; g += blockDim.x) {
    if (load_before) load_before[b * m + g] = li[g];
    if (load_after) load_after[b * m + g] = keep ? lg[g] : li[g];
  }
  if (threadIdx.x == 0) {
    if (kept) kept[b] = keep ? 1 : 0;
    if (wide_flag) wide_flag[b] = 1u;  // consumers read the 32-bit tokens
  }
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const int src = keep ? flat[k] : k;
    order_out[first + k] = src;
    if (tok32_staged != nullptr && tok32 != nullptr) tok32_staged[first + k] = tok32[first + src];
  }
}

cudaError_t launch_batch_tokens(const int* io, const int* it, const int* ao, const int* at,
                                long long first, int n, int* tok32, double* sizes, DevErr* err,
                                int bidx, cudaStream_t stream) {
  batch_tokens_kernel<<<(n + 255) / 256, 256, 0, stream>>>(io, it, ao, at, first, n, tok32,
                                                          sizes, err, bidx);
  return cudaGetLastError();
}

cudaError_t launch_generic_decide(const double* li, const double* lg, int m, int n, long long b,
                                  int intra, const int* flat, const int* tok32, int* order_out,
                                  int* tok32_staged, double* load_before, double* load_after,
                                  unsigned char* kept, unsigned* wide_flag, cudaStream_t stream) {
  generic_decide_kernel<<<1, 1024, 0, stream>>>(li, lg, m, n, b, intra, flat, tok32, order_out,
                                                tok32_staged, load_before, load_after, kept,
                                                wide_flag);
  return cudaGetLastError();
}

// select_min / select_closest (reorder.cpp:121-175) for one pending list.
// One warp: each pick is a warp argmin under the reference's comparator;
// `pool` flags live in global scratch (out buffer holds picks).
__global__ void select_kernel(const double* keys, const int* pending, int np, int k,
                              int closest, double target, int* out, unsigned char* taken) {
  const int lane = threadIdx.x;
  for (int q = lane; q < np; q += 32) taken[q] = 0;
  __syncwarp();
  double residual = target;
  for (int pick = 0; pick < k; ++pick) {
    // candidate: (position q in pending, index, key)
    int best_q = -1;
    for (int q = lane; q < np; q += 32) {
      if (taken[q]) continue;
      if (best_q < 0) {
        best_q = q;
        continue;
      }
      const int a = pending[q], b = pending[best_q];
      bool better;
      if (!closest) {
        better = keys[a] != keys[b] ? keys[a] < keys[b] : a < b;
      } else {
        const double da = fabs(residual - keys[a]), db = fabs(residual - keys[b]);
        if (da != db) better = da < db;
        else {
          const bool au = keys[a] <= residual, bu = keys[b] <= residual;
          better = au != bu ? au : a < b;
        }
      }
      if (better) best_q = q;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const int oq = __shfl_xor_sync(kFull, best_q, o);
      if (oq < 0) continue;
      if (best_q < 0) {
        best_q = oq;
        continue;
      }
      const int a = pending[oq], b = pending[best_q];
      bool better;
      if (!closest) {
        better = keys[a] != keys[b] ? keys[a] < keys[b] : a < b;
      } else {
        const double da = fabs(residual - keys[a]), db = fabs(residual - keys[b]);
        if (da != db) better = da < db;
        else {
          const bool au = keys[a] <= residual, bu = keys[b] <= residual;
          better = au != bu ? au : a < b;
        }
      }
      if (better) best_q = oq;
    }
    const int idx = pending[best_q];
    if (lane == 0) {
      out[pick] = idx;
      taken[best_q] = 1;
    }
    residual -= keys[idx];
    __syncwarp();
  }
}

cudaError_t launch_select(const double* keys, const int* pending, int np, int k, int closest,
                          double target, int* out, cudaStream_t stream) {
  auto* taken = reinterpret_cast<unsigned char*>(out + (k > 0 ? k : 1));
  select_kernel<<<1, 32, 0, stream>>>(keys, pending, np, k, closest, target, out, taken);
  return cudaGetLastError();
}

// assemble_microbatches (workload.cpp:179-204) as token sums: microbatch i of
// coupled group e = samples at positions (e*span + j)*per_group + i, j < span.
__global__ void assemble_kernel(long long n_batches, int n, int dp_lm, int dp_me, TokSrc tok,
                                bool staged, int* mbsum) {
  const int per_group = n / dp_lm;
  const int span = dp_lm / dp_me;
  const long long per_batch = static_cast<long long>(dp_me) * per_group;
  const long long x = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (x >= n_batches * per_batch) return;
  const long long b = x / per_batch;
  const int r = static_cast<int>(x % per_batch);  // r = e * per_group + i
  const int e = r / per_group, i = r % per_group;
  long long s = 0;
  for (int j = 0; j < span; ++j) s += tok.get(b, (e * span + j) * per_group + i, staged);
  mbsum[x] = static_cast<int>(s);
}

cudaError_t launch_assemble(long long n_batches, int n, int dp_lm, int dp_me, TokSrc tok,
                            bool staged, int* mbsum, cudaStream_t stream) {
  const long long total = n_batches * dp_me * static_cast<long long>(n / dp_lm);
  if (total == 0) return cudaSuccess;
  assemble_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, stream>>>(
      n_batches, n, dp_lm, dp_me, tok, staged, mbsum);
  return cudaGetLastError();
}

// output_order composition (reorder.cpp:380-390): position
// (e*span + j)*per_group + i takes intra[(e*span + j)*per_group + order_e[i]].
// Positions no coupled group covers keep 0, as the reference's assign(n, 0).
__global__ void compose_kernel(long long n_batches, int n, int dp_lm, int dp_me,
                               const int* intra, const int* inter, int* out) {
  const long long x = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (x >= n_batches * n) return;
  const long long b = x / n;
  const int pos = static_cast<int>(x % n);
  const int per_group = n / dp_lm;
  const int span = dp_lm / dp_me;
  const int blk = per_group ? pos / per_group : 0;
  const int i = per_group ? pos % per_group : 0;
  const int e = span ? blk / span : 0;
  if (per_group == 0 || e >= dp_me) {
    out[x] = 0;
    return;
  }
  const int src_i = inter ? inter[(b * dp_me + e) * per_group + i] : i;
  out[x] = intra[b * n + static_cast<long long>(blk) * per_group + src_i];
}

cudaError_t launch_compose(long long n_batches, int n, int dp_lm, int dp_me, const int* intra,
                           const int* inter, int* out, cudaStream_t stream) {
  const long long total = n_batches * n;
  if (total == 0) return cudaSuccess;
  compose_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, stream>>>(
      n_batches, n, dp_lm, dp_me, intra, inter, out);
  return cudaGetLastError();
}

}  // namespace dtb

// Intra-microbatch reordering kernels (Alg. 2).
//
//  * intra_generic_kernel — intra_partition(sizes, m, order, equal_counts)
//    for arbitrary doubles (reference: src/reorder.cpp:30-90).  One CTA per
//    problem after a stable device radix sort of (orderable key, index).
//  * intra_fused_kernel — the disaggregated hot path after the cost pass
//    (k_cost.cu): persistent CTAs of 1024 threads over the global batches the
//    cost pass left undecided.  Per batch, in shared memory: token histogram
//    of the u16 per-sample tokens -> the sorted size sequence (histogram
//    expansion) -> greedy equal-count partition (greedy_fused.cuh) ->
//    block_group_loads of the greedy and the identity order ->
//    keep-greedy-if-no-worse (src/reorder.cpp:340-354); only a kept batch
//    needs the stable radix sort of its sample indices (src/reorder.cpp:30-42)
//    for its output order.  With few batches the two CTAs of a cluster share
//    one: the sort runs on the peer and is read through DSMEM.
//
// Narrow layout: 16-bit keys, 16-bit sample indices and 16-bit (group, slot)
// cells.  A batch whose costs or (group, slot) ranges do not fit 16 bits is
// processed by the same algorithm with 32-bit arrays in a global scratch slot
// (`fused_wide`).
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include "block_ops.cuh"
#include "greedy.cuh"
#include "greedy_fused.cuh"
#include "greedy_warp.cuh"
#include "kernels.cuh"
#include "pdl.cuh"
#include "tma.cuh"

namespace dtb {

namespace cg = cooperative_groups;

// Orderable bits of a double: -0.0 folds onto +0.0 (the reference
// comparator treats them as equal, src/reorder.cpp:34-40).
__device__ __forceinline__ unsigned long long ord_bits(double x) {
  if (x == 0.0) x = 0.0;
  const unsigned long long b = __double_as_longlong(x);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

// ------------------------------------------------------------------ generic
constexpr int kGenT = 1024;
constexpr int kGenEmax = 4;  // m <= 4096

__global__ void __launch_bounds__(kGenT)
intra_keys_kernel(const double* __restrict__ sizes, int n, int order,
                  unsigned long long* __restrict__ keys, int* __restrict__ vals) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned long long k = ord_bits(sizes[i]);
    keys[i] = order == DTB_DESCENDING ? ~k : k;
    vals[i] = i;
  }
}

__global__ void __launch_bounds__(kGenT)
intra_generic_kernel(const double* __restrict__ sizes, int n, int m, int order,
                     int equal_counts, const int* __restrict__ vals, int* __restrict__ g_of,
                     int* __restrict__ slot_of, int* __restrict__ flat_out,
                     long long* __restrict__ offsets_out, GreedyState<double> st) {
  __shared__ int s_tmp[kGenT / 32 + 2];
  // the zero run in sorted order (zeros are contiguous; -0.0 == 0.0)
  int below = 0, zeros = 0;
  for (int i = threadIdx.x; i < n; i += kGenT) {
    const double x = sizes[i];
    zeros += x == 0.0;
    below += order == DTB_DESCENDING ? (x > 0.0) : (x < 0.0);
  }
  int tot_below, tot_zeros;
  block_excl_scan<kGenT>(below, s_tmp, &tot_below);
  block_excl_scan<kGenT>(zeros, s_tmp, &tot_zeros);
  const int cap = equal_counts ? (n + m - 1) / m : n;
  auto size_at = [&](int k) { return sizes[vals[k]]; };
  auto assign = [&](int k, int g, int slot) {
    g_of[k] = g;
    slot_of[k] = slot;
  };
  greedy_rounds<kGenT, kGenEmax, double>(n, m, cap, tot_below, tot_below + tot_zeros, size_at,
                                         assign, st);
  // group offsets (exclusive scan of counts) and the flat order
  const int E = (m + kGenT - 1) / kGenT;
  int local = 0;
  for (int e = 0; e < E; ++e) {
    const int g = threadIdx.x * E + e;
    if (g < m) local += st.cnt[g];
  }
  int total;
  int pre = block_excl_scan<kGenT>(local, s_tmp, &total);
  for (int e = 0; e < E; ++e) {
    const int g = threadIdx.x * E + e;
    if (g < m) {
      st.TG[g] = pre;
      offsets_out[g] = pre;
      pre += st.cnt[g];
    }
  }
  if (threadIdx.x == 0) offsets_out[m] = total;
  __syncthreads();
  for (int k = threadIdx.x; k < n; k += kGenT) flat_out[st.TG[g_of[k]] + slot_of[k]] = vals[k];
}

// -------------------------------------------------------------------- fused
// 1024 threads x 16 items per CTA, one CTA per SM (64 registers per thread).
constexpr int kFusedT = 1024;
constexpr int kFusedMaxN = 16384;  // samples per batch
constexpr int kFusedItems = ((kFusedMaxN + kFusedT - 1) / kFusedT + 3) / 4 * 4;  // 16
constexpr int kNarrowMaxM = kNarrowGroups;          // groups in the smem path
constexpr int kWideMaxM = 512;                      // groups in the global path
constexpr int kRB = 7;                              // radix digit bits
#ifndef DTB_FUSED_MIN_BLOCKS
#define DTB_FUSED_MIN_BLOCKS 1  // one CTA of 1024 threads per SM (64 registers per thread)
#endif

// Narrow (shared-memory) state.
//   kbi[i]   = sort key of sample i: modality tokens (asc) or 0x7fff - tokens
//              (desc); cost_size = 2 * tokens, so sorting by key is sorting
//              by cost.  Slots past n hold the padding key 0xffff.
//   idx16[k] = sample index of sorted position k (after the last pass: at
//              swizzled slot swz(k)).
//   out16[g * capP + slot] = sorted position of the item the greedy put in
//              slot `slot` of group g (capP = cap padded to 2 mod 4: bank
//              spread); the sort passes park their per-item ranks here.
constexpr int kFusedSlots = kFusedT * kFusedItems;  // sort slots incl. padding
constexpr int kCells = kFusedMaxN + 4 * kNarrowMaxM;  // (group, slot) cells, padded groups
// Per-batch state of the histogram path's greedy and decision.
struct BatchState {
  FusedGreedySmem G;
  WarpGreedySmem WG;
  unsigned blk_ident[kNarrowMaxM], blk_greedy[kNarrowMaxM];
  int off[kNarrowMaxM];
  unsigned keep_flag;  // the decision, broadcast from warp 0
  int zc;              // zero-cost samples
};
struct NarrowSmem {
  unsigned short kbi[kFusedSlots];
  alignas(16) unsigned short idx16[kFusedSlots];
  alignas(16) unsigned short out16[kCells];
  BatchState A;  // every single-batch path
  // a second batch whose greedy runs next to A's (descending order, one
  // warp each): its cells, its state
  alignas(16) unsigned short cellsB[kCells];
  BatchState B;
  int tmp[kFusedT / 32 + 3];
  long long tmpll[kFusedT / 32 + 1];
  unsigned int s_and, s_or;
  unsigned deferred;  // cluster pair (rank 1): epoch of a kept batch whose order this CTA writes
  // cluster pair: rank 0 stores the pair's batch epoch into rank 1's
  // sort_abort once the batch is decided NOT kept (rank 1's speculative sort
  // is then useless and stops at its next pass)
  unsigned pair_epoch, sort_abort, sort_go;
};
constexpr int kSortRB = 5;  // narrow-path digit bits (per-thread counters)
// per-thread radix counters of the narrow path (their own space, so the
// greedy's cells in out16 survive a sort that runs after the greedy)
struct SortSmem {
  NarrowSmem N;
  alignas(16) unsigned cnt[blocked_cnt_words(kFusedT, kSortRB)];
};

constexpr size_t kFusedSmem = sizeof(SortSmem);
static_assert(kFusedSmem + 1024 <= 227 * 1024, "one partition CTA per SM: 227 KB of shared memory");

// The kernel's dynamic shared memory as NarrowSmem.  Non-inlined device
// functions re-derive it here instead of taking a reference argument, so the
// compiler keeps the shared address space (LDS/STS instead of generic LD/ST).
__device__ __forceinline__ NarrowSmem& shared_state() {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  return reinterpret_cast<SortSmem*>(smem_raw)->N;
}
__device__ __forceinline__ unsigned* sort_counters() {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  return reinterpret_cast<SortSmem*>(smem_raw)->cnt;
}
// Wide fallback (any cost <= 2^32-1, m <= 512) in a global scratch slot.
constexpr size_t kWidePerBatch = static_cast<size_t>(kFusedMaxN) * (4 + 2 + 4) +
                                 static_cast<size_t>(kWideMaxM) * (8 * 5 + 4 * 4) + 1024;

size_t fused_smem_bytes() { return kFusedSmem; }
int fused_max_n() { return kFusedMaxN; }
int fused_max_m() { return kWideMaxM; }
size_t fused_wide_scratch_bytes(long long n_batches) { return kWidePerBatch * n_batches; }

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Microbatch key of position pos (span == 1 stream layout [b][pg][dp_me]).
__device__ __forceinline__ long long mb_index(const FusedArgs& a, long long b, int pos) {
  const unsigned qd = a.div_pg.div(static_cast<unsigned>(pos));
  return (b * a.pg + (static_cast<unsigned>(pos) - qd * a.pg)) * a.dp_me + qd;
}

__device__ __forceinline__ void write_outputs_common(const FusedArgs& a, long long b, int g,
                                                     unsigned long long ident,
                                                     unsigned long long after) {
  if (a.load_before) a.load_before[b * a.m + g] = static_cast<double>(ident);
  if (a.load_after) a.load_after[b * a.m + g] = static_cast<double>(after);
}

// ---- wide path: 32-bit keys, (group, slot) assignments, global scratch.
__device__ __noinline__ void fused_wide(const FusedArgs& a, long long b, NarrowSmem&) {
  NarrowSmem& S = shared_state();  // shared address space: LDS/STS, not generic
  const int n = a.n, m = a.m, tid = threadIdx.x;
  const long long first = b * n;
  const bool desc = a.order == DTB_DESCENDING;
  unsigned char* slot = a.wide_scratch + static_cast<size_t>(b) * kWidePerBatch;
  auto* keys = reinterpret_cast<unsigned int*>(slot);
  auto* vals = reinterpret_cast<unsigned short*>(slot + 4ull * kFusedMaxN);
  auto* asg = reinterpret_cast<unsigned int*>(slot + 6ull * kFusedMaxN);
  char* st_mem = reinterpret_cast<char*>(slot + 10ull * kFusedMaxN);
  GreedyState<long long> st;
  st.AL = reinterpret_cast<long long*>(st_mem);
  st.TL = st.AL + kWideMaxM;
  st.gload = st.TL + kWideMaxM;
  auto* blk_g = reinterpret_cast<unsigned long long*>(st.gload + kWideMaxM);
  auto* blk_i = blk_g + kWideMaxM;
  st.AG = reinterpret_cast<int*>(blk_i + kWideMaxM);
  st.TG = st.AG + kWideMaxM;
  st.cnt = st.TG + kWideMaxM;
  int* off = st.cnt + kWideMaxM;
  st.tmp = S.tmp;
  unsigned int kand = ~0u, kor = 0u;
  int zeros = 0;
  for (int g = tid; g < m; g += kFusedT) blk_i[g] = blk_g[g] = 0ull;
  __syncthreads();
  const int pg = n / m;
  for (int i = tid; i < n; i += kFusedT) {
    const long long gi = first + i;
    long long t = 0;
    for (int x = a.img_off[gi]; x < a.img_off[gi + 1]; ++x) t += a.img_tok[x];
    if (a.aud_off != nullptr)
      for (int x = a.aud_off[gi]; x < a.aud_off[gi + 1]; ++x) t += a.aud_tok[x];
    const unsigned int c = static_cast<unsigned int>(t + t);
    const unsigned int key = desc ? ~c : c;
    keys[i] = key;
    vals[i] = static_cast<unsigned short>(i);
    kand &= key;
    kor |= key;
    zeros += c == 0;
    atomicAdd(&blk_i[min(i / pg, m - 1)], static_cast<unsigned long long>(c));
    // (after the cost pass, its finalize kernel already wrote them)
    if (a.tok32_orig != nullptr && a.state == nullptr) a.tok32_orig[first + i] = static_cast<int>(t);
  }
  if (tid == 0) {
    S.s_and = ~0u;
    S.s_or = 0u;
  }
  __syncthreads();
  atomicAnd(&S.s_and, kand);
  atomicOr(&S.s_or, kor);
  int tot_zeros;
  block_excl_scan<kFusedT>(zeros, S.tmp, &tot_zeros);
  const unsigned int varying = S.s_and ^ S.s_or;
  if (a.intra) {
    const int lo = varying ? __ffs(static_cast<int>(varying)) - 1 : 0;
    const int hi = varying ? 32 - __clz(static_cast<int>(varying)) : 0;
    tile_radix_sort<kFusedT, kFusedItems, kRB>(keys, vals, n, lo, hi, reinterpret_cast<int*>(sort_counters()), S.tmp);
    const int z0 = desc ? n - tot_zeros : 0;
    const int z1 = desc ? n : tot_zeros;
    const int cap = (n + m - 1) / m;
    auto size_at = [&](int k) -> long long {
      return static_cast<long long>(desc ? ~keys[k] : keys[k]);
    };
    auto assign = [&](int k, int g, int sl) {
      asg[k] = (static_cast<unsigned>(g) << 16) | static_cast<unsigned>(sl);
    };
    st.tmpll = S.tmpll;
    if (desc)
      greedy_rounds<kFusedT, 2, long long, false>(n, m, cap, z0, z1, size_at, assign, st);
    else
      greedy_rounds<kFusedT, 2, long long, true>(n, m, cap, z0, z1, size_at, assign, st);
    // group offsets (blocked: thread owns groups 2*tid, 2*tid + 1)
    const int g0 = 2 * tid;
    const int c0 = g0 < m ? st.cnt[g0] : 0, c1 = g0 + 1 < m ? st.cnt[g0 + 1] : 0;
    int total;
    const int pre = block_excl_scan<kFusedT>(c0 + c1, S.tmp, &total);
    if (g0 < m) off[g0] = pre;
    if (g0 + 1 < m) off[g0 + 1] = pre + c0;
    __syncthreads();
    for (int k = tid; k < n; k += kFusedT) {
      const unsigned as = asg[k];
      const int pos = off[as >> 16] + static_cast<int>(as & 0xffffu);
      atomicAdd(&blk_g[min(pos / pg, m - 1)], static_cast<unsigned long long>(size_at(k)));
    }
    __syncthreads();
  }
  long long mg = 0, mi = 0;
  for (int g = tid; g < m; g += kFusedT) {
    mg = max(mg, static_cast<long long>(blk_g[g]));
    mi = max(mi, static_cast<long long>(blk_i[g]));
  }
  mg = block_max_ll<kFusedT>(mg, S.tmpll);
  mi = block_max_ll<kFusedT>(mi, S.tmpll);
  const bool keep = a.intra && mg <= mi;
  if (tid == 0 && a.kept != nullptr) a.kept[b] = keep ? 1 : 0;
  for (int g = tid; g < m; g += kFusedT) write_outputs_common(a, b, g, blk_i[g], keep ? blk_g[g] : blk_i[g]);
  for (int k = tid; k < n; k += kFusedT) {
    const unsigned int key = keys[k];
    const int tok = static_cast<int>((desc ? ~key : key) >> 1);
    int pos = vals[k];
    if (keep) {
      const unsigned as = asg[k];
      pos = off[as >> 16] + static_cast<int>(as & 0xffffu);
    }
    a.order_out[first + pos] = keep ? vals[k] : pos;
    if (a.tok32_staged != nullptr) a.tok32_staged[first + pos] = tok;
  }
}

constexpr int kHistBins = 8192;  // token sums below this take the histogram path
constexpr int kProfSlots = 64;   // debug timestamps per batch
static_assert(kHistBins * 2 <= sizeof(NarrowSmem::kbi), "the histogram fits kbi");

// Inclusive "last non-zero" scan of one value per thread (all threads get
// their inclusive value; *carry gets the exclusive one).
__device__ __forceinline__ unsigned block_last_nz(unsigned v, int* s, unsigned* excl) {
  constexpr int W = kFusedT / 32;
  const int lane = lane_id(), w = warp_id();
  unsigned x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(kFull, x, o);
    if (lane >= o && x == 0u) x = y;
  }
  __syncthreads();
  if (lane == 31) s[w] = static_cast<int>(x);
  __syncthreads();
  unsigned carry = 0u;
  for (int k = 0; k < w; ++k) {
    const unsigned c = static_cast<unsigned>(s[k]);
    if (c) carry = c;
  }
  const unsigned up = __shfl_up_sync(kFull, x, 1);
  *excl = lane == 0 ? carry : (up ? up : carry);
  return x ? x : carry;
}

// Outputs of a batch whose order stays the identity.
__device__ __forceinline__ void identity_order_out(const FusedArgs& a, long long first, int n) {
  int* out = a.order_out + first;
  if (aligned16(out)) {
    int4* o4 = reinterpret_cast<int4*>(out);
    for (int q = threadIdx.x; q < (n >> 2); q += kFusedT)
      o4[q] = make_int4(4 * q, 4 * q + 1, 4 * q + 2, 4 * q + 3);
  } else {
    for (int i = threadIdx.x; i < n; i += kFusedT) out[i] = i;
  }
}

// The permutation of a kept batch: stable LSD radix sort of the sample
// indices by key (the u16 tokens; descending keys 0x7fff - tok) in kbi /
// idx16, counters in their own space so the greedy's cells in out16
// survive.  Sorted position k (the greedy's k: the same stable order of the
// sizes) is then idx16[swz(k)].
// Stable sort of a batch's samples by key (u16 tokens from the cost pass;
// descending: 0x7fff - tokens) as packed (key << 16 | index) items in the
// 64 KB of kbi + idx16 (`batch_kv`): 3 blocked passes of 5-bit digits over
// the 13-bit keys; the last writes swizzled positions.  abort_epoch != 0: a
// cluster peer's speculative sort, stopped between passes once the peer
// decided the batch is not kept.
__device__ __forceinline__ unsigned* batch_kv(NarrowSmem& S) { return reinterpret_cast<unsigned*>(S.kbi); }
static_assert(offsetof(NarrowSmem, idx16) == sizeof(NarrowSmem::kbi) &&
                  sizeof(NarrowSmem::kbi) + sizeof(NarrowSmem::idx16) == 4 * kFusedSlots,
              "kbi and idx16 form one array of packed (key, index) items");
__device__ __noinline__ void sort_batch_keys(const FusedArgs& a, long long b, NarrowSmem&,
                                             unsigned abort_epoch = 0u) {
  NarrowSmem& S = shared_state();
  const int n = a.n, tid = threadIdx.x;
  const long long first = b * n;
  const bool desc = a.order == DTB_DESCENDING;
  unsigned* kv = batch_kv(S);
  const uint4* src = reinterpret_cast<const uint4*>(a.tok16 + first);
  for (int q = tid; q < (n >> 3); q += kFusedT) {
    const uint4 v = __ldg(src + q);
    const unsigned wd[4] = {v.x, v.y, v.z, v.w};
    unsigned o[8];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const unsigned t0 = wd[h] & 0xffffu, t1 = wd[h] >> 16;
      const unsigned k0 = desc ? 0x7fffu - t0 : t0, k1 = desc ? 0x7fffu - t1 : t1;
      const unsigned i0 = static_cast<unsigned>(8 * q + 2 * h);
      o[2 * h] = (k0 << 16) | i0;
      o[2 * h + 1] = (k1 << 16) | (i0 + 1);
    }
    reinterpret_cast<uint4*>(kv)[2 * q] = make_uint4(o[0], o[1], o[2], o[3]);
    reinterpret_cast<uint4*>(kv)[2 * q + 1] = make_uint4(o[4], o[5], o[6], o[7]);
  }
  for (int i = n + tid; i < kFusedSlots; i += kFusedT)  // padding: largest digits
    kv[i] = 0xffff0000u | static_cast<unsigned>(i);
  __syncthreads();
  // every token < kHistBins: ascending keys vary in bits [0, 13), descending
  // keys (0x7fff - tok > 0x5fff) in bits [0, 13) too; padding is 0xffff
  constexpr int kKeyBits = 13;
  static_assert(kHistBins <= (1 << kKeyBits), "keys of the histogram path fit 13 bits");
  unsigned* cw = sort_counters();
  for (int sh = 0; sh < kKeyBits; sh += kSortRB) {
    if (abort_epoch != 0u) {  // the cluster peer decided the batch: not kept
      if (tid == 0) S.sort_go = *reinterpret_cast<volatile unsigned*>(&S.sort_abort) != abort_epoch;
      __syncthreads();
      if (!S.sort_go) return;
    }
    const int bits = min(kSortRB, kKeyBits - sh);
    const unsigned mask = (1u << bits) - 1u;
    auto dig = [&](unsigned key) { return (key >> sh) & mask; };
    if (sh + kSortRB >= kKeyBits)
      tile_pass_kv<kFusedT, kFusedItems, kSortRB, true>(kv, dig, cw, S.tmp);
    else
      tile_pass_kv<kFusedT, kFusedItems, kSortRB, false>(kv, dig, cw, S.tmp);
  }
}

// The histogram path's buffers of batch slot W (0: A — every
// single-batch path; 1: B — the second batch of a two-batch descending step):
// token histogram (8,192 bins as u16 pairs), sorted sizes, the greedy's
// (group, slot) cells, the batch state.  B's histogram and sorted sizes live
// where A's are dead by then (the sort counters, A's histogram).
template <int W>
__device__ __forceinline__ unsigned* fp_hist_buf() {
  if constexpr (W) return sort_counters();
  else return reinterpret_cast<unsigned*>(shared_state().kbi);
}
template <int W>
__device__ __forceinline__ unsigned short* fp_skey() {
  if constexpr (W) return shared_state().kbi;
  else return shared_state().idx16;
}
template <int W>
__device__ __forceinline__ unsigned short* fp_cells() {
  if constexpr (W) return shared_state().cellsB;
  else return shared_state().out16;
}
template <int W>
__device__ __forceinline__ BatchState& fp_state() {
  if constexpr (W) return shared_state().B;
  else return shared_state().A;
}
static_assert(kHistBins * 2 <= 4 * blocked_cnt_words(kFusedT, kSortRB),
              "batch B's histogram fits the sort counters");

// Outputs of a kept batch from the greedy's cells of slot W and the
// sorted (key, index) items `kv` (this CTA's, or a cluster peer's handed
// over): the intra order and its staged tokens, coalesced per group.
template <int W>
__device__ __noinline__ void kept_output(const FusedArgs& a, long long b, const unsigned* kv) {
  const unsigned short* cells = fp_cells<W>();
  BatchState& T = fp_state<W>();
  const int n = a.n, m = a.m, lane = lane_id(), w = warp_id();
  const long long first = b * n;
  const bool desc = a.order == DTB_DESCENDING;
  const int cap = (n + m - 1) / m;
  const int capP = ((cap + 1) | 3) - 1;
  // the output pointers in registers: stores through them cannot then force
  // reloads of the (generic-addressed) kernel parameters every iteration
  int* __restrict__ order_out = a.order_out + first;
  unsigned short* __restrict__ tok_out = a.tok16_staged != nullptr ? a.tok16_staged + first : nullptr;
  for (int g = w; g < m; g += kFusedT / 32) {
    const int base = T.off[g], cnt = T.G.gcnt[g];
    for (int slot = lane; slot < cnt; slot += 32) {
      DTB_CHECK(g * capP + slot < kCells && base + slot < n);
      DTB_CHECK(cells[g * capP + slot] < n);
      const unsigned item = kv[swz(cells[g * capP + slot])];
      DTB_CHECK(static_cast<int>(item & 0xffffu) < n);
      order_out[base + slot] = static_cast<int>(item & 0xffffu);
      if (tok_out != nullptr) {
        const unsigned k = item >> 16;
        tok_out[base + slot] = static_cast<unsigned short>(desc ? 0x7fffu - k : k);
      }
    }
  }
}

// Histogram path (every token sum < kHistBins).  The greedy's decisions
// depend only on the SORTED SIZES, and equal sizes are interchangeable, so
// the sorted size sequence is the histogram's expansion: the greedy, its
// block loads and the keep decision (src/reorder.cpp:340-354) need no
// permutation.  Only a batch whose greedy split is kept needs the stable
// sort of its samples (sort_batch_keys; src/reorder.cpp:30-42).
//
// Phases (slot W): fp_hist (histogram of the cost pass's u16 tokens,
// identity block loads), fp_prep (sorted sizes), the greedy (ascending: 8
// warps over named barrier 1; descending: one warp), fp_decide (keep
// decision), fp_output (loads, kept flag, kept order).

// Token histogram of batch b and its identity block loads (from the cost
// pass).  All threads.
template <int W>
__device__ __forceinline__ void fp_hist(const FusedArgs& a, long long b) {
  unsigned* hist = fp_hist_buf<W>();
  BatchState& T = fp_state<W>();
  const int n = a.n, m = a.m, tid = threadIdx.x;
  const long long first = b * n;
  for (int q = tid; q < kHistBins / 8; q += kFusedT)
    reinterpret_cast<uint4*>(hist)[q] = make_uint4(0, 0, 0, 0);
  for (int g = tid; g < m; g += kFusedT) T.blk_ident[g] = a.blk_ident[b * m + g];
  __syncthreads();
  constexpr int V = 3;  // 128-bit loads in flight per thread and round
  const uint4* src = reinterpret_cast<const uint4*>(a.tok16 + first);
  const int nv = n >> 3;
  unsigned z = 0u;
  for (int v0 = 0; v0 * kFusedT < nv; v0 += V) {
    uint4 q[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int idx = tid + (v0 + v) * kFusedT;
      q[v] = idx < nv ? __ldg(src + idx) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int idx = tid + (v0 + v) * kFusedT;
      if (idx >= nv) break;
      const unsigned words[4] = {q[v].x, q[v].y, q[v].z, q[v].w};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const unsigned t = (words[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
        DTB_CHECK(t < static_cast<unsigned>(kHistBins));
        if (t == 0u)
          ++z;
        else
          atomicAdd(hist + (t >> 1), 1u << ((t & 1u) << 4));
      }
    }
  }
  z = __reduce_add_sync(kFull, z);
  if (lane_id() == 0 && z) atomicAdd(hist, z);
  __syncthreads();
}

// Sorted sizes skey[p] = token of sorted position p: starts of every token
// value (ascending: exclusive prefix; descending: n - inclusive prefix), run
// heads skey[start] = tok + 1 over a zeroed skey, then a "last non-zero"
// fill-forward scan.  All threads.
template <int W>
__device__ __forceinline__ void fp_prep(const FusedArgs& a, long long b) {
  NarrowSmem& S = shared_state();
  const unsigned* hist = fp_hist_buf<W>();
  unsigned short* skey = fp_skey<W>();
  BatchState& T = fp_state<W>();
  const int n = a.n, tid = threadIdx.x;
  const bool desc = a.order == DTB_DESCENDING;
  if (tid == 0) T.zc = static_cast<int>(hist[0] & 0xffffu);
  for (int q = tid; q < kFusedSlots / 8; q += kFusedT)
    reinterpret_cast<uint4*>(skey)[q] = make_uint4(0, 0, 0, 0);
  constexpr int kWordsPer = kHistBins / 2 / kFusedT;  // 4 words = 8 bins per thread
  static_assert(kWordsPer % 4 == 0 && kWordsPer >= 4, "scan layout");
  int sum = 0;
#pragma unroll
  for (int q = 0; q < kWordsPer / 4; ++q) {
    const uint4 v = reinterpret_cast<const uint4*>(hist + tid * kWordsPer)[q];
    sum += static_cast<int>((v.x & 0xffffu) + (v.x >> 16) + (v.y & 0xffffu) + (v.y >> 16) +
                            (v.z & 0xffffu) + (v.z >> 16) + (v.w & 0xffffu) + (v.w >> 16));
  }
  int tot;
  int base = block_excl_scan<kFusedT>(sum, S.tmp, &tot);  // also orders the zeroing
  {
    unsigned c[kWordsPer];  // re-read: nothing held across the scan
#pragma unroll
    for (int q = 0; q < kWordsPer / 4; ++q) {
      const uint4 v = reinterpret_cast<const uint4*>(hist + tid * kWordsPer)[q];
      c[4 * q] = v.x, c[4 * q + 1] = v.y, c[4 * q + 2] = v.z, c[4 * q + 3] = v.w;
    }
#pragma unroll
    for (int q = 0; q < kWordsPer; ++q) {
      const int lo = static_cast<int>(c[q] & 0xffffu), hi = static_cast<int>(c[q] >> 16);
      const unsigned v0 = static_cast<unsigned>(tid * 2 * kWordsPer + 2 * q);
      const int s0 = desc ? n - (base + lo) : base;
      const int s1 = desc ? n - (base + lo + hi) : base + lo;
      base += lo + hi;
      DTB_CHECK(!lo || (s0 >= 0 && s0 < n));
      DTB_CHECK(!hi || (s1 >= 0 && s1 < n));
      if (lo) skey[s0] = static_cast<unsigned short>(v0 + 1);
      if (hi) skey[s1] = static_cast<unsigned short>(v0 + 2);
    }
  }
  __syncthreads();
  constexpr int C = kFusedSlots / kFusedT;  // positions per thread (16 = 2 x 16 bytes)
  static_assert(C % 8 == 0, "fill-forward chunks of 16 bytes");
  const int p0 = tid * C;
  unsigned last = 0u;
#pragma unroll
  for (int q = 0; q < C / 8; ++q) {
    const uint4 v = reinterpret_cast<const uint4*>(skey + p0)[q];
    const unsigned wd[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      const unsigned e = (wd[h >> 1] >> ((h & 1) * 16)) & 0xffffu;
      if (e) last = e;
    }
  }
  unsigned run;
  block_last_nz(last, S.tmp, &run);
#pragma unroll
  for (int q = 0; q < C / 8; ++q) {
    const uint4 v = reinterpret_cast<const uint4*>(skey + p0)[q];  // re-read: no registers held across the scan
    unsigned wd[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      const unsigned e = (wd[h >> 1] >> ((h & 1) * 16)) & 0xffffu;
      if (e) run = e;
      const unsigned val = (run - 1u) & 0xffffu;
      wd[h >> 1] = (h & 1) ? ((wd[h >> 1] & 0xffffu) | (val << 16)) : ((wd[h >> 1] & 0xffff0000u) | val);
    }
    reinterpret_cast<uint4*>(skey + p0)[q] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
  }
  __syncthreads();
}

// The equal-count greedy over slot W's sorted sizes (reference:
// src/reorder.cpp:70-90): descending on warp W; ascending on all threads
// (greedy_asc_block).  The caller brackets it with __syncthreads.
// (each variant its own function: separate register allocation)
template <int W, bool DESC>
__device__ __noinline__ void fp_greedy_run(const FusedArgs& a, long long b) {
  const unsigned short* skey = fp_skey<W>();
  unsigned short* cells = fp_cells<W>();
  BatchState& T = fp_state<W>();
  const int n = a.n, m = a.m;
  const int cap = (n + m - 1) / m;
  const int capP = ((cap + 1) | 3) - 1;
  const int zc = T.zc;
  auto size_at = [&](int k) -> unsigned {
    const unsigned t = skey[k];
    return t + t;
  };
  auto emit = [&](int k, int g, int slot) {
    DTB_CHECK(g >= 0 && g < m && slot >= 0 && slot < cap && g * capP + slot < kCells && k >= 0 && k < n);
    cells[g * capP + slot] = static_cast<unsigned short>(k);
  };
  // u32 keys (load << 8 | gid) while every load stays below 2^24
  const bool k32 = static_cast<long long>(cap) * 2 * (kHistBins - 1) < (1ll << 24);
  if constexpr (DESC) {  // warp W
    unsigned long long* gprof = a.prof ? a.prof + b * kProfSlots + 6 : nullptr;
    if (k32)
      greedy_warp<unsigned>(n, m, cap, n - zc, n, size_at, emit, T.WG, T.G.gload, T.G.gcnt, gprof);
    else
      greedy_warp<unsigned long long>(n, m, cap, n - zc, n, size_at, emit, T.WG, T.G.gload,
                                      T.G.gcnt, gprof);
  } else {  // threads [0, 256), named barrier 1 (8-warp barriers: much cheaper than 32-warp ones)
    constexpr int kGT = 256;
    unsigned long long* gprof = a.prof ? a.prof + b * kProfSlots + 6 : nullptr;
    if (threadIdx.x < kGT)
      greedy_fused<kGT, true, 1>(n, m, cap, 0, zc, size_at, emit, T.G, shared_state().tmp,
                                 shared_state().tmpll, gprof);
  }
}

template <int W>
__device__ __forceinline__ void fp_greedy(const FusedArgs& a, long long b) {
  if (a.order == DTB_DESCENDING) {
    if (warp_id() == W) fp_greedy_run<W, true>(a, b);
  } else {
    fp_greedy_run<W, false>(a, b);  // (slot A only)
  }
}

// Group offsets of the flat order, greedy block loads and the keep
// decision (src/reorder.cpp:340-354, exact integer loads) on one warp; the
// caller's __syncthreads publishes T.keep_flag.  Needs the slot's sorted
// sizes (n % m != 0) and cells.
template <int W>
__device__ __forceinline__ void fp_decide(const FusedArgs& a) {
  const unsigned short* skey = fp_skey<W>();
  const unsigned short* cells = fp_cells<W>();
  BatchState& T = fp_state<W>();
  const int n = a.n, m = a.m, lane = lane_id(), w = warp_id();
  const int pg = n / m;
  const int cap = (n + m - 1) / m;
  const int capP = ((cap + 1) | 3) - 1;
  {
    if (w == 0) {  // m <= 128 groups: 4 per lane, no block barriers
      int cnt[4], sum = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int g = 4 * lane + e;
        cnt[e] = g < m ? T.G.gcnt[g] : 0;
        sum += cnt[e];
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      int base = incl - sum;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int g = 4 * lane + e;
        if (g < m) T.off[g] = base;
        base += cnt[e];
      }
      unsigned mg = 0u, mi = 0u;
      if (n % m == 0) {  // blocks == groups
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int g = 4 * lane + e;
          if (g < m) {
            const unsigned l = T.G.gload[g];
            T.blk_greedy[g] = l;
            mg = max(mg, l);
            mi = max(mi, T.blk_ident[g]);
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (4 * lane + e < m) T.blk_greedy[4 * lane + e] = 0u;
        __syncwarp();
        for (int g = 0; g < m; ++g)
          for (int slot = lane; slot < T.G.gcnt[g]; slot += 32) {
            const int pos = T.off[g] + slot;
            const unsigned t = skey[cells[g * capP + slot]];
            atomicAdd(&T.blk_greedy[min(pos / pg, m - 1)], t + t);
          }
        __syncwarp();
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int g = 4 * lane + e;
          if (g < m) {
            mg = max(mg, T.blk_greedy[g]);
            mi = max(mi, T.blk_ident[g]);
          }
        }
      }
      mg = __reduce_max_sync(kFull, mg);
      mi = __reduce_max_sync(kFull, mi);
      if (lane == 0) T.keep_flag = mg <= mi ? 1u : 0u;
    }
  }
}

// The outputs after fp_decide (and a __syncthreads): loads, kept flag, and
// for a kept batch its order — sorted here (the sort reuses kbi / idx16 and
// the counters), or (defer_kept, cluster pair) handed to the peer that
// sorted it.  All threads.
template <int W>
__device__ __forceinline__ void fp_output(const FusedArgs& a, long long b, bool defer_kept) {
  NarrowSmem& S = shared_state();
  BatchState& T = fp_state<W>();
  const int n = a.n, m = a.m, tid = threadIdx.x;
  const long long first = b * n;
  const bool keep = a.intra && T.keep_flag != 0u;
  if (tid == 0 && a.kept != nullptr) a.kept[b] = keep ? 1 : 0;
  for (int g = tid; g < m; g += kFusedT)
    write_outputs_common(a, b, g, T.blk_ident[g], keep ? T.blk_greedy[g] : T.blk_ident[g]);
  if (a.prof && tid == 0) a.prof[b * kProfSlots + 4] = globaltimer();
  if (!keep) {
    if (defer_kept && tid == 0)  // stop the peer's speculative sort
      *reinterpret_cast<volatile unsigned*>(cg::this_cluster().map_shared_rank(&S.sort_abort, 1)) =
          S.pair_epoch;
    if (a.state == nullptr) identity_order_out(a, first, n);  // else written by the cost pass
  } else if (defer_kept) {  // (slot A)
    // hand this CTA's cells, group offsets and counts to the cluster peer,
    // which holds the sorted items (DSMEM stores: no round trips), and mark
    // the batch there; the peer writes the kept order after the cluster sync
    cg::cluster_group cl = cg::this_cluster();
    uint4* dst = reinterpret_cast<uint4*>(cl.map_shared_rank(S.out16, 1));
    const uint4* src = reinterpret_cast<const uint4*>(S.out16);
    constexpr int kCellWords = static_cast<int>(sizeof(NarrowSmem::out16) / 16);
    for (int q = tid; q < kCellWords; q += kFusedT) dst[q] = src[q];
    int* doff = cl.map_shared_rank(S.A.off, 1);
    int* dcnt = cl.map_shared_rank(S.A.G.gcnt, 1);
    for (int g = tid; g < m; g += kFusedT) {
      doff[g] = S.A.off[g];
      dcnt[g] = S.A.G.gcnt[g];
    }
    if (tid == 0) *cl.map_shared_rank(&S.deferred, 1) = S.pair_epoch;
  } else {  // the permutation, here
    __syncthreads();
    sort_batch_keys(a, b, S);
    kept_output<W>(a, b, batch_kv(S));
  }
  if (a.prof) {
    __syncthreads();
    if (tid == 0) a.prof[b * kProfSlots + 5] = globaltimer();
  }
}

// One batch on the histogram path (slot A).
__device__ __noinline__ void fast_path(const FusedArgs& a, long long b, NarrowSmem&,
                                      bool defer_kept) {
  if (a.intra) {
    fp_prep<0>(a, b);
    if (a.prof && threadIdx.x == 0) a.prof[b * kProfSlots + 2] = globaltimer();
    fp_greedy<0>(a, b);
    __syncthreads();
    if (a.prof && threadIdx.x == 0) a.prof[b * kProfSlots + 3] = globaltimer();
    fp_decide<0>(a);
    __syncthreads();
  }
  fp_output<0>(a, b, defer_kept);
}

// Two batches on the histogram path, descending order: their one-warp
// greedies (all rounds general: ~95% of a batch's time) run side by side on
// warps 0 and 1; everything else is block-wide, one batch after the other.
__device__ __noinline__ void fast_path_two_desc(const FusedArgs& a, long long b0, long long b1) {
  fp_hist<0>(a, b0);
  fp_prep<0>(a, b0);
  fp_hist<1>(a, b1);
  fp_prep<1>(a, b1);
  if (warp_id() == 0) fp_greedy_run<0, true>(a, b0);
  else if (warp_id() == 1) fp_greedy_run<1, true>(a, b1);
  __syncthreads();
  fp_decide<0>(a);
  fp_decide<1>(a);  // (warp 0 both: before A's sort reuses B's sorted sizes)
  __syncthreads();
  fp_output<0>(a, b0, false);
  __syncthreads();
  fp_output<1>(a, b1, false);
}

// Sort path of the 16-bit layout (token sums up to 0x7fff, or the separate
// cost pass): keys from the u16 tokens `tok` (written earlier — by this CTA
// or by the cost pass; read through L2), stable LSD radix sort, greedy,
// decision, outputs.
__device__ __noinline__ void narrow_sort_path(const FusedArgs& a, long long b, NarrowSmem&,
                                              const unsigned short* tok) {
  NarrowSmem& S = shared_state();
  const int n = a.n, m = a.m, tid = threadIdx.x;
  const int lane = lane_id(), w = warp_id();
  const long long first = b * n;
  const int pg = n / m;
  const bool desc = a.order == DTB_DESCENDING;
  __syncthreads();
  for (int g = tid; g < m; g += kFusedT) S.A.blk_ident[g] = 0u;
  if (tid == 0) {
    S.s_and = ~0u;
    S.s_or = 0u;
  }
  __syncthreads();
  unsigned int kand = ~0u, kor = 0u;
  int zeros = 0;
  auto take_sample = [&](int i, unsigned t) {
    const unsigned key = desc ? 0x7fffu - t : t;
    kand &= key;
    kor |= key;
    zeros += t == 0;
    S.kbi[i] = static_cast<unsigned short>(key);
    S.idx16[i] = static_cast<unsigned short>(i);
  };
  {
    // 8 samples per 128-bit load, all loads issued before use
    constexpr int V = (kFusedMaxN / 8 + kFusedT - 1) / kFusedT;
    const uint4* src = reinterpret_cast<const uint4*>(tok + first);
    const int nv = n >> 3;
    uint4 q[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int idx = tid + v * kFusedT;
      q[v] = idx < nv ? __ldcg(src + idx) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int idx = tid + v * kFusedT;
      if (idx >= nv) break;
      const unsigned words[4] = {q[v].x, q[v].y, q[v].z, q[v].w};
      const int i0 = idx * 8;
      const unsigned blk0 = min(a.div_pg.div(static_cast<unsigned>(i0)), static_cast<unsigned>(m - 1));
      const unsigned blk7 = min(a.div_pg.div(static_cast<unsigned>(i0 + 7)), static_cast<unsigned>(m - 1));
      unsigned run = 0u;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = i0 + j;
        const unsigned t = (words[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
        take_sample(i, t);
        if (blk0 == blk7) {
          run += 2u * t;
        } else {
          const unsigned qd = a.div_pg.div(static_cast<unsigned>(i));
          atomicAdd(&S.A.blk_ident[min(qd, static_cast<unsigned>(m - 1))], 2u * t);
        }
      }
      if (blk0 == blk7) atomicAdd(&S.A.blk_ident[blk0], run);
    }
  }
  // sort padding: key 0xffff has the largest digit in every pass
  for (int i = n + tid; i < kFusedSlots; i += kFusedT) {
    S.kbi[i] = 0xffffu;
    S.idx16[i] = static_cast<unsigned short>(i);
  }
  atomicAnd(&S.s_and, kand);
  atomicOr(&S.s_or, kor);
  int tot_zeros;
  block_excl_scan<kFusedT>(zeros, S.tmp, &tot_zeros);
  bool keep = false;
  const int cap = (n + m - 1) / m;
  const int capP = ((cap + 1) | 3) - 1;  // >= cap, == 2 mod 4
  if (a.intra) {
    if (a.prof && tid == 0) a.prof[b * kProfSlots + 1] = globaltimer();
    // ---- stable LSD radix sort by key over its varying bit window; the
    // last pass writes swizzled positions (at least one pass always runs)
    const unsigned varying = S.s_and ^ S.s_or;
    const int lo = varying ? __ffs(static_cast<int>(varying)) - 1 : 0;
    const int hi = varying ? 32 - __clz(static_cast<int>(varying)) : 1;
    for (int sh = lo; sh < hi; sh += kSortRB) {
      const int bits = min(kSortRB, hi - sh);
      const unsigned mask = (1u << bits) - 1u;
      auto dig = [&](unsigned key) { return (key >> sh) & mask; };
      unsigned* cw = sort_counters();
      if (sh + kSortRB >= hi)
        tile_pass_blocked<kFusedT, kFusedItems, kSortRB, true>(S.idx16, S.kbi, dig, cw, S.tmp);
      else
        tile_pass_blocked<kFusedT, kFusedItems, kSortRB, false>(S.idx16, S.kbi, dig, cw, S.tmp);
    }
    if (a.prof && tid == 0) a.prof[b * kProfSlots + 2] = globaltimer();
    // ---- greedy equal-count partition (sizes = 2 * tokens), emitted
    // straight into the flat order's (group, slot) cells
    const int z0 = desc ? n - tot_zeros : 0;
    const int z1 = desc ? n : tot_zeros;
    auto size_at = [&](int k) -> unsigned {
      const unsigned key = S.kbi[S.idx16[swz(k)]];
      const unsigned t = desc ? 0x7fffu - key : key;
      return t + t;
    };
    auto emit = [&](int k, int g, int slot) {
      S.out16[g * capP + slot] = static_cast<unsigned short>(k);
    };
    // ascending: the greedy runs on 8 warps over named barrier 1 (its full
    // rounds are block-parallel; 8-warp barriers are much cheaper than
    // 32-warp ones); descending (every round a general one): on one warp
    constexpr int kGT = 256;
    unsigned long long* gprof = a.prof ? a.prof + b * kProfSlots + 6 : nullptr;
    if (desc) {
      // u32 keys (load << 8 | gid) while every load stays below 2^24
      if (w == 0) {
        if (static_cast<long long>(cap) * 2 * 0x7fff < (1ll << 24))
          greedy_warp<unsigned>(n, m, cap, z0, z1, size_at, emit, S.A.WG, S.A.G.gload, S.A.G.gcnt, gprof);
        else
          greedy_warp<unsigned long long>(n, m, cap, z0, z1, size_at, emit, S.A.WG, S.A.G.gload, S.A.G.gcnt,
                                          gprof);
      }
    } else if (tid < kGT) {
      greedy_fused<kGT, true, 1>(n, m, cap, z0, z1, size_at, emit, S.A.G, S.tmp, S.tmpll, gprof);
    }
    __syncthreads();
    if (a.prof && tid == 0) a.prof[b * kProfSlots + 3] = globaltimer();
    // ---- group offsets of the flat order and the greedy block loads
    int c = tid < m ? S.A.G.gcnt[tid] : 0, tot;
    const int o = block_excl_scan<kFusedT>(c, S.tmp, &tot);
    if (tid < m) S.A.off[tid] = o;
    if (n % m == 0) {
      // blocks are the groups (every group holds cap = n / m items)
      for (int g = tid; g < m; g += kFusedT) S.A.blk_greedy[g] = S.A.G.gload[g];
    } else {
      for (int g = tid; g < m; g += kFusedT) S.A.blk_greedy[g] = 0u;
      __syncthreads();
      for (int g = w; g < m; g += kFusedT / 32) {
        for (int slot = lane; slot < S.A.G.gcnt[g]; slot += 32) {
          const int pos = S.A.off[g] + slot;
          atomicAdd(&S.A.blk_greedy[min(pos / pg, m - 1)], size_at(S.out16[g * capP + slot]));
        }
      }
    }
    __syncthreads();
    unsigned mg = 0u, mi = 0u;
    for (int g = tid; g < m; g += kFusedT) {
      mg = max(mg, S.A.blk_greedy[g]);
      mi = max(mi, S.A.blk_ident[g]);
    }
    mg = static_cast<unsigned>(block_max_ll<kFusedT>(mg, S.tmpll));
    mi = static_cast<unsigned>(block_max_ll<kFusedT>(mi, S.tmpll));
    // src/reorder.cpp:350-353: keep the greedy split when its max block load
    // is no worse than the incoming order's (integer loads: exact).
    keep = mg <= mi;
  } else {
    __syncthreads();
  }
  if (tid == 0 && a.kept != nullptr) a.kept[b] = keep ? 1 : 0;
  for (int g = tid; g < m; g += kFusedT)
    write_outputs_common(a, b, g, S.A.blk_ident[g], keep ? S.A.blk_greedy[g] : S.A.blk_ident[g]);
  if (a.prof && tid == 0) a.prof[b * kProfSlots + 4] = globaltimer();
  // ---- outputs, coalesced: one warp per group, lanes over its slots — the
  // intra order and, when the greedy split is kept, its per-position tokens
  // (identity batches reuse the input-order tokens, see TokSrc)
  if (keep) {
    for (int g = w; g < m; g += kFusedT / 32) {
      const int base = S.A.off[g], cnt = S.A.G.gcnt[g];
      for (int slot = lane; slot < cnt; slot += 32) {
        const unsigned idx = S.idx16[swz(S.out16[g * capP + slot])];
        const unsigned key = S.kbi[idx];
        a.order_out[first + base + slot] = static_cast<int>(idx);
        if (a.tok16_staged != nullptr)
          a.tok16_staged[first + base + slot] = static_cast<unsigned short>(desc ? 0x7fffu - key : key);
      }
    }
  } else if (a.state == nullptr) {  // else written by the cost pass
    identity_order_out(a, first, n);
  }
  if (a.prof) {
    __syncthreads();
    if (tid == 0) a.prof[b * kProfSlots + 5] = globaltimer();
  }
}

// Per global batch, after the streaming cost pass (cost_stream_kernel,
// k_cost.cu): batches it already decided exit at once; the rest take the
// histogram path, the sort path (token sums >= kHistBins) or the 32-bit path.
__device__ __forceinline__ void process_batch(const FusedArgs& a, long long b, NarrowSmem& S,
                                              bool defer_kept = false) {
  const int n = a.n, m = a.m, tid = threadIdx.x;
  const long long first = b * n;
  const unsigned st = a.state != nullptr ? a.state[b] : kBatchSort;
  if (st == kBatchDecided) return;

  if (a.prof && tid == 0) a.prof[b * kProfSlots + 0] = globaltimer();
  // Batches outside the 16-bit layout's limits take the 32-bit path.
  if (st == kBatchWide || m > kNarrowMaxM || n > kFusedMaxN || (n & 7) ||
      (a.state == nullptr && a.wide_flag[b])) {
    // consumers (TokSrc) then read this batch's 32-bit token copies
    if (tid == 0 && a.state == nullptr) a.wide_flag[b] = 1u;  // else set by the cost pass
    fused_wide(a, b, S);
    return;
  }
  if (st == kBatchSort) {
    narrow_sort_path(a, b, S, a.tok16);
    return;
  }
  // ---- histogram path: token histogram from the cost pass's u16 tokens;
  // identity block loads from the cost pass
  fp_hist<0>(a, b);
  if (a.prof && tid == 0) a.prof[b * kProfSlots + 1] = globaltimer();
  fast_path(a, b, S, defer_kept);
}

// One CTA per batch, or (with the cost pass's list) persistent CTAs over the
// batches it left undecided.
__global__ void __launch_bounds__(kFusedT, DTB_FUSED_MIN_BLOCKS)
intra_fused_kernel(const __grid_constant__ FusedArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  NarrowSmem& S = *reinterpret_cast<NarrowSmem*>(smem_raw);
  pdl_wait();  // the cost pass's list and batch states
  if (a.prof && threadIdx.x == 0) {  // debug: first CTA entry, last CTA exit
    atomicMin(a.prof + 62, globaltimer());
    atomicMax(a.prof + 63, 0ull);
  }
  if (a.list == nullptr) {
    process_batch(a, blockIdx.x, S);
    return;
  }
  const unsigned count = a.list[0];
  const unsigned pairs = gridDim.x / 2;  // launched as clusters of two CTAs
  if (count > pairs) {  // many batches: every CTA takes its own
    const bool desc = a.order == DTB_DESCENDING && a.intra && a.m <= kNarrowMaxM &&
                      a.n <= kFusedMaxN && (a.n & 7) == 0;
    auto fast = [&](long long b) { return a.state[b] == kBatchFast; };
    unsigned q = blockIdx.x;
    if (desc) {  // two histogram-path batches at a time: their greedies side by side
      for (; q + gridDim.x < count; q += 2 * gridDim.x) {
        const long long b0 = a.list[1 + q], b1 = a.list[1 + q + gridDim.x];
        if (fast(b0) && fast(b1)) {
          if (a.prof && threadIdx.x == 0) a.prof[b0 * kProfSlots + 0] = globaltimer();
          fast_path_two_desc(a, b0, b1);
        } else {
          process_batch(a, b0, S);
          __syncthreads();
          process_batch(a, b1, S);
        }
        __syncthreads();  // the shared state is reused by the next batches
      }
    }
    for (; q < count; q += gridDim.x) {
      process_batch(a, a.list[1 + q], S);
      __syncthreads();  // the shared state is reused by the next batch
    }
    if (a.prof && threadIdx.x == 0) atomicMax(a.prof + 63, globaltimer());
    return;
  }
  // Few batches (latency-bound): the two CTAs of a cluster share one.  Rank 0
  // runs the histogram, greedy and keep decision while rank 1 runs the
  // stable radix sort; for a kept batch rank 0 stores its (group, slot)
  // cells into rank 1's shared memory (DSMEM) and rank 1 writes the order.
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  if (blockIdx.x / 2 >= count) return;  // the whole pair is idle
  if (threadIdx.x == 0) S.sort_abort = S.deferred = 0u;
  cl.sync();
  for (unsigned q = blockIdx.x / 2; q < count; q += pairs) {
    const long long b = a.list[1 + q];
    const bool fast = a.state[b] == kBatchFast && a.m <= kNarrowMaxM && a.n <= kFusedMaxN &&
                      (a.n & 7) == 0;
    if (threadIdx.x == 0) S.pair_epoch = q + 1;
    __syncthreads();
    if (rank == 1) {
      if (fast) sort_batch_keys(a, b, S, q + 1);
      if (a.prof && threadIdx.x == 0) a.prof[b * kProfSlots + 57] = globaltimer();
    } else {
      process_batch(a, b, S, fast);
    }
    cl.sync();  // rank 1: its sorted items and (kept) rank 0's cells are ready
    if (a.prof && rank == 0 && threadIdx.x == 0) a.prof[b * kProfSlots + 58] = globaltimer();
    if (rank == 1 && S.deferred == q + 1) {
      if (a.prof && threadIdx.x == 0) a.prof[b * kProfSlots + 61] = globaltimer();
      kept_output<0>(a, b, batch_kv(S));
      if (a.prof) {
        __syncthreads();
        if (threadIdx.x == 0) a.prof[b * kProfSlots + 60] = globaltimer();
      }
    }
    cl.sync();  // rank 1's shared memory is free for the next batch's cells
    if (a.prof && rank == 1 && threadIdx.x == 0) a.prof[b * kProfSlots + 59] = globaltimer();
    if (a.prof && rank == 0 && threadIdx.x == 0) a.prof[b * kProfSlots + 59] = globaltimer();
  }
  if (a.prof && threadIdx.x == 0) atomicMax(a.prof + 63, globaltimer());
}

// ------------------------------------------------------------- host glue
cudaError_t launch_intra_fused(const FusedArgs& a, long long n_batches, cudaStream_t stream,
                               bool pdl) {
  // the opt-in is per device: set it on every launch (cheap), so contexts on
  // several devices and several host threads need no shared state
  cudaError_t e = cudaFuncSetAttribute(intra_fused_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(kFusedSmem));
  if (e != cudaSuccess) return e;
  long long grid = n_batches;
  if (a.list != nullptr) {  // persistent: one CTA per SM
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid = static_cast<long long>(sms) * DTB_FUSED_MIN_BLOCKS / 2 * 2;  // clusters of two
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(kFusedT);
    cfg.dynamicSmemBytes = kFusedSmem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    // programmatic launch right behind the cost pass's finalize kernel (same
    // stream, no event wait in between)
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, intra_fused_kernel, a);
  }
  intra_fused_kernel<<<static_cast<unsigned>(grid), kFusedT, kFusedSmem, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_intra_generic(const double* sizes, int n, int m, int order, int equal_counts,
                                 void* scratch, size_t scratch_bytes, int* flat_out,
                                 long long* offsets_out, cudaStream_t stream) {
  // scratch: keys[n] u64 x2, vals[n] x2, g_of[n], slot_of[n], greedy state, cub temp
  char* p = static_cast<char*>(scratch);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) & ~size_t(255);
    return r;
  };
  auto* keys = reinterpret_cast<unsigned long long*>(take(sizeof(unsigned long long) * n));
  auto* keys2 = reinterpret_cast<unsigned long long*>(take(sizeof(unsigned long long) * n));
  auto* vals = reinterpret_cast<int*>(take(sizeof(int) * n));
  auto* vals2 = reinterpret_cast<int*>(take(sizeof(int) * n));
  auto* g_of = reinterpret_cast<int*>(take(sizeof(int) * n));
  auto* slot_of = reinterpret_cast<int*>(take(sizeof(int) * n));
  GreedyState<double> st;
  st.AL = reinterpret_cast<double*>(take(sizeof(double) * m));
  st.TL = reinterpret_cast<double*>(take(sizeof(double) * m));
  st.AG = reinterpret_cast<int*>(take(sizeof(int) * m));
  st.TG = reinterpret_cast<int*>(take(sizeof(int) * m));
  st.cnt = reinterpret_cast<int*>(take(sizeof(int) * m));
  st.tmp = reinterpret_cast<int*>(take(sizeof(int) * (kGenT / 32 + 2)));
  st.gload = nullptr;
  st.tmpll = nullptr;
  const size_t used = static_cast<size_t>(p - static_cast<char*>(scratch));
  if (used > scratch_bytes) return cudaErrorMemoryAllocation;
  const int grid = (n + kGenT - 1) / kGenT;
  intra_keys_kernel<<<grid > 0 ? grid : 1, kGenT, 0, stream>>>(sizes, n, order, keys, vals);
  // Stable device-wide radix sort of (orderable key, index) pairs: ties keep
  // index order, i.e. the reference's (size, index) comparator.
  size_t temp = scratch_bytes - used;
  cub::DoubleBuffer<unsigned long long> dk(keys, keys2);
  cub::DoubleBuffer<int> dv(vals, vals2);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(p, temp, dk, dv, n, 0, 64, stream);
  if (e != cudaSuccess) return e;
  intra_generic_kernel<<<1, kGenT, 0, stream>>>(sizes, n, m, order, equal_counts, dv.Current(),
                                                g_of, slot_of, flat_out, offsets_out, st);
  return cudaGetLastError();
}

size_t intra_generic_scratch(int n, int m) {
  size_t b = 0;
  auto add = [&](size_t x) { b += (x + 255) & ~size_t(255); };
  add(8ull * n); add(8ull * n); add(4ull * n); add(4ull * n); add(4ull * n); add(4ull * n);
  add(8ull * m); add(8ull * m); add(4ull * m); add(4ull * m); add(4ull * m);
  add(4ull * (kGenT / 32 + 2));
  size_t temp = 0;
  cub::DoubleBuffer<unsigned long long> dk(nullptr, nullptr);
  cub::DoubleBuffer<int> dv(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, temp, dk, dv, n, 0, 64);
  return b + temp + 1024;
}

int intra_generic_max_m() { return kGenT * kGenEmax; }

}  // namespace dtb

// Streaming cost pass of the disaggregated reorder (K0).
//
// Per sample: Sample::cost_size (include/core.hpp:160-167, src/core.cpp:90-95)
// = 2 x (image + audio subsequence tokens), kept as u16 tokens for the
// simulations and the partition kernel.  Per global batch: the identity
// order's block_group_loads (src/reorder.cpp:111-119), and — when the last
// chunk of a batch is done — the keep decision of disaggregated_reorder
// (src/reorder.cpp:340-354) whenever an averaging bound already settles it.
//
// One CTA of 128 threads per chunk of 1024 consecutive samples; ~20 KB of
// shared memory, so eleven CTAs share an SM.
// A chunk's CSR offsets and the CONTIGUOUS token spans its samples own
// ([io[c0], io[c0 + 1024]) — a batch's tokens are one span of the CSR) are
// brought in by bulk asynchronous copies (TMA, cp.async.bulk, completed on an
// mbarrier); an in-place exclusive prefix sum over the staged tokens turns
// every sample's sum into two shared-memory reads (no per-sample loops, no
// divergence, no dependent global loads).
//
// The bound: with ascending sizes and equal counts (cap = n / m), the z
// zero-cost items fill groups 0, 1, ... to cap first (every load is 0 and ties
// go to the lowest group, src/reorder.cpp:80-88), so floor(z / cap) groups
// hold no positive item and the positive total T is spread over at most
// m - floor(z / cap) groups: the greedy's max block load (blocks == groups
// when n % m == 0) is >= T / (m - floor(z / cap)).  If that exceeds the
// identity's max block load, the reference keeps the identity order
// (`<=` keeps the greedy) — exactly, in integers.  Every other batch goes to
// the partition kernel.
#include <algorithm>

#include "block_ops.cuh"
#include "kernels.cuh"
#include "pdl.cuh"
#include "tma.cuh"

namespace dtb {

#ifndef DTB_COST_Q
#define DTB_COST_Q 1024
#endif
#ifndef DTB_COST_MINB
#define DTB_COST_MINB 11
#endif
#ifndef DTB_COST_T
#define DTB_COST_T 128
#endif
#ifndef DTB_COST_SCAN_L
#define DTB_COST_SCAN_L 4
#endif
constexpr int kCostT = DTB_COST_T;          // threads per chunk CTA
constexpr int kCostQ = DTB_COST_Q;          // samples per chunk
constexpr int kCostOff = kCostQ + 4;        // offsets + the next boundary, padded
#ifndef DTB_COST_TOKQ
#define DTB_COST_TOKQ 11
#endif
constexpr int kCostTok = DTB_COST_TOKQ * kCostQ / 4;  // token slots (image + audio + spares; ~2.1 per sample used)
constexpr int kCostPer = kCostQ / kCostT;   // samples per thread

struct CostSmem {
  alignas(16) int io[kCostOff];
  alignas(16) int ao[kCostOff];
  alignas(16) int tk[kCostTok];
  alignas(8) unsigned long long bar[2];  // offsets, tokens
  int bnd[6];  // lo, hi, alo, ahi, image / audio token counts of the stream
  int tmp[2 * (kCostT / 32)];
};

// Token slots: image tokens [fl, ceil4(hi)) at [0, ilen), a zero spare slot,
// audio tokens [afl, ceil4(ahi)) at [abase, abase + alen), a zero spare slot.
// After the exclusive prefix sum E, a sample's image sum is E[hi - fl] -
// E[lo - fl].  Copies end at ceil4(hi) unless that passes the stream's last
// token (tend): then the last < 4 tokens are read by thread 0.
struct ChunkLayout {
  int fl, ilen, ilen_tma;
  int afl, alen, alen_tma, abase;
  int len;    // slots in the prefix sum
  bool fits;  // else: per-sample sums from global memory
};
__device__ __forceinline__ ChunkLayout chunk_layout(int lo, int hi, int alo, int ahi, int tend,
                                                    int aend, bool audio) {
  ChunkLayout L;
  L.fl = lo & ~3;
  const int c4 = (hi + 3) & ~3;
  L.ilen = c4 - L.fl;
  L.ilen_tma = (c4 <= tend ? c4 : (hi & ~3)) - L.fl;
  L.abase = (L.ilen + 4) & ~3;
  if (audio) {
    L.afl = alo & ~3;
    const int ac4 = (ahi + 3) & ~3;
    L.alen = ac4 - L.afl;
    L.alen_tma = (ac4 <= aend ? ac4 : (ahi & ~3)) - L.afl;
  } else {
    L.afl = L.alen = L.alen_tma = 0;
  }
  L.len = L.abase + L.alen + 1;
  L.fits = L.len <= kCostTok;
  return L;
}

// In-place exclusive prefix sum of tk[0, len).  Returns true when a slot lies
// outside [0, 0x7fff] (the int32 sums could overflow, or a sample's sum be
// negative): the chunk then uses the int64 per-sample path.  Warp w scans a
// contiguous quarter of the slots, lanes on consecutive 16-byte words
// (conflict-free: one word per lane and step — two words per lane put the
// lanes 32 B apart, 2-way bank conflicts, 76 vs 70 µs for the pass): a first
// pass sums the quarter, one barrier exchanges the four sums, a second pass
// scans with the carry-in.
__device__ __forceinline__ bool chunk_prefix(int* tk, int len, int* tmp) {
  constexpr int W = kCostT / 32;
  constexpr int L = DTB_COST_SCAN_L;  // consecutive slots per lane and step (16-byte words)
  const int lane = lane_id(), w = warp_id();
  const int R = (len + W * 32 * L - 1) / (W * 32 * L) * (32 * L);  // slots per warp
  const int beg = w * R, end = min(beg + R, len);
  auto load = [&](int p, int* v) {
    if (p + L <= end) {
#pragma unroll
      for (int q = 0; q < L / 4; ++q) {
        const int4 x = *reinterpret_cast<const int4*>(tk + p + 4 * q);
        v[4 * q] = x.x, v[4 * q + 1] = x.y, v[4 * q + 2] = x.z, v[4 * q + 3] = x.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < L; ++k) v[k] = p + k < end ? tk[p + k] : 0;
    }
  };
  int sum = 0;
  unsigned orv = 0u;
  for (int p = beg + L * lane; p < end; p += 32 * L) {
    int v[L];
    load(p, v);
#pragma unroll
    for (int k = 0; k < L; ++k) {
      sum += v[k];
      orv |= static_cast<unsigned>(v[k]);
    }
  }
  sum = static_cast<int>(__reduce_add_sync(kFull, static_cast<unsigned>(sum)));
  orv = __reduce_or_sync(kFull, orv);
  if (lane == 0) {
    tmp[w] = sum;
    tmp[W + w] = static_cast<int>(orv);
  }
  __syncthreads();
  int carry = 0;
  unsigned all_or = 0u;
#pragma unroll
  for (int k = 0; k < W; ++k) {
    if (k < w) carry += tmp[k];
    all_or |= static_cast<unsigned>(tmp[W + k]);
  }
  const bool bad = all_or > 0x7fffu;
  if (!bad) {
    for (int base = beg; base < end; base += 32 * L) {
      const int p = base + L * lane;
      int v[L];
      load(p, v);
#pragma unroll
      for (int k = 1; k < L; ++k) v[k] += v[k - 1];  // inclusive within the lane
      int incl = v[L - 1];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      const int e = carry + incl - v[L - 1];  // exclusive carry-in of the lane
      if (p + L <= end) {
        *reinterpret_cast<int4*>(tk + p) = make_int4(e, e + v[0], e + v[1], e + v[2]);
#pragma unroll
        for (int q = 1; q < L / 4; ++q)
          *reinterpret_cast<int4*>(tk + p + 4 * q) =
              make_int4(e + v[4 * q - 1], e + v[4 * q], e + v[4 * q + 1], e + v[4 * q + 2]);
      } else {
        for (int k = 0; k < L && p + k < end; ++k) tk[p + k] = k ? e + v[k - 1] : e;
      }
      carry += __shfl_sync(kFull, incl, 31);
    }
  }
  __syncthreads();
  return bad;
}

// A whole small batch (n <= kSmallN samples, m <= kSmallN groups) in one
// warp, exactly as the reference: stable order by (cost, index) — descending:
// (-cost, index) — (src/reorder.cpp:30-42), the equal-count greedy (each
// item to the least loaded group with room, ties to the lowest group,
// src/reorder.cpp:70-90; integer loads: exact), its block loads and the
// keep decision (src/reorder.cpp:340-354).  Batches of a few dozen samples
// (BASELINE config 2: 32 per iteration) need no partition kernel.
constexpr int kSmallN = 128;
__device__ __noinline__ void small_batch(const CostArgs& a, long long b, unsigned short* tk,
                                         unsigned short* sorted, unsigned* load,
                                         unsigned char* cnt, unsigned short* flat_of,
                                         unsigned* blk) {
  const int n = a.n, m = a.m, lane = threadIdx.x & 31;
  const long long first = b * n;
  const bool desc = a.order == DTB_DESCENDING;
  for (int i = lane; i < n; i += 32) tk[i] = a.tok16[first + i];
  for (int g = lane; g < m; g += 32) load[g] = 0u, cnt[g] = 0, blk[g] = 0u;
  __syncwarp();
  // stable rank of every item
  for (int i = lane; i < n; i += 32) {
    const unsigned ki = tk[i];
    int r = 0;
    for (int j = 0; j < n; ++j) {
      const unsigned kj = tk[j];
      r += desc ? (kj > ki || (kj == ki && j < i)) : (kj < ki || (kj == ki && j < i));
    }
    sorted[r] = static_cast<unsigned short>(i);
  }
  __syncwarp();
  // equal-count greedy, item by item; the group of every sorted item
  const int cap = (n + m - 1) / m;
  unsigned char* group_of = reinterpret_cast<unsigned char*>(flat_of);  // reused below
  for (int k = 0; k < n; ++k) {
    const unsigned size = 2u * tk[sorted[k]];
    unsigned bl = 0xffffffffu;
    int bg = 0x7fffffff;
    for (int g = lane; g < m; g += 32)
      if (cnt[g] < cap && (load[g] < bl || (load[g] == bl && g < bg))) bl = load[g], bg = g;
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned ol = __shfl_xor_sync(0xffffffffu, bl, o);
      const int og = __shfl_xor_sync(0xffffffffu, bg, o);
      if (ol < bl || (ol == bl && og < bg)) bl = ol, bg = og;
    }
    if (lane == 0) {
      load[bg] += size;
      ++cnt[bg];
      group_of[k] = static_cast<unsigned char>(bg);
    }
    __syncwarp();
  }
  // flat order (IntraPartition::flat): groups in order, items in sorted order
  if (lane == 0) {
    int off = 0;
    for (int g = 0; g < m; ++g) {
      const int c = cnt[g];
      cnt[g] = static_cast<unsigned char>(0);
      load[g] = static_cast<unsigned>(off);  // group offset (loads are no longer needed)
      off += c;
    }
  }
  __syncwarp();
  unsigned short* flat = tk + kSmallN;  // tk[kSmallN .. 2 kSmallN): flat order (sample indices)
  if (lane == 0)
    for (int k = 0; k < n; ++k) {
      const int g = group_of[k];
      flat[load[g] + cnt[g]] = sorted[k];
      ++cnt[g];
    }
  __syncwarp();
  // block loads of the greedy flat order and of the identity
  const int per = n / m;
  unsigned mg = 0u, mi = 0u;
  for (int g = lane; g < m; g += 32) {
    const int lo = g * per, hi = g == m - 1 ? n : lo + per;
    unsigned sg = 0u, si = 0u;
    for (int q = lo; q < hi; ++q) {
      sg += 2u * tk[flat[q]];
      si += 2u * tk[q];
    }
    blk[g] = sg;
    mg = max(mg, sg);
    mi = max(mi, si);
    if (a.load_before) a.load_before[b * m + g] = static_cast<double>(si);
  }
  mg = __reduce_max_sync(0xffffffffu, mg);
  mi = __reduce_max_sync(0xffffffffu, mi);
  const bool keep = mg <= mi;
  for (int g = lane; g < m; g += 32) {
    const int lo = g * per, hi = g == m - 1 ? n : lo + per;
    unsigned si = 0u;
    for (int q = lo; q < hi; ++q) si += 2u * tk[q];
    if (a.load_after) a.load_after[b * m + g] = static_cast<double>(keep ? blk[g] : si);
  }
  for (int q = lane; q < n; q += 32) {
    const int src = keep ? flat[q] : q;
    a.order_out[first + q] = src;
    if (a.tok16_staged != nullptr && keep) a.tok16_staged[first + q] = tk[src];
  }
  if (lane == 0 && a.kept) a.kept[b] = keep ? 1 : 0;
}

// Per batch, after the cost pass: identity loads, averaging bound, batch
// state; batches the partition kernel must process are appended to `list`.
__global__ void __launch_bounds__(kCostT) cost_finalize_kernel(const __grid_constant__ CostArgs a) {
  __shared__ long long red[kCostT / 32 + 1];
  pdl_wait();  // the cost pass's statistics
  const int m = a.m, tid = threadIdx.x;
  const long long b = blockIdx.x;
  const unsigned* st = a.bstat + 4 * b;
  const unsigned z = st[0], total = st[1], flags = st[2];
  unsigned mi = 0u;
  for (int g = tid; g < m; g += kCostT) mi = max(mi, a.blk_ident[b * m + g]);
  mi = static_cast<unsigned>(block_max_ll<kCostT>(mi, red));
  const bool wide = flags & 1u, big = flags & 2u;
  bool decided = false;
  if (!wide) {
    if (!a.intra) {
      decided = true;
    } else if (a.order == DTB_ASCENDING && a.n % m == 0) {
      const int cap = a.n / m;
      const long long m_pos = m - static_cast<long long>(z) / cap;
      decided = static_cast<long long>(total) > static_cast<long long>(mi) * m_pos;
    }
  }
  if (decided) {
    for (int g = tid; g < m; g += kCostT) {
      const double l = static_cast<double>(a.blk_ident[b * m + g]);
      if (a.load_before) a.load_before[b * m + g] = l;
      if (a.load_after) a.load_after[b * m + g] = l;
    }
  } else if (!wide && a.order_out != nullptr && a.n <= kSmallN && m <= kSmallN) {
    __shared__ unsigned short s_tk[2 * kSmallN], s_sorted[kSmallN], s_flat[kSmallN];
    __shared__ unsigned s_load[kSmallN], s_blk[kSmallN];
    __shared__ unsigned char s_cnt[kSmallN];
    if (tid < 32) small_batch(a, b, s_tk, s_sorted, s_load, s_cnt, s_flat, s_blk);
    if (tid == 0) {  // decided and all outputs written
      a.wide_flag[b] = 0u;
      a.state[b] = kBatchDecided;
    }
    return;
  }
  // a batch the partition kernel runs on 32-bit arrays gets its 32-bit tokens
  // (input order) here, so everything that reads the input order's tokens
  // (the t_iter_before simulations) depends on this pass only and can run
  // concurrently with the partition kernel
  const bool route_wide = !decided && (wide || m > kNarrowGroups || (a.n & 7));
  if (route_wide && a.tok32_orig != nullptr) {
    const long long first = b * a.n;
    for (int i = tid; i < a.n; i += kCostT) {
      const long long gi = first + i;
      long long t = 0;
      for (int x = a.img_off[gi]; x < a.img_off[gi + 1]; ++x) t += a.img_tok[x];
      if (a.aud_off != nullptr)
        for (int x = a.aud_off[gi]; x < a.aud_off[gi + 1]; ++x) t += a.aud_tok[x];
      a.tok32_orig[first + i] = static_cast<int>(t);  // in [0, 2^31): checked by the cost pass
    }
  }
  if (tid == 0) {
    if (decided && a.kept) a.kept[b] = 0;
    a.wide_flag[b] = route_wide ? 1u : 0u;
    a.state[b] = decided ? kBatchDecided : route_wide ? kBatchWide : big ? kBatchSort : kBatchFast;
    if (!decided) a.list[1 + atomicAdd(a.list, 1u)] = static_cast<unsigned>(b);
  }
}

// Chunk c of the stream: batch b = c / cpb, samples [q0, q0 + qs) of it.
struct ChunkPos {
  long long b, s0;
  int q0, qs;
};
__device__ __forceinline__ ChunkPos chunk_pos(const CostArgs& a, unsigned c) {
  const unsigned b = a.div_cpb.div(c);  // grid < 2^31 chunks
  ChunkPos P;
  P.b = b;
  P.q0 = static_cast<int>(c - b * a.div_cpb.d) * kCostQ;
  P.qs = min(kCostQ, a.n - P.q0);
  P.s0 = P.b * a.n + P.q0;
  return P;
}

// Thread 0: bulk copies of chunk c's offsets (no bounds needed) ...
__device__ __forceinline__ void issue_offsets(const CostArgs& a, CostSmem& S, const ChunkPos& P) {
  const unsigned ob = 4u * static_cast<unsigned>(P.qs);
  const bool audio = a.aud_off != nullptr;
  mbar_arrive_expect_tx(&S.bar[0], ob * (audio ? 2u : 1u));
  bulk_g2s(S.io, a.img_off + P.s0, ob, &S.bar[0]);
  if (audio) bulk_g2s(S.ao, a.aud_off + P.s0, ob, &S.bar[0]);
}
// ... and of its token spans, given the chunk's bounds (lo, hi, alo, ahi)
// and the stream's token ends (tend, aend).
__device__ __forceinline__ void issue_tokens(const CostArgs& a, CostSmem& S, const ChunkPos& P, int lo,
                                             int hi, int alo, int ahi, int tend, int aend) {
  const bool audio = a.aud_off != nullptr;
  S.bnd[0] = lo, S.bnd[1] = hi, S.bnd[2] = alo, S.bnd[3] = ahi, S.bnd[4] = tend, S.bnd[5] = aend;
  const ChunkLayout L = chunk_layout(lo, hi, alo, ahi, tend, aend, audio);
  S.io[P.qs] = hi;  // the next boundary (outside the copied range)
  if (audio) S.ao[P.qs] = ahi;
  const unsigned ib = L.fits ? 4u * static_cast<unsigned>(L.ilen_tma) : 0u;
  const unsigned ab = L.fits ? 4u * static_cast<unsigned>(L.alen_tma) : 0u;
  if (L.fits) {  // slots the prefix sum reads but no copy writes
    for (int k = L.ilen; k < L.abase; ++k) S.tk[k] = 0;
    S.tk[L.abase + L.alen] = 0;
  }
  mbar_arrive_expect_tx(&S.bar[1], ib + ab);
  if (ib) bulk_g2s(S.tk, a.img_tok + L.fl, ib, &S.bar[1]);
  if (ab) bulk_g2s(S.tk + L.abase, a.aud_tok + L.afl, ab, &S.bar[1]);
}
struct Bounds {
  int lo, hi, alo, ahi;
};
__device__ __forceinline__ Bounds load_bounds(const CostArgs& a, const ChunkPos& P) {
  const bool audio = a.aud_off != nullptr;
  Bounds B;
  B.lo = __ldg(a.img_off + P.s0);
  B.hi = __ldg(a.img_off + P.s0 + P.qs);
  B.alo = audio ? __ldg(a.aud_off + P.s0) : 0;
  B.ahi = audio ? __ldg(a.aud_off + P.s0 + P.qs) : 0;
  return B;
}

// Everything after the copies are issued (all threads): wait for them
// (mbarrier phase `parity`), prefix sums, per-sample tokens, identity loads
// and order, per-batch statistics.  STAGED == false: per-sample sums straight
// from global memory (unaligned CSR).
template <bool STAGED>
__device__ __forceinline__ void cost_consume(const CostArgs& a, CostSmem& S, const ChunkPos& P,
                                             unsigned parity) {
  const int m = a.m, tid = threadIdx.x, lane = lane_id();
  const long long b = P.b, s0 = P.s0;
  const int q0 = P.q0, qs = P.qs;
  const bool audio = a.aud_off != nullptr;
  const int* io_s = STAGED ? S.io : a.img_off + s0;
  const int* ao_s = STAGED ? S.ao : (audio ? a.aud_off + s0 : nullptr);
  ChunkLayout L{};
  bool pre = false;
  if (STAGED) {
    L = chunk_layout(S.bnd[0], S.bnd[1], S.bnd[2], S.bnd[3], S.bnd[4], S.bnd[5], audio);
    mbar_wait(&S.bar[1], parity);
    if (L.fits) {
      if (L.ilen_tma < L.ilen || L.alen_tma < L.alen) {  // the stream's last tokens
        if (tid == 0) {
          for (int k = L.ilen_tma; k < L.ilen; ++k)
            S.tk[k] = L.fl + k < S.bnd[1] ? __ldg(a.img_tok + L.fl + k) : 0;
          for (int k = L.alen_tma; k < L.alen; ++k)
            S.tk[L.abase + k] = L.afl + k < S.bnd[3] ? __ldg(a.aud_tok + L.afl + k) : 0;
        }
        __syncthreads();
      }
      pre = !chunk_prefix(S.tk, L.len, S.tmp);
    }
    mbar_wait(&S.bar[0], parity);
  }
  // ---- per sample: thread t takes 4 consecutive samples per round (5
  // boundaries, one 8-byte token store)
  unsigned zeros = 0u, total = 0u;
  bool wide = false, big = false;
  unsigned short* tok_out = a.tok16 + s0;
  unsigned* blk = a.blk_ident + b * m;
  auto store4 = [&](int j0, unsigned* t4) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool ok = j0 + k < qs;
      const bool bad = t4[k] > 0x7fffu;  // negative sums mapped above 0x7fff
      wide |= ok && bad;
      const unsigned tok = ok ? (bad ? 0x7fffu : t4[k]) : 0u;
      t4[k] = tok;
      big |= tok >= 8192u;
      zeros += ok && tok == 0u;
    }
    if (j0 + 3 < qs && (reinterpret_cast<uintptr_t>(tok_out + j0) & 7u) == 0) {
      uint2 pk;
      pk.x = t4[0] | (t4[1] << 16);
      pk.y = t4[2] | (t4[3] << 16);
      *reinterpret_cast<uint2*>(tok_out + j0) = pk;
    } else {
      for (int k = 0; k < 4 && j0 + k < qs; ++k) tok_out[j0 + k] = static_cast<unsigned short>(t4[k]);
    }
  };
  if (STAGED && pre) {
    // a sample's sum is a difference of two prefix entries (image + audio);
    // so is a block's: the identity block loads and the chunk total come from
    // the prefix at block boundaries, not from per-sample reductions (a wide
    // batch's loads are recomputed by the partition kernel)
    const int* E = S.tk - L.fl;
    const int* F = S.tk + L.abase - L.afl;
    // every lane in range (qs % 4 == 0): a sample's clamp, the chunk's wide /
    // big flags and zero count from one running max and one compare per sample
    const bool al8 = (reinterpret_cast<uintptr_t>(tok_out) & 7u) == 0;
    unsigned mx = 0u;
    for (int j0 = 4 * tid; j0 < qs; j0 += 4 * kCostT) {  // qs % 4 == 0 when STAGED
      const int4 o = *reinterpret_cast<const int4*>(io_s + j0);
      DTB_CHECK(o.x - L.fl >= 0 && io_s[j0 + 4] - L.fl < L.abase);
      const int e0 = E[o.x], e1 = E[o.y], e2 = E[o.z], e3 = E[o.w], e4 = E[io_s[j0 + 4]];
      int v[4] = {e1 - e0, e2 - e1, e3 - e2, e4 - e3};
      if (audio) {
        const int4 p = *reinterpret_cast<const int4*>(ao_s + j0);
        DTB_CHECK(p.x - L.afl >= 0 && L.abase + ao_s[j0 + 4] - L.afl < L.len);
        const int f0 = F[p.x], f1 = F[p.y], f2 = F[p.z], f3 = F[p.w], f4 = F[ao_s[j0 + 4]];
        v[0] += f1 - f0, v[1] += f2 - f1, v[2] += f3 - f2, v[3] += f4 - f3;
      }
      unsigned t4[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const unsigned t = static_cast<unsigned>(v[k]);  // in [0, 0x7fff * len]
        mx = max(mx, t);
        zeros += t == 0u;
        t4[k] = min(t, 0x7fffu);
      }
      if (al8) {
        *reinterpret_cast<uint2*>(tok_out + j0) = make_uint2(t4[0] | (t4[1] << 16), t4[2] | (t4[3] << 16));
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) tok_out[j0 + k] = static_cast<unsigned short>(t4[k]);
      }
    }
    wide = mx > 0x7fffu;
    big = mx >= 8192u;  // a clamped token (0x7fff) is big too
    auto span = [&](int lo, int hi) {  // tokens of local samples [lo, hi)
      int t = E[io_s[hi]] - E[io_s[lo]];
      if (audio) t += F[ao_s[hi]] - F[ao_s[lo]];
      return 2u * static_cast<unsigned>(t);
    };
    const int per = static_cast<int>(a.div_pg.d);
    const int g0 = min(static_cast<int>(a.div_pg.div(static_cast<unsigned>(q0))), m - 1);
    const int g1 = min(static_cast<int>(a.div_pg.div(static_cast<unsigned>(q0 + qs - 1))), m - 1);
    for (int g = g0 + tid; g <= g1; g += kCostT) {
      const int lo = max(g * per, q0) - q0;
      const int hi = g == m - 1 ? qs : min((g + 1) * per, q0 + qs) - q0;
      const unsigned s = span(lo, hi);
      if (s) atomicAdd(blk + g, s);
    }
    if (tid == 0) total = span(0, qs);
  } else {
    for (int j0 = 4 * tid; j0 < qs; j0 += 4 * kCostT) {
      unsigned t4[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int j = j0 + k;
        long long t = 0;
        if (j < qs) {
          for (int x = io_s[j]; x < io_s[j + 1]; ++x) t += __ldg(a.img_tok + x);
          if (audio)
            for (int y = ao_s[j]; y < ao_s[j + 1]; ++y) t += __ldg(a.aud_tok + y);
        }
        // the 32-bit path orders 2 * tokens as u32 keys: a negative sum or one
        // of 2^31 or more is rejected (Sample::valid, src/core.cpp:97, never
        // admits negative tokens) instead of silently misordered
        if (t < 0 || t >= (1ll << 31)) dev_fail(a.err, E_COST_RANGE, static_cast<int>(b));
        t4[k] = t < 0 ? 0xffffffffu : t > 0xfffffffell ? 0xfffffffeu : static_cast<unsigned>(t);
      }
      store4(j0, t4);
      unsigned s2 = 0u;
#pragma unroll
      for (int k = 0; k < 4; ++k) s2 += 2u * t4[k];
      total += s2;
      // identity block loads: one atomic per warp when its 128 samples share
      // a block, else per sample
      const unsigned bl0 = min(a.div_pg.div(static_cast<unsigned>(q0 + j0)), static_cast<unsigned>(m - 1));
      const unsigned bl3 =
          min(a.div_pg.div(static_cast<unsigned>(q0 + min(j0 + 3, qs - 1))), static_cast<unsigned>(m - 1));
      const unsigned am = __activemask();
      const unsigned w0 = __shfl_sync(am, bl0, __ffs(am) - 1);
      if (__all_sync(am, bl0 == w0 && bl3 == w0)) {
        const unsigned sum = __reduce_add_sync(am, s2);
        if (lane == __ffs(am) - 1) atomicAdd(blk + w0, sum);
      } else if (bl0 == bl3) {
        atomicAdd(blk + bl0, s2);
      } else {
        for (int k = 0; k < 4 && j0 + k < qs; ++k)
          atomicAdd(blk + min(a.div_pg.div(static_cast<unsigned>(q0 + j0 + k)),
                              static_cast<unsigned>(m - 1)),
                    2u * t4[k]);
      }
    }
  }
  // ---- identity order for the chunk (kept batches are overwritten later)
  if (a.order_out != nullptr) {
    int* out = a.order_out + s0;
    if (aligned16(out) && (qs & 3) == 0) {
      for (int v = tid; v < (qs >> 2); v += kCostT)
        reinterpret_cast<int4*>(out)[v] =
            make_int4(q0 + 4 * v, q0 + 4 * v + 1, q0 + 4 * v + 2, q0 + 4 * v + 3);
    } else {
      for (int j = tid; j < qs; j += kCostT) out[j] = q0 + j;
    }
  }
  // ---- per-batch reductions; the last chunk of the batch finalizes it
  zeros = __reduce_add_sync(kFull, zeros);
  total = __reduce_add_sync(kFull, total);
  const unsigned fl = __reduce_or_sync(kFull, (wide ? 1u : 0u) | (big ? 2u : 0u));
  unsigned* st = a.bstat + 4 * b;
  if (lane == 0) {
    if (zeros) atomicAdd(st + 0, zeros);
    if (total) atomicAdd(st + 1, total);
    if (fl) atomicOr(st + 2, fl);
  }
}

// One chunk per CTA.
template <bool STAGED>
__device__ __forceinline__ void cost_chunk(const CostArgs& a, CostSmem& S) {
  const ChunkPos P = chunk_pos(a, blockIdx.x);
  if (threadIdx.x == 0) {
    if (STAGED) {  // the offsets need no bounds: their copy overlaps the bounds loads
      mbar_init(&S.bar[0], 1);
      mbar_init(&S.bar[1], 1);
      mbar_init_fence();
      issue_offsets(a, S, P);
    }
    const Bounds B = load_bounds(a, P);
    const long long last = a.n_batches * a.n;
    const int tend = STAGED ? __ldg(a.img_off + last) : 0;
    const int aend = STAGED && a.aud_off != nullptr ? __ldg(a.aud_off + last) : 0;
    if (STAGED) {
      issue_tokens(a, S, P, B.lo, B.hi, B.alo, B.ahi, tend, aend);
    } else {
      S.bnd[0] = B.lo, S.bnd[1] = B.hi, S.bnd[2] = B.alo, S.bnd[3] = B.ahi;
    }
  }
  __syncthreads();
  cost_consume<STAGED>(a, S, P, 0u);
}

__global__ void __launch_bounds__(kCostT, DTB_COST_MINB) cost_stream_kernel(const __grid_constant__ CostArgs a) {
  __shared__ CostSmem S;
  if (a.staged)
    cost_chunk<true>(a, S);
  else
    cost_chunk<false>(a, S);  // unaligned CSR: per-sample sums from global memory
}

size_t cost_scratch_bytes(long long n_batches, int m) {
  // blk_ident [nb * m], bstat [nb * 4], list [1 + nb], state [nb]
  return 4ull * (n_batches * (static_cast<unsigned long long>(m) + 4 + 2) + 1);
}

cudaError_t launch_cost_stream(const CostArgs& a, cudaStream_t stream) {
  const long long cpb = (a.n + kCostQ - 1) / kCostQ;
  const long long grid = a.n_batches * cpb;
  if (grid == 0) return cudaSuccess;
  // blk_ident, bstat and the list count are contiguous and zeroed here
  cudaError_t e = cudaMemsetAsync(a.blk_ident, 0, 4ull * (a.n_batches * (a.m + 4) + 1), stream);
  if (e != cudaSuccess) return e;
  // all of the unified L1 / shared memory as shared: eleven 20.6 KB chunk CTAs
  // per SM (token slots for 2.75 subsequences per sample: the mixed stream's
  // chunks peak at 2.30, the dense stream's at 2.60; a chunk that does not fit
  // sums its samples from global memory; ten 21.6 KB CTAs: 77.7 vs 76.3 µs)
  // (a persistent double-buffered variant — 5 CTAs of two stages per SM,
  // copies of chunk i + 1 in flight while chunk i computes — measured
  // slower: 95 µs at 128 threads, 101-105 µs at 256, vs 80 µs)
  // (set on every launch: the attribute is per device, like the partition
  // kernel's shared-memory opt-in)
  e = cudaFuncSetAttribute(cost_stream_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  CostArgs k = a;
  k.div_cpb = FastDiv::make(static_cast<unsigned>(cpb));
  cost_stream_kernel<<<static_cast<unsigned>(grid), kCostT, 0, stream>>>(k);
  e = launch_pdl(cost_finalize_kernel, dim3(static_cast<unsigned>(a.n_batches)), dim3(kCostT), 0,
                 stream, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace dtb

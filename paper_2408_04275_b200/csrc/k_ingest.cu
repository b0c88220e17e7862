// Trace ingest on the device: JSONL bytes -> sample CSR (SURVEY.md §8(f)
// row 3; reference: ingest_trace, src/workload.cpp:115-153).
//
// HBM-bound byte work, four launches over a byte buffer resident in HBM:
//   1. nl_count_kernel: 16-byte vector loads, newline bytes counted with
//      __vcmpeq4 + popc, one count per 16 KB tile;
//   2. (cub ExclusiveSum over the tile counts)
//   3. nl_write_kernel: the same pass again, block scans turn counts into the
//      ordered newline positions (= the getline line boundaries);
//   4. ingest_parse_kernel: one thread per line runs the validating parser
//      (csrc/jsonl.cuh) — status, text tokens, subsequence counts and the
//      byte offsets of the last image / audio arrays; the first failing line
//      is found with atomicMin (the reference throws at the first one);
//   5. (cub ExclusiveScan over (sample, image, audio) counts per line)
//   6. ingest_write_kernel: one thread per valid line writes its CSR row.
#include <cub/cub.cuh>

#include "jsonl.cuh"
#include "kernels.cuh"

namespace dtb {

namespace {

struct JDev {
  const unsigned char* p;
  int n;
  __device__ __forceinline__ int operator()(int i) const {
    return i < n ? static_cast<int>(__ldg(p + i)) : -1;
  }
};

constexpr int kNlT = 256;
constexpr int kNlRounds = 4;                        // 16-byte chunks per thread
constexpr long long kNlTile = 16ll * kNlT * kNlRounds;  // bytes per block

// newline mask (bit i of the result = byte i of the chunk is '\n')
__device__ __forceinline__ unsigned nl_mask16(const unsigned char* b, long long off, long long len,
                                              bool aligned) {
  unsigned w[4] = {0u, 0u, 0u, 0u};
  if (aligned && off + 16 <= len) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(b + off));
    w[0] = v.x;
    w[1] = v.y;
    w[2] = v.z;
    w[3] = v.w;
  } else {
    for (int k = 0; k < 16 && off + k < len; ++k)
      w[k >> 2] |= static_cast<unsigned>(__ldg(b + off + k)) << (8 * (k & 3));
  }
  unsigned m = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    unsigned e = __vcmpeq4(w[q], 0x0a0a0a0au);  // 0xff per equal byte
    // bytes beyond len were zero-filled, never '\n'
    e &= 0x80808080u;
    // compress the four byte flags to 4 bits
    const unsigned bits = ((e >> 7) & 1u) | ((e >> 14) & 2u) | ((e >> 21) & 4u) | ((e >> 28) & 8u);
    m |= bits << (4 * q);
  }
  return m;
}

__global__ void __launch_bounds__(kNlT)
nl_count_kernel(const unsigned char* __restrict__ b, long long len, unsigned* __restrict__ cnt) {
  const bool aligned = (reinterpret_cast<uintptr_t>(b) & 15) == 0;
  const long long tile = blockIdx.x * kNlTile;
  unsigned c = 0;
#pragma unroll
  for (int r = 0; r < kNlRounds; ++r) {
    const long long off = tile + 16ll * (r * kNlT + threadIdx.x);
    if (off < len) c += __popc(nl_mask16(b, off, len, aligned));
  }
  using BR = cub::BlockReduce<unsigned, kNlT>;
  __shared__ typename BR::TempStorage ts;
  const unsigned tot = BR(ts).Sum(c);
  if (threadIdx.x == 0) cnt[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kNlT)
nl_write_kernel(const unsigned char* __restrict__ b, long long len,
                const unsigned long long* __restrict__ base, long long* __restrict__ nl) {
  const bool aligned = (reinterpret_cast<uintptr_t>(b) & 15) == 0;
  const long long tile = blockIdx.x * kNlTile;
  using BS = cub::BlockScan<unsigned, kNlT>;
  __shared__ typename BS::TempStorage ts;
  unsigned long long at = base[blockIdx.x];
#pragma unroll
  for (int r = 0; r < kNlRounds; ++r) {
    const long long off = tile + 16ll * (r * kNlT + threadIdx.x);
    unsigned m = off < len ? nl_mask16(b, off, len, aligned) : 0u;
    unsigned ex, tot;
    BS(ts).ExclusiveSum(__popc(m), ex, tot);
    long long* dst = nl + at + ex;
    while (m) {
      const int k = __ffs(m) - 1;
      *dst++ = off + k;
      m &= m - 1;
    }
    at += tot;
    __syncthreads();
  }
}

struct Tri {
  int s, i, a;
};
struct TriSum {
  __device__ __forceinline__ Tri operator()(const Tri& x, const Tri& y) const {
    return Tri{x.s + y.s, x.i + y.i, x.a + y.a};
  }
};

__device__ __forceinline__ void line_span(const long long* nl, long long n_nl, long long len,
                                          long long k, long long* s, long long* e) {
  *s = k == 0 ? 0 : nl[k - 1] + 1;
  *e = k < n_nl ? nl[k] : len;
}

// A block's lines are contiguous in the buffer: the block stages the byte
// window of its 128 lines in shared memory with coalesced 16-byte loads, and
// each thread parses its line from there (bytes past the staged window, on
// rare long lines, are read from global memory).
constexpr int kPT = 128;
constexpr int kFastBit = 1 << 16;  // status flag: the line took the canonical fast path
constexpr int kStage = 16384;

struct JStaged {
  const unsigned char* sm;  // the line's first byte in the staged window
  int sn;                   // staged bytes of the line
  const unsigned char* g;   // the line in global memory
  int n;
  __device__ __forceinline__ int operator()(int i) const {
    return i < sn ? static_cast<int>(sm[i]) : i < n ? static_cast<int>(__ldg(g + i)) : -1;
  }
};

struct StageWin {
  long long w0, wn;
};

__device__ __forceinline__ StageWin stage_lines(const unsigned char* __restrict__ b, long long len,
                                                const long long* nl, long long n_nl,
                                                long long n_lines, unsigned char* sm) {
  __shared__ long long s_w0, s_wn;
  const long long k0 = blockIdx.x * static_cast<long long>(kPT);
  if (threadIdx.x == 0) {
    long long s, e, s1, e1;
    line_span(nl, n_nl, len, k0, &s, &e);
    const long long kl = min(k0 + kPT, n_lines) - 1;
    line_span(nl, n_nl, len, kl, &s1, &e1);
    s_w0 = s & ~15ll;
    s_wn = min(e1 - s_w0, static_cast<long long>(kStage));
  }
  __syncthreads();
  const long long w0 = s_w0, wn = s_wn;
  if ((reinterpret_cast<uintptr_t>(b) & 15) == 0) {
    for (long long v = threadIdx.x; 16 * v < wn; v += kPT) {
      const long long off = w0 + 16 * v;
      if (off + 16 <= len) {
        *reinterpret_cast<uint4*>(sm + 16 * v) = __ldg(reinterpret_cast<const uint4*>(b + off));
      } else {
        for (long long q = off; q < len; ++q) sm[q - w0] = __ldg(b + q);
      }
    }
  } else {
    for (long long q = threadIdx.x; q < wn; q += kPT) sm[q] = __ldg(b + w0 + q);
  }
  __syncthreads();
  return StageWin{w0, wn};
}

// a line entirely inside the staged window
struct JSmem {
  const unsigned char* sm;
  int n;
  __device__ __forceinline__ int operator()(int i) const {
    return i < n ? static_cast<int>(sm[i]) : -1;
  }
};

__device__ __forceinline__ JStaged staged_line(const unsigned char* b, const unsigned char* sm,
                                               StageWin w, long long s, long long e) {
  const long long rel = s - w.w0;
  long long sn = w.wn - rel;
  sn = sn < 0 ? 0 : sn > e - s ? e - s : sn;
  return JStaged{sm + (rel < w.wn ? rel : 0), static_cast<int>(sn), b + s, static_cast<int>(e - s)};
}

__global__ void __launch_bounds__(kPT)
ingest_parse_kernel(const unsigned char* __restrict__ b, long long len,
                    const long long* __restrict__ nl, long long n_nl, long long n_lines,
                    long long cap, IngestLines L, unsigned long long* __restrict__ first_bad) {
  __shared__ alignas(16) unsigned char sm[kStage];
  const StageWin w = stage_lines(b, len, nl, n_nl, n_lines, sm);
  const long long k = blockIdx.x * static_cast<long long>(kPT) + threadIdx.x;
  if (k >= n_lines) return;
  long long s, e;
  line_span(nl, n_nl, len, k, &s, &e);
  JLine r;
  bool fast = false;
  if (e - s > 0x7fffffffll) {
    r.status = J_UNSUPPORTED;
    r.reason = JR_INT32;
    r.text = 0;
    r.n_img = r.n_aud = 0;
    r.img_at = r.aud_at = -1;
  } else {
    const JStaged at = staged_line(b, sm, w, s, e);
    r = at.sn == at.n ? j_parse_record(JSmem{at.sm, at.n}, at.n, cap, &fast)
                      : j_parse_record(at, at.n, cap, &fast);
  }
  L.status[k] = r.status | (r.reason << 8) | (fast ? kFastBit : 0);
  const bool ok = r.status == J_OK;
  L.text[k] = r.text;
  L.img_at[k] = r.img_at;
  L.aud_at[k] = r.aud_at;
  reinterpret_cast<Tri*>(L.counts)[k] = Tri{ok ? 1 : 0, ok ? r.n_img : 0, ok ? r.n_aud : 0};
  if (r.status >= J_PARSE) atomicMin(first_bad, static_cast<unsigned long long>(k));
}

__global__ void __launch_bounds__(kPT)
ingest_write_kernel(const unsigned char* __restrict__ b, long long len,
                    const long long* __restrict__ nl, long long n_nl, long long n_lines,
                    IngestLines L, IngestOut o) {
  __shared__ alignas(16) unsigned char sm[kStage];
  const long long k = blockIdx.x * static_cast<long long>(kPT) + threadIdx.x;
  const Tri* sc = reinterpret_cast<const Tri*>(L.scan);
  if (k == 0) {
    const Tri t = sc[n_lines];
    o.image_offsets[t.s] = t.i;
    o.audio_offsets[t.s] = t.a;
  }
  if (n_lines == 0) return;
  const StageWin w = stage_lines(b, len, nl, n_nl, n_lines, sm);
  if (k >= n_lines || (L.status[k] & 0xffff) != J_OK) return;
  const bool fast = (L.status[k] & kFastBit) != 0;
  long long s, e;
  line_span(nl, n_nl, len, k, &s, &e);
  const JStaged at = staged_line(b, sm, w, s, e);
  const Tri t = sc[k];
  o.text_tokens[t.s] = static_cast<int>(L.text[k]);
  o.image_offsets[t.s] = t.i;
  o.audio_offsets[t.s] = t.a;
  if (fast && at.sn == at.n) {
    const JSmem as{at.sm, at.n};
    if (L.img_at[k] >= 0) j_write_array_fast(as, L.img_at[k], o.image_tokens + t.i);
    if (L.aud_at[k] >= 0) j_write_array_fast(as, L.aud_at[k], o.audio_tokens + t.a);
  } else if (fast) {
    if (L.img_at[k] >= 0) j_write_array_fast(at, L.img_at[k], o.image_tokens + t.i);
    if (L.aud_at[k] >= 0) j_write_array_fast(at, L.aud_at[k], o.audio_tokens + t.a);
  } else {
    if (L.img_at[k] >= 0) j_write_array(at, L.img_at[k], o.image_tokens + t.i);
    if (L.aud_at[k] >= 0) j_write_array(at, L.aud_at[k], o.audio_tokens + t.a);
  }
}

}  // namespace

// ------------------------------------------------------------------ host glue
size_t ingest_lines_scratch(long long len) {
  const long long tiles = (len + kNlTile - 1) / kNlTile;
  size_t temp = 0, t2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, temp, static_cast<unsigned*>(nullptr),
                                static_cast<unsigned long long*>(nullptr),
                                static_cast<int>(tiles > 0 ? tiles : 1));
  cub::DeviceScan::ExclusiveScan(nullptr, t2, static_cast<Tri*>(nullptr), static_cast<Tri*>(nullptr),
                                 TriSum(), Tri{0, 0, 0}, 1 << 30);
  return (temp > t2 ? temp : t2) + 4096 + 12ull * (tiles + 1);
}

// scratch: tile counts | tile bases | cub temp
static void nl_layout(void* scratch, long long tiles, unsigned** cnt, unsigned long long** base,
                      char** temp) {
  char* p = static_cast<char*>(scratch);
  *cnt = reinterpret_cast<unsigned*>(p);
  *base = reinterpret_cast<unsigned long long*>(p + ((4 * (tiles + 1) + 255) & ~255ll));
  *temp = reinterpret_cast<char*>(*base) + ((8 * (tiles + 1) + 255) & ~255ll);
}

cudaError_t launch_nl_count(const unsigned char* b, long long len, void* scratch,
                            size_t scratch_bytes, long long* n_nl, cudaStream_t st) {
  const long long tiles = (len + kNlTile - 1) / kNlTile;
  *n_nl = 0;
  if (tiles == 0) return cudaSuccess;
  unsigned* cnt;
  unsigned long long* base;
  char* temp;
  nl_layout(scratch, tiles, &cnt, &base, &temp);
  size_t tb = scratch_bytes - static_cast<size_t>(temp - static_cast<char*>(scratch));
  nl_count_kernel<<<static_cast<unsigned>(tiles), kNlT, 0, st>>>(b, len, cnt);
  cudaError_t e = cub::DeviceScan::ExclusiveSum(temp, tb, cnt, base, static_cast<int>(tiles), st);
  if (e != cudaSuccess) return e;
  unsigned long long last_base = 0;
  unsigned last_cnt = 0;
  e = cudaMemcpyAsync(&last_base, base + tiles - 1, 8, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&last_cnt, cnt + tiles - 1, 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return e;
  *n_nl = static_cast<long long>(last_base + last_cnt);
  return cudaGetLastError();
}

cudaError_t launch_nl_write(const unsigned char* b, long long len, void* scratch, long long* nl,
                            cudaStream_t st) {
  const long long tiles = (len + kNlTile - 1) / kNlTile;
  if (tiles == 0) return cudaSuccess;
  unsigned* cnt;
  unsigned long long* base;
  char* temp;
  nl_layout(scratch, tiles, &cnt, &base, &temp);
  nl_write_kernel<<<static_cast<unsigned>(tiles), kNlT, 0, st>>>(b, len, base, nl);
  return cudaGetLastError();
}

cudaError_t launch_ingest_parse(const unsigned char* b, long long len, const long long* nl,
                                long long n_nl, long long n_lines, long long cap,
                                const IngestLines& L, unsigned long long* first_bad, void* scratch,
                                size_t scratch_bytes, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>((n_lines + kPT - 1) / kPT);
  if (n_lines > 0)
    ingest_parse_kernel<<<grid, kPT, 0, st>>>(b, len, nl, n_nl, n_lines, cap, L, first_bad);
  // counts[n_lines] = 0, so scan[n_lines] = totals
  cudaError_t e = cudaMemsetAsync(reinterpret_cast<Tri*>(L.counts) + n_lines, 0, sizeof(Tri), st);
  if (e != cudaSuccess) return e;
  size_t tb = scratch_bytes;
  e = cub::DeviceScan::ExclusiveScan(scratch, tb, reinterpret_cast<const Tri*>(L.counts),
                                     reinterpret_cast<Tri*>(L.scan), TriSum(), Tri{0, 0, 0},
                                     static_cast<int>(n_lines + 1), st);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_ingest_write(const unsigned char* b, long long len, const long long* nl,
                                long long n_nl, long long n_lines, const IngestLines& L,
                                const IngestOut& o, cudaStream_t st) {
  const long long grid = (n_lines + kPT - 1) / kPT;
  ingest_write_kernel<<<static_cast<unsigned>(grid > 0 ? grid : 1), kPT, 0, st>>>(
      b, len, nl, n_nl, n_lines, L, o);
  return cudaGetLastError();
}

}  // namespace dtb

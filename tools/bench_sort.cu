// Microbenchmark of the fused kernel's block radix-sort passes (debug tool):
// 2 CTAs per SM, each sorts 16384 u16 indices by random 15-bit keys; reports
// SM cycles per pass (CTA thread 0, clock64) for each variant.
#include <cstdio>
#include <cuda_runtime.h>
#include "block_ops.cuh"
using namespace dtb;
namespace dtb {
template <int T, int ITEMS, int RB, bool SWZ, typename DigitFn>
__device__ void tile_pass_prof(unsigned short* idx, const unsigned short* key,
                                  const DigitFn& digit, unsigned short* cnt, int* scan_tmp, long long* ph) {
  constexpr int D = 1 << RB;
  constexpr int WORDS = D * T / 2;
  constexpr int G = 4;
  constexpr int W = T / 32;
  static_assert(ITEMS % G == 0 && WORDS % (32 * W) == 0, "shape");
  const int t = threadIdx.x, lane = lane_id(), w = warp_id();
  auto* cntw = reinterpret_cast<unsigned*>(cnt);
  for (int i = t; i < WORDS; i += T) cntw[i] = 0u;
  __syncthreads();
  long long c0 = clock64();
  const uint2* mine = reinterpret_cast<const uint2*>(idx + t * ITEMS);
  // histogram straight from shared memory
#pragma unroll 1
  for (int g = 0; g < ITEMS / G; ++g) {
    const uint2 p = mine[g];
    const unsigned v[G] = {p.x & 0xffffu, p.x >> 16, p.y & 0xffffu, p.y >> 16};
    unsigned d[G];
#pragma unroll
    for (int j = 0; j < G; ++j) d[j] = static_cast<unsigned>(digit(key[v[j]]));
#pragma unroll
    for (int j = 0; j < G; ++j) {
      unsigned short* c = cnt + d[j] * T + t;
      *c = static_cast<unsigned short>(*c + 1);
    }
  }
  // this thread's items, two per register, held across the scan (the
  // scatter is in place)
  uint2 it[ITEMS / G];
#pragma unroll
  for (int g = 0; g < ITEMS / G; ++g) {
    it[g] = mine[g];
    asm volatile("" : "+r"(it[g].x), "+r"(it[g].y));  // keep them packed
  }
  __syncthreads();
  long long c1 = clock64();
  // exclusive scan over (d, t) = word order: warp w scans its WORDS / W
  // consecutive words 32 at a time (conflict-free), then warps combine
  constexpr int SPAN = WORDS / W;
  int carry = 0;
#pragma unroll 1
  for (int q = 0; q < SPAN; q += 32) {
    const unsigned x = cntw[w * SPAN + q + lane];
    int s = static_cast<int>((x & 0xffffu) + (x >> 16));
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, s, o);
      if (lane >= o) s += y;
    }
    carry += __shfl_sync(kFull, s, 31);
  }
  if (lane == 0) scan_tmp[w] = carry;
  __syncthreads();
  int base = 0;
  for (int i = 0; i < w; ++i) base += scan_tmp[i];
#pragma unroll 1
  for (int q = 0; q < SPAN; q += 32) {
    const int widx = w * SPAN + q + lane;
    const unsigned x = cntw[widx];
    const int lo = static_cast<int>(x & 0xffffu), hi = static_cast<int>(x >> 16);
    int s = lo + hi;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, s, o);
      if (lane >= o) s += y;
    }
    const int ex = base + s - (lo + hi);
    cntw[widx] = static_cast<unsigned>(ex) | (static_cast<unsigned>(ex + lo) << 16);
    base += __shfl_sync(kFull, s, 31);
  }
  __syncthreads();
  long long c2 = clock64();
#pragma unroll
  for (int g = 0; g < ITEMS / G; ++g) {
    const unsigned v[G] = {it[g].x & 0xffffu, it[g].x >> 16, it[g].y & 0xffffu, it[g].y >> 16};
    unsigned d[G];
#pragma unroll
    for (int j = 0; j < G; ++j) d[j] = static_cast<unsigned>(digit(key[v[j]]));
#pragma unroll
    for (int j = 0; j < G; ++j) {
      unsigned short* c = cnt + d[j] * T + t;
      const int dst = *c;
      *c = static_cast<unsigned short>(dst + 1);
      idx[SWZ ? swz(dst) : dst] = static_cast<unsigned short>(v[j]);
    }
  }
  __syncthreads();
  long long c3 = clock64();
  if (threadIdx.x == 0) { ph[0] += c1 - c0; ph[1] += c2 - c1; ph[2] += c3 - c2; }
}

}

constexpr int T = 384, ITEMS = 44, SLOTS = T * ITEMS, N = 16384;
struct Smem {
  unsigned short key[SLOTS];
  alignas(16) unsigned short idx[SLOTS];
  alignas(16) unsigned short aux[SLOTS];
  int cnt[128 * (T / 32) + 1];
  int tmp[T / 32 + 3];
};
template <int VARIANT>
__global__ void __launch_bounds__(T, 2) k(const unsigned short* keys, long long* cyc, int bits) {
  extern __shared__ __align__(16) unsigned char raw[];
  Smem& S = *reinterpret_cast<Smem*>(raw);
  for (int i = threadIdx.x; i < SLOTS; i += T) {
    S.key[i] = i < N ? keys[blockIdx.x * N + i] : 0xffff;
    S.idx[i] = i;
  }
  __syncthreads();
  long long ph[3] = {0, 0, 0};
  long long t0 = clock64();
  constexpr int RB = VARIANT == 0 ? 5 : 7;
  for (int sh = 0; sh < bits; sh += RB) {
    const unsigned mask = (1u << min(RB, bits - sh)) - 1u;
    auto dig = [&](unsigned kk) { return (kk >> sh) & mask; };
    if (VARIANT == 0)
      tile_pass_blocked<T, ITEMS, 5, false>(S.idx, S.key, dig, reinterpret_cast<unsigned*>(S.aux), S.tmp);
    else
      tile_pass_idx16<T, ITEMS, 7, false>(S.idx, S.key, dig, S.cnt, S.tmp, S.aux);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[blockIdx.x] = t1 - t0; if (VARIANT == 0 && blockIdx.x == 0) printf("phases hist %lld scan %lld scatter %lld\n", ph[0], ph[1], ph[2]); }
  // check sortedness
  for (int i = threadIdx.x + 1; i < N; i += T)
    if ((S.key[S.idx[i - 1]] & ((1 << bits) - 1)) > (S.key[S.idx[i]] & ((1 << bits) - 1))) cyc[blockIdx.x] = -1;
}
int main() {
  const int grid = 296;
  unsigned short* h = new unsigned short[grid * N];
  unsigned s = 12345;
  for (int i = 0; i < grid * N; ++i) { s = s * 1664525u + 1013904223u; h[i] = (s >> 9) & 0x1fff; }
  unsigned short* d; long long* c;
  cudaMalloc(&d, 2ull * grid * N); cudaMalloc(&c, 8 * grid);
  cudaMemcpy(d, h, 2ull * grid * N, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(Smem));
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(Smem));
  long long hc[296];
  for (int v = 0; v < 2; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      if (v == 0) k<0><<<grid, T, sizeof(Smem)>>>(d, c, 13);
      else k<1><<<grid, T, sizeof(Smem)>>>(d, c, 13);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      cudaMemcpy(hc, c, 8 * grid, cudaMemcpyDeviceToHost);
      long long mx = 0, bad = 0; double avg = 0;
      for (int i = 0; i < grid; ++i) { if (hc[i] < 0) bad++; mx = hc[i] > mx ? hc[i] : mx; avg += hc[i]; }
      if (rep) printf("variant %s: kernel %.1f us, CTA sort cycles avg %.0f max %lld (%s) smem %zu err %s\n",
                      v ? "warp-striped ballot RB7" : "blocked RB5", ms * 1e3, avg / grid, mx,
                      bad ? "UNSORTED" : "sorted", sizeof(Smem), cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}

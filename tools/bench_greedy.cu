// Microbenchmark of the equal-count greedy variants on one descending-sorted
// 16,384-item batch, m = 128 (debug tool): SM cycles (clock64) of the one-warp
// greedy (greedy_warp.cuh), of its 128-key warp sort alone, and of the
// 8-warp block version (greedy_fused.cuh); checks both agree.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include "greedy_fused.cuh"
#include "greedy_warp.cuh"
using namespace dtb;

struct Sm {
  FusedGreedySmem G;
  WarpGreedySmem WG;
  int tmp[64];
  long long tmpll[64];
  unsigned short out[16384 + 512];
  unsigned short sz[16384];
};

__global__ void k_greedy(const unsigned short* sizes, int n, int m, int zc, int which,
                         long long* cyc, unsigned* gl, int* gc, unsigned short* out) {
  extern __shared__ __align__(16) unsigned char raw[];
  Sm& S = *reinterpret_cast<Sm*>(raw);
  for (int i = threadIdx.x; i < n; i += blockDim.x) S.sz[i] = sizes[i];
  __syncthreads();
  const int cap = (n + m - 1) / m, capP = ((cap + 1) | 3) - 1;
  auto size_at = [&](int k) -> unsigned { return 2u * S.sz[k]; };
  auto emit = [&](int k, int g, int slot) { S.out[g * capP + slot] = (unsigned short)k; };
  const int z0 = which >= 3 ? 0 : n - zc, z1 = which >= 3 ? (which == 4 ? 0 : zc) : n;
  long long c0 = clock64();
  if (which == 3 || which == 4) {  // ascending (sizes reversed: read from the end)
    auto size_asc = [&](int k) -> unsigned { return 2u * S.sz[n - 1 - k]; };
    if (threadIdx.x < 256) greedy_fused<256, true, 1>(n, m, cap, z0, z1, size_asc, emit, S.G, S.tmp, S.tmpll);
  } else if (which == 5) {
    if (threadIdx.x < 256) {
      int tot = 0, acc = 0;
      for (int it = 0; it < 100; ++it) acc += block_excl_scan<256, 1>(threadIdx.x + it, S.tmp, &tot);
      if (acc == 12345) cyc[7] = tot;
    }
  } else if (which == 6) {
    if (threadIdx.x < 256)
      for (int it = 0; it < 100; ++it) bar_sync<1, 256>();
  } else if (which == 0) {
    if (threadIdx.x < 32) greedy_warp<unsigned>(n, m, cap, z0, z1, size_at, emit, S.WG, S.G.gload, S.G.gcnt);
  } else if (which == 1) {
    if (threadIdx.x < 256) greedy_fused<256, false, 1>(n, m, cap, z0, z1, size_at, emit, S.G, S.tmp, S.tmpll);
  } else {
    if (threadIdx.x < 32) {
      unsigned v[4];
      for (int e = 0; e < 4; ++e) v[e] = (threadIdx.x * 2654435761u + e * 97u) & 0xffffu;
      for (int it = 0; it < 100; ++it) { wg_sort128(v); v[0] ^= it; }
      if (v[0] == 12345) cyc[5] = 1;
    }
  }
  __syncthreads();
  long long c1 = clock64();
  if (threadIdx.x == 0) cyc[which] = c1 - c0;
  if (which >= 3) return;
  for (int g = threadIdx.x; g < m; g += blockDim.x) { gl[which * 128 + g] = S.G.gload[g]; gc[which * 128 + g] = S.G.gcnt[g]; }
  for (int i = threadIdx.x; i < m * capP; i += blockDim.x) out[which * 17000 + i] = S.out[i];
}

int main() {
  const int n = 16384, m = 128;
  std::vector<unsigned short> h(n);
  srand(7);
  int zc = 0;
  for (int i = 0; i < n; ++i) {
    int r = rand() % 100;
    h[i] = r < 25 ? 0 : (unsigned short)(200 + rand() % 3000);
  }
  std::sort(h.begin(), h.end(), [](unsigned short a, unsigned short b) { return a > b; });
  for (int i = 0; i < n; ++i) zc += h[i] == 0;
  unsigned short* d; long long* cyc; unsigned* gl; int* gc; unsigned short* out;
  cudaMalloc(&d, 2 * n); cudaMalloc(&cyc, 128); cudaMalloc(&gl, 4 * 3 * 128); cudaMalloc(&gc, 4 * 3 * 128);
  cudaMalloc(&out, 2 * 3 * 17000);
  cudaMemcpy(d, h.data(), 2 * n, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_greedy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Sm));
  for (int rep = 0; rep < 3; ++rep)
    for (int which = 0; which < 7; ++which)
      k_greedy<<<1, 1024, sizeof(Sm)>>>(d, n, m, zc, which, cyc, gl, gc, out);
  cudaError_t e = cudaDeviceSynchronize();
  long long c[16];
  cudaMemcpy(c, cyc, 128, cudaMemcpyDeviceToHost);
  std::vector<unsigned> hg(3 * 128); std::vector<int> hc(3 * 128); std::vector<unsigned short> ho(3 * 17000);
  cudaMemcpy(hg.data(), gl, 4 * 3 * 128, cudaMemcpyDeviceToHost);
  cudaMemcpy(hc.data(), gc, 4 * 3 * 128, cudaMemcpyDeviceToHost);
  cudaMemcpy(ho.data(), out, 2 * 3 * 17000, cudaMemcpyDeviceToHost);
  bool same = true;
  for (int g = 0; g < m; ++g) same &= hg[g] == hg[128 + g] && hc[g] == hc[128 + g];
  for (int i = 0; i < 17000; ++i) same &= ho[i] == ho[17000 + i];
  printf("{\"err\": \"%s\", \"zeros\": %d, \"warp_greedy_cycles\": %lld, \"block_greedy_cycles\": %lld, "
         "\"sort128_cycles_per_call\": %.1f, \"agree\": %s, \"asc_block_greedy_cycles\": %lld, "
         "\"asc_block_greedy_no_zero_run_cycles\": %lld, \"block_excl_scan_256_cycles\": %.1f, "
         "\"bar_sync_256_cycles\": %.1f}\n", cudaGetErrorString(e), zc, c[0], c[1],
         c[2] / 100.0, same ? "true" : "false", c[3], c[4], c[5] / 100.0, c[6] / 100.0);
  return 0;
}

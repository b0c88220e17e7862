// Multi-GPU exchange of the reorder stream's output: every
// rank reorders a contiguous range of global batches and the concatenated
// ordering must end up on every rank.  Each rank holds a replica buffer of
// the whole ordering (u16 in-batch sample indices: a global batch has at most
// 16,384 samples, so half the bytes of int32) opened by every peer over CUDA
// IPC; this kernel stores the rank's shard straight into all replicas over
// NVLink (peer stores, 16 bytes per store) and ends with a flag barrier over
// the group in device memory, so the stream that runs it continues only once
// every rank's shard has arrived everywhere.
#include <algorithm>

#include "kernels.cuh"

namespace dtb {

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(256) peer_broadcast_kernel(const __grid_constant__ PeerBcast a) {
  // this phase's batches (a packet of 8 samples never straddles two batches:
  // the packed path requires n % 8 == 0)
  auto mine = [&](long long i) -> bool {
    if (a.phase == 0) return true;
    const bool decided = a.state[i / a.n] == kBatchDecided;
    return a.phase == 1 ? decided : !decided;
  };
  // ---- data: 8 samples per thread and step (two 16-byte loads, one 16-byte
  // store per replica)
  const long long n8 = a.aligned ? a.count >> 3 : 0;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  const long long t0 = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  for (long long q = t0; q < n8; q += stride) {
    if (!mine(8 * q)) continue;
    const int4 x0 = reinterpret_cast<const int4*>(a.src)[2 * q];
    const int4 x1 = reinterpret_cast<const int4*>(a.src)[2 * q + 1];
    const uint4 v = make_uint4(static_cast<unsigned>(x0.x) | (static_cast<unsigned>(x0.y) << 16),
                               static_cast<unsigned>(x0.z) | (static_cast<unsigned>(x0.w) << 16),
                               static_cast<unsigned>(x1.x) | (static_cast<unsigned>(x1.y) << 16),
                               static_cast<unsigned>(x1.z) | (static_cast<unsigned>(x1.w) << 16));
#pragma unroll 1
    for (int p = 0; p < a.world; ++p) reinterpret_cast<uint4*>(a.dst[p])[q] = v;
  }
  for (long long i = (n8 << 3) + t0; i < a.count; i += stride)  // tail / unaligned
    if (mine(i))
      for (int p = 0; p < a.world; ++p) a.dst[p][i] = static_cast<unsigned short>(a.src[i]);
  if (a.phase == 1) return;  // the barrier closes phase 2
  // ---- barrier: every thread's peer stores precede its CTA's arrival; the
  // last CTA releases this rank's flag in every replica and acquires every
  // peer's flag in the local one
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(a.done, 1u);
    if (prev == gridDim.x - 1) {
      const unsigned ep = *a.epoch + 1;  // every rank counts its calls the same way
      *a.epoch = ep;
      __threadfence_system();
      for (int p = 0; p < a.world; ++p) st_release_sys(a.flags[p] + a.rank, ep);
      for (int p = 0; p < a.world; ++p)
        while (static_cast<int>(ld_acquire_sys(a.flags_local + p) - ep) < 0) {
        }
    }
  }
}

cudaError_t launch_peer_broadcast(const PeerBcast& a, cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(a.done, 0, sizeof(unsigned), stream);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long n8 = a.count >> 3;
  const long long want = (n8 + 255) / 256;
  const unsigned grid = static_cast<unsigned>(std::max<long long>(1, std::min<long long>(want, 2ll * sms)));
  peer_broadcast_kernel<<<grid, 256, 0, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace dtb

// Programmatic dependent launch (PDL): a kernel launched with
// launch_pdl may start while the previous kernel of its stream drains (its
// CTAs fill the SMs the predecessor frees, its launch latency overlaps the
// predecessor's tail); pdl_wait() — griddepcontrol.wait, a no-op without PDL —
// blocks until the predecessor's memory is visible, so a kernel calls it
// before its first read of a predecessor's output.  Kept in CUDA graph
// captures as programmatic edges.
#pragma once

#include <cuda_runtime.h>

namespace dtb {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace dtb

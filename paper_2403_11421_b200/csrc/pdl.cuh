// Programmatic dependent launch for the decode step's kernel chain: every
// kernel signals `launch_dependents` on entry and calls `pdl_wait()` after
// its global-memory-free prologue (barrier init, TMEM alloc, smem zero-fill)
// and before it reads anything a previous kernel wrote. griddepcontrol.wait
// returns once the preceding grid has completed and its writes are visible,
// so the ordering of a plain stream launch is kept while the next kernel's
// launch latency and prologue overlap the previous kernel's tail. On a launch
// without the attribute both instructions are no-ops.
#pragma once

#include <cuda_runtime.h>

#include "sd_common.h"

namespace sd {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() { return tuning().pdl != 0; }

// cudaLaunchKernelEx with the programmatic-serialization attribute (and an
// optional cluster dimension)
template <typename... K, typename... A>
cudaError_t launch_pdl(void (*kernel)(K...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, unsigned cluster,
                       A&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (cluster > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<A&&>(args)...);
}

}  // namespace sd

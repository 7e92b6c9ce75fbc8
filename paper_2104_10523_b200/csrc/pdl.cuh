// Programmatic dependent launch (PDL) for every kernel of the hot path.
//
// A slice program is a chain of ~30 dependent kernels per slice, most
// of them short; without PDL each boundary costs a full drain + launch + prologue.  Every
// kernel is launched with programmaticStreamSerializationAllowed and begins with
// pdl_wait() (griddepcontrol.wait: returns once the preceding grid of the stream has
// completed and its memory is visible; a no-op when launched without the attribute), so a
// kernel's launch and the CTA rasterisation overlap its predecessor's tail.  pdl_wait() is
// the FIRST statement of every kernel (before any early return), which makes the ordering
// transitive along the chain: grid i+1 cannot complete before grid i has.
// TNQVM_PDL=0 launches without the attribute (the kernels are unchanged).
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace tnqvm {
namespace dev {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// SM count of the CURRENT device (cached per device ordinal)
inline int sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cache[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

inline bool pdl_enabled() {
  static const int on = getenv("TNQVM_PDL") ? atoi(getenv("TNQVM_PDL")) : 1;
  return on != 0;
}

// kernel<<<grid, block, smem, st>>>(args...) with the PDL attribute
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// the same with a thread-block cluster of `cx` CTAs along x (CTA pairs for cta_group::2)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                      unsigned cx, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cx;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace dev
}  // namespace tnqvm

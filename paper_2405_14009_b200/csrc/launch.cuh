// launch.cuh — kernel launch with Programmatic Dependent Launch (PDL).
//
// Every libslip kernel starts its dependent work after ptx::grid_dep_wait(), so it may be
// launched with cudaLaunchAttributeProgrammaticStreamSerialization: its CTAs become
// resident and run their prologue (barrier init, TMEM allocation, tensor-map prefetch)
// while the previous kernel in the stream drains, instead of after a full launch gap.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>

namespace slip {

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       int cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int n = 0;
  attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  static const bool no_pdl = std::getenv("SLIP_NO_PDL") != nullptr;  // debugging aid
  attr[n].val.programmaticStreamSerializationAllowed = no_pdl ? 0 : 1;
  ++n;
  if (cluster_x > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster_x;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace slip

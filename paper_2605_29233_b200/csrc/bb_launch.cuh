// Host-side kernel launch with programmatic dependent launch (PDL) enabled.
#pragma once
#include <cuda_runtime.h>
#include <stdlib.h>

#include <utility>

namespace bb {

inline bool pdl_enabled() {
  static const int on = [] {
    const char* e = getenv("BB_PDL");
    return e == nullptr ? 1 : atoi(e);
  }();
  return on != 0;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace bb

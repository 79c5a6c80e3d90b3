// Kernel launch with programmatic dependent launch (PDL) enabled: the kernel
// may begin (prologue, smem / TMEM setup) while the previous kernel on the
// stream finishes; it orders its global-memory work with griddepcontrol.wait.
// Captured into CUDA graphs as programmatic dependency edges.
#pragma once

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>
#include <utility>

namespace dpl {

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
  if (e != cudaSuccess) throw std::runtime_error(std::string("dpl: launch failed: ") + cudaGetErrorString(e));
}

}  // namespace dpl

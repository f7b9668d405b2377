// fuseplan-b200 — programmatic-dependent-launch helper for the small kernels.
//
// A kernel launched through launch_pdl() may start while its stream
// predecessor is still running (once every CTA of the predecessor executed
// griddepcontrol.launch_dependents), so its CTAs are resident and past their
// prologue when the predecessor ends. Such a kernel MUST execute pdl_wait()
// (griddepcontrol.wait) before it touches anything a predecessor kernel wrote;
// reads of data uploaded before the first kernel of the chain are safe earlier.
#pragma once

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

namespace fpk {

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
  if (e != cudaSuccess) throw std::runtime_error(std::string("kernel launch: ") + cudaGetErrorString(e));
}

}  // namespace fpk

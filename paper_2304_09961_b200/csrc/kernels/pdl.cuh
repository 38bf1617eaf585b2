// Programmatic dependent launch (PDL) for the stream-ordered layer kernels.
//
// Every kernel of a step is launched with programmatic stream serialization,
// so kernel k+1 is scheduled while kernel k drains (its CTAs run their
// prologue -- barrier init, TMEM allocation, tensor-map prefetch, weight
// loads -- on SMs that k has released) and park in griddepcontrol.wait until
// k has completed and its memory is visible. Rules that keep this exact:
//   * every kernel issues launch_dependents() at entry, by every CTA, so a
//     dependent grid is only scheduled once all CTAs of the current grid are
//     resident (dependents can never starve it of SMs);
//   * every kernel calls wait() before it reads or writes anything another
//     kernel produces or consumes (activations, blob tables, split-K
//     workspace); only immutable inputs (weights, bias) may be touched before.
//     Since every kernel waits, completion stays ordered along the stream and
//     kernel k+2 transitively sees kernel k.
// Outside a PDL launch both instructions are no-ops. BS_PDL=0 disables it.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace bs200 {
namespace pdl {

__device__ __forceinline__ void launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

inline bool enabled() {
  static const bool on = [] {
    const char* e = std::getenv("BS_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
cudaError_t launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                   Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace pdl
}  // namespace bs200

// Programmatic dependent launch (PDL) for the stream-ordered layer kernels.
//
// Every kernel of a step is launched with programmatic stream serialization,
// so kernel k+1 is scheduled while kernel k drains (its CTAs run their
// prologue -- barrier init, TMEM allocation, tensor-map prefetch, weight
// loads -- on SMs that k has released) and park in griddepcontrol.wait until
// k has completed and its memory is visible. Rules that keep this exact:
//   * every kernel issues launch_dependents() in every CTA, so a dependent
//     grid is only scheduled once all CTAs of the current grid are resident
//     (dependents can never starve it of SMs). The conv kernel triggers after
//     its last gather, not at entry: entry triggers let every kernel of a
//     step become resident at once (each parked in griddepcontrol.wait) and
//     starve other streams of SMs;
//   * every kernel calls wait() before it reads or writes anything another
//     kernel produces or consumes (activations, blob tables, split-K
//     workspace); only immutable inputs (weights, bias) may be touched before.
//     Since every kernel waits, completion stays ordered along the stream and
//     kernel k+2 transitively sees kernel k.
// Outside a PDL launch both instructions are no-ops.
//
// On by default (BS_PDL=0 disables). Measured on B200 (profiles/r02/pdl/,
// profiles/r02/anatomy/): whole-network passes GoogLeNet b=1 360 -> 252 us,
// ResNet-50 b=1 765 -> 557 us, GoogLeNet b=8 509 -> 412 us, b=90 unchanged.
// The per-layer latency tables are scaled to the measured whole-pass time
// (live.cu measure_profile): layer timings with events between the layers
// break this overlap, and with unscaled tables the Pareto configs 3 / 5
// served less on time with PDL (their schedulers planned on step costs the
// GPU no longer had); with scaled tables PDL serves more on every config
// (config 3 5.7k -> 7.3k req/s, config 5 12.6k -> 13.9k).
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

// A launch right after a cross-stream event wait (admission ready events,
// slot-release events) or on the admission copy stream goes without PDL:
// measured, PDL launches behind cudaStreamWaitEvent made the e2e (H2D
// admission) serving path ~3x slower. Host-thread local, consumed by the next
// launch on this thread.
inline bool& suppressed() {
  thread_local bool s = false;
  return s;
}
inline void suppress_next() { suppressed() = true; }

// cluster > 1: a thread-block cluster launch of `cluster` CTAs along x.
template <typename... KArgs, typename... Args>
cudaError_t launch_ex(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                      int cluster, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  const bool skip = suppressed();
  suppressed() = false;
  attr[0].val.programmaticStreamSerializationAllowed = enabled() && !skip ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cluster > 1) {
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = static_cast<unsigned>(cluster);
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.numAttrs = 2;
  }
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
cudaError_t launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                   Args&&... args) {
  return launch_ex(kernel, grid, block, smem, stream, 1, std::forward<Args>(args)...);
}

}  // namespace pdl
}  // namespace bs200

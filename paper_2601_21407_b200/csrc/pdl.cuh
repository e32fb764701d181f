// pdl.cuh -- programmatic dependent launch (PDL) for the layer-step kernel chain.
//
// A kernel launched with the programmatic-stream-serialization attribute may
// start while its predecessor on the stream is still draining: its CTAs are
// scheduled once every predecessor CTA has issued griddepcontrol.launch_dependents
// (or exited), run their prologue (barrier init, TMEM allocation, tensor-map
// prefetch) on the SMs the predecessor's finished CTAs freed, and block in
// griddepcontrol.wait until the predecessor grid has completed and its memory
// is visible.  Rule kept by every kernel launched this way: pdl_wait() comes
// before its first global-memory access (read or write) in every thread, so a
// PDL kernel never completes before its predecessor and the stream order stays
// transitive.  Outside a PDL launch both instructions are no-ops.
// On by default (HHB_PDL=0 turns it off): three same-box A/B pairs, config 3
// 0.567 -> 0.561 ms (bf16x3) and 0.471 -> 0.462 ms (bf16), config 4 2.450 ->
// 2.446 ms, configs 1 / 2 / 5 unchanged.  (Before the
// GEMMs walked column tiles fastest it cost config 4 1.3 %: CTAs parked in the
// wait held SM resources the side-stream weight-gradient GEMM needed.)
#pragma once

#include <cstdlib>
#include <cuda_runtime.h>
#include <utility>

namespace hhb {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HHB_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
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
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace hhb

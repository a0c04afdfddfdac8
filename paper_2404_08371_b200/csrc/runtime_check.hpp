// runtime_check.hpp -- CUDA error checks that throw tetmf::DeviceError.
#pragma once

#include <cstdlib>
#include <string>
#include <utility>

#include <cuda_runtime.h>

#include "common.hpp"

namespace tetmf {

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}
void count_launch(int k);  // runtime.cpp: process-wide kernel launch counter
inline void check_launch(const char* kernel) {
  cuda_check(cudaGetLastError(), kernel);
  count_launch(1);
}

// Programmatic dependent launch (PDL) of a kernel that follows another one on
// the stream: its CTAs may become resident while the previous grid drains
// (after that grid's griddepcontrol.launch_dependents, or its end), and the
// kernel itself orders its first global access behind the previous grid with
// pdl_wait(). Hides the launch bubble between the element kernel and K4 and
// between applies (config 4: two boundaries per ~100 us apply).
// TETMF_PDL=0 launches with full stream serialization (A/B).
#ifndef TETMF_PDL_DEFAULT
#define TETMF_PDL_DEFAULT 3
#endif
// TETMF_PDL: bit 0 = K4 (interface sum), bit 1 = K1 (stencil); 0 = off.
constexpr int kPdlK4 = 1, kPdlK1 = 2;
inline int pdl_mask() {
  static const int m = [] {
    const char* e = std::getenv("TETMF_PDL");
    return e ? std::atoi(e) : TETMF_PDL_DEFAULT;
  }();
  return m;
}
template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(int which, void (*kern)(KArgs...), dim3 grid, dim3 block, std::size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = (pdl_mask() & which) ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, KArgs(std::forward<Args>(args))...);
}
#ifdef __CUDACC__
// every thread that goes on to touch global memory written by the previous
// grid calls this first (no-op when the kernel was launched without PDL)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// lets the next PDL kernel's CTAs be scheduled as this grid's CTAs retire
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;"); }
#endif

} // namespace tetmf

#define TETMF_CUDA(call) ::tetmf::cuda_check((call), #call)

// runtime_check.hpp -- CUDA error checks that throw tetmf::DeviceError.
#pragma once

#include <string>

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

} // namespace tetmf

#define TETMF_CUDA(call) ::tetmf::cuda_check((call), #call)

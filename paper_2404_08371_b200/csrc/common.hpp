// common.hpp -- error model shared by the host library.
//
// The reference throws std::invalid_argument for bad arguments (forms.cpp:
// 58-67, 198-200; mesh.cpp:76-94) and std::logic_error for internal
// inconsistency (fespace.cpp:330, 400). The C ABI maps these to TETMF_EINVAL
// and TETMF_EINTERNAL; CUDA / NCCL failures map to TETMF_EDEVICE / TETMF_ECOMM.
#pragma once

#include <stdexcept>
#include <string>

namespace tetmf {

struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CommError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

[[noreturn]] inline void fail_arg(const std::string& msg) { throw std::invalid_argument(msg); }
[[noreturn]] inline void fail_internal(const std::string& msg) { throw std::logic_error(msg); }

} // namespace tetmf

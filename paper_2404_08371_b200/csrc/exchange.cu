// exchange.cu -- device side of the interface exchange: pack, transport
// (NCCL send/recv over NVLink, or loopback copies), combine (exchange.hpp).
#include <cstring>

#include "exchange.hpp"
#include "runtime_check.hpp"

namespace tetmf {

namespace {

__global__ void pack_kernel(const double* y, const i64* send_index, double* send, i64 count, bool sgn) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < count) exchange_pack_one(y, send_index, send, i, sgn);
}

__global__ void combine_kernel(double* y, const double* recv, const i64* offsets, const i64* entries, i64 ngroups,
                               bool sgn, bool owner) {
  const i64 g = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (g < ngroups) exchange_combine_one(y, recv, offsets, entries, g, sgn, owner);
}

template <typename T>
T* upload(const std::vector<T>& v) {
  if (v.empty()) return nullptr;
  T* p = nullptr;
  TETMF_CUDA(cudaMalloc(&p, v.size() * sizeof(T)));
  TETMF_CUDA(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return p;
}

} // namespace

Exchange::Exchange(ExchangePlan plan, Transport* transport) : plan_(std::move(plan)), transport_(transport) {
  d_send_index_ = upload(plan_.send_index);
  d_group_offsets_ = upload(plan_.group_offsets);
  d_group_entries_ = upload(plan_.group_entries);
  if (plan_.send_total() > 0) TETMF_CUDA(cudaMalloc(&d_send_, plan_.send_total() * sizeof(double)));
  if (plan_.recv_total() > 0) TETMF_CUDA(cudaMalloc(&d_recv_, plan_.recv_total() * sizeof(double)));
}

Exchange::~Exchange() {
  cudaFree(d_send_index_);
  cudaFree(d_group_offsets_);
  cudaFree(d_group_entries_);
  cudaFree(d_send_);
  cudaFree(d_recv_);
}

void Exchange::run(double* y, cudaStream_t stream, bool signed_values) { run_mode(y, stream, signed_values, false); }

void Exchange::broadcast_owner(double* y, cudaStream_t stream) { run_mode(y, stream, true, true); }

void Exchange::run_mode(double* y, cudaStream_t stream, bool signed_values, bool owner) {
  if (!transport_) throw CommError("exchange: no transport attached to the context");
  const i64 ns = plan_.send_total();
  if (ns > 0) {
    pack_kernel<<<static_cast<unsigned>((ns + 255) / 256), 256, 0, stream>>>(y, d_send_index_, d_send_, ns,
                                                                                 signed_values);
    check_launch("exchange_pack");
  }
  transport_->exchange(ExchangeIO{&plan_.peers, &plan_.send_offsets, &plan_.recv_offsets, d_send_, d_recv_}, stream);
  const i64 ng = plan_.num_groups();
  if (ng > 0) {
    combine_kernel<<<static_cast<unsigned>((ng + 255) / 256), 256, 0, stream>>>(y, d_recv_, d_group_offsets_,
                                                                                 d_group_entries_, ng,
                                                                                 signed_values, owner);
    check_launch("exchange_combine");
  }
}

} // namespace tetmf

// exchange.cu -- device side of the interface exchange: pack, NCCL
// send/recv over NVLink, combine (see exchange.hpp).
#include <cstring>

#include <nccl.h>

#include "exchange.hpp"
#include "runtime_check.hpp"

namespace tetmf {

namespace {

__global__ void pack_kernel(const double* y, const i64* send_index, double* send, i64 count, bool sgn) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < count) exchange_pack_one(y, send_index, send, i, sgn);
}

__global__ void combine_kernel(double* y, const double* recv, const i64* offsets, const i64* entries, i64 ngroups,
                               bool sgn) {
  const i64 g = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (g < ngroups) exchange_combine_one(y, recv, offsets, entries, g, sgn);
}

template <typename T>
T* upload(const std::vector<T>& v) {
  if (v.empty()) return nullptr;
  T* p = nullptr;
  TETMF_CUDA(cudaMalloc(&p, v.size() * sizeof(T)));
  TETMF_CUDA(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return p;
}

inline void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw CommError(std::string(what) + ": " + ncclGetErrorString(r));
}

} // namespace

Exchange::Exchange(ExchangePlan plan, void* nccl_comm) : plan_(std::move(plan)), comm_(nccl_comm) {
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

void Exchange::run(double* y, cudaStream_t stream, bool signed_values) {
  if (plan_.peers.empty()) return;
  if (!comm_) throw CommError("exchange: no NCCL communicator attached to the context");
  const i64 ns = plan_.send_total();
  if (ns > 0) {
    pack_kernel<<<static_cast<unsigned>((ns + 255) / 256), 256, 0, stream>>>(y, d_send_index_, d_send_, ns,
                                                                                 signed_values);
    check_launch("exchange_pack");
  }
  auto comm = static_cast<ncclComm_t>(comm_);
  nccl_check(ncclGroupStart(), "ncclGroupStart");
  for (std::size_t p = 0; p < plan_.peers.size(); ++p) {
    const i64 so = plan_.send_offsets[p], sc = plan_.send_offsets[p + 1] - so;
    const i64 ro = plan_.recv_offsets[p], rc = plan_.recv_offsets[p + 1] - ro;
    if (sc > 0) nccl_check(ncclSend(d_send_ + so, sc, ncclDouble, plan_.peers[p], comm, stream), "ncclSend");
    if (rc > 0) nccl_check(ncclRecv(d_recv_ + ro, rc, ncclDouble, plan_.peers[p], comm, stream), "ncclRecv");
  }
  nccl_check(ncclGroupEnd(), "ncclGroupEnd");
  const i64 ng = plan_.num_groups();
  if (ng > 0) {
    combine_kernel<<<static_cast<unsigned>((ng + 255) / 256), 256, 0, stream>>>(y, d_recv_, d_group_offsets_,
                                                                                 d_group_entries_, ng,
                                                                                 signed_values);
    check_launch("exchange_combine");
  }
}

} // namespace tetmf

namespace tetmf {

void nccl_get_unique_id(void* out) {
  ncclUniqueId id;
  nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof(id));
}

void* nccl_comm_create(int nranks, const void* unique_id, int rank) {
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  ncclComm_t comm = nullptr;
  nccl_check(ncclCommInitRank(&comm, nranks, id, rank), "ncclCommInitRank");
  return comm;
}

void nccl_comm_destroy(void* comm) {
  if (comm) ncclCommDestroy(static_cast<ncclComm_t>(comm));
}

// out[r * count + k] = in_r[k] for every rank r (solver scalars, solver.hpp)
void nccl_allgather_doubles(void* comm, const double* d_in, double* d_out, int count, cudaStream_t stream) {
  if (!comm) throw CommError("allgather: no NCCL communicator attached to the context");
  nccl_check(ncclAllGather(d_in, d_out, count, ncclDouble, static_cast<ncclComm_t>(comm), stream), "ncclAllGather");
}

} // namespace tetmf

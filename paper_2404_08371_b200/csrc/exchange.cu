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

__global__ void put_kernel(const double* y, const i64* send_index, const i64* dst_off, const int* dst_peer,
                           double* const* peer_win, i64 count, bool sgn) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < count) exchange_put_one(y, send_index, dst_off, dst_peer, peer_win, i, sgn);
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

Exchange::Exchange(ExchangePlan plan, Transport* transport, bool put) : plan_(std::move(plan)), transport_(transport) {
  d_send_index_ = upload(plan_.send_index);
  d_group_offsets_ = upload(plan_.group_offsets);
  d_group_entries_ = upload(plan_.group_entries);
  if (put) {
    if (!transport_) throw CommError("exchange: no transport attached to the context");
    put_ = transport_->open_put(plan_.peers, plan_.send_offsets, plan_.recv_offsets);
    if (!put_) fail_arg("exchange: the context's transport cannot store into peer memory (put mode)");
    std::vector<i64> dst_off;
    std::vector<int> dst_peer;
    exchange_put_targets(plan_, put_->peer_off, dst_off, dst_peer);
    d_dst_off_ = upload(dst_off);
    d_dst_peer_ = upload(dst_peer);
    const std::size_t np = plan_.peers.size();
    std::vector<double*> wins(2 * np);
    for (std::size_t k = 0; k < np; ++k) {
      wins[k] = put_->peer_base[k];
      wins[np + k] = put_->peer_base[k] + put_->half;
    }
    d_peer_win_ = upload(wins);
    return;
  }
  if (plan_.send_total() > 0) TETMF_CUDA(cudaMalloc(&d_send_, plan_.send_total() * sizeof(double)));
  if (plan_.recv_total() > 0) TETMF_CUDA(cudaMalloc(&d_recv_, plan_.recv_total() * sizeof(double)));
}

Exchange::~Exchange() {
  cudaFree(d_send_index_);
  cudaFree(d_group_offsets_);
  cudaFree(d_group_entries_);
  cudaFree(d_send_);
  cudaFree(d_recv_);
  cudaFree(d_dst_off_);
  cudaFree(d_dst_peer_);
  cudaFree(d_peer_win_);
  cudaFree(d_first_);
  cudaFree(d_chain_);
  cudaFree(d_dst_);
}

bool Exchange::fusable() const {
  if (!put_ || plan_.peers.size() > static_cast<std::size_t>(kFusedMaxPeers)) return false;
  for (i64 e : plan_.send_index)
    if (e & 1) return false;
  return true;
}

FusedPut Exchange::fused_begin(i64 storage_size) {
  if (!fusable()) fail_internal("exchange: fused put without a put channel or with signed entries");
  if (first_size_ != storage_size) {
    const i64 ns = plan_.send_total();
    if (ns >= (i64(1) << 31)) fail_arg("exchange: too many send entries for the fused put");
    std::vector<int> first(static_cast<std::size_t>(storage_size), -1), chain(static_cast<std::size_t>(ns), -1);
    for (i64 e = ns - 1; e >= 0; --e) {
      const i64 j = plan_.send_index[e] >> 1;
      if (j < 0 || j >= storage_size) fail_internal("exchange: send slot outside the level buffer");
      chain[e] = first[j];
      first[j] = static_cast<int>(e);
    }
    std::vector<i64> dst(static_cast<std::size_t>(ns)), off;
    std::vector<int> peer;
    exchange_put_targets(plan_, put_->peer_off, off, peer);
    for (i64 e = 0; e < ns; ++e) {
      if (off[e] >= (i64(1) << 48)) fail_arg("exchange: window too large for the fused put");
      dst[e] = (static_cast<i64>(peer[e]) << 48) | off[e];
    }
    cudaFree(d_first_);
    cudaFree(d_chain_);
    cudaFree(d_dst_);
    d_first_ = upload(first);
    d_chain_ = upload(chain);
    d_dst_ = upload(dst);
    first_size_ = storage_size;
  }
  FusedPut fp;
  fp.first = d_first_;
  fp.chain = d_chain_;
  fp.dst = d_dst_;
  for (std::size_t k = 0; k < plan_.peers.size(); ++k) fp.win[k] = put_->peer_base[k] + parity_ * put_->half;
  return fp;
}

void Exchange::fused_finish(double* y, cudaStream_t stream) {
  const int par = parity_;
  parity_ ^= 1;
  put_->fence(stream);
  const i64 ng = plan_.num_groups();
  if (ng > 0) {
    combine_kernel<<<static_cast<unsigned>((ng + 255) / 256), 256, 0, stream>>>(
        y, put_->local + par * put_->half, d_group_offsets_, d_group_entries_, ng, true, false);
    check_launch("exchange_combine");
  }
}

void exchange_put_targets(const ExchangePlan& plan, const std::vector<i64>& peer_off, std::vector<i64>& dst_off,
                          std::vector<int>& dst_peer) {
  if (peer_off.size() != plan.peers.size()) fail_internal("exchange_put_targets: one offset per peer");
  dst_off.resize(static_cast<std::size_t>(plan.send_total()));
  dst_peer.resize(dst_off.size());
  for (std::size_t k = 0; k < plan.peers.size(); ++k)
    for (i64 i = plan.send_offsets[k]; i < plan.send_offsets[k + 1]; ++i) {
      dst_off[i] = peer_off[k] + (i - plan.send_offsets[k]);
      dst_peer[i] = static_cast<int>(k);
    }
}

void Exchange::run(double* y, cudaStream_t stream, bool signed_values) { run_mode(y, stream, signed_values, false); }

void Exchange::broadcast_owner(double* y, cudaStream_t stream) { run_mode(y, stream, true, true); }

void Exchange::run_mode(double* y, cudaStream_t stream, bool signed_values, bool owner) {
  if (!transport_) throw CommError("exchange: no transport attached to the context");
  const i64 ns = plan_.send_total();
  const i64 ng = plan_.num_groups();
  if (put_) {
    // pack straight into the peers' windows (this exchange's parity half),
    // fence, combine from this rank's own half
    const int par = parity_;
    parity_ ^= 1;
    if (ns > 0) {
      put_kernel<<<static_cast<unsigned>((ns + 255) / 256), 256, 0, stream>>>(
          y, d_send_index_, d_dst_off_, d_dst_peer_, d_peer_win_ + par * plan_.peers.size(), ns, signed_values);
      check_launch("exchange_put");
    }
    put_->fence(stream);
    if (ng > 0) {
      combine_kernel<<<static_cast<unsigned>((ng + 255) / 256), 256, 0, stream>>>(
          y, put_->local + par * put_->half, d_group_offsets_, d_group_entries_, ng, signed_values, owner);
      check_launch("exchange_combine");
    }
    return;
  }
  if (ns > 0) {
    pack_kernel<<<static_cast<unsigned>((ns + 255) / 256), 256, 0, stream>>>(y, d_send_index_, d_send_, ns,
                                                                                 signed_values);
    check_launch("exchange_pack");
  }
  transport_->exchange(ExchangeIO{&plan_.peers, &plan_.send_offsets, &plan_.recv_offsets, d_send_, d_recv_}, stream);
  if (ng > 0) {
    combine_kernel<<<static_cast<unsigned>((ng + 255) / 256), 256, 0, stream>>>(y, d_recv_, d_group_offsets_,
                                                                                 d_group_entries_, ng,
                                                                                 signed_values, owner);
    check_launch("exchange_combine");
  }
}

} // namespace tetmf

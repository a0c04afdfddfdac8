// transport.cpp -- NCCL and loopback transports (transport.hpp).
#include "transport.hpp"

#include <algorithm>
#include <chrono>
#include <cstring>
#include <string>

#include <nccl.h>

#include "common.hpp"
#include "nccl_put.hpp"
#include "runtime_check.hpp"

namespace tetmf {

namespace {

inline void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw CommError(std::string(what) + ": " + ncclGetErrorString(r));
}

// ---------------------------------------------------------------- NCCL
class NcclTransport final : public Transport {
public:
  NcclTransport(int nranks, const void* unique_id, int rank) : rank_(rank), nranks_(nranks) {
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    nccl_check(ncclCommInitRank(&comm_, nranks, id, rank), "ncclCommInitRank");
    int count = 0;
    nccl_check(ncclCommCount(comm_, &count), "ncclCommCount");
    if (count != nranks) throw CommError("NCCL communicator has " + std::to_string(count) + " ranks, expected " +
                                         std::to_string(nranks));
  }
  ~NcclTransport() override {
    if (comm_) ncclCommDestroy(comm_);
  }
  int rank() const override { return rank_; }
  int nranks() const override { return nranks_; }

  void exchange(const ExchangeIO& io, cudaStream_t s) override {
    poll_async_error();
    nccl_check(ncclGroupStart(), "ncclGroupStart");
    for (std::size_t p = 0; p < io.peers->size(); ++p) {
      const i64 so = (*io.send_off)[p], sc = (*io.send_off)[p + 1] - so;
      const i64 ro = (*io.recv_off)[p], rc = (*io.recv_off)[p + 1] - ro;
      const int peer = (*io.peers)[p];
      if (sc > 0) nccl_check(ncclSend(io.send + so, static_cast<size_t>(sc), ncclDouble, peer, comm_, s), "ncclSend");
      if (rc > 0) nccl_check(ncclRecv(io.recv + ro, static_cast<size_t>(rc), ncclDouble, peer, comm_, s), "ncclRecv");
    }
    nccl_check(ncclGroupEnd(), "ncclGroupEnd");
  }

  void allgather(const double* d_in, double* d_out, int count, cudaStream_t s) override {
    poll_async_error();
    nccl_check(ncclAllGather(d_in, d_out, static_cast<size_t>(count), ncclDouble, comm_, s), "ncclAllGather");
  }

  std::unique_ptr<PutChannel> open_put(const std::vector<int>& peers, const std::vector<i64>& send_off,
                                       const std::vector<i64>& recv_off) override {
    poll_async_error();
    return nccl_open_put(comm_, rank_, nranks_, peers, send_off, recv_off);
  }

  std::string describe() const override {
    int count = 0, dev = -1, r = -1;
    ncclCommCount(comm_, &count);
    ncclCommCuDevice(comm_, &dev);
    ncclCommUserRank(comm_, &r);
    return "nccl rank " + std::to_string(r) + " of " + std::to_string(count) + " (cuda device " +
           std::to_string(dev) + ")";
  }

private:
  // a failed peer / link surfaces here instead of as a hang on the next call
  void poll_async_error() {
    ncclResult_t st = ncclSuccess;
    nccl_check(ncclCommGetAsyncError(comm_, &st), "ncclCommGetAsyncError");
    if (st != ncclSuccess && st != ncclInProgress)
      throw CommError(std::string("NCCL asynchronous error: ") + ncclGetErrorString(st));
  }

  ncclComm_t comm_ = nullptr;
  int rank_, nranks_;
};

// ---------------------------------------------------------------- loopback
class LoopbackTransport final : public Transport {
public:
  LoopbackTransport(std::shared_ptr<LoopbackHub> hub, int rank) : hub_(std::move(hub)), rank_(rank) {
    if (!hub_ || rank < 0 || rank >= hub_->nranks()) fail_arg("loopback: bad rank for the group");
  }
  int rank() const override { return rank_; }
  int nranks() const override { return hub_->nranks(); }

  // publish -> barrier -> copy from every peer's send buffer -> barrier ->
  // wait for the peers' copies out of OUR send buffer (so the next pack on
  // this stream cannot overwrite it while a peer still reads it)
  void exchange(const ExchangeIO& io, cudaStream_t s) override {
    guarded([&] { exchange_impl(io, s); });
  }
  void allgather(const double* d_in, double* d_out, int count, cudaStream_t s) override {
    guarded([&] { allgather_impl(d_in, d_out, count, s); });
  }

private:
  // a rank that fails inside a collective step releases its peers from the
  // barriers at once (they throw "aborted") instead of leaving them to the timeout
  template <typename F>
  void guarded(F&& f) {
    try {
      f();
    } catch (...) {
      hub_->barrier().abort();
      throw;
    }
  }

  void exchange_impl(const ExchangeIO& io, cudaStream_t s) {
    int dev = 0;
    TETMF_CUDA(cudaGetDevice(&dev));
    hub_->ensure_events(rank_, dev);
    auto& me = hub_->slot(rank_);
    me.send = io.send;
    me.peers = io.peers;
    me.send_off = io.send_off;
    TETMF_CUDA(cudaEventRecord(me.ready, s));
    hub_->barrier().wait(hub_->timeout_s);
    for (std::size_t p = 0; p < io.peers->size(); ++p) {
      const int peer = (*io.peers)[p];
      const auto& ps = hub_->slot(peer);
      if (ps.device != dev) fail_internal("loopback: virtual ranks must share one device");
      i64 so = -1, sc = 0;
      for (std::size_t q = 0; q < ps.peers->size(); ++q)
        if ((*ps.peers)[q] == rank_) {
          so = (*ps.send_off)[q];
          sc = (*ps.send_off)[q + 1] - so;
        }
      const i64 ro = (*io.recv_off)[p], rc = (*io.recv_off)[p + 1] - ro;
      if (so < 0 || sc != rc)
        fail_internal("loopback: peer " + std::to_string(peer) + " sends " + std::to_string(sc) + " values, rank " +
                      std::to_string(rank_) + " expects " + std::to_string(rc));
      if (rc == 0) continue;
      TETMF_CUDA(cudaStreamWaitEvent(s, ps.ready, 0));
      TETMF_CUDA(cudaMemcpyAsync(io.recv + ro, ps.send + so, static_cast<size_t>(rc) * sizeof(double),
                                 cudaMemcpyDeviceToDevice, s));
    }
    finish(*io.peers, s);
  }

  void allgather_impl(const double* d_in, double* d_out, int count, cudaStream_t s) {
    int dev = 0;
    TETMF_CUDA(cudaGetDevice(&dev));
    hub_->ensure_events(rank_, dev);
    auto& me = hub_->slot(rank_);
    me.send = d_in;
    TETMF_CUDA(cudaEventRecord(me.ready, s));
    hub_->barrier().wait(hub_->timeout_s);
    std::vector<int> all;
    for (int q = 0; q < nranks(); ++q) {
      const auto& ps = hub_->slot(q);
      if (q != rank_) {
        all.push_back(q);
        TETMF_CUDA(cudaStreamWaitEvent(s, ps.ready, 0));
      }
      TETMF_CUDA(cudaMemcpyAsync(d_out + static_cast<i64>(q) * count, ps.send, sizeof(double) * count,
                                 cudaMemcpyDeviceToDevice, s));
    }
    finish(all, s);
  }

public:
  std::unique_ptr<PutChannel> open_put(const std::vector<int>& peers, const std::vector<i64>& send_off,
                                       const std::vector<i64>& recv_off) override {
    std::unique_ptr<PutChannel> ch;
    guarded([&] { ch = open_put_impl(peers, send_off, recv_off); });
    return ch;
  }

  std::string describe() const override {
    return "loopback virtual rank " + std::to_string(rank_) + " of " + std::to_string(nranks()) +
           " (device-to-device copies on one GPU)";
  }

private:
  // the virtual ranks' windows are device buffers of the same GPU; the peers'
  // stores become visible through stream order: fence = record this rank's
  // event after its put kernel, host barrier, wait for every peer's event
  class LoopbackPut final : public PutChannel {
  public:
    LoopbackPut(LoopbackTransport* t, std::vector<int> peers) : t_(t), peers_(std::move(peers)) {}
    ~LoopbackPut() override { cudaFree(local); }
    void fence(cudaStream_t s) override {
      t_->guarded([&] {
        auto& me = t_->hub_->slot(t_->rank_);
        TETMF_CUDA(cudaEventRecord(me.ready, s));
        t_->hub_->barrier().wait(t_->hub_->timeout_s);
        for (int p : peers_) TETMF_CUDA(cudaStreamWaitEvent(s, t_->hub_->slot(p).ready, 0));
      });
    }

  private:
    LoopbackTransport* t_;
    std::vector<int> peers_;
  };

  std::unique_ptr<PutChannel> open_put_impl(const std::vector<int>& peers, const std::vector<i64>& send_off,
                                            const std::vector<i64>& recv_off) {
    int dev = 0;
    TETMF_CUDA(cudaGetDevice(&dev));
    hub_->ensure_events(rank_, dev);
    auto ch = std::make_unique<LoopbackPut>(this, peers);
    auto& me = hub_->slot(rank_);
    me.peers = &peers;
    me.send_off = &send_off;
    me.recv_off = &recv_off;
    me.recv_total = recv_off.empty() ? 0 : recv_off.back();
    hub_->barrier().wait(hub_->timeout_s);  // every rank's receive layout is published
    const int P = nranks();
    std::vector<i64> counts(static_cast<std::size_t>(P) * P, 0);
    i64 half = 0;
    for (int q = 0; q < P; ++q) {
      const auto& qs = hub_->slot(q);
      half = std::max(half, qs.recv_total);
      for (std::size_t k = 0; k < qs.peers->size(); ++k)
        counts[static_cast<std::size_t>(q) * P + (*qs.peers)[k]] = (*qs.send_off)[k + 1] - (*qs.send_off)[k];
    }
    ch->half = half;
    ch->peer_off = put_peer_offsets(P, counts.data(), rank_, peers);
    // cross-check against the peers' own receive layouts
    for (std::size_t k = 0; k < peers.size(); ++k) {
      const auto& ps = hub_->slot(peers[k]);
      i64 expect = -1;
      for (std::size_t q = 0; q < ps.peers->size(); ++q)
        if ((*ps.peers)[q] == rank_) expect = (*ps.recv_off)[q];
      if (expect != ch->peer_off[k])
        fail_internal("loopback put: peer " + std::to_string(peers[k]) + " receives rank " + std::to_string(rank_) +
                      " at " + std::to_string(expect) + ", computed " + std::to_string(ch->peer_off[k]));
    }
    if (half > 0) TETMF_CUDA(cudaMalloc(&ch->local, sizeof(double) * 2 * half));
    me.window = ch->local;
    hub_->barrier().wait(hub_->timeout_s);  // every window exists
    for (int p : peers) {
      if (hub_->slot(p).device != dev) fail_internal("loopback: virtual ranks must share one device");
      ch->peer_base.push_back(hub_->slot(p).window);
    }
    hub_->barrier().wait(hub_->timeout_s);  // the slots may be reused by the next setup
    return ch;
  }

  void finish(const std::vector<int>& peers, cudaStream_t s) {
    auto& me = hub_->slot(rank_);
    TETMF_CUDA(cudaEventRecord(me.done, s));
    hub_->barrier().wait(hub_->timeout_s);
    for (int p : peers) TETMF_CUDA(cudaStreamWaitEvent(s, hub_->slot(p).done, 0));
  }

  std::shared_ptr<LoopbackHub> hub_;
  int rank_;
};

} // namespace

std::vector<i64> put_peer_offsets(int nranks, const i64* counts, int me, const std::vector<int>& peers) {
  std::vector<i64> off;
  off.reserve(peers.size());
  for (int p : peers) {
    if (p < 0 || p >= nranks || p == me) fail_internal("put_peer_offsets: bad peer rank");
    i64 o = 0;
    for (int q = 0; q < me; ++q)
      if (q != p) o += counts[static_cast<std::size_t>(q) * nranks + p];
    off.push_back(o);
  }
  return off;
}

std::unique_ptr<Transport> make_nccl_transport(int nranks, const void* unique_id, int rank) {
  return std::make_unique<NcclTransport>(nranks, unique_id, rank);
}

void nccl_get_unique_id(void* out) {
  ncclUniqueId id;
  nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof(id));
}

void HostBarrier::wait(double timeout_s) {
  std::unique_lock<std::mutex> lk(mu_);
  if (aborted_) throw CommError("loopback group aborted by a failed rank");
  const std::uint64_t gen = generation_;
  if (++arrived_ == n_) {
    arrived_ = 0;
    ++generation_;
    cv_.notify_all();
    return;
  }
  const bool ok = cv_.wait_for(lk, std::chrono::duration<double>(timeout_s),
                               [&] { return generation_ != gen || aborted_; });
  if (aborted_) throw CommError("loopback group aborted by a failed rank");
  if (!ok) {
    aborted_ = true;
    cv_.notify_all();
    throw CommError("loopback barrier timeout: a virtual rank did not reach the collective step");
  }
}

void HostBarrier::abort() {
  std::lock_guard<std::mutex> lk(mu_);
  aborted_ = true;
  cv_.notify_all();
}

LoopbackHub::LoopbackHub(int nranks) : nranks_(nranks), slots_(nranks), barrier_(nranks) {
  if (nranks < 1) fail_arg("loopback: nranks must be >= 1");
}

LoopbackHub::~LoopbackHub() {
  for (auto& s : slots_) {
    if (s.ready) cudaEventDestroy(s.ready);
    if (s.done) cudaEventDestroy(s.done);
  }
}

void LoopbackHub::ensure_events(int rank, int device) {
  Slot& s = slots_[rank];
  if (s.ready) return;
  TETMF_CUDA(cudaEventCreateWithFlags(&s.ready, cudaEventDisableTiming));
  TETMF_CUDA(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
  s.device = device;
}

std::unique_ptr<Transport> make_loopback_transport(std::shared_ptr<LoopbackHub> hub, int rank) {
  return std::make_unique<LoopbackTransport>(std::move(hub), rank);
}

} // namespace tetmf

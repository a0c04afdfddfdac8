// transport.hpp -- how the interface exchange and the solver's scalar
// all-gather move bytes between ranks.
//
// The path has ONE real exchange step per apply: the neighbour SUM-exchange
// of partial y values on carriers shared with macros of other ranks
// (exchange.hpp), plus the solver's all-gather of per-rank
// inner-product partials. Both go through a Transport:
//
//  * NcclTransport     one process per GPU, grouped ncclSend / ncclRecv and
//                      ncclAllGather on the context stream (NVLink / NVSwitch)
//  * LoopbackTransport P "virtual ranks" of ONE process on ONE device, one
//                      host thread per rank: every transfer is a
//                      device-to-device cudaMemcpyAsync from the peer's send
//                      buffer, ordered by CUDA events and two host barriers
//                      per step. No kernel ever waits on another kernel, so
//                      the virtual ranks are safe on a single GPU. It runs the
//                      product's own pack / combine kernels, the K4 local sum
//                      and the solver all-gather, so the multi-rank path is
//                      testable bitwise against the single-rank apply with
//                      one B200 (layer 3).
//
// Semantics are those of a collective: every rank of the group must make the
// matching call (same plan step), in the same order.
#pragma once

#include <condition_variable>
#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

namespace tetmf {

using i64 = std::int64_t;

// One rank's side of a neighbour exchange: for every peer (ascending rank),
// send[send_off[p] .. send_off[p+1]) goes to peers[p] and
// recv[recv_off[p] .. recv_off[p+1]) comes from peers[p].
struct ExchangeIO {
  const std::vector<int>* peers;
  const std::vector<i64>* send_off;
  const std::vector<i64>* recv_off;
  const double* send;
  double* recv;
};

// Direct-put channel of one exchange plan (Exchange put mode): every rank
// owns a receive window of two parity halves (consecutive exchanges alternate
// halves, so a peer's next puts never land in the half this rank is still
// combining); the pack kernel stores each value straight into the peer's
// window (NVLink stores through NCCL LSA pointers, or plain device pointers
// between loopback virtual ranks), then fence() makes all peers' stores into
// this rank's window visible on `s`.
class PutChannel {
public:
  virtual ~PutChannel() = default;
  double* local = nullptr;          // this rank's window: 2 * half doubles
  i64 half = 0;                     // doubles per parity half (max receive total over the ranks)
  std::vector<double*> peer_base;   // per plan peer: device address of the peer's window
  std::vector<i64> peer_off;        // per plan peer: first position of this rank's values in a half
  virtual void fence(cudaStream_t s) = 0;
};

// where this rank's values start in each peer's receive buffer: a receive
// buffer concatenates its peers' contributions in ascending rank order, so
// for peer p it is the sum of counts[q][p] over ranks q < me
// (counts[src * nranks + dst] = number of values src sends to dst)
std::vector<i64> put_peer_offsets(int nranks, const i64* counts, int me, const std::vector<int>& peers);

class Transport {
public:
  virtual ~Transport() = default;
  // collective over the group: the put channel of one plan, or nullptr when
  // the transport cannot store into peer memory
  virtual std::unique_ptr<PutChannel> open_put(const std::vector<int>& peers, const std::vector<i64>& send_off,
                                               const std::vector<i64>& recv_off) {
    (void)peers, (void)send_off, (void)recv_off;
    return nullptr;
  }
  virtual int rank() const = 0;
  virtual int nranks() const = 0;
  virtual void exchange(const ExchangeIO& io, cudaStream_t s) = 0;
  // out[r * count + k] = in_r[k] for every rank r
  virtual void allgather(const double* d_in, double* d_out, int count, cudaStream_t s) = 0;
  virtual std::string describe() const = 0;
};

// ---------------------------------------------------------------- NCCL
std::unique_ptr<Transport> make_nccl_transport(int nranks, const void* unique_id, int rank);
void nccl_get_unique_id(void* out128);

// ---------------------------------------------------------------- loopback
// Host barrier with a timeout: a virtual rank that fails (throws) before a
// collective step would otherwise leave its peers waiting forever.
class HostBarrier {
public:
  explicit HostBarrier(int n) : n_(n) {}
  void wait(double timeout_s);
  void abort();

private:
  std::mutex mu_;
  std::condition_variable cv_;
  int n_, arrived_ = 0;
  std::uint64_t generation_ = 0;
  bool aborted_ = false;
};

// State shared by the P virtual ranks of one loopback group (one device).
class LoopbackHub {
public:
  explicit LoopbackHub(int nranks);
  ~LoopbackHub();
  int nranks() const { return nranks_; }
  double timeout_s = 300.0;

  struct Slot {
    const double* send = nullptr;          // exchange: send buffer, allgather: input
    const std::vector<int>* peers = nullptr;
    const std::vector<i64>* send_off = nullptr;
    cudaEvent_t ready = nullptr;           // recorded after the rank's send buffer is written
    cudaEvent_t done = nullptr;            // recorded after the rank's copies from its peers
    int device = -1;
    // put channel setup (open_put): the rank's window and its plan's receive layout
    double* window = nullptr;
    i64 recv_total = 0;
    const std::vector<i64>* recv_off = nullptr;
  };
  Slot& slot(int r) { return slots_[r]; }
  HostBarrier& barrier() { return barrier_; }
  void ensure_events(int rank, int device);

private:
  int nranks_;
  std::vector<Slot> slots_;
  HostBarrier barrier_;
};

std::unique_ptr<Transport> make_loopback_transport(std::shared_ptr<LoopbackHub> hub, int rank);

} // namespace tetmf

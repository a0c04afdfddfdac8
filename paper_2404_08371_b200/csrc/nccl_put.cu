// nccl_put.cu -- PutChannel over the NCCL device API (nccl_put.hpp).
//
// Setup (collective, once per exchange plan):
//   1. all-gather every rank's receive total and per-destination send counts
//      (ncclAllGather); the window half is the largest receive total, so all
//      windows have the same size (symmetric registration);
//   2. ncclMemAlloc + ncclCommWindowRegister(NCCL_WIN_COLL_SYMMETRIC);
//   3. a device communicator with one LSA barrier (ncclDevCommCreate);
//   4. one tiny kernel resolves every peer's window base with
//      ncclGetLsaPointer -- the pack kernel then stores through plain device
//      pointers (NVLink P2P stores), the same kernel as the loopback mode.
// fence(): one CTA runs an LSA barrier session (release / acquire at system
// scope) after the put kernel; every rank's stores into this rank's window
// precede its arrival, so the combine that follows on the stream sees them.
#include "nccl_put.hpp"

#include <algorithm>
#include <string>

#include <nccl_device.h>

#include "runtime_check.hpp"

namespace tetmf {

namespace {

inline void nc(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw CommError(std::string(what) + ": " + ncclGetErrorString(r));
}

__global__ void lsa_bases_kernel(ncclWindow_t win, ncclDevComm dc, const int* peers, int npeers, double** out) {
  const int i = threadIdx.x + blockIdx.x * blockDim.x;
  if (i < npeers)
    out[i] = static_cast<double*>(ncclGetLsaPointer(win, 0, ncclTeamRankToLsa(dc, ncclTeamWorld(dc), peers[i])));
}

__global__ void lsa_barrier_kernel(ncclDevComm dc) {
  __threadfence_system();
  ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), 0);
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}

class NcclPut final : public PutChannel {
public:
  NcclPut(ncclComm_t comm) : comm_(comm) {}
  ~NcclPut() override {
    if (dev_ok_) ncclDevCommDestroy(comm_, &dc_);
    if (win_) ncclCommWindowDeregister(comm_, win_);
    if (local) ncclMemFree(local);
  }
  void fence(cudaStream_t s) override {
    lsa_barrier_kernel<<<1, 32, 0, s>>>(dc_);
    check_launch("lsa_barrier");
  }

  ncclComm_t comm_;
  ncclWindow_t win_ = nullptr;
  ncclDevComm dc_{};
  bool dev_ok_ = false;
};

} // namespace

std::unique_ptr<PutChannel> nccl_open_put(ncclComm_t comm, int rank, int nranks, const std::vector<int>& peers,
                                          const std::vector<i64>& send_off, const std::vector<i64>& recv_off) {
  cudaStream_t s = nullptr;
  TETMF_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } sg{s};
  // 1. counts: row of this rank = [recv total, send count to rank 0 .. P-1]
  const int W = nranks + 1;
  std::vector<double> row(W, 0.0), all(static_cast<std::size_t>(W) * nranks, 0.0);
  row[0] = static_cast<double>(recv_off.empty() ? 0 : recv_off.back());
  for (std::size_t k = 0; k < peers.size(); ++k) row[1 + peers[k]] = static_cast<double>(send_off[k + 1] - send_off[k]);
  double *d_row = nullptr, *d_all = nullptr;
  TETMF_CUDA(cudaMalloc(&d_row, sizeof(double) * W));
  TETMF_CUDA(cudaMalloc(&d_all, sizeof(double) * W * nranks));
  TETMF_CUDA(cudaMemcpyAsync(d_row, row.data(), sizeof(double) * W, cudaMemcpyHostToDevice, s));
  nc(ncclAllGather(d_row, d_all, W, ncclDouble, comm, s), "ncclAllGather (put counts)");
  TETMF_CUDA(cudaMemcpyAsync(all.data(), d_all, sizeof(double) * W * nranks, cudaMemcpyDeviceToHost, s));
  TETMF_CUDA(cudaStreamSynchronize(s));
  cudaFree(d_row);
  cudaFree(d_all);
  std::vector<i64> counts(static_cast<std::size_t>(nranks) * nranks);
  i64 half = 0;
  for (int q = 0; q < nranks; ++q) {
    half = std::max(half, static_cast<i64>(all[static_cast<std::size_t>(q) * W]));
    for (int p = 0; p < nranks; ++p)
      counts[static_cast<std::size_t>(q) * nranks + p] = static_cast<i64>(all[static_cast<std::size_t>(q) * W + 1 + p]);
  }
  for (std::size_t k = 0; k < peers.size(); ++k)  // symmetric plans: what peer p sends is what we expect
    if (counts[static_cast<std::size_t>(peers[k]) * nranks + rank] != recv_off[k + 1] - recv_off[k])
      throw CommError("nccl put: rank " + std::to_string(peers[k]) + " sends a different count than rank " +
                      std::to_string(rank) + " receives");

  auto ch = std::make_unique<NcclPut>(comm);
  ch->half = half;
  ch->peer_off = put_peer_offsets(nranks, counts.data(), rank, peers);
  // 2. symmetric window (same size on every rank)
  const size_t bytes = std::max<size_t>(static_cast<size_t>(2 * half) * sizeof(double), NCCL_WIN_REQUIRED_ALIGNMENT);
  const size_t size = (bytes + NCCL_WIN_REQUIRED_ALIGNMENT - 1) / NCCL_WIN_REQUIRED_ALIGNMENT * NCCL_WIN_REQUIRED_ALIGNMENT;
  void* buf = nullptr;
  nc(ncclMemAlloc(&buf, size), "ncclMemAlloc");
  ch->local = static_cast<double*>(buf);
  nc(ncclCommWindowRegister(comm, buf, size, &ch->win_, NCCL_WIN_COLL_SYMMETRIC), "ncclCommWindowRegister");
  // 3. device communicator with one LSA barrier
  ncclDevCommRequirements req{};
  req.lsaBarrierCount = 1;
  nc(ncclDevCommCreate(comm, &req, &ch->dc_), "ncclDevCommCreate");
  ch->dev_ok_ = true;
  const ncclTeam_t lsa = ncclTeamLsa(comm), world = ncclTeamWorld(comm);
  for (int p : peers)
    if (!ncclTeamRankIsMember(lsa, world, p))
      throw CommError("nccl put: rank " + std::to_string(p) +
                      " is not load/store reachable (outside the NVLink domain); use the send/recv exchange");
  // 4. peers' window bases
  if (!peers.empty()) {
    int* d_peers = nullptr;
    double** d_bases = nullptr;
    TETMF_CUDA(cudaMalloc(&d_peers, sizeof(int) * peers.size()));
    TETMF_CUDA(cudaMalloc(&d_bases, sizeof(double*) * peers.size()));
    TETMF_CUDA(cudaMemcpyAsync(d_peers, peers.data(), sizeof(int) * peers.size(), cudaMemcpyHostToDevice, s));
    lsa_bases_kernel<<<1, 256, 0, s>>>(ch->win_, ch->dc_, d_peers, static_cast<int>(peers.size()), d_bases);
    check_launch("lsa_bases");
    ch->peer_base.resize(peers.size());
    TETMF_CUDA(cudaMemcpyAsync(ch->peer_base.data(), d_bases, sizeof(double*) * peers.size(),
                               cudaMemcpyDeviceToHost, s));
    TETMF_CUDA(cudaStreamSynchronize(s));
    cudaFree(d_peers);
    cudaFree(d_bases);
  }
  return ch;
}

} // namespace tetmf

// exchange.hpp -- cross-rank interface exchange (the path's one collective).
//
// After the element kernels, every rank holds macro-local partial sums on
// the carriers its macros share with macros of other ranks. The exchange is
// a sparse neighbour SUM-exchange (not an all-reduce):
//   1. pack:    send[p][k] = +-y[local copy]      (owner orientation)
//   2. NCCL grouped send/recv with every peer rank over NVLink
//   3. combine: per shared carrier, sum ALL copies in ascending global macro
//               id order (local values or receive-buffer entries), write the
//               total back to the local copies.
// Summation order depends only on global macro ids, so every rank (and the
// single-rank run) produces bitwise-identical totals.
//
// The pack / combine bodies are __host__ __device__ so the exact product code
// also runs on the CPU for the world_size-2 gloo tests (tests/test_dist.py).
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include <cuda_runtime.h>

#include "lattice.hpp"
#include "layout.hpp"
#include "mesh.hpp"
#include "device.hpp"
#include "transport.hpp"

namespace tetmf {

struct ExchangePlan {
  // peers and per-peer send / receive counts (entries of doubles)
  std::vector<int> peers;
  std::vector<i64> send_offsets;  // size peers+1
  std::vector<i64> recv_offsets;  // size peers+1
  // send entries: (storage index << 1) | negative
  std::vector<i64> send_index;
  // combine CSR over cross-rank carriers; entry = (v << 2) | (remote << 1) | negative
  // v = storage index (local) or position in the concatenated receive buffer
  std::vector<i64> group_offsets;
  std::vector<i64> group_entries;
  i64 num_groups() const { return static_cast<i64>(group_offsets.size()) - 1; }
  i64 send_total() const { return send_offsets.empty() ? 0 : send_offsets.back(); }
  i64 recv_total() const { return recv_offsets.empty() ? 0 : recv_offsets.back(); }
};

// rank_of[m] = rank storing macro m. Local-only groups are excluded here
// (they are summed by the interface kernel, K4).
ExchangePlan build_exchange_plan(const MacroMesh& mesh, const Topology& topo, const LevelLayout& lay,
                                 const std::vector<int>& rank_of, int rank);

// Interface groups whose copies are all on this rank.
InterfaceGroups local_groups_only(const MacroMesh& mesh, const Topology& topo, const LevelLayout& lay,
                                  const std::vector<int>& rank_of, int rank);

// ---- (macro, z-slab) partition (SURVEY.md 8(e), config 4 strong scaling).
// A unit is a range of lattice planes [za, zb) of one macro; rank r computes
// y at the P1 points of its units (the stencil kernel needs x of the ghost
// planes za - 1 and zb, read from the rank's own copy). Cuts lie on multiples
// of the K1 box height (8 planes); units are contiguous in (macro, plane)
// order with balanced point counts. Every rank stores every macro (the
// storage outside its units is not computed).
struct SlabUnit {
  int macro, za, zb;
};
constexpr int kSlabAlign = 8;  // K1 box planes (k_p1_stencil5.cu kBoxPlanes6)
// all ranks' units: result[r] = the units of rank r (ascending macro)
std::vector<std::vector<SlabUnit>> slab_partition(int num_macros, int n, int nranks);
// rank computing the P1 point of plane z in macro m
int slab_rank(const std::vector<std::vector<SlabUnit>>& units, int macro, int z);

// Exchange plan and rank-local groups when every rank stores every macro and
// each copy belongs to copy_rank(macro, z) (slab partition)
ExchangePlan build_exchange_plan_slab(const MacroMesh& mesh, const Topology& topo, const LevelLayout& lay,
                                      const std::vector<std::vector<SlabUnit>>& units, int rank);
InterfaceGroups local_groups_slab(const MacroMesh& mesh, const Topology& topo, const LevelLayout& lay,
                                  const std::vector<std::vector<SlabUnit>>& units, int rank);

// signed_values = false: orientation signs ignored (operator diagonals)
TM_HD void exchange_pack_one(const double* y, const i64* send_index, double* send, i64 i,
                             bool signed_values = true) {
  const i64 e = send_index[i];
  const double v = y[e >> 1];
  send[i] = (signed_values && (e & 1)) ? -v : v;
}

// put mode: entry i goes straight into the receive window of peer slot
// dst_peer[i] at position dst_off[i] (exchange_put_offsets), same value as the pack
TM_HD void exchange_put_one(const double* y, const i64* send_index, const i64* dst_off, const int* dst_peer,
                            double* const* peer_win, i64 i, bool signed_values = true) {
  const i64 e = send_index[i];
  const double v = y[e >> 1];
  peer_win[dst_peer[i]][dst_off[i]] = (signed_values && (e & 1)) ? -v : v;
}

// per send entry: the peer slot it goes to and its position in that peer's
// receive buffer (peer_off from put_peer_offsets)
void exchange_put_targets(const ExchangePlan& plan, const std::vector<i64>& peer_off, std::vector<i64>& dst_off,
                          std::vector<int>& dst_peer);

// owner = true: ghost update instead of a sum -- every local copy takes the
// owner copy's value (the first entry: entries are in ascending macro id)
TM_HD void exchange_combine_one(double* y, const double* recv, const i64* offsets, const i64* entries, i64 g,
                                bool signed_values = true, bool owner = false) {
  const i64 b = offsets[g], e = offsets[g + 1];
  double s = 0.0;
  for (i64 k = b; k < (owner ? b + 1 : e); ++k) {
    const i64 c = entries[k];
    const double v = (c & 2) ? recv[c >> 2] : y[c >> 2];
    s += (signed_values && (c & 1)) ? -v : v;
  }
  for (i64 k = b; k < e; ++k) {
    const i64 c = entries[k];
    if (c & 2) continue;
    y[c >> 2] = (signed_values && (c & 1)) ? -s : s;
  }
}

// K4 body for rank-local groups (same arithmetic as interface_sum_kernel)
TM_HD void interface_sum_one(double* y, const i64* offsets, const i64* copies, i64 g) {
  const i64 b = offsets[g], e = offsets[g + 1];
  double s = 0.0;
  for (i64 k = b; k < e; ++k) {
    const i64 c = copies[k];
    const double v = y[c >> 1];
    s += (c & 1) ? -v : v;
  }
  for (i64 k = b; k < e; ++k) {
    const i64 c = copies[k];
    y[c >> 1] = (c & 1) ? -s : s;
  }
}

// Device side of one level's plan; the bytes move through a Transport
// (NCCL send/recv, or device-to-device copies between loopback virtual ranks).
class Exchange {
public:
  // put = true: direct-put mode (transport PutChannel: the pack kernel stores
  // into the peers' receive windows; no send buffer, no send/recv calls)
  Exchange(ExchangePlan plan, Transport* transport, bool put = false);
  ~Exchange();
  // pack -> send/recv -> combine on `stream` (signed_values = false: ND1
  // orientation signs ignored, for operator diagonals). Collective: every
  // rank calls it, also ranks without cross-rank carriers.
  void run(double* y, cudaStream_t stream, bool signed_values = true);
  // ghost update: every copy of a cross-rank carrier := its owner's value
  void broadcast_owner(double* y, cudaStream_t stream);
  const ExchangePlan& plan() const { return plan_; }

  // Fused put (put mode, unsigned send entries): the producing kernel stores
  // every sent value straight into the peers' windows (FusedPut) while it
  // computes y, and fused_finish() does what run() does after its put
  // kernel: fence, combine, flip the window half. fused_begin() returns the
  // targets of the current half; storage_size = doubles of the level buffer
  // (the slot map is built on the first call). No put channel or a signed
  // entry: fusable() is false and the caller uses run().
  bool fusable() const;
  FusedPut fused_begin(i64 storage_size);
  void fused_finish(double* y, cudaStream_t stream);

private:
  void run_mode(double* y, cudaStream_t stream, bool signed_values, bool owner);
  ExchangePlan plan_;
  Transport* transport_;
  i64* d_send_index_ = nullptr;
  i64* d_group_offsets_ = nullptr;
  i64* d_group_entries_ = nullptr;
  double* d_send_ = nullptr;
  double* d_recv_ = nullptr;
  // put mode
  std::unique_ptr<PutChannel> put_;
  i64* d_dst_off_ = nullptr;
  int* d_dst_peer_ = nullptr;
  double** d_peer_win_ = nullptr;  // [2 parities][peers]: window half bases
  int parity_ = 0;
  // fused put: per storage slot the first send entry, per entry the next of the same slot
  int* d_first_ = nullptr;
  int* d_chain_ = nullptr;
  i64* d_dst_ = nullptr;  // per entry: (peer slot << 48) | offset in the window half
  i64 first_size_ = -1;
};

} // namespace tetmf

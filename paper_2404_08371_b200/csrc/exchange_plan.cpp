// exchange_plan.cpp -- host-side exchange planning (no CUDA calls).
#include "exchange.hpp"

#include <algorithm>
#include <map>

#include "common.hpp"

namespace tetmf {

namespace {

template <typename F>
void for_each_group(const std::vector<SharedCarrier>& sc, F&& f) {
  for (std::size_t i = 0; i < sc.size();) {
    std::size_t j = i;
    while (j < sc.size() && sc[j].owner == sc[i].owner && sc[j].owner_slot == sc[i].owner_slot) ++j;
    f(i, j);
    i = j;
  }
}

} // namespace

InterfaceGroups local_groups_only(const MacroMesh& mesh, const Topology& topo, const LevelLayout& lay,
                                  const std::vector<int>& rank_of, int rank) {
  const auto sc = shared_carriers(mesh, topo, lay);
  InterfaceGroups g;
  g.offsets.push_back(0);
  for_each_group(sc, [&](std::size_t i, std::size_t j) {
    const auto& sharers = topo.sharers[sc[i].macro][sc[i].mask];
    for (int s : sharers)
      if (rank_of[s] != rank) return;  // cross-rank: exchange plan
    if (j - i != sharers.size()) fail_internal("interface: copy count does not match sharers");
    for (std::size_t k = i; k < j; ++k) {
      g.copies.push_back((sc[k].index << 1) | (sc[k].negative ? 1 : 0));
      g.copy_macro.push_back(sc[k].macro);
    }
    g.offsets.push_back(static_cast<i64>(g.copies.size()));
  });
  return g;
}

ExchangePlan build_exchange_plan(const MacroMesh& mesh, const Topology& topo, const LevelLayout& lay,
                                 const std::vector<int>& rank_of, int rank) {
  const auto sc = shared_carriers(mesh, topo, lay);
  // pass 1: peers and per-peer send / receive entries (in group key order)
  std::map<int, std::vector<i64>> send;   // peer -> send entries
  std::map<int, i64> recvCount;           // peer -> received values
  struct Pending {
    std::size_t i, j;
    std::vector<int> sharers;
    std::vector<i64> recvPos;  // per remote sharer: position within its peer's stream
  };
  std::vector<Pending> groups;
  for_each_group(sc, [&](std::size_t i, std::size_t j) {
    const auto& sharers = topo.sharers[sc[i].macro][sc[i].mask];
    bool cross = false;
    for (int s : sharers) cross |= rank_of[s] != rank;
    if (!cross) return;
    Pending p{i, j, sharers, {}};
    std::vector<int> peersHere;
    for (int s : sharers)
      if (rank_of[s] != rank && std::find(peersHere.begin(), peersHere.end(), rank_of[s]) == peersHere.end())
        peersHere.push_back(rank_of[s]);
    for (int peer : peersHere)
      for (std::size_t k = i; k < j; ++k)
        send[peer].push_back((sc[k].index << 1) | (sc[k].negative ? 1 : 0));
    for (int s : sharers)
      if (rank_of[s] != rank) p.recvPos.push_back(recvCount[rank_of[s]]++);
    groups.push_back(std::move(p));
  });

  ExchangePlan plan;
  for (const auto& [peer, _] : send) plan.peers.push_back(peer);
  for (const auto& [peer, _] : recvCount)
    if (!send.count(peer)) fail_internal("exchange: asymmetric peer relation");
  plan.send_offsets.push_back(0);
  plan.recv_offsets.push_back(0);
  std::map<int, i64> recvBase;
  for (int peer : plan.peers) {
    const auto& s = send[peer];
    plan.send_index.insert(plan.send_index.end(), s.begin(), s.end());
    plan.send_offsets.push_back(static_cast<i64>(plan.send_index.size()));
    recvBase[peer] = plan.recv_offsets.back();
    plan.recv_offsets.push_back(plan.recv_offsets.back() + recvCount[peer]);
  }
  // pass 2: combine entries, all sharers in ascending global macro order
  plan.group_offsets.push_back(0);
  for (const auto& p : groups) {
    std::size_t k = p.i, r = 0;
    for (int s : p.sharers) {
      if (rank_of[s] == rank) {
        if (k >= p.j || sc[k].macro != s) fail_internal("exchange: local copy order mismatch");
        plan.group_entries.push_back((sc[k].index << 2) | (sc[k].negative ? 1 : 0));
        ++k;
      } else {
        plan.group_entries.push_back(((recvBase[rank_of[s]] + p.recvPos[r]) << 2) | 2);
        ++r;
      }
    }
    plan.group_offsets.push_back(static_cast<i64>(plan.group_entries.size()));
  }
  return plan;
}

} // namespace tetmf

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

std::vector<std::vector<SlabUnit>> slab_partition(int num_macros, int n, int nranks) {
  if (nranks < 1 || num_macros < 1) fail_arg("slab partition: bad rank / macro count");
  // blocks of kSlabAlign planes, work = P1 points in the block
  struct Block {
    int macro, za, zb;
    double work;
  };
  std::vector<Block> blocks;
  double total = 0.0;
  for (int m = 0; m < num_macros; ++m)
    for (int za = 0; za <= n; za += kSlabAlign) {
      const int zb = std::min(za + kSlabAlign, n + 1);
      double w = 0.0;
      for (int z = za; z < zb; ++z) w += 0.5 * double(n + 1 - z) * double(n + 2 - z);
      blocks.push_back({m, za, zb, w});
      total += w;
    }
  std::vector<std::vector<SlabUnit>> out(nranks);
  double cum = 0.0;
  for (const Block& b : blocks) {
    const double mid = cum + 0.5 * b.work;  // the block goes to the rank whose share holds its midpoint
    cum += b.work;
    const int r = std::min(nranks - 1, static_cast<int>(mid / total * nranks));
    auto& u = out[r];
    if (!u.empty() && u.back().macro == b.macro && u.back().zb == b.za)
      u.back().zb = b.zb;
    else
      u.push_back({b.macro, b.za, b.zb});
  }
  return out;
}

int slab_rank(const std::vector<std::vector<SlabUnit>>& units, int macro, int z) {
  for (std::size_t r = 0; r < units.size(); ++r)
    for (const SlabUnit& u : units[r])
      if (u.macro == macro && z >= u.za && z < u.zb) return static_cast<int>(r);
  fail_internal("slab partition: no rank holds macro " + std::to_string(macro) + " plane " + std::to_string(z));
}

namespace {

// groups of all copies of each shared carrier, with each copy's rank
template <typename F>
void for_each_slab_group(const std::vector<SharedCarrier>& sc, const std::vector<std::vector<SlabUnit>>& units,
                         F&& f) {
  for_each_group(sc, [&](std::size_t i, std::size_t j) {
    std::vector<int> ranks;
    for (std::size_t k = i; k < j; ++k) ranks.push_back(slab_rank(units, sc[k].macro, sc[k].z));
    f(i, j, ranks);
  });
}

} // namespace

InterfaceGroups local_groups_slab(const MacroMesh& mesh, const Topology& topo, const LevelLayout& lay,
                                  const std::vector<std::vector<SlabUnit>>& units, int rank) {
  if (lay.space != Space::P1) fail_arg("slab partition: P1 functions only");
  const auto sc = shared_carriers(mesh, topo, lay);
  InterfaceGroups g;
  g.offsets.push_back(0);
  for_each_slab_group(sc, units, [&](std::size_t i, std::size_t j, const std::vector<int>& ranks) {
    for (int r : ranks)
      if (r != rank) return;  // some copy elsewhere (exchange), or none here
    if (j - i != topo.sharers[sc[i].macro][sc[i].mask].size())
      fail_internal("interface: copy count does not match sharers");
    for (std::size_t k = i; k < j; ++k) {
      g.copies.push_back((sc[k].index << 1) | (sc[k].negative ? 1 : 0));
      g.copy_macro.push_back(sc[k].macro);
    }
    g.offsets.push_back(static_cast<i64>(g.copies.size()));
  });
  return g;
}

ExchangePlan build_exchange_plan_slab(const MacroMesh& mesh, const Topology& topo, const LevelLayout& lay,
                                      const std::vector<std::vector<SlabUnit>>& units, int rank) {
  if (lay.space != Space::P1) fail_arg("slab partition: P1 functions only");
  const auto sc = shared_carriers(mesh, topo, lay);  // every rank stores every macro: all copies, same order
  std::map<int, std::vector<i64>> send;  // peer -> my copies of the groups it shares, in group order
  std::map<int, i64> recvCount;
  struct Pending {
    std::size_t i, j;
    std::vector<int> ranks;
    std::vector<i64> recvPos;  // per copy: position within its peer's stream (-1 local)
  };
  std::vector<Pending> groups;
  for_each_slab_group(sc, units, [&](std::size_t i, std::size_t j, const std::vector<int>& ranks) {
    bool mine = false, other = false;
    for (int r : ranks) (r == rank ? mine : other) = true;
    if (!mine || !other) return;
    std::vector<int> peers;
    for (int r : ranks)
      if (r != rank && std::find(peers.begin(), peers.end(), r) == peers.end()) peers.push_back(r);
    for (int p : peers)
      for (std::size_t k = i; k < j; ++k)
        if (ranks[k - i] == rank) send[p].push_back((sc[k].index << 1) | (sc[k].negative ? 1 : 0));
    Pending pd{i, j, ranks, {}};
    for (std::size_t k = i; k < j; ++k) pd.recvPos.push_back(ranks[k - i] == rank ? -1 : recvCount[ranks[k - i]]++);
    groups.push_back(std::move(pd));
  });
  ExchangePlan plan;
  for (const auto& [peer, _] : send) plan.peers.push_back(peer);
  for (const auto& [peer, _] : recvCount)
    if (!send.count(peer)) fail_internal("exchange: asymmetric peer relation");
  plan.send_offsets.push_back(0);
  plan.recv_offsets.push_back(0);
  std::map<int, i64> recvBase;
  for (int peer : plan.peers) {
    const auto& v = send[peer];
    plan.send_index.insert(plan.send_index.end(), v.begin(), v.end());
    plan.send_offsets.push_back(static_cast<i64>(plan.send_index.size()));
    recvBase[peer] = plan.recv_offsets.back();
    plan.recv_offsets.push_back(plan.recv_offsets.back() + recvCount[peer]);
  }
  // combine: all copies in ascending macro order (sc order within a group)
  plan.group_offsets.push_back(0);
  for (const auto& pd : groups) {
    for (std::size_t k = pd.i; k < pd.j; ++k) {
      const int r = pd.ranks[k - pd.i];
      if (r == rank)
        plan.group_entries.push_back((sc[k].index << 2) | (sc[k].negative ? 1 : 0));
      else
        plan.group_entries.push_back(((recvBase[r] + pd.recvPos[k - pd.i]) << 2) | 2);
    }
    plan.group_offsets.push_back(static_cast<i64>(plan.group_entries.size()));
  }
  return plan;
}

} // namespace tetmf

// layout.cpp -- storage layout, reference numbering, interface groups.
#include "layout.hpp"

#include <algorithm>
#include <atomic>
#include <memory>
#include <numeric>
#include <string>
#include <thread>
#include <tuple>

#include "common.hpp"

namespace tetmf {

LevelLayout LevelLayout::make(Space s, int level, int num_macros_global, const std::vector<int>& macros) {
  if (level < 0 || level > 14) fail_arg("level out of range (0..14)");
  // level 0 (n = 1): the edge lattices have extent 0, one anchor per class
  LevelLayout l;
  l.space = s;
  l.level = level;
  l.n = 1 << level;
  if (s == Space::P1) {
    l.class_stride = 0;
    l.macro_stride = round_up(tet_count(l.n), 32);
  } else {
    l.class_stride = round_up(tet_count(l.n - 1), 32);
    l.macro_stride = 7 * l.class_stride + (s == Space::P2 ? p2_vertex_stride(l.n) : 0);
  }
  l.macros = macros;
  std::sort(l.macros.begin(), l.macros.end());
  l.local_of.assign(num_macros_global, -1);
  for (std::size_t i = 0; i < l.macros.size(); ++i) {
    const int m = l.macros[i];
    if (m < 0 || m >= num_macros_global) fail_arg("layout: macro id out of range");
    if (l.local_of[m] >= 0) fail_arg("layout: duplicate macro id");
    l.local_of[m] = static_cast<int>(i);
  }
  return l;
}

std::array<int, 3> map_point(const MacroMesh& mesh, int n, int m, std::array<int, 3> p, int m2) {
  const auto w = bary(n, p[0], p[1], p[2]);
  const auto& t = mesh.tets[m];
  const auto& t2 = mesh.tets[m2];
  int w2[4] = {0, 0, 0, 0};
  for (int i = 0; i < 4; ++i) {
    if (w[i] == 0) continue;
    int j = 0;
    while (j < 4 && t2[j] != t[i]) ++j;
    if (j == 4) fail_internal("map_point: carrier not contained in target macro");
    w2[j] = w[i];
  }
  return {w2[1], w2[2], w2[3]};
}

namespace {

// carriers based at lattice point (x,y,z): calls f(cls, mask, anchor, slot)
template <typename F>
void point_carriers(Space s, int n, i64 cs, int x, int y, int z, F&& f) {
  const unsigned mb = support_mask(bary(n, x, y, z));
  if (s == Space::P1 || s == Space::P2) {
    f(-1, mb, std::array<int, 3>{x, y, z}, lattice_index(n, x, y, z));
    if (s == Space::P1) return;
  }
  const i64 eoff = s == Space::P2 ? p2_vertex_stride(n) : 0;
  for (int c = 0; c < 7; ++c) {
    const int tx = x + kEdgeDir[c][0], ty = y + kEdgeDir[c][1], tz = z + kEdgeDir[c][2];
    if (tx < 0 || ty < 0 || tz < 0 || tx + ty + tz > n) continue;
    const Off3 b = edge_base_from_anchor(c);
    const std::array<int, 3> a = {x - b.x, y - b.y, z - b.z};
    f(c, mb | support_mask(bary(n, tx, ty, tz)), a, eoff + c * cs + lattice_index(n - 1, a[0], a[1], a[2]));
  }
}

// boundary base points (any barycentric weight zero), any order
template <typename F>
void for_each_boundary_point(int n, F&& f) {
  for (int z = 0; z <= n; ++z)
    for (int y = 0; y <= n - z; ++y) {
      const int len = n - z - y + 1;
      if (z == 0 || y == 0) {
        for (int x = 0; x < len; ++x) f(x, y, z);
      } else {
        f(0, y, z);
        if (len > 1) f(len - 1, y, z);
      }
    }
}

// Owned-carrier prefix counts of one macro in reference record order
// (z, y, x, kindClass): rowPrefix[r] = owned carriers in rows before r.
struct OwnedPrefix {
  Space s;
  int n;
  i64 cs;
  std::array<bool, 16> owned;
  std::vector<i64> rowPrefix;

  int count_at(int x, int y, int z) const {
    int c = 0;
    point_carriers(s, n, cs, x, y, z, [&](int, unsigned mask, const std::array<int, 3>&, i64) {
      c += owned[mask] ? 1 : 0;
    });
    return c;
  }
  // owned carriers with base x' < x in row (y,z)
  i64 row_count_before(int x, int y, int z) const {
    const int len = n - z - y + 1;
    i64 c = 0;
    const int lo = std::min(x, 2);
    for (int xx = 0; xx < lo; ++xx) c += count_at(xx, y, z);
    const int midEnd = std::min(x, std::max(2, len - 3));
    if (midEnd > 2) c += static_cast<i64>(midEnd - 2) * count_at(2, y, z);
    for (int xx = std::max(2, len - 3); xx < x; ++xx) c += count_at(xx, y, z);
    return c;
  }
  static i64 row_id(int n, int z, int y) { return static_cast<i64>(z) * (n + 1) - static_cast<i64>(z) * (z - 1) / 2 + y; }

  OwnedPrefix(Space s_, int n_, i64 cs_, const std::array<bool, 16>& own) : s(s_), n(n_), cs(cs_), owned(own) {
    const i64 rows = tri_count(n);
    rowPrefix.assign(rows + 1, 0);
    i64 r = 0;
    for (int z = 0; z <= n; ++z)
      for (int y = 0; y <= n - z; ++y, ++r)
        rowPrefix[r + 1] = rowPrefix[r] + row_count_before(n - z - y + 1, y, z);
  }
  i64 total() const { return rowPrefix.back(); }
  // rank of the carrier (cls at base point) among owned carriers
  i64 rank(int x, int y, int z, int cls) const {
    i64 c = rowPrefix[row_id(n, z, y)] + row_count_before(x, y, z);
    point_carriers(s, n, cs, x, y, z, [&](int cc, unsigned mask, const std::array<int, 3>&, i64) {
      if (cc < cls && owned[mask]) ++c;
    });
    return c;
  }
};

std::array<bool, 16> owned_masks(const Topology& topo, int m) {
  std::array<bool, 16> o{};
  for (unsigned mask = 0; mask < 16; ++mask) o[mask] = topo.owner(m, mask) == m;
  return o;
}

// Reference vertex key of lattice point p of macro m: (global vertex id,
// weight) pairs of nonzero weights, sorted by id (fespace.cpp:124-142).
struct VKey {
  int k = 0;
  std::array<std::pair<int, int>, 4> e;
  bool operator<(const VKey& o) const {
    const int kk = std::min(k, o.k);
    for (int i = 0; i < kk; ++i) {
      if (e[i] != o.e[i]) return e[i] < o.e[i];
    }
    return k < o.k;
  }
};
VKey vkey(const MacroMesh& mesh, int m, int n, int x, int y, int z) {
  const auto w = bary(n, x, y, z);
  VKey key;
  for (int v = 0; v < 4; ++v)
    if (w[v] > 0) key.e[key.k++] = {mesh.tets[m][v], w[v]};
  std::sort(key.e.begin(), key.e.begin() + key.k);
  return key;
}

// base and tip (unshifted) of an edge carrier given its anchor
inline void edge_endpoints(int cls, const std::array<int, 3>& a, std::array<int, 3>& b, std::array<int, 3>& t) {
  const Off3 bo = edge_base_from_anchor(cls);
  b = {a[0] + bo.x, a[1] + bo.y, a[2] + bo.z};
  t = {b[0] + kEdgeDir[cls][0], b[1] + kEdgeDir[cls][1], b[2] + kEdgeDir[cls][2]};
}

struct Mapped {
  int x, y, z, cls;  // base point (P1) or anchor (ND1) in the target macro
  i64 slot;
  bool flipped;      // direction reversed relative to the target's canonical
};

Mapped map_carrier(const MacroMesh& mesh, const LevelLayout& lay, int m, int cls,
                   const std::array<int, 3>& pa, int m2) {
  const int n = lay.n;
  if (cls < 0) {
    const auto q = map_point(mesh, n, m, pa, m2);
    return {q[0], q[1], q[2], -1, lattice_index(n, q[0], q[1], q[2]), false};
  }
  std::array<int, 3> b, t;
  edge_endpoints(cls, pa, b, t);
  const auto b2 = map_point(mesh, n, m, b, m2);
  const auto t2 = map_point(mesh, n, m, t, m2);
  bool flipped = false;
  const int c2 = edge_class_of(t2[0] - b2[0], t2[1] - b2[1], t2[2] - b2[2], &flipped);
  if (c2 < 0) fail_internal("map_carrier: not a lattice edge after mapping");
  const std::array<int, 3> a2 = {std::min(b2[0], t2[0]), std::min(b2[1], t2[1]), std::min(b2[2], t2[2])};
  const bool p2 = lay.space == Space::P2;  // P2 edge DoFs are unsigned
  return {a2[0], a2[1], a2[2], c2,
          (p2 ? p2_vertex_stride(n) : 0) + c2 * lay.class_stride + lattice_index(n - 1, a2[0], a2[1], a2[2]),
          p2 ? false : flipped};
}

// unshifted base (record coordinates) of a carrier given its anchor
inline std::array<int, 3> record_base(int cls, const std::array<int, 3>& a) {
  if (cls < 0) return a;
  const Off3 bo = edge_base_from_anchor(cls);
  return {a[0] + bo.x, a[1] + bo.y, a[2] + bo.z};
}

} // namespace

bool carrier_interior(const Topology& topo, int m, int n, const Carrier& c) {
  // boundary iff the carrier lies in a boundary face plane of any macro that
  // holds it (fespace.cpp:207-214; flags OR-merged over copies, :226)
  (void)n;
  return !((topo.dirichlet_mask[m] >> (c.mask & 15u)) & 1u);
}

RefNumbering build_ref_numbering(const MacroMesh& mesh, const Topology& topo, const LevelLayout& lay) {
  const int M = mesh.num_tets();
  const int n = lay.n;
  const i64 cs = lay.class_stride;
  // per-mask carrier histogram of one macro (identical for every macro)
  std::array<i64, 16> hist{};
  {
    for (int z = 0; z <= n; ++z)
      for (int y = 0; y <= n - z; ++y) {
        const int len = n - z - y + 1;
        auto add_point = [&](int x, i64 mult) {
          point_carriers(lay.space, n, cs, x, y, z,
                         [&](int, unsigned mask, const std::array<int, 3>&, i64) { hist[mask] += mult; });
        };
        for (int x = 0; x < std::min(len, 2); ++x) add_point(x, 1);
        const int midEnd = std::max(2, len - 3);
        if (midEnd > 2) add_point(2, midEnd - 2);
        for (int x = std::max(2, len - 3); x < len; ++x) add_point(x, 1);
      }
  }
  std::vector<i64> base(M + 1, 0);
  for (int m = 0; m < M; ++m) {
    const auto own = owned_masks(topo, m);
    i64 c = 0;
    for (unsigned mask = 0; mask < 16; ++mask)
      if (own[mask]) c += hist[mask];
    base[m + 1] = base[m] + c;
  }
  RefNumbering out;
  out.num_dofs = base[M];
  out.map.assign(lay.total(), -1);

  // lazily built owned-prefix tables of owner macros
  std::vector<std::unique_ptr<OwnedPrefix>> prefix(M);
  auto prefix_of = [&](int m) -> const OwnedPrefix& {
    if (!prefix[m]) prefix[m] = std::make_unique<OwnedPrefix>(lay.space, n, cs, owned_masks(topo, m));
    return *prefix[m];
  };
  // owners needed by the stored macros' boundary carriers (build serially)
  for (int m : lay.macros)
    for (unsigned mask = 0; mask < 16; ++mask) prefix_of(topo.owner(m, mask));

  auto vkl = [&](int m, const std::array<int, 3>& p, const std::array<int, 3>& q) {
    return vkey(mesh, m, n, p[0], p[1], p[2]) < vkey(mesh, m, n, q[0], q[1], q[2]);
  };

  auto fill_macro = [&](int li) {
    const int m = lay.macros[li];
    i64* map = out.map.data() + static_cast<i64>(li) * lay.macro_stride;
    const auto own = owned_masks(topo, m);
    i64 next = base[m];
    // (1) owned carriers: consecutive ids in record order. Interior carriers
    // of ND1 are sign-constant per class: cache the
    // key-order comparison per class for edges with both endpoints interior.
    int signCache[7];
    for (int c = 0; c < 7; ++c) signCache[c] = -1;
    for_each_carrier(lay.space, n, [&](const Carrier& c) {
      bool neg = false;
      if (c.cls >= 0 && lay.space == Space::ND1) {  // P2 edge DoFs carry no orientation
        std::array<int, 3> b, t;
        edge_endpoints(c.cls, {c.x, c.y, c.z}, b, t);
        const bool inner = support_mask(bary(n, b[0], b[1], b[2])) == 15u &&
                           support_mask(bary(n, t[0], t[1], t[2])) == 15u;
        if (inner && signCache[c.cls] >= 0) {
          neg = signCache[c.cls] == 1;
        } else {
          neg = !vkl(m, b, t);
          if (inner) signCache[c.cls] = neg ? 1 : 0;
        }
      }
      if (own[c.mask]) {
        map[c.slot] = (next << 2) | (neg ? 2 : 0) | 1;
        ++next;
      } else {
        map[c.slot] = neg ? -2 : -3;  // provisional: resolved below
      }
    });
    if (next != base[m + 1]) fail_internal("ref numbering: owned count mismatch");
    // (2) non-owned copies: id of the owner's record
    for_each_boundary_point(n, [&](int x, int y, int z) {
      point_carriers(lay.space, n, cs, x, y, z, [&](int cls, unsigned mask, const std::array<int, 3>& a, i64 slot) {
        if (own[mask]) return;
        const int o = topo.owner(m, mask);
        const Mapped mp = map_carrier(mesh, lay, m, cls, a, o);
        const auto rb = record_base(mp.cls, {mp.x, mp.y, mp.z});
        const i64 id = base[o] + prefix_of(o).rank(rb[0], rb[1], rb[2], mp.cls);
        const bool neg = map[slot] == -2;
        map[slot] = (id << 2) | (neg ? 2 : 0);
      });
    });
  };

  const int nthreads = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 32u));
  std::vector<std::thread> pool;
  std::atomic<int> nextMacro{0};
  for (int t = 0; t < nthreads; ++t)
    pool.emplace_back([&] {
      for (int li; (li = nextMacro.fetch_add(1)) < static_cast<int>(lay.macros.size());) fill_macro(li);
    });
  for (auto& th : pool) th.join();
  return out;
}

std::vector<SharedCarrier> shared_carriers(const MacroMesh& mesh, const Topology& topo, const LevelLayout& lay) {
  std::vector<SharedCarrier> out;
  const int n = lay.n;
  for (std::size_t li = 0; li < lay.macros.size(); ++li) {
    const int m = lay.macros[li];
    const i64 baseIdx = static_cast<i64>(li) * lay.macro_stride;
    for_each_boundary_point(n, [&](int x, int y, int z) {
      point_carriers(lay.space, n, lay.class_stride, x, y, z,
                     [&](int cls, unsigned mask, const std::array<int, 3>& a, i64 slot) {
                       if (topo.sharers[m][mask].size() < 2) return;
                       const int o = topo.owner(m, mask);
                       const Mapped mp = o == m ? Mapped{a[0], a[1], a[2], cls, slot, false}
                                                : map_carrier(mesh, lay, m, cls, a, o);
                       out.push_back({o, mp.slot, m, baseIdx + slot, mp.flipped, mask, a[2]});
                     });
    });
  }
  std::sort(out.begin(), out.end(), [](const SharedCarrier& a, const SharedCarrier& b) {
    return std::tie(a.owner, a.owner_slot, a.macro) < std::tie(b.owner, b.owner_slot, b.macro);
  });
  return out;
}

InterfaceGroups build_interface_groups(const MacroMesh& mesh, const Topology& topo, const LevelLayout& lay) {
  const auto sc = shared_carriers(mesh, topo, lay);
  InterfaceGroups g;
  g.offsets.push_back(0);
  for (std::size_t i = 0; i < sc.size();) {
    std::size_t j = i;
    while (j < sc.size() && sc[j].owner == sc[i].owner && sc[j].owner_slot == sc[i].owner_slot) ++j;
    if (j - i >= 2) {  // only groups with >= 2 local copies need a local sum
      for (std::size_t k = i; k < j; ++k) {
        g.copies.push_back((sc[k].index << 1) | (sc[k].negative ? 1 : 0));
        g.copy_macro.push_back(sc[k].macro);
      }
      g.offsets.push_back(static_cast<i64>(g.copies.size()));
    }
    i = j;
  }
  return g;
}

} // namespace tetmf

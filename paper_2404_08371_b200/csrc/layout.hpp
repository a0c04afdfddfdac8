// layout.hpp -- level-indexed function storage layout and the host-side
// index machinery around it (host C++).
//
// A Function of space S at level L stores, for every macro-tetrahedron it
// holds, the complete closure of the macro's lattice (interior plus its own
// copies of face/edge/vertex carriers). Carriers that several macros share
// (macro-primitive faces, edges, vertices) are therefore stored once per
// sharing macro; the apply's interface step (K4) keeps the copies equal.
//
// Reference anchors:
//  * global numbering / interface merge: DoFIndexer::build fespace.cpp:182-307
//  * slot maps with +-(id+1) signs:    DoFIndexer::fill_map fespace.cpp:320-376
//  * ND1 key-ascending orientation:     vertex_key_less fespace.cpp:151-169
//  * interior (Dirichlet) mask:         fespace.cpp:207-214, 304-306
#pragma once

#include <array>
#include <cstdint>
#include <vector>

#include "lattice.hpp"
#include "mesh.hpp"

namespace tetmf {

enum class Space : int { P1 = 0, P2 = 1, ND1 = 2 };  // reference enum order (fespace.hpp:15)

inline i64 round_up(i64 v, i64 a) { return (v + a - 1) / a * a; }

struct LevelLayout {
  Space space = Space::P1;
  int level = 0;
  int n = 1;
  i64 class_stride = 0;  // ND1: padded entries per edge class block
  i64 macro_stride = 0;  // padded entries per macro
  std::vector<int> macros;      // global macro ids stored here, ascending
  std::vector<int> local_of;    // global macro id -> local index or -1
  i64 total() const { return macro_stride * static_cast<i64>(macros.size()); }

  static LevelLayout make(Space s, int level, int num_macros_global, const std::vector<int>& macros);
};

// One carrier (a DoF-carrying lattice point or lattice edge) of a macro.
struct Carrier {
  i64 slot;       // index inside the macro's block
  int x, y, z;    // base point (P1) or anchor (ND1)
  int cls;        // -1 for vertices, else edge class
  unsigned mask;  // support mask: local vertices with nonzero weight
};

// barycentric weights (w0..w3) of lattice point p at extent n
inline std::array<int, 4> bary(int n, int x, int y, int z) { return {n - x - y - z, x, y, z}; }
inline unsigned support_mask(const std::array<int, 4>& w) {
  return (w[0] > 0 ? 1u : 0u) | (w[1] > 0 ? 2u : 0u) | (w[2] > 0 ? 4u : 0u) | (w[3] > 0 ? 8u : 0u);
}

// Maps lattice point p of macro m to the lattice of macro m2 (which must
// contain the support simplex of p). Identical barycentric weights on shared
// global vertices (conforming mesh).
std::array<int, 3> map_point(const MacroMesh& mesh, int n, int m, std::array<int, 3> p, int m2);

// Interior mask of a carrier (1 = not on the domain boundary).
bool carrier_interior(const Topology& topo, int m, int n, const Carrier& c);

// Visits every carrier of macro m in the reference's record order
// (z, y, x, kindClass) with the unshifted base point (fespace.cpp:236-281).
// P2 storage: the vertex block (P1 layout) then the 7 edge-class blocks (ND1
// layout), both 32-padded; edge DoFs are unsigned (midpoint values).
inline i64 p2_vertex_stride(int n) { return round_up(tet_count(n), 32); }

template <typename F>
void for_each_carrier(Space s, int n, F&& f) {
  if (s == Space::P1) {
    i64 slot = 0;
    for (int z = 0; z <= n; ++z)
      for (int y = 0; y <= n - z; ++y)
        for (int x = 0; x <= n - z - y; ++x, ++slot)
          f(Carrier{slot, x, y, z, -1, support_mask(bary(n, x, y, z))});
    return;
  }
  const i64 cs = round_up(tet_count(n - 1), 32);
  const i64 eoff = s == Space::P2 ? p2_vertex_stride(n) : 0;  // edge blocks follow the P2 vertex block
  for (int z = 0; z <= n; ++z)
    for (int y = 0; y <= n - z; ++y)
      for (int x = 0; x <= n - z - y; ++x) {
        const unsigned mb = support_mask(bary(n, x, y, z));
        if (s == Space::P2) f(Carrier{lattice_index(n, x, y, z), x, y, z, -1, mb});  // kindClass 0 first
        for (int c = 0; c < 7; ++c) {
          const int tx = x + kEdgeDir[c][0], ty = y + kEdgeDir[c][1], tz = z + kEdgeDir[c][2];
          if (tx < 0 || ty < 0 || tz < 0 || tx + ty + tz > n) continue;
          const Off3 b = edge_base_from_anchor(c);
          const int ax = x - b.x, ay = y - b.y, az = z - b.z;
          const unsigned mask = mb | support_mask(bary(n, tx, ty, tz));
          f(Carrier{eoff + c * cs + lattice_index(n - 1, ax, ay, az), ax, ay, az, c, mask});
        }
      }
}

// Reference global numbering of every slot of the stored macros:
// entry = (id << 2) | (negative_sign << 1) | is_owner_copy, or -1 for unused
// padding slots. sign = ND1 factor between this macro's canonical edge
// direction and the reference's key-ascending orientation.
struct RefNumbering {
  i64 num_dofs = 0;
  std::vector<i64> map;  // LevelLayout::total() entries
};
RefNumbering build_ref_numbering(const MacroMesh& mesh, const Topology& topo, const LevelLayout& lay);

// Interface groups (K4 input): every carrier shared by >= 2 macros, with all
// stored copies. entry = (storage index << 1) | negative_sign, where sign is
// relative to the owner macro's canonical orientation (ND1 only).
struct InterfaceGroups {
  std::vector<i64> offsets;  // CSR, size groups+1
  std::vector<i64> copies;   // encoded storage indices, copies sorted by macro id
  // multi-rank: per copy, the global macro id (to order sums identically)
  std::vector<int> copy_macro;
  i64 num_groups() const { return static_cast<i64>(offsets.size()) - 1; }
};
// Groups among the macros of `lay` only (single-rank or rank-local part).
InterfaceGroups build_interface_groups(const MacroMesh& mesh, const Topology& topo, const LevelLayout& lay);

// Cross-rank interface description: for every carrier shared with macros
// stored on other ranks, a stable global key (owner macro, owner slot) and
// the sharer macros. Used by the exchange planner (exchange.hpp).
struct SharedCarrier {
  int owner;
  i64 owner_slot;
  int macro;      // holding macro (local)
  i64 index;      // storage index in the local function
  bool negative;  // sign relative to the owner orientation
  unsigned mask;  // support mask in the holding macro (sharers: topo.sharers[macro][mask])
  int z;          // base point (P1) / anchor (ND1) plane in the holding macro
};
std::vector<SharedCarrier> shared_carriers(const MacroMesh& mesh, const Topology& topo, const LevelLayout& lay);

} // namespace tetmf

// lattice.hpp -- index functions of a uniformly refined macro-tetrahedron.
//
// Shared by host C++ and CUDA device code. Everything here is analytic: no
// lookup maps (the reference uses per-macro int32 slot maps, fespace.cpp:
// 309-389; on the GPU they are replaced by these closed forms).
//
// Conventions (identical to the reference):
//  * level L, n = 2^L intervals per macro edge; lattice points p = (x,y,z)
//    with x,y,z >= 0 and x+y+z <= n (mesh.cpp:183-194).
//  * six micro orientations WU, WD, BU, BD, GU, GD with vertex offsets
//    kOffsets (mesh.cpp:22-29); local vertex order = table order.
//  * local edges (0,1),(0,2),(0,3),(1,2),(1,3),(2,3) (fespace.hpp:27-28).
//  * seven edge classes kEdgeDirs (fespace.hpp:32-33), canonical direction
//    = first nonzero component positive.
//
// Storage (this library's own layout):
//  * vertex lattice of extent n: P(n) = (n+1)(n+2)(n+3)/6 doubles, x fastest,
//    then y, then z (row (y,z) holds n+1-y-z points).
//  * edge lattice: 7 class blocks, each a vertex lattice of extent n-1 indexed
//    by the edge's ANCHOR = componentwise min of its two endpoints. The anchor
//    of every edge of the unit cube [a, a+1]^3 that is "owned" by cube a is a
//    itself, so one index serves all 7 classes (class 6 leaves the outermost
//    layer x+y+z = n-1 unused).
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define TM_HD __host__ __device__ __forceinline__
#else
#define TM_HD inline
#endif

namespace tetmf {

using i64 = std::int64_t;

enum Orient : int { WU = 0, WD = 1, BU = 2, BD = 3, GU = 4, GD = 5 };

struct Off3 { int x, y, z; };

// number of lattice points with x+y+z <= k (0 for k < 0)
TM_HD i64 tet_count(i64 k) { return k < 0 ? 0 : (k + 1) * (k + 2) * (k + 3) / 6; }
// number of points in a triangle x+y <= k
TM_HD i64 tri_count(i64 k) { return k < 0 ? 0 : (k + 1) * (k + 2) / 2; }

// first index of plane z in a lattice of extent n
TM_HD i64 plane_offset(i64 n, i64 z) { return tet_count(n) - tet_count(n - z); }
// first index of row y inside plane z (relative to the plane start)
TM_HD i64 row_offset(i64 n, i64 z, i64 y) { return y * (n - z + 1) - y * (y - 1) / 2; }
// flat index of (x,y,z) in a lattice of extent n
TM_HD i64 lattice_index(i64 n, i64 x, i64 y, i64 z) {
  return plane_offset(n, z) + row_offset(n, z, y) + x;
}

// vertex offsets of the six orientations (mesh.cpp:22-29)

TM_HD constexpr Off3 orient_offset(int o, int i) {
  // packed: per orientation 4 vertices, bits x|y<<1|z<<2
  // WU {0,e1,e2,e3}; WD {e12,e23,e13,e123}; BU {e1,e2,e3,e12};
  // BD {e2,e3,e12,e23}; GU {e1,e3,e12,e13}; GD {e3,e12,e23,e13}
  constexpr unsigned char kPacked[6][4] = {{0, 1, 2, 4}, {3, 6, 5, 7}, {1, 2, 4, 3},
                                           {2, 4, 3, 6}, {1, 4, 3, 5}, {4, 3, 6, 5}};
  const unsigned b = kPacked[o][i];
  return {int(b & 1u), int((b >> 1) & 1u), int((b >> 2) & 1u)};
}

constexpr int kLocalEdge[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
constexpr int kEdgeDir[7][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {1, -1, 0},
                                {1, 0, -1}, {0, 1, -1}, {1, 1, -1}};

// device-usable accessors of the two tables above
TM_HD constexpr int local_edge_vertex(int le, int k) {
  // a = {0,0,0,1,1,2}, b = {1,2,3,2,3,3}
  return k == 0 ? (le < 3 ? 0 : (le < 5 ? 1 : 2)) : (le == 0 ? 1 : (le == 1 || le == 3 ? 2 : 3));
}
TM_HD Off3 edge_dir(int c) {
  switch (c) {
    case 0: return {1, 0, 0};
    case 1: return {0, 1, 0};
    case 2: return {0, 0, 1};
    case 3: return {1, -1, 0};
    case 4: return {1, 0, -1};
    case 5: return {0, 1, -1};
    default: return {1, 1, -1};
  }
}

// class of a lattice direction; *flipped = direction is -canonical.
// returns -1 if not an edge direction (fespace.cpp:60-70)
TM_HD constexpr int edge_class_of(int dx, int dy, int dz, bool* flipped) {
  bool f = false;
  if (dx < 0 || (dx == 0 && dy < 0) || (dx == 0 && dy == 0 && dz < 0)) {
    dx = -dx; dy = -dy; dz = -dz; f = true;
  }
  int c = -1;
  if (dx == 1 && dy == 0 && dz == 0) c = 0;
  else if (dx == 0 && dy == 1 && dz == 0) c = 1;
  else if (dx == 0 && dy == 0 && dz == 1) c = 2;
  else if (dx == 1 && dy == -1 && dz == 0) c = 3;
  else if (dx == 1 && dy == 0 && dz == -1) c = 4;
  else if (dx == 0 && dy == 1 && dz == -1) c = 5;
  else if (dx == 1 && dy == 1 && dz == -1) c = 6;
  if (flipped) *flipped = f;
  return c;
}

// Base and tip of the class-c edge whose anchor is a (see header comment).
TM_HD Off3 edge_base_from_anchor(int c) {
  // c=3: base a+e2; c=4,5,6: base a+e3; else a
  return c == 3 ? Off3{0, 1, 0} : (c >= 4 ? Off3{0, 0, 1} : Off3{0, 0, 0});
}

// Local-edge descriptor of one orientation: which edge of the cube (anchor
// offset in {0,1}^3, class) it is, and whether the local direction a->b is
// opposite to the class direction.
struct LocalEdgeRef {
  int ax, ay, az;  // anchor offset relative to the element's anchor
  int cls;
  bool flipped;
};

TM_HD constexpr LocalEdgeRef local_edge_ref(int o, int le) {
  const Off3 pa = orient_offset(o, local_edge_vertex(le, 0));
  const Off3 pb = orient_offset(o, local_edge_vertex(le, 1));
  bool f = false;
  const int c = edge_class_of(pb.x - pa.x, pb.y - pa.y, pb.z - pa.z, &f);
  LocalEdgeRef r{0, 0, 0, 0, false};
  r.ax = pa.x < pb.x ? pa.x : pb.x;
  r.ay = pa.y < pb.y ? pa.y : pb.y;
  r.az = pa.z < pb.z ? pa.z : pb.z;
  r.cls = c;
  r.flipped = f;
  return r;
}

// Sizes of one macro's storage at extent n.
TM_HD i64 p1_macro_size(i64 n) { return tet_count(n); }
TM_HD i64 nd1_class_size(i64 n) { return tet_count(n - 1); }
TM_HD i64 nd1_macro_size(i64 n) { return 7 * tet_count(n - 1); }

// Loop bounds per orientation (mesh.cpp:66-74): the element anchored at a
// exists iff a.x+a.y+a.z <= n-1 (WU), n-3 (WD), n-2 (others).
TM_HD int orient_sum_limit(int o, int n) { return o == WU ? n - 1 : (o == WD ? n - 3 : n - 2); }

// SplitMix64 and the layout-independent seeded input generator
// (SURVEY.md 8(d)): vertex key = integer world-lattice coordinates; edge key
// = ordered pair of endpoint keys (lexicographically ascending); the edge
// value is defined along the ascending direction.
TM_HD std::uint64_t splitmix64(std::uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
TM_HD std::uint64_t key_hash_vertex(i64 X, i64 Y, i64 Z) {
  std::uint64_t h = splitmix64(static_cast<std::uint64_t>(X) ^ 0x5851F42D4C957F2Dull);
  h = splitmix64(h ^ static_cast<std::uint64_t>(Y));
  return splitmix64(h ^ static_cast<std::uint64_t>(Z));
}
// endpoints must already be in ascending lexicographic order
TM_HD std::uint64_t key_hash_edge(i64 X0, i64 Y0, i64 Z0, i64 X1, i64 Y1, i64 Z1) {
  return splitmix64(key_hash_vertex(X0, Y0, Z0) ^
                    (key_hash_vertex(X1, Y1, Z1) * 0x9E3779B97F4A7C15ull) ^ 0xED6Eull);
}
TM_HD double seeded_uniform(std::uint64_t seed, std::uint64_t h) {
  const std::uint64_t r = splitmix64(seed ^ h);
  return 2.0 * (static_cast<double>(r >> 11) * (1.0 / 9007199254740992.0)) - 1.0;
}
TM_HD bool lex_less(i64 X0, i64 Y0, i64 Z0, i64 X1, i64 Y1, i64 Z1) {
  return X0 != X1 ? X0 < X1 : (Y0 != Y1 ? Y0 < Y1 : Z0 < Z1);
}

} // namespace tetmf

// mesh.hpp -- macro mesh and macro-primitive topology (host C++).
//
// Mirrors the reference's MacroMesh (mesh.hpp:37-56, mesh.cpp:76-181):
// same built-ins (single-tet, cube6), same text format ("v x y z" /
// "t i0 i1 i2 i3"), same validation errors (std::invalid_argument class ->
// TETMF_EINVAL at the C ABI). Adds the K x K x K Kuhn cube meshes of the
// BASELINE configs (cube6's vertex-ordering rule applied per unit cube) and
// the macro-primitive topology (which macros contain a given vertex / edge /
// face primitive) that the interface exchange needs.
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

namespace tetmf {

struct MacroMesh {
  std::vector<std::array<double, 3>> vertices;
  std::vector<std::array<int, 4>> tets;

  int num_tets() const { return static_cast<int>(tets.size()); }
  void validate() const;  // throws std::invalid_argument (mesh.cpp:76-94)
  std::vector<std::array<int, 3>> boundary_faces() const;  // mesh.cpp:96-112

  static MacroMesh single_tet();        // mesh.cpp:114-120
  static MacroMesh cube6();             // mesh.cpp:122-141
  static MacroMesh kuhn_cubes(int kx, int ky, int kz);  // K^3 unit cubes, cube6 rule each
  static MacroMesh load_text(const std::string& text);  // mesh.cpp:143-169
  static MacroMesh load_file(const std::string& path);
  std::string to_text() const;          // reference text format
};

// "single-tet", "cube6", "cubes<K>" / "cubes<Kx>x<Ky>x<Kz>", or a file path
MacroMesh mesh_by_name(const std::string& name);

double tet_volume6(const MacroMesh& m, int macroId);

// Macro-primitive topology. A carrier (lattice point or lattice edge) of
// macro m lies on the sub-simplex spanned by the local vertices with nonzero
// barycentric weight ("support mask", bit i = local vertex i). The macros
// that contain that sub-simplex hold a copy of the carrier.
struct Topology {
  // [macro][mask] -> sorted macro ids containing the global vertices of mask
  std::vector<std::array<std::vector<int>, 16>> sharers;
  // [macro][local face f (opposite local vertex f)] -> true if domain boundary
  std::vector<std::array<bool, 4>> boundary_face;
  // [macro] bit `mask`: the sub-simplex of that support mask lies in a domain
  // boundary face (of ANY macro), i.e. its carriers are Dirichlet carriers.
  // The reference OR-merges the per-copy boundary flag over all macros that
  // hold a carrier (fespace.cpp:207-214, 226).
  std::vector<unsigned> dirichlet_mask;
  // integer scale D such that D * vertex coordinates are integers (0 if none)
  std::int64_t coord_scale = 0;
  std::vector<std::array<std::int64_t, 3>> int_vertices;  // D * vertices

  explicit Topology(const MacroMesh& mesh);
  int owner(int macro, unsigned mask) const { return sharers[macro][mask & 15u].front(); }
};

} // namespace tetmf

// mesh.cpp -- macro mesh, built-in meshes, text format and primitive topology.
#include "mesh.hpp"

#include <algorithm>
#include <cmath>
#include <fstream>
#include <map>
#include <set>
#include <sstream>

#include "common.hpp"

namespace tetmf {

double tet_volume6(const MacroMesh& m, int macroId) {
  const auto& t = m.tets[macroId];
  double a[3][3];
  for (int c = 0; c < 3; ++c)
    for (int r = 0; r < 3; ++r) a[r][c] = m.vertices[t[c + 1]][r] - m.vertices[t[0]][r];
  return a[0][0] * (a[1][1] * a[2][2] - a[2][1] * a[1][2]) -
         a[1][0] * (a[0][1] * a[2][2] - a[2][1] * a[0][2]) +
         a[2][0] * (a[0][1] * a[1][2] - a[1][1] * a[0][2]);
}

namespace {
std::array<int, 3> face_of(const std::array<int, 4>& t, int f) {
  std::array<int, 3> face;
  int k = 0;
  for (int i = 0; i < 4; ++i)
    if (i != f) face[k++] = t[i];
  std::sort(face.begin(), face.end());
  return face;
}
} // namespace

void MacroMesh::validate() const {
  const int nv = static_cast<int>(vertices.size());
  std::map<std::array<int, 3>, int> faceCount;
  for (int m = 0; m < num_tets(); ++m) {
    const auto& t = tets[m];
    for (int i : t)
      if (i < 0 || i >= nv) fail_arg("mesh: vertex id out of range");
    if (tet_volume6(*this, m) <= 0.0) fail_arg("mesh: tet with non-positive volume");
    for (int f = 0; f < 4; ++f)
      if (++faceCount[face_of(t, f)] > 2) fail_arg("mesh: face shared by more than two tets");
  }
  if (tets.empty()) fail_arg("mesh: no tetrahedra");
}

std::vector<std::array<int, 3>> MacroMesh::boundary_faces() const {
  std::map<std::array<int, 3>, int> faceCount;
  for (const auto& t : tets)
    for (int f = 0; f < 4; ++f) ++faceCount[face_of(t, f)];
  std::vector<std::array<int, 3>> out;
  for (const auto& [face, count] : faceCount)
    if (count == 1) out.push_back(face);
  return out;
}

MacroMesh MacroMesh::single_tet() {
  MacroMesh m;
  m.vertices = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  m.tets = {{0, 1, 2, 3}};
  m.validate();
  return m;
}

MacroMesh MacroMesh::kuhn_cubes(int kx, int ky, int kz) {
  if (kx < 1 || ky < 1 || kz < 1) fail_arg("kuhn_cubes: cube counts must be >= 1");
  MacroMesh m;
  for (int z = 0; z <= kz; ++z)
    for (int y = 0; y <= ky; ++y)
      for (int x = 0; x <= kx; ++x) m.vertices.push_back({double(x), double(y), double(z)});
  auto id = [&](int x, int y, int z) { return x + (kx + 1) * (y + (ky + 1) * z); };
  // Kuhn split of every unit cube with the vertex-ordering rule of cube6
  // (mesh.cpp:128-139): t = {c, c+e_p0, c+e_p0+e_p1, c+(1,1,1)}, swap the last
  // two if the volume is negative.
  const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  for (int cz = 0; cz < kz; ++cz)
    for (int cy = 0; cy < ky; ++cy)
      for (int cx = 0; cx < kx; ++cx)
        for (const auto& p : perms) {
          int a[3] = {0, 0, 0};
          a[p[0]] = 1;
          int b[3] = {a[0], a[1], a[2]};
          b[p[1]] = 1;
          std::array<int, 4> t = {id(cx, cy, cz), id(cx + a[0], cy + a[1], cz + a[2]),
                                  id(cx + b[0], cy + b[1], cz + b[2]), id(cx + 1, cy + 1, cz + 1)};
          m.tets.push_back(t);
          if (tet_volume6(m, m.num_tets() - 1) < 0.0) std::swap(m.tets.back()[2], m.tets.back()[3]);
        }
  m.validate();
  return m;
}

MacroMesh MacroMesh::cube6() { return kuhn_cubes(1, 1, 1); }

MacroMesh MacroMesh::load_text(const std::string& text) {
  MacroMesh m;
  std::istringstream in(text);
  std::string line;
  int lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    std::istringstream ls(line);
    std::string tag;
    if (!(ls >> tag) || tag[0] == '#') continue;
    if (tag == "v") {
      double x, y, z;
      if (!(ls >> x >> y >> z)) fail_arg("mesh file: bad vertex at line " + std::to_string(lineno));
      m.vertices.push_back({x, y, z});
    } else if (tag == "t") {
      std::array<int, 4> t;
      if (!(ls >> t[0] >> t[1] >> t[2] >> t[3]))
        fail_arg("mesh file: bad tet at line " + std::to_string(lineno));
      m.tets.push_back(t);
    } else {
      fail_arg("mesh file: unknown tag '" + tag + "' at line " + std::to_string(lineno));
    }
  }
  m.validate();
  return m;
}

MacroMesh MacroMesh::load_file(const std::string& path) {
  std::ifstream f(path);
  if (!f) fail_arg("mesh file: cannot open " + path);
  std::stringstream ss;
  ss << f.rdbuf();
  return load_text(ss.str());
}

std::string MacroMesh::to_text() const {
  std::ostringstream os;
  os.precision(17);
  for (const auto& v : vertices) os << "v " << v[0] << ' ' << v[1] << ' ' << v[2] << '\n';
  for (const auto& t : tets) os << "t " << t[0] << ' ' << t[1] << ' ' << t[2] << ' ' << t[3] << '\n';
  return os.str();
}

MacroMesh mesh_by_name(const std::string& name) {
  if (name == "single-tet") return MacroMesh::single_tet();
  if (name == "cube6") return MacroMesh::cube6();
  if (name.rfind("cubes", 0) == 0 && name.size() > 5) {
    int kx = 0, ky = 0, kz = 0;
    const std::string s = name.substr(5);
    if (std::sscanf(s.c_str(), "%dx%dx%d", &kx, &ky, &kz) == 3) return MacroMesh::kuhn_cubes(kx, ky, kz);
    if (std::sscanf(s.c_str(), "%d", &kx) == 1 && s.find_first_not_of("0123456789") == std::string::npos)
      return MacroMesh::kuhn_cubes(kx, kx, kx);
  }
  return MacroMesh::load_file(name);
}

Topology::Topology(const MacroMesh& mesh) {
  const int nt = mesh.num_tets();
  // vertex -> macros
  std::vector<std::vector<int>> vmac(mesh.vertices.size());
  for (int m = 0; m < nt; ++m)
    for (int v : mesh.tets[m]) vmac[v].push_back(m);
  sharers.resize(nt);
  for (int m = 0; m < nt; ++m) {
    for (unsigned mask = 0; mask < 16; ++mask) {
      std::vector<int> cand;
      bool first = true;
      for (int i = 0; i < 4; ++i) {
        if (!(mask & (1u << i))) continue;
        const auto& l = vmac[mesh.tets[m][i]];
        if (first) {
          cand = l;
          first = false;
        } else {
          std::vector<int> out;
          std::set_intersection(cand.begin(), cand.end(), l.begin(), l.end(), std::back_inserter(out));
          cand.swap(out);
        }
      }
      if (first) cand = {m};  // empty mask: cell interior, only this macro
      sharers[m][mask] = cand;
    }
  }
  const auto bf = mesh.boundary_faces();
  std::set<std::array<int, 3>> bset(bf.begin(), bf.end());
  boundary_face.assign(nt, {false, false, false, false});
  for (int m = 0; m < nt; ++m)
    for (int f = 0; f < 4; ++f) boundary_face[m][f] = bset.count(face_of(mesh.tets[m], f)) > 0;
  dirichlet_mask.assign(nt, 0u);
  for (int m = 0; m < nt; ++m)
    for (unsigned mask = 1; mask < 16; ++mask) {
      bool on = false;
      for (int m2 : sharers[m][mask])
        for (int f = 0; f < 4 && !on; ++f) {
          if (!boundary_face[m2][f]) continue;
          const int skip = mesh.tets[m2][f];  // the face is tet m2 without this vertex
          bool inside = true;
          for (int v = 0; v < 4; ++v)
            if ((mask >> v) & 1u) {
              const int g = mesh.tets[m][v];
              bool in_tet = false;
              for (int w = 0; w < 4; ++w) in_tet = in_tet || mesh.tets[m2][w] == g;
              if (!in_tet || g == skip) inside = false;
            }
          on = inside;
        }
      if (on) dirichlet_mask[m] |= 1u << mask;
    }

  // integer coordinate scale (world keys of the seeded input generator)
  coord_scale = 0;
  for (std::int64_t d = 1; d <= (1 << 20); d *= 2) {
    bool ok = true;
    for (const auto& v : mesh.vertices)
      for (double c : v) {
        const double s = c * static_cast<double>(d);
        if (std::fabs(s - std::nearbyint(s)) > 1e-9 || std::fabs(s) > 1e12) ok = false;
      }
    if (ok) {
      coord_scale = d;
      break;
    }
  }
  int_vertices.resize(mesh.vertices.size());
  for (std::size_t i = 0; i < mesh.vertices.size(); ++i)
    for (int c = 0; c < 3; ++c)
      int_vertices[i][c] =
          coord_scale ? static_cast<std::int64_t>(std::nearbyint(mesh.vertices[i][c] * coord_scale)) : 0;
}

} // namespace tetmf

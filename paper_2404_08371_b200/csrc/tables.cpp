// tables.cpp -- exact per-orientation tensors (host).
#include "tables.hpp"
#include "quadrature.hpp"

#include <cmath>
#include <cstring>
#include <map>
#include <mutex>

#include "common.hpp"

namespace tetmf {

namespace {

using V3 = std::array<double, 3>;

constexpr double kGradRef[4][3] = {{-1, -1, -1}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}};

V3 mat_vec(const double M[3][3], const double v[3]) {
  return {M[0][0] * v[0] + M[0][1] * v[1] + M[0][2] * v[2], M[1][0] * v[0] + M[1][1] * v[1] + M[1][2] * v[2],
          M[2][0] * v[0] + M[2][1] * v[1] + M[2][2] * v[2]};
}
double dot(const V3& a, const V3& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
V3 cross(const double a[3], const double b[3]) {
  return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}

// int over the element of lambda_m lambda_p lambda_q = 6 vol a!b!c!d!/6!
double triple(double vol, int m, int p, int q) {
  int cnt[4] = {0, 0, 0, 0};
  ++cnt[m]; ++cnt[p]; ++cnt[q];
  static const int fact[4] = {1, 1, 2, 6};
  int f = 1;
  for (int i = 0; i < 4; ++i) f *= fact[cnt[i]];
  return vol * 6.0 * f / 720.0;
}

int stencil_index(int dx, int dy, int dz) {
  if (dx == 0 && dy == 0 && dz == 0) return 0;
  bool f = false;
  const int c = edge_class_of(dx, dy, dz, &f);
  if (c < 0) fail_internal("stencil_index: not a lattice edge");
  return 2 * c + (f ? 2 : 1);
}

} // namespace

OrientGeom orient_geometry(const MacroMesh& mesh, int macro, int level, int o) {
  if (macro < 0 || macro >= mesh.num_tets()) fail_arg("orient_geometry: macro id out of range");
  const auto& t = mesh.tets[macro];
  double A[3][3], D[3][3];
  for (int c = 0; c < 3; ++c)
    for (int r = 0; r < 3; ++r) A[r][c] = mesh.vertices[t[c + 1]][r] - mesh.vertices[t[0]][r];
  const Off3 o0 = orient_offset(o, 0);
  for (int c = 0; c < 3; ++c) {
    const Off3 oc = orient_offset(o, c + 1);
    D[0][c] = oc.x - o0.x;
    D[1][c] = oc.y - o0.y;
    D[2][c] = oc.z - o0.z;
  }
  const double h = 1.0 / static_cast<double>(1 << level);
  OrientGeom g;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s += A[r][k] * D[k][c];
      g.J[r][c] = s * h;
    }
  auto det3 = [](const double M[3][3]) {
    return M[0][0] * (M[1][1] * M[2][2] - M[2][1] * M[1][2]) - M[1][0] * (M[0][1] * M[2][2] - M[2][1] * M[0][2]) +
           M[2][0] * (M[0][1] * M[1][2] - M[1][1] * M[0][2]);
  };
  const double detA = det3(A);
  if (detA <= 0.0) fail_arg("micro_jacobian: degenerate macro");
  const double detD = det3(D);
  g.det = detA * detD * h * h * h;
  const auto& J = g.J;
  double adj[3][3];
  adj[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
  adj[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
  adj[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
  adj[1][0] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
  adj[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
  adj[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
  adj[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  adj[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
  adj[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
  const double detJ = J[0][0] * adj[0][0] + J[0][1] * adj[1][0] + J[0][2] * adj[2][0];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) g.JinvT[r][c] = adj[c][r] / detJ;
  g.vol = std::fabs(g.det) / 6.0;
  return g;
}

P1Tables p1_tables(const MacroMesh& mesh, int macro, int level) {
  P1Tables t;
  std::memset(&t, 0, sizeof(t));
  for (int o = 0; o < 6; ++o) {
    const OrientGeom g = orient_geometry(mesh, macro, level, o);
    V3 G[4];
    for (int i = 0; i < 4; ++i) G[i] = mat_vec(g.JinvT, kGradRef[i]);
    for (int j = 0; j < 4; ++j)
      for (int i = 0; i < 4; ++i) t.K[o][j][i] = g.vol * dot(G[i], G[j]);
  }
  for (int type = 0; type < 16; ++type)
    for (int o = 0; o < 6; ++o)
      for (int i = 0; i < 4; ++i) {
        const Off3 pi = orient_offset(o, i);
        bool in = true;
        for (int j = 0; j < 4; ++j) {
          const Off3 pj = orient_offset(o, j);
          const int rx = pj.x - pi.x, ry = pj.y - pi.y, rz = pj.z - pi.z;
          if ((type & 1) && rx < 0) in = false;
          if ((type & 2) && ry < 0) in = false;
          if ((type & 4) && rz < 0) in = false;
          if ((type & 8) && rx + ry + rz > 0) in = false;
        }
        if (!in) continue;
        for (int j = 0; j < 4; ++j) {
          const Off3 pj = orient_offset(o, j);
          t.stencil[type][stencil_index(pj.x - pi.x, pj.y - pi.y, pj.z - pi.z)] += t.K[o][i][j];
        }
      }
  return t;
}

N1Tables n1_tables(const MacroMesh& mesh, int macro, int level) {
  N1Tables t;
  std::memset(&t, 0, sizeof(t));
  for (int o = 0; o < 6; ++o) {
    const OrientGeom g = orient_geometry(mesh, macro, level, o);
    V3 G[4];
    for (int i = 0; i < 4; ++i) G[i] = mat_vec(g.JinvT, kGradRef[i]);
    V3 curl[6];
    double s[6];
    for (int e = 0; e < 6; ++e) {
      const int a = kLocalEdge[e][0], b = kLocalEdge[e][1];
      const V3 c = cross(kGradRef[a], kGradRef[b]);
      const double cr[3] = {2.0 * c[0], 2.0 * c[1], 2.0 * c[2]};
      const V3 w = mat_vec(g.J, cr);
      curl[e] = {w[0] / g.det, w[1] / g.det, w[2] / g.det};
      s[e] = local_edge_ref(o, e).flipped ? -1.0 : 1.0;
    }
    for (int j = 0; j < 6; ++j)
      for (int i = 0; i < 6; ++i) {
        t.Kc[o][j][i] = s[i] * s[j] * 0.25 * g.vol * dot(curl[i], curl[j]);
        const int a = kLocalEdge[i][0], b = kLocalEdge[i][1];
        const int c = kLocalEdge[j][0], d = kLocalEdge[j][1];
        for (int m = 0; m < 4; ++m) {
          const double v = triple(g.vol, m, a, c) * dot(G[b], G[d]) - triple(g.vol, m, a, d) * dot(G[b], G[c]) -
                           triple(g.vol, m, b, c) * dot(G[a], G[d]) + triple(g.vol, m, b, d) * dot(G[a], G[c]);
          t.T[o][m][j][i] = s[i] * s[j] * v;
        }
      }
  }
  return t;
}

P1DeviceTable pack_p1(const P1Tables& t) {
  P1DeviceTable d;
  std::memset(&d, 0, sizeof(d));
  for (int ty = 0; ty < 16; ++ty)
    for (int k = 0; k < 15; ++k) d.stencil[ty][k] = t.stencil[ty][k];
  for (int o = 0; o < 6; ++o)
    for (int i = 0; i < 4; ++i)
      for (int j = i; j < 4; ++j) d.K[o][sym4(i, j)] = t.K[o][i][j];
  return d;
}

N1DeviceTable pack_n1(const N1Tables& t) {
  N1DeviceTable d;
  for (int o = 0; o < 6; ++o)
    for (int i = 0; i < 6; ++i)
      for (int j = i; j < 6; ++j) {
        d.e[o][0][sym6(i, j)] = t.Kc[o][i][j];
        for (int m = 0; m < 4; ++m) d.e[o][1 + m][sym6(i, j)] = t.T[o][m][i][j];
      }
  return d;
}

N1GramTable n1_gram_table(const MacroMesh& mesh, int macro, int level) {
  N1GramTable out;
  std::memset(&out, 0, sizeof(out));
  const N1Tables t = n1_tables(mesh, macro, level);
  for (int o = 0; o < 6; ++o) {
    for (int i = 0; i < 6; ++i)
      for (int j = i; j < 6; ++j) out.o[o][sym6(i, j)] = t.Kc[o][i][j];
    const OrientGeom g = orient_geometry(mesh, macro, level, o);
    V3 G[4];
    for (int i = 0; i < 4; ++i) G[i] = mat_vec(g.JinvT, kGradRef[i]);
    for (int x = 0; x < 4; ++x)
      for (int y = x; y < 4; ++y) out.o[o][22 + sym4(x, y)] = g.vol / 120.0 * dot(G[x], G[y]);
    for (int e = 0; e < 6; ++e)
      out.o[o][32 + e] = -2.0 * out.o[o][22 + sym4(local_edge_vertex(e, 0), local_edge_vertex(e, 1))];
    out.o[o][21] = 7200.0 / g.vol;  // kappa of the ZW form (curl-curl folded into B)
  }
  return out;
}

namespace {

// polynomials in the four barycentric coordinates (exponent tuple -> coeff)
using Mono = std::array<int, 4>;
using Poly = std::map<Mono, double>;

Poly pmul(const Poly& a, const Poly& b) {
  Poly c;
  for (const auto& [ea, ca] : a)
    for (const auto& [eb, cb] : b) {
      Mono e{ea[0] + eb[0], ea[1] + eb[1], ea[2] + eb[2], ea[3] + eb[3]};
      c[e] += ca * cb;
    }
  return c;
}

double fact(int k) {
  double f = 1.0;
  for (int i = 2; i <= k; ++i) f *= i;
  return f;
}

// int over a tetrahedron of volume vol of prod lambda_i^e_i = 6 vol prod e_i! / (sum e_i + 3)!
double pint(const Poly& p, double vol) {
  double s = 0.0;
  for (const auto& [e, c] : p)
    s += c * 6.0 * vol * fact(e[0]) * fact(e[1]) * fact(e[2]) * fact(e[3]) / fact(e[0] + e[1] + e[2] + e[3] + 3);
  return s;
}

Mono unit(int i) {
  Mono e{0, 0, 0, 0};
  e[i] = 1;
  return e;
}

// P2 basis (vertices 0-3, edges 4-9) and d phi_i / d lambda_p
Poly p2_basis(int i) {
  Poly p;
  if (i < 4) {
    Mono e2 = unit(i);
    e2[i] = 2;
    p[e2] = 2.0;
    p[unit(i)] = -1.0;
  } else {
    const int a = kLocalEdge[i - 4][0], b = kLocalEdge[i - 4][1];
    Mono e = unit(a);
    e[b] += 1;
    p[e] = 4.0;
  }
  return p;
}
Poly p2_dbasis(int i, int pvar) {
  Poly p;
  if (i < 4) {
    if (pvar == i) {
      p[unit(i)] = 4.0;
      p[Mono{0, 0, 0, 0}] = -1.0;
    }
  } else {
    const int a = kLocalEdge[i - 4][0], b = kLocalEdge[i - 4][1];
    if (pvar == a) p[unit(b)] = 4.0;
    if (pvar == b) p[unit(a)] = 4.0;
  }
  return p;
}

} // namespace

P2VTable p2v_table(const MacroMesh& mesh, int macro, int level) {
  P2VTable out;
  std::memset(&out, 0, sizeof(out));
  // orientation-independent reference integrals: I[m][i][j][p][q] = int psi_m
  // d_p phi_i d_q phi_j over a unit-volume element (scaled by vol below)
  static std::vector<double> ref;  // [m][i][j][p][q]
  static std::once_flag once;
  std::call_once(once, [] {
    ref.assign(10 * 10 * 10 * 16, 0.0);
    for (int m = 0; m < 10; ++m) {
      const Poly psi = p2_basis(m);
      for (int i = 0; i < 10; ++i)
        for (int p = 0; p < 4; ++p) {
          const Poly di = p2_dbasis(i, p);
          if (di.empty()) continue;
          const Poly pd = pmul(psi, di);
          for (int j = 0; j < 10; ++j)
            for (int q = 0; q < 4; ++q) {
              const Poly dj = p2_dbasis(j, q);
              if (dj.empty()) continue;
              ref[(((m * 10 + i) * 10 + j) * 4 + p) * 4 + q] = pint(pmul(pd, dj), 1.0);
            }
        }
    }
  });
  for (int o = 0; o < 6; ++o) {
    const OrientGeom g = orient_geometry(mesh, macro, level, o);
    V3 G[4];
    for (int i = 0; i < 4; ++i) G[i] = mat_vec(g.JinvT, kGradRef[i]);
    double GG[4][4];
    for (int p = 0; p < 4; ++p)
      for (int q = 0; q < 4; ++q) GG[p][q] = dot(G[p], G[q]);
    for (int p = 0; p < 4; ++p)
      for (int q = p; q < 4; ++q) out.G[o][sym4(p, q)] = g.vol * GG[p][q];
    for (int m = 0; m < 10; ++m)
      for (int i = 0; i < 10; ++i)
        for (int j = i; j < 10; ++j) {
          double v = 0.0;
          for (int p = 0; p < 4; ++p)
            for (int q = 0; q < 4; ++q) v += GG[p][q] * ref[(((m * 10 + i) * 10 + j) * 4 + p) * 4 + q];
          out.T[o][m][sym10(i, j)] = g.vol * v;
        }
  }
  return out;
}

namespace {
// barycentric coordinates of a reference point
void bary(double x, double y, double z, double l[4]) {
  l[0] = 1.0 - x - y - z;
  l[1] = x;
  l[2] = y;
  l[3] = z;
}
} // namespace

void p2v_rule_moments(int degree, double C[10][10]) {
  if (degree == 0) {
    p2v_moments(C);
    return;
  }
  const QuadRule r = quadrature_rule(degree);
  for (int m = 0; m < 10; ++m)
    for (int k = 0; k < 10; ++k) C[m][k] = 0.0;
  for (int q = 0; q < r.size(); ++q) {
    double l[4];
    bary(r.x[q], r.y[q], r.z[q], l);
    for (int m = 0; m < 10; ++m) {
      const double psi = m < 4 ? l[m] * (2.0 * l[m] - 1.0)
                               : 4.0 * l[kLocalEdge[m - 4][0]] * l[kLocalEdge[m - 4][1]];
      for (int a = 0; a < 4; ++a)
        for (int b = a; b < 4; ++b) C[m][sym4(a, b)] += 6.0 * r.w[q] * psi * l[a] * l[b];
    }
  }
}

void n1_rule_moments(int degree, double R[4][10]) {
  for (int m = 0; m < 4; ++m)
    for (int k = 0; k < 10; ++k) R[m][k] = 0.0;
  if (degree == 0) {  // exact: 120 (1/vol) int lambda_m lambda_p lambda_q = alpha!
    for (int m = 0; m < 4; ++m)
      for (int a = 0; a < 4; ++a)
        for (int b = a; b < 4; ++b) {
          int e[4] = {0, 0, 0, 0};
          ++e[m];
          ++e[a];
          ++e[b];
          double f = 1.0;
          for (int i = 0; i < 4; ++i)
            for (int j = 2; j <= e[i]; ++j) f *= j;
          R[m][sym4(a, b)] = f;
        }
    return;
  }
  const QuadRule r = quadrature_rule(degree);
  for (int q = 0; q < r.size(); ++q) {
    double l[4];
    bary(r.x[q], r.y[q], r.z[q], l);
    for (int m = 0; m < 4; ++m)
      for (int a = 0; a < 4; ++a)
        for (int b = a; b < 4; ++b) R[m][sym4(a, b)] += 720.0 * r.w[q] * l[m] * l[a] * l[b];
  }
}

void p2v_moments(double C[10][10]) {
  for (int m = 0; m < 10; ++m) {
    const Poly psi = p2_basis(m);
    for (int r = 0; r < 4; ++r)
      for (int s = r; s < 4; ++s) {
        Mono e = unit(r);
        e[s] += 1;
        C[m][sym4(r, s)] = pint(pmul(psi, Poly{{e, 1.0}}), 1.0);
      }
  }
}

std::vector<int> geometry_groups(const MacroMesh& mesh, const std::vector<int>& macros, int* num_groups) {
  std::map<std::array<double, 9>, int> seen;
  std::vector<int> out;
  for (int m : macros) {
    const auto& t = mesh.tets[m];
    std::array<double, 9> key;
    for (int c = 0; c < 3; ++c)
      for (int r = 0; r < 3; ++r) key[3 * c + r] = mesh.vertices[t[c + 1]][r] - mesh.vertices[t[0]][r];
    auto it = seen.find(key);
    if (it == seen.end()) it = seen.emplace(key, static_cast<int>(seen.size())).first;
    out.push_back(it->second);
  }
  if (num_groups) *num_groups = static_cast<int>(seen.size());
  return out;
}

} // namespace tetmf

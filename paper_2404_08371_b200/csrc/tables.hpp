// tables.hpp -- per (macro, level, orientation) micro-invariant tables.
//
// This is the paper's tabulation "T" plus loop-invariant hoisting "I"
// (PAPER.md:884-903), evaluated once per macro on the host:
//  * micro Jacobian J = A * D * 2^-L, det = detA * detD * 2^-3L
//    (micro_jacobian mesh.cpp:243-262)
//  * P1 stiffness K_o[i][j] = vol * (J^-T grad_i) . (J^-T grad_j) -- the
//    reference's starA summed over an exact rule (forms.cpp:110-116)
//  * P1 15-point stencil variants: per lattice-point type (which of the four
//    macro faces the point lies on) the sum of K_o over the incident micro
//    elements that belong to the macro
//  * N1: Kc_o = s_i s_j vol/4 curl_i.curl_j and T_o[m] = s_i s_j
//    int lambda_m phi_i.phi_j (exact), so that
//      A_e = (sum_m alpha_m) Kc_o + sum_m beta_m T_o[m]
//    equals the reference's starA/starB contraction (forms.cpp:93-108,
//    233-243) for P1 coefficients; s_i = -1 where the local edge runs
//    against its class direction (ND1 signs folded into the table).
#pragma once

#include <array>
#include <vector>

#include "lattice.hpp"
#include "mesh.hpp"

namespace tetmf {

struct OrientGeom {
  double J[3][3];
  double det;
  double JinvT[3][3];
  double vol;  // |det| / 6
};

OrientGeom orient_geometry(const MacroMesh& mesh, int macro, int level, int o);

// 15-point stencil offsets: 0 = centre, 2c+1 = +dir_c, 2c+2 = -dir_c
TM_HD Off3 stencil_offset(int k) {
  if (k == 0) return {0, 0, 0};
  const int c = (k - 1) >> 1;
  const int s = (k & 1) ? 1 : -1;
  const Off3 d = edge_dir(c);
  return {s * d.x, s * d.y, s * d.z};
}

struct P1Tables {
  double K[6][4][4];        // per orientation local stiffness
  double stencil[16][15];   // per point type (bit0 x=0, bit1 y=0, bit2 z=0, bit3 x+y+z=n)
};
P1Tables p1_tables(const MacroMesh& mesh, int macro, int level);

struct N1Tables {
  double Kc[6][6][6];       // [o][j][i] curl-curl / 4, signs folded
  double T[6][4][6][6];     // [o][m][j][i] mass moments, signs folded
};
N1Tables n1_tables(const MacroMesh& mesh, int macro, int level);

// Device table image of one distinct macro geometry, as consumed by the
// kernels (packed symmetric storage, see kernels_*.cu).
struct P1DeviceTable {
  double stencil[16][16];   // 16 slots per type (last unused) for alignment
  double K[6][10];          // packed upper triangle (i<=j) of K_o
};
struct N1DeviceTable {
  // per orientation: 21 packed entries of Kc, then 4 x 21 of T[m]
  double e[6][5][21];
};
P1DeviceTable pack_p1(const P1Tables& t);
N1DeviceTable pack_n1(const N1Tables& t);

// Gram form of the N1 element matrix (K3): per orientation
//   Kc[q]  = s_i s_j vol/4 curl_i . curl_j        (21 packed, + 1 pad)
//   g[xy]  = vol/120 G_x . G_y, G = J^-T grad lambda (10 packed, sym4)
// and for edges i = (a,b), j = (c,d), beta in P1, S = sum_m beta_m:
//   int beta phi_i.phi_j = Bt_ac g_bd - Bt_ad g_bc - Bt_bc g_ad + Bt_bd g_ac
//   Bt_pq = S + beta_p + beta_q (p != q),  Bt_pp = 2 S + 4 beta_p
// (exact: int lambda_m lambda_p lambda_q = 6 vol a!b!c!d!/6!). The local
// signs s_i s_j of the mass term are compile-time constants in the kernel.
// Diagonal entries i = (a,b) use  Bt_aa g_bb + Bt_bb g_aa + Bt_ab (-2 g_ab),
// with -2 g_ab stored per local edge (one FP64 op fewer per diagonal entry).
constexpr int kGramRow = 40;
struct N1GramTable {
  double o[6][kGramRow];  // [orientation][Kc 0..20, kappa = 7200/vol 21, g 22..31, -2 g_ab 32..37, pad]
};
N1GramTable n1_gram_table(const MacroMesh& mesh, int macro, int level);

// packed index of (i, j), i <= j < 6 (row-major upper triangle)
TM_HD constexpr int sym6(int i, int j) {
  if (i > j) { const int t = i; i = j; j = t; }
  return i * 6 - i * (i - 1) / 2 + (j - i);
}
TM_HD constexpr int sym4(int i, int j) {
  if (i > j) { const int t = i; i = j; j = t; }
  return i * 4 - i * (i - 1) / 2 + (j - i);
}

// P2V form (P2 trial/test, k in P2; forms.cpp:12): per orientation o the ten
// coefficient-basis tables T_m[ij] = int psi_m grad phi_i . grad phi_j over
// the micro element (exact; local DoFs 0-3 vertices, 4-9 edges in local-edge
// order (0,1),(0,2),(0,3),(1,2),(1,3),(2,3); psi = phi = the P2 basis
// lambda_i (2 lambda_i - 1), 4 lambda_a lambda_b), so A_e = sum_m k_m T_m.
//
// The factored kernel (k_p2v.cu) uses instead, per orientation, the metric
// G[o][sym4(p, q)] = vol grad lambda_p . grad lambda_q and the universal
// moments C[m][sym4(r, s)] = (1 / vol) int psi_m lambda_r lambda_s (p2v_moments):
// int k grad u . grad phi_i = sum_pq G_pq int k (du/dlambda_p)(dphi_i/dlambda_q)
// (chain rule in barycentrics; any polynomial representation of u works
// because sum_p grad lambda_p = 0).
struct P2VTable {
  double T[6][10][56];  // [orientation][coefficient DoF m][packed upper triangle (55) + pad]
  double G[6][10];      // [orientation][sym4(p, q)]
};
P2VTable p2v_table(const MacroMesh& mesh, int macro, int level);
void p2v_moments(double C[10][10]);
// the same moments under quadrature(degree) (degree 0: exact): C[m][sym4(r, s)]
// = 6 sum_q w_q psi_m lambda_r lambda_s at the rule's points
void p2v_rule_moments(int degree, double C[10][10]);
// N1 mass moments: R[m][sym4(p, q)] = 120 (1/vol) int lambda_m lambda_p lambda_q
// (exact: alpha!, so sum_m beta_m R[m][pq] = S + beta_p + beta_q, 2S + 4 beta_p
// on the diagonal -- the Gram form's B); degree > 0: under quadrature(degree)
void n1_rule_moments(int degree, double R[4][10]);
// packed index of (i, j), i <= j < 10
TM_HD constexpr int sym10(int i, int j) {
  if (i > j) { const int t = i; i = j; j = t; }
  return i * 10 - i * (i - 1) / 2 + (j - i);
}

// Groups macros with bitwise-identical tables (translated copies, e.g. all
// cubes of a Kuhn mesh share six geometries). Returns per-macro group id.
std::vector<int> geometry_groups(const MacroMesh& mesh, const std::vector<int>& macros, int* num_groups);

} // namespace tetmf

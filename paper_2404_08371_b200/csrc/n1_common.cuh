// n1_common.cuh -- pieces shared by the N1 cube kernels (k_n1_cubes.cu,
// k_n1_fold.cu): cube edge / vertex numbering, the Gram-form element, and the
// cp.async / shared-memory helpers of the staged input paths.
#pragma once

#include "device.hpp"

namespace tetmf {
namespace n1 {

// cube edge numbering: (owner offset, class)
//  0..6: (000, c)   7: (100,1)  8: (100,2)  9: (100,5)
// 10: (010,0) 11: (010,2) 12: (010,4) 13: (110,2)
// 14: (001,0) 15: (001,1) 16: (001,3) 17: (101,1) 18: (011,0)
__host__ __device__ constexpr int cube_edge_id(int ox, int oy, int oz, int c) {
  return (ox == 0 && oy == 0 && oz == 0) ? c
         : (ox == 1 && oy == 0 && oz == 0) ? (c == 1 ? 7 : c == 2 ? 8 : 9)
         : (ox == 0 && oy == 1 && oz == 0) ? (c == 0 ? 10 : c == 2 ? 11 : 12)
         : (ox == 1 && oy == 1 && oz == 0) ? 13
         : (ox == 0 && oy == 0 && oz == 1) ? (c == 0 ? 14 : c == 1 ? 15 : 16)
         : (ox == 1 && oy == 0 && oz == 1) ? 17
                                           : 18;
}

__host__ __device__ constexpr int cube_edge(int o, int le) {
  // local edge (a,b) of orientation o -> cube edge id (lattice.hpp conventions)
  return cube_edge_id(local_edge_ref(o, le).ax, local_edge_ref(o, le).ay, local_edge_ref(o, le).az,
                      local_edge_ref(o, le).cls);
}

__host__ __device__ constexpr int cube_vertex(int o, int i) {
  return orient_offset(o, i).x + 2 * orient_offset(o, i).y + 4 * orient_offset(o, i).z;
}

__device__ __forceinline__ void prefetch_l1(const double* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// volatile shared load: not CSE'd across elements, so values are re-read
// where used instead of being held in registers for the whole step
__device__ __forceinline__ double lds(const double* p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p))));
  return v;
}

// (i, j) of the P-th packed upper-triangle entry of a symmetric 6x6
__host__ __device__ constexpr int pair_i(int p) { return p < 6 ? 0 : p < 11 ? 1 : p < 15 ? 2 : p < 18 ? 3 : p < 20 ? 4 : 5; }
__host__ __device__ constexpr int pair_j(int p) {
  return p < 6 ? p : p < 11 ? p - 5 : p < 15 ? p - 9 : p < 18 ? p - 12 : p < 20 ? p - 14 : 5;
}

// Gram table of one orientation in shared memory (tables.hpp N1GramTable row)
struct SmemTab {
  const double* p;
  template <int I>
  __device__ __forceinline__ double get() const { return p[I]; }
};

// entry P of A_e x_e (template recursion: every table index is a compile-
// time constant, so a constant-bank table becomes a DFMA operand)
template <int O, int P, typename Tab>
__device__ __forceinline__ void gram_pairs(const Tab& tb, const double (&Bt)[4][4], double sa, const double (&xe)[6],
                                           double (&Y)[19]) {
  constexpr int i = pair_i(P), j = pair_j(P);
  constexpr int a = local_edge_vertex(i, 0), b = local_edge_vertex(i, 1);
  constexpr int c = local_edge_vertex(j, 0), d = local_edge_vertex(j, 1);
  constexpr bool neg = local_edge_ref(O, i).flipped != local_edge_ref(O, j).flipped;
  double m;
  if constexpr (i == j) {  // Bt_aa g_bb + Bt_bb g_aa - 2 Bt_ab g_ab
    m = Bt[a][a] * tb.template get<22 + sym4(b, b)>();
    m = fma(Bt[b][b], tb.template get<22 + sym4(a, a)>(), m);
    m = fma(Bt[a][b], tb.template get<32 + i>(), m);
  } else {
    m = Bt[a][c] * tb.template get<22 + sym4(b, d)>();
    m = fma(-Bt[a][d], tb.template get<22 + sym4(b, c)>(), m);
    m = fma(-Bt[b][c], tb.template get<22 + sym4(a, d)>(), m);
    m = fma(Bt[b][d], tb.template get<22 + sym4(a, c)>(), m);
  }
  const double aij = fma(sa, tb.template get<sym6(i, j)>(), neg ? -m : m);
  constexpr int ei = cube_edge(O, i), ej = cube_edge(O, j);
  Y[ei] = fma(aij, xe[j], Y[ei]);
  if constexpr (i != j) Y[ej] = fma(aij, xe[i], Y[ej]);
  if constexpr (P + 1 < 21) gram_pairs<O, P + 1>(tb, Bt, sa, xe, Y);
}

// Gram-form element (tables.hpp N1GramTable): Y[cube edges] += A_e x_e with
//   A_ij = sa Kc_ij + s_ij (B_ac g_bd - B_ad g_bc - B_bc g_ad + B_bd g_ac)
// In: accessor with  template <int K> double x()  (cube edge K) and
//     template <int V, int W> double c()  (cube vertex V; W 0 alpha, 1 beta).
// Tab: template <int I> double get()  (entry I of the orientation's row).
// An invalid element gets zero coefficients -> A_e = 0 (inputs are finite).
// N1 mass moments under quadrature(1) / quadrature(2) (tables.hpp
// n1_rule_moments; degrees >= 3 integrate the N1 form exactly): with rule R
// the Gram form's B_pq = sum_m beta_m R[m][pq]. Filled by the launching TU.
__constant__ double kN1Rule[2][4][10];

template <int O, int RULE = 0, typename Tab, typename In>
__device__ __forceinline__ void element_gram(const Tab& tb, const In& in, double (&Y)[19], bool valid) {
  constexpr int v0 = cube_vertex(O, 0), v1 = cube_vertex(O, 1), v2 = cube_vertex(O, 2), v3 = cube_vertex(O, 3);
  const double a4 = (in.template c<v0, 0>() + in.template c<v1, 0>()) +
                    (in.template c<v2, 0>() + in.template c<v3, 0>());
  const double sa = valid ? a4 : 0.0;
  const double bv[4] = {valid ? in.template c<v0, 1>() : 0.0, valid ? in.template c<v1, 1>() : 0.0,
                        valid ? in.template c<v2, 1>() : 0.0, valid ? in.template c<v3, 1>() : 0.0};
  double Bt[4][4];
  if constexpr (RULE == 0) {
    const double S = (bv[0] + bv[1]) + (bv[2] + bv[3]);
    const double S2 = S + S;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const double u = S + bv[p];
#pragma unroll
      for (int q = p + 1; q < 4; ++q) Bt[p][q] = Bt[q][p] = u + bv[q];
      Bt[p][p] = fma(4.0, bv[p], S2);
    }
  } else {
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int q = p; q < 4; ++q) {
        double b = bv[0] * kN1Rule[RULE - 1][0][sym4(p, q)];
#pragma unroll
        for (int m = 1; m < 4; ++m) b = fma(bv[m], kN1Rule[RULE - 1][m][sym4(p, q)], b);
        Bt[p][q] = Bt[q][p] = b;
      }
  }
  double xe[6];
  xe[0] = in.template x<cube_edge(O, 0)>();
  xe[1] = in.template x<cube_edge(O, 1)>();
  xe[2] = in.template x<cube_edge(O, 2)>();
  xe[3] = in.template x<cube_edge(O, 3)>();
  xe[4] = in.template x<cube_edge(O, 4)>();
  xe[5] = in.template x<cube_edge(O, 5)>();
  gram_pairs<O, 0>(tb, Bt, sa, xe, Y);
}

// ---------------------------------------------------------------------------
// ZW form of the same element (default since round 2, session 2). With
// X_pq = +-x (local edge (p,q), antisymmetric, orientation signs folded in),
// g the Gram table and B the coefficient moments above, the Gram-form matvec
// is   y_(a,b) = (B X g)_ab - (B X g)_ba,
// and the curl-curl term folds into B: all micro-elements of a macro have the
// same volume, curl_i . curl_j = 4 (D_ac D_bd - D_ad D_bc) with D = 120 g / vol,
// so  sa Kc_ij  is the Gram expression of  t g  with  t = sa * kappa,
// kappa = 7200 / vol (table slot 21). Per element:
//   B' = B + t g                     10 FMA
//   Z  = X g  (rows sum to zero: Z_p3 = -(Z_p0 + Z_p1 + Z_p2))   36 + 8
//   Y_e += s_e sum_p (B'_ap Z_pb - B'_bp Z_pa)                    48 FMA
// ~123 FP64 instructions and 11 table values per element (Gram: ~155 and 38).
__host__ __device__ constexpr int edge_of_pair(int p, int q) {  // p < q
  return p == 0 ? q - 1 : p == 1 ? q + 1 : 5;
}
__host__ __device__ constexpr int other_q(int p, int k) { return k < p ? k : k + 1; }  // k-th vertex != p
// X_PQ = (neg ? -1 : 1) * x of the cube edge
template <int O, int P, int Q>
__host__ __device__ constexpr bool x_neg() {
  return (P > Q) != local_edge_ref(O, P < Q ? edge_of_pair(P, Q) : edge_of_pair(Q, P)).flipped;
}
template <int O, int P, int Q>
__device__ __forceinline__ double xpq(const double (&xe)[6]) {
  constexpr int e = P < Q ? edge_of_pair(P, Q) : edge_of_pair(Q, P);
  return x_neg<O, P, Q>() ? -xe[e] : xe[e];
}
// Z_PB (B < 3) = sum_{q != P, ascending} X_Pq g_qB
template <int O, int P, int B, typename Tab>
__device__ __forceinline__ double zw_z(const Tab& tb, const double (&xe)[6]) {
  constexpr int q0 = other_q(P, 0), q1 = other_q(P, 1), q2 = other_q(P, 2);
  double z = xpq<O, P, q0>(xe) * tb.template get<22 + sym4(q0, B)>();
  z = fma(xpq<O, P, q1>(xe), tb.template get<22 + sym4(q1, B)>(), z);
  return fma(xpq<O, P, q2>(xe), tb.template get<22 + sym4(q2, B)>(), z);
}
// one term s * B'_AP Z_PC of edge output (A, C); Z_P3 = -Z3[P]
template <bool NEG, int A, int P, int C>
__device__ __forceinline__ double zw_term(const double (&Bp)[10], const double (&Z)[4][3], const double (&Z3)[4],
                                          double acc) {
  constexpr bool neg = NEG != (C == 3);
  const double z = C == 3 ? Z3[P] : Z[P][C < 3 ? C : 0];
  return fma(neg ? -Bp[sym4(A, P)] : Bp[sym4(A, P)], z, acc);
}
// element order of cube_elements; a cube edge's first contribution starts its
// accumulator (no zero-initialised Y)
constexpr int kCubeOrder[6] = {WU, BU, BD, GU, GD, WD};
__host__ __device__ constexpr bool touched_before(int o, int ce) {
  for (int k = 0; k < 6 && kCubeOrder[k] != o; ++k)
    for (int le = 0; le < 6; ++le)
      if (cube_edge(kCubeOrder[k], le) == ce) return true;
  return false;
}
// SEED: the cube's bottom-face accumulators 0, 1, 3, 7, 10 arrive holding the
// top-face sums of the cube below (k_n1_fold2.cu)
__host__ __device__ constexpr bool seeded_edge(int ce) { return ce == 0 || ce == 1 || ce == 3 || ce == 7 || ce == 10; }
template <int O, int I, bool SEED = false>
__device__ __forceinline__ void zw_out(const double (&Bp)[10], const double (&Z)[4][3], const double (&Z3)[4],
                                       double (&Y)[19]) {
  constexpr int a = local_edge_vertex(I, 0), b = local_edge_vertex(I, 1);
  constexpr bool s = local_edge_ref(O, I).flipped;  // Y_e += s_e y_ab
  constexpr int ce = cube_edge(O, I);
  double acc;
  constexpr bool prior = touched_before(O, ce) || (SEED && seeded_edge(ce));
  if constexpr (prior) {
    acc = zw_term<s, a, 0, b>(Bp, Z, Z3, Y[ce]);
  } else {
    constexpr bool neg = s != (b == 3);
    acc = (neg ? -Bp[sym4(a, 0)] : Bp[sym4(a, 0)]) * (b == 3 ? Z3[0] : Z[0][b < 3 ? b : 0]);
  }
  acc = zw_term<!s, b, 0, a>(Bp, Z, Z3, acc);
  acc = zw_term<s, a, 1, b>(Bp, Z, Z3, acc);
  acc = zw_term<!s, b, 1, a>(Bp, Z, Z3, acc);
  acc = zw_term<s, a, 2, b>(Bp, Z, Z3, acc);
  acc = zw_term<!s, b, 2, a>(Bp, Z, Z3, acc);
  acc = zw_term<s, a, 3, b>(Bp, Z, Z3, acc);
  acc = zw_term<!s, b, 3, a>(Bp, Z, Z3, acc);
  Y[ce] = acc;
  if constexpr (I + 1 < 6) zw_out<O, I + 1, SEED>(Bp, Z, Z3, Y);
}
template <int O, int P, typename Tab>
__device__ __forceinline__ void zw_rows(const Tab& tb, const double (&xe)[6], double (&Z)[4][3], double (&Z3)[4]) {
  Z[P][0] = zw_z<O, P, 0>(tb, xe);
  Z[P][1] = zw_z<O, P, 1>(tb, xe);
  Z[P][2] = zw_z<O, P, 2>(tb, xe);
  Z3[P] = (Z[P][0] + Z[P][1]) + Z[P][2];
  if constexpr (P + 1 < 4) zw_rows<O, P + 1>(tb, xe, Z, Z3);
}

template <int O, int RULE = 0, bool SEED = false, typename Tab, typename In>
__device__ __forceinline__ void element_zw(const Tab& tb, const In& in, double (&Y)[19], bool valid) {
  constexpr int v0 = cube_vertex(O, 0), v1 = cube_vertex(O, 1), v2 = cube_vertex(O, 2), v3 = cube_vertex(O, 3);
  const double a4 = (in.template c<v0, 0>() + in.template c<v1, 0>()) +
                    (in.template c<v2, 0>() + in.template c<v3, 0>());
  const double t = (valid ? a4 : 0.0) * tb.template get<21>();
  const double bv[4] = {valid ? in.template c<v0, 1>() : 0.0, valid ? in.template c<v1, 1>() : 0.0,
                        valid ? in.template c<v2, 1>() : 0.0, valid ? in.template c<v3, 1>() : 0.0};
  double Bp[10];
  if constexpr (RULE == 0) {
    const double S = (bv[0] + bv[1]) + (bv[2] + bv[3]);
    const double S2 = S + S;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const double u = S + bv[p];
#pragma unroll
      for (int q = p + 1; q < 4; ++q) Bp[sym4(p, q)] = u + bv[q];
      Bp[sym4(p, p)] = fma(4.0, bv[p], S2);
    }
  } else {
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int q = p; q < 4; ++q) {
        double b = bv[0] * kN1Rule[RULE - 1][0][sym4(p, q)];
#pragma unroll
        for (int m = 1; m < 4; ++m) b = fma(bv[m], kN1Rule[RULE - 1][m][sym4(p, q)], b);
        Bp[sym4(p, q)] = b;
      }
  }
  Bp[0] = fma(t, tb.template get<22 + 0>(), Bp[0]);
  Bp[1] = fma(t, tb.template get<22 + 1>(), Bp[1]);
  Bp[2] = fma(t, tb.template get<22 + 2>(), Bp[2]);
  Bp[3] = fma(t, tb.template get<22 + 3>(), Bp[3]);
  Bp[4] = fma(t, tb.template get<22 + 4>(), Bp[4]);
  Bp[5] = fma(t, tb.template get<22 + 5>(), Bp[5]);
  Bp[6] = fma(t, tb.template get<22 + 6>(), Bp[6]);
  Bp[7] = fma(t, tb.template get<22 + 7>(), Bp[7]);
  Bp[8] = fma(t, tb.template get<22 + 8>(), Bp[8]);
  Bp[9] = fma(t, tb.template get<22 + 9>(), Bp[9]);
  double xe[6];
  xe[0] = in.template x<cube_edge(O, 0)>();
  xe[1] = in.template x<cube_edge(O, 1)>();
  xe[2] = in.template x<cube_edge(O, 2)>();
  xe[3] = in.template x<cube_edge(O, 3)>();
  xe[4] = in.template x<cube_edge(O, 4)>();
  xe[5] = in.template x<cube_edge(O, 5)>();
  double Z[4][3], Z3[4];
  zw_rows<O, 0>(tb, xe, Z, Z3);
  zw_out<O, 0, SEED>(Bp, Z, Z3, Y);
}

#ifndef TETMF_N1_ZW
#define TETMF_N1_ZW 1  // 0: the Gram-form element (round 1)
#endif

// ZW cube: validity by table choice -- an element outside the macro reads an
// all-zero table (Z = X 0 = 0, so its contribution is exactly 0 for finite
// inputs): three table bases per step instead of selects on every input.
// Every cube edge's accumulator is set by its first contribution.
template <int RULE = 0, bool SEED = false, typename Tabs, typename In>
__device__ __forceinline__ void cube_elements_zw(const Tabs& ts, const In& in, double (&Y)[19]) {
  element_zw<WU, RULE, SEED>(ts.template tab<WU>(), in, Y, true);
  element_zw<BU, RULE, SEED>(ts.template tab<BU>(), in, Y, true);
  element_zw<BD, RULE, SEED>(ts.template tab<BD>(), in, Y, true);
  element_zw<GU, RULE, SEED>(ts.template tab<GU>(), in, Y, true);
  element_zw<GD, RULE, SEED>(ts.template tab<GD>(), in, Y, true);
  element_zw<WD, RULE, SEED>(ts.template tab<WD>(), in, Y, true);
}
// one orientation row of a table at a 32-bit shared address; entries are
// loaded in 16-byte pairs (ld.shared.v2.f64 with an immediate offset; the
// asm is pure, so the two halves of a pair come from one load). Pure asm may
// be reordered freely, so it must only read memory that no later code writes
// and that is complete before its address operand exists: the tables are
// written before the kernel's __syncthreads and never again, and the address
// (a table-base select) depends on the task loaded after that barrier.
template <int O>
struct SmemTabA {
  unsigned a;
  template <int I>
  __device__ __forceinline__ double get() const {
    double lo, hi;
    asm("ld.shared.v2.f64 {%0, %1}, [%2+%3];" : "=d"(lo), "=d"(hi) : "r"(a), "n"((O * kGramRow + (I & ~1)) * 8));
    return (I & 1) ? hi : lo;
  }
};
// an opaque copy: keeps the compiler from pushing a select into every address
__device__ __forceinline__ unsigned opaque_u32(unsigned v) {
  unsigned r;
  asm("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}
// three table bases (real or zero table, shared addresses) for the validity
// classes WU / middle / WD
struct SmemTabs3 {
  unsigned wu, mid, wd;
  template <int O>
  __device__ __forceinline__ SmemTabA<O> tab() const {
    return SmemTabA<O>{O == WU ? wu : O == WD ? wd : mid};
  }
};

// the six elements of the cube (validity by anchor sum class); Tabs:
// template <int O> tab() -> the orientation's table accessor
template <int RULE = 0, typename Tabs, typename In>
__device__ __forceinline__ void cube_elements(const Tabs& ts, const In& in, double (&Y)[19], bool vWU, bool vMid,
                                              bool vWD) {
#if TETMF_N1_ZW
  element_zw<WU, RULE>(ts.template tab<WU>(), in, Y, vWU);
  element_zw<BU, RULE>(ts.template tab<BU>(), in, Y, vMid);
  element_zw<BD, RULE>(ts.template tab<BD>(), in, Y, vMid);
  element_zw<GU, RULE>(ts.template tab<GU>(), in, Y, vMid);
  element_zw<GD, RULE>(ts.template tab<GD>(), in, Y, vMid);
  element_zw<WD, RULE>(ts.template tab<WD>(), in, Y, vWD);
#else
  element_gram<WU, RULE>(ts.template tab<WU>(), in, Y, vWU);
  element_gram<BU, RULE>(ts.template tab<BU>(), in, Y, vMid);
  element_gram<BD, RULE>(ts.template tab<BD>(), in, Y, vMid);
  element_gram<GU, RULE>(ts.template tab<GU>(), in, Y, vMid);
  element_gram<GD, RULE>(ts.template tab<GD>(), in, Y, vMid);
  element_gram<WD, RULE>(ts.template tab<WD>(), in, Y, vWD);
#endif
}

// the six orientation rows of an N1GramTable in shared memory
struct SmemTabs {
  const N1GramTable& sg;
  template <int O>
  __device__ __forceinline__ SmemTab tab() const { return SmemTab{sg.o[O]}; }
};

} // namespace n1

// kernel variant of the N1 apply (TETMF_N1_TABLE, read once):
// 0 assembled tables, 1 Gram + direct loads, 2 Gram + row ring, 3 folded walk
int n1_kernel_mode();

} // namespace tetmf

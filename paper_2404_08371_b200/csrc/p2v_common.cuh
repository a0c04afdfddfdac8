// p2v_common.cuh -- P2V element pieces shared by the cube kernel (k_p2v.cu)
// and the folded cube walk (k_p2v_fold.cu).
#pragma once

#include "device.hpp"
#include "lattice.hpp"
#include "tables.hpp"

namespace tetmf {

// K_rs = int k lambda_r lambda_s / vol for k in P2 (exact rule, RULE 0) in
// closed form: with k = sum_{a<=b} kap_ab lambda_a lambda_b (kap_aa = k_a,
// kap_ab = 4 k_ab - k_a - k_b) and int lambda^alpha = 6 vol alpha!/7!,
// summing alpha! over the permutations that fix the index multiset gives
//   K_rs = (base + 2 (Q_r + Q_s) + kap_rs) / 840            (r != s)
//   K_rr = (2 base + 8 R_r + 12 kap_rr) / 840
// with R_r = kap_rr + sum_{s != r} kap_rs / 2, Q_r = R_r + kap_rr,
// base = sum_r R_r + sum_r kap_rr: 66 FP64 instructions and no constant-bank
// operands instead of the 10 x 10 moment matrix (100 FP64 + 100 constants).
__device__ __forceinline__ void p2v_exact_moments(const double (&kv)[10], double (&K)[10]) {
  constexpr double c = 1.0 / 840.0;
  double kd[4], ke[6];
#pragma unroll
  for (int a = 0; a < 4; ++a) kd[a] = kv[a] * c;
#pragma unroll
  for (int e = 0; e < 6; ++e) ke[e] = fma(4.0 * c, kv[4 + e], -(kd[local_edge_vertex(e, 0)] + kd[local_edge_vertex(e, 1)]));
  double R[4];  // local edges (0,1),(0,2),(0,3),(1,2),(1,3),(2,3)
  R[0] = fma(0.5, (ke[0] + ke[1]) + ke[2], kd[0]);
  R[1] = fma(0.5, (ke[0] + ke[3]) + ke[4], kd[1]);
  R[2] = fma(0.5, (ke[1] + ke[3]) + ke[5], kd[2]);
  R[3] = fma(0.5, (ke[2] + ke[4]) + ke[5], kd[3]);
  const double base = ((R[0] + R[1]) + (R[2] + R[3])) + ((kd[0] + kd[1]) + (kd[2] + kd[3]));
  const double b2 = base + base;
  double Q[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    Q[r] = R[r] + kd[r];
    K[sym4(r, r)] = fma(12.0, kd[r], fma(8.0, R[r], b2));
  }
#pragma unroll
  for (int e = 0; e < 6; ++e) {
    const int a = local_edge_vertex(e, 0), b = local_edge_vertex(e, 1);
    K[sym4(a, b)] = fma(2.0, Q[a] + Q[b], base) + ke[e];
  }
}

} // namespace tetmf

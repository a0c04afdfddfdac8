// solver.hpp -- Dirichlet-masked matrix-free CG over Operator::apply
// (the reference's missing cg_solve).
//
//   solve  A x = b  on the interior (non-Dirichlet) carriers, homogeneous
//   Dirichlet values (the reference's interior() mask, fespace.hpp:95-96),
// with A = P A_full P (P zeroes Dirichlet carriers). Vectors are level-
// indexed Functions whose interface copies stay equal; inner products weight
// each carrier once (owner copy, solver.cu). Multi-rank: per-rank partial
// sums are all-gathered and added in rank order, so every rank (and any rank
// count with the same partition) sees bitwise-identical scalars.
#pragma once

#include <cuda_runtime.h>

#include "lattice.hpp"

namespace tetmf {

// geometry of a function's storage as the slot-class kernels see it
struct SlotSpace {
  int n;             // lattice extent (2^level)
  int nd1;           // 0 P1 points, 1 ND1 edges, 2 P2 (vertex block, then edge blocks)
  i64 macro_stride;  // entries per macro
  i64 class_stride;  // ND1: entries per edge-class block
};

int masked_dot_partials();
void launch_masked_dot(const double* a, const double* b, const SlotSpace& sp, const unsigned char* d_table, i64 count,
                       double* d_partials, double* d_out, cudaStream_t s);
void launch_sum_ordered(const double* d_values, int count, double* d_out, cudaStream_t s);
void launch_mask_dirichlet(double* y, const SlotSpace& sp, const unsigned char* d_table, i64 count, cudaStream_t s);
void launch_xpby(double* y, const double* x, double beta, i64 count, cudaStream_t s);
void launch_jacobi(double* z, const double* r, const double* d, i64 count, cudaStream_t s);
void launch_axpby(double* y, const double* x, double a, double b, i64 count, cudaStream_t s);
void launch_mul(double* z, const double* x, const double* d, i64 count, cudaStream_t s);
void launch_scale(double* y, double a, i64 count, cudaStream_t s);

class Context;
class Function;
class Operator;

// <a, b> over the interior carriers, each counted once (all ranks)
double masked_dot(const Function& a, const Function& b, int level);
// zero the Dirichlet carriers of f
void mask_dirichlet(Function& f, int level);

// P1 <-> ND1 discrete gradient (k_transfer.cu): nd1 = G p1, p1 = G^T nd1
void gradient(const Function& p1, Function& nd1, int level);
void gradient_transpose(const Function& nd1, Function& p1, int level);

struct CgResult {
  int iterations = 0;
  double rel_residual = 0.0;  // ||r_k|| / ||r_0|| (masked norm)
  bool converged = false;
};
// x: initial guess in, solution out (Dirichlet carriers forced to 0); b is
// read-only (its Dirichlet carriers are ignored). Stops when
// ||r_k|| <= rtol ||r_0|| or after max_iter iterations. diag (optional): the
// operator diagonal (Operator::diagonal) -> Jacobi-preconditioned CG.
CgResult cg_solve(Operator& op, const Function& b, Function& x, int level, double rtol, int max_iter,
                  const Function* diag = nullptr);

// Largest eigenvalue of D^-1 A on the interior carriers (power iteration with
// the Rayleigh quotient <v, A v> / <v, D v>, seeded start vector).
double estimate_lambda_max(Operator& op, const Function& diag, int level, int iterations);

// Chebyshev-Jacobi smoother (the smoother of the reference paper's
// multigrid): `degree` steps of the Chebyshev iteration for
// D^-1 A targeting [lambda_max / eig_ratio, lambda_max]; x updated in place.
void chebyshev_smooth(Operator& op, const Function& diag, const Function& b, Function& x, int level, int degree,
                      double lambda_max, double eig_ratio);

} // namespace tetmf

// cg.cpp -- host driver of the Dirichlet-masked matrix-free CG (solver.hpp).
//
// Plain CG (Hestenes-Stiefel) on P A P with P the Dirichlet mask:
//   r = P(b - A x), p = r
//   repeat: q = P A p;  alpha = <r,r> / <p,q>;  x += alpha p;  r -= alpha q
//           beta = <r_new,r_new> / <r,r>;  p = r + beta p
// Every vector op is a kernel on the context stream; the two inner products
// per iteration are read back to the host (the iteration count decision).
#include <cmath>
#include <memory>

#include "exchange.hpp"
#include "runtime.hpp"
#include "runtime_check.hpp"
#include "solver.hpp"

namespace tetmf {

namespace {

SlotSpace slot_space(const Context::LevelData& ld) {
  const int kind = ld.lay.space == Space::ND1 ? 1 : (ld.lay.space == Space::P2 ? 2 : 0);
  return SlotSpace{ld.lay.n, kind, ld.lay.macro_stride, ld.lay.class_stride};
}

} // namespace

double masked_dot(const Function& a, const Function& b, int level) {
  if (a.space() != b.space() || &a.ctx() != &b.ctx()) fail_arg("dot: functions of different spaces / contexts");
  Context& ctx = a.ctx();
  if (ctx.partition() == Context::kPartitionSlab)
    fail_arg("dot / solvers: slab partitions hold unowned macro storage (apply only)");
  auto& ld = ctx.level(a.space(), level);
  const cudaStream_t s = ctx.stream();
  double* scratch = ld.dot_scratch.get();
  const int np = masked_dot_partials();
  double* local = scratch + np;          // this rank's sum
  double* gathered = local + 1;          // nranks sums
  double* total = gathered + ctx.nranks();
  if (ld.lay.macros.empty()) {
    TETMF_CUDA(cudaMemsetAsync(local, 0, sizeof(double), s));
  } else {
    launch_masked_dot(a.data(level), b.data(level), slot_space(ld), ld.slot_table.get(), ld.lay.total(), scratch,
                      local, s);
  }
  double out = 0.0;
  if (ctx.nranks() > 1) {
    if (!ctx.transport()) throw CommError("dot: no transport attached to the multi-rank context");
    ctx.transport()->allgather(local, gathered, 1, s);
    launch_sum_ordered(gathered, ctx.nranks(), total, s);
    TETMF_CUDA(cudaMemcpyAsync(&out, total, sizeof(double), cudaMemcpyDeviceToHost, s));
  } else {
    TETMF_CUDA(cudaMemcpyAsync(&out, local, sizeof(double), cudaMemcpyDeviceToHost, s));
  }
  TETMF_CUDA(cudaStreamSynchronize(s));
  return out;
}

void mask_dirichlet(Function& f, int level) {
  auto& ld = f.ctx().level(f.space(), level);
  if (ld.lay.macros.empty()) return;
  launch_mask_dirichlet(f.data(level), slot_space(ld), ld.slot_table.get(), ld.lay.total(), f.ctx().stream());
}

void gradient(const Function& p1, Function& nd1, int level) {
  if (p1.space() != Space::P1 || nd1.space() != Space::ND1 || &p1.ctx() != &nd1.ctx())
    fail_arg("gradient: expects a P1 and an ND1 function of one context");
  Context& ctx = p1.ctx();
  auto& le = ctx.level(Space::ND1, level);
  auto& lp = ctx.level(Space::P1, level);
  launch_gradient(p1.data(level), nd1.data(level), static_cast<int>(le.lay.macros.size()), le.lay.macro_stride,
                  le.lay.class_stride, lp.lay.macro_stride, le.lay.n, ctx.stream());
}

void gradient_transpose(const Function& nd1, Function& p1, int level) {
  if (p1.space() != Space::P1 || nd1.space() != Space::ND1 || &p1.ctx() != &nd1.ctx())
    fail_arg("gradient_transpose: expects an ND1 and a P1 function of one context");
  Context& ctx = p1.ctx();
  auto& le = ctx.level(Space::ND1, level);
  auto& lp = ctx.level(Space::P1, level);
  double* y = p1.data(level);
  launch_gradient_t(nd1.data(level), y, static_cast<int>(le.lay.macros.size()), le.lay.macro_stride,
                    le.lay.class_stride, lp.lay.macro_stride, le.lay.n, le.slot_table.get(), ctx.stream());
  lp.interface_sum(y, ctx.stream());
  if (lp.exchange) lp.exchange->run(y, ctx.stream());
}

CgResult cg_solve(Operator& op, const Function& b, Function& x, int level, double rtol, int max_iter,
                  const Function* diag) {
  const Space sp = op.info().trial;
  if (b.space() != sp || x.space() != sp) fail_arg("cg: b and x must be in the operator's trial space");
  if (diag && (diag->space() != sp || !diag->has_level(level))) fail_arg("cg: diagonal not in the trial space");
  if (!(rtol > 0.0) || max_iter < 0) fail_arg("cg: rtol must be > 0 and max_iter >= 0");
  Context& ctx = x.ctx();
  const cudaStream_t s = ctx.stream();
  const i64 count = x.size(level);
  Function r(ctx, sp), p(ctx, sp), q(ctx, sp);
  std::unique_ptr<Function> zf;
  double* X = x.data(level);
  double* R = r.data(level);
  double* P = p.data(level);
  double* Q = q.data(level);
  const double* B = b.data(level);
  const double* Dg = diag ? diag->data(level) : nullptr;
  double* Z = R;  // unpreconditioned: z = r
  if (Dg) {
    zf = std::make_unique<Function>(ctx, sp);
    Z = zf->data(level);
  }
  const Function& z = Dg ? *zf : r;

  mask_dirichlet(x, level);
  op.apply(x, q, level, Update::Replace);  // q = A x
  TETMF_CUDA(cudaMemcpyAsync(R, B, sizeof(double) * count, cudaMemcpyDeviceToDevice, s));
  launch_axpy(R, Q, -1.0, count, s);       // r = b - A x
  mask_dirichlet(r, level);
  if (Dg) launch_jacobi(Z, R, Dg, count, s);  // z = D^-1 r
  TETMF_CUDA(cudaMemcpyAsync(P, Z, sizeof(double) * count, cudaMemcpyDeviceToDevice, s));
  double rr = masked_dot(r, r, level);
  double rz = Dg ? masked_dot(r, z, level) : rr;
  const double rr0 = rr;
  CgResult res;
  res.rel_residual = rr0 > 0.0 ? 1.0 : 0.0;
  if (rr0 == 0.0) {
    res.converged = true;
    return res;
  }
  const double stop = rtol * rtol * rr0;
  for (int it = 0; it < max_iter; ++it) {
    op.apply(p, q, level, Update::Replace);
    mask_dirichlet(q, level);
    const double pq = masked_dot(p, q, level);
    if (!(pq > 0.0)) fail_internal("cg: operator is not positive definite on the interior carriers");
    const double alpha = rz / pq;
    launch_axpy(X, P, alpha, count, s);
    launch_axpy(R, Q, -alpha, count, s);
    rr = masked_dot(r, r, level);
    res.iterations = it + 1;
    res.rel_residual = std::sqrt(rr / rr0);
    if (rr <= stop) {
      res.converged = true;
      break;
    }
    double rz_new = rr;
    if (Dg) {
      launch_jacobi(Z, R, Dg, count, s);
      rz_new = masked_dot(r, z, level);
    }
    launch_xpby(P, Z, rz_new / rz, count, s);  // p = z + beta p
    rz = rz_new;
  }
  return res;
}

double estimate_lambda_max(Operator& op, const Function& diag, int level, int iterations) {
  const Space sp = op.info().trial;
  if (diag.space() != sp || !diag.has_level(level)) fail_arg("lambda_max: diagonal not in the trial space");
  if (iterations < 1) fail_arg("lambda_max: iterations must be >= 1");
  Context& ctx = diag.ctx();
  const cudaStream_t s = ctx.stream();
  const i64 count = diag.size(level);
  Function v(ctx, sp), q(ctx, sp), w(ctx, sp);
  const double* D = diag.data(level);
  v.fill_seeded(level, 0x5eedULL, true);
  mask_dirichlet(v, level);
  double lambda = 0.0;
  for (int it = 0; it < iterations; ++it) {
    op.apply(v, q, level, Update::Replace);  // q = A v
    mask_dirichlet(q, level);
    launch_mul(w.data(level), v.data(level), D, count, s);  // w = D v
    const double vav = masked_dot(v, q, level), vdv = masked_dot(v, w, level);
    if (!(vdv > 0.0)) fail_internal("lambda_max: degenerate start vector");
    lambda = vav / vdv;
    launch_jacobi(v.data(level), q.data(level), D, count, s);  // v = D^-1 A v
    launch_mul(w.data(level), v.data(level), D, count, s);
    const double nrm = std::sqrt(masked_dot(v, w, level));  // ||v||_D
    if (!(nrm > 0.0)) break;
    launch_scale(v.data(level), 1.0 / nrm, count, s);
  }
  return lambda;
}

void chebyshev_smooth(Operator& op, const Function& diag, const Function& b, Function& x, int level, int degree,
                      double lambda_max, double eig_ratio) {
  const Space sp = op.info().trial;
  if (diag.space() != sp || b.space() != sp || x.space() != sp) fail_arg("chebyshev: functions not in the trial space");
  if (degree < 1 || !(lambda_max > 0.0) || !(eig_ratio > 1.0)) fail_arg("chebyshev: bad degree / eigenvalue bounds");
  Context& ctx = x.ctx();
  const cudaStream_t s = ctx.stream();
  const i64 count = x.size(level);
  const double hi = lambda_max, lo = lambda_max / eig_ratio;
  const double theta = 0.5 * (hi + lo), delta = 0.5 * (hi - lo), sigma = theta / delta;
  Function r(ctx, sp), z(ctx, sp), d(ctx, sp), q(ctx, sp);
  const double* D = diag.data(level);
  double* X = x.data(level);
  double* R = r.data(level);
  double* Z = z.data(level);
  double* Dd = d.data(level);
  double* Q = q.data(level);
  mask_dirichlet(x, level);
  op.apply(x, q, level, Update::Replace);
  TETMF_CUDA(cudaMemcpyAsync(R, b.data(level), sizeof(double) * count, cudaMemcpyDeviceToDevice, s));
  launch_axpy(R, Q, -1.0, count, s);  // r = b - A x
  mask_dirichlet(r, level);
  launch_jacobi(Z, R, D, count, s);
  launch_axpby(Dd, Z, 1.0 / theta, 0.0, count, s);  // d = z / theta
  double rho = 1.0 / sigma;
  for (int k = 0; k < degree; ++k) {
    launch_axpy(X, Dd, 1.0, count, s);  // x += d
    if (k + 1 == degree) break;
    op.apply(d, q, level, Update::Replace);
    mask_dirichlet(q, level);
    launch_axpy(R, Q, -1.0, count, s);  // r -= A d
    launch_jacobi(Z, R, D, count, s);
    const double rho_new = 1.0 / (2.0 * sigma - rho);
    launch_axpby(Dd, Z, 2.0 * rho_new / delta, rho_new * rho, count, s);  // d = rho' rho d + 2 rho' / delta z
    rho = rho_new;
  }
}

} // namespace tetmf

// quadrature.cpp -- quadrature rules by degree (quadrature.hpp; the
// reference's quadrature.cpp:19-147 restated).
#include "quadrature.hpp"

#include <cmath>

#include "runtime_check.hpp"

namespace tetmf {

namespace {

// eigenvalues (ascending) and first eigenvector components of a symmetric
// tridiagonal n x n matrix (n <= 8) by cyclic Jacobi rotations
void tridiag_eigen(int n, const double* diag, const double* off, double* vals, double* v0) {
  double a[8][8] = {}, v[8][8] = {};
  for (int i = 0; i < n; ++i) {
    a[i][i] = diag[i];
    v[i][i] = 1.0;
    if (i + 1 < n) a[i][i + 1] = a[i + 1][i] = off[i];
  }
  for (int sweep = 0; sweep < 100; ++sweep) {
    double offn = 0.0;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) offn += a[p][q] * a[p][q];
    if (offn < 1e-300) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        if (std::fabs(a[p][q]) < 1e-300) continue;
        const double th = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
        const double t = (th >= 0.0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double kp = a[k][p], kq = a[k][q];
          a[k][p] = c * kp - s * kq;
          a[k][q] = s * kp + c * kq;
        }
        for (int k = 0; k < n; ++k) {
          const double pk = a[p][k], qk = a[q][k];
          a[p][k] = c * pk - s * qk;
          a[q][k] = s * pk + c * qk;
        }
        for (int k = 0; k < n; ++k) {
          const double kp = v[k][p], kq = v[k][q];
          v[k][p] = c * kp - s * kq;
          v[k][q] = s * kp + c * kq;
        }
      }
  }
  int order[8];
  for (int i = 0; i < n; ++i) order[i] = i;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j)
      if (a[order[j]][order[j]] < a[order[i]][order[i]]) {
        const int t = order[i];
        order[i] = order[j];
        order[j] = t;
      }
  for (int j = 0; j < n; ++j) {
    vals[j] = a[order[j]][order[j]];
    v0[j] = v[0][order[j]];
  }
}

// n-point Gauss-Jacobi rule on [0, 1] for the weight (1 - x)^alpha: Golub-
// Welsch on the Jacobi matrix of the Jacobi polynomials P^(alpha, 0)
void gauss_jacobi01(int n, int alpha, double* x, double* w) {
  const double a = alpha, b = 0.0;
  double diag[8], off[8];
  for (int i = 0; i < n; ++i) {
    const double k = i;
    diag[i] = i == 0 ? (b - a) / (a + b + 2.0) : (b * b - a * a) / ((2.0 * k + a + b) * (2.0 * k + a + b + 2.0));
    if (i + 1 < n) {
      const double m = i + 1, s = 2.0 * m + a + b;
      off[i] = std::sqrt(4.0 * m * (m + a) * (m + b) * (m + a + b) / (s * s * (s + 1.0) * (s - 1.0)));
    }
  }
  double vals[8], v0[8];
  tridiag_eigen(n, diag, off, vals, v0);
  const double mu0 = std::pow(2.0, a + 1.0) / (a + 1.0);  // mass of (1-t)^a on [-1, 1]
  for (int i = 0; i < n; ++i) {
    x[i] = 0.5 * (1.0 + vals[i]);
    w[i] = mu0 * v0[i] * v0[i] / std::pow(2.0, a + 1.0);  // to [0, 1]: dt / 2, (1-t)^a -> 2^a (1-x)^a
  }
}

void push(QuadRule& r, double x, double y, double z, double w) {
  r.x.push_back(x);
  r.y.push_back(y);
  r.z.push_back(z);
  r.w.push_back(w);
}

} // namespace

QuadRule quadrature_rule(int degree) {
  QuadRule r;
  if (degree == 1) {
    push(r, 0.25, 0.25, 0.25, 1.0 / 6.0);
  } else if (degree == 2) {
    const double a = 0.58541019662496845446, b = 0.13819660112501051518, w = 1.0 / 24.0;
    push(r, a, b, b, w);
    push(r, b, a, b, w);
    push(r, b, b, a, w);
    push(r, b, b, b, w);
  } else if (degree == 4) {  // Keast: centroid, 4 points near the vertices, 6 near the edge midpoints
    push(r, 0.25, 0.25, 0.25, -148.0 / 11250.0);
    const double a = 11.0 / 14.0, b = 1.0 / 14.0, wa = 343.0 / 45000.0;
    push(r, a, b, b, wa);
    push(r, b, a, b, wa);
    push(r, b, b, a, wa);
    push(r, b, b, b, wa);
    const double t = std::sqrt(5.0 / 14.0), c = 0.25 * (1.0 + t), d = 0.25 * (1.0 - t), wc = 28.0 / 1125.0;
    const double l[6][3] = {{c, d, d}, {d, c, d}, {d, d, c}, {c, c, d}, {c, d, c}, {d, c, c}};
    for (const auto& p : l) push(r, p[0], p[1], p[2], wc);
  } else if (degree == 3 || degree == 5 || degree == 6) {  // conical (collapsed) product rule
    const int n = degree == 3 ? 2 : degree == 5 ? 3 : 4;
    double x2[8], w2[8], x1[8], w1[8], x0[8], w0[8];
    gauss_jacobi01(n, 2, x2, w2);
    gauss_jacobi01(n, 1, x1, w1);
    gauss_jacobi01(n, 0, x0, w0);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        for (int k = 0; k < n; ++k) {
          const double x = x2[i], y = x1[j] * (1.0 - x), z = x0[k] * (1.0 - x - y);
          push(r, x, y, z, w2[i] * w1[j] * w0[k]);
        }
  } else {
    fail_arg("quadrature: unsupported degree (supported: 1..6)");
  }
  return r;
}

} // namespace tetmf

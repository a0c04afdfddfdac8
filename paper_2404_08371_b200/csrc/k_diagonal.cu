// k_diagonal.cu -- operator diagonals (the inverse diagonal
// of Jacobi / Chebyshev smoothing; tetmf_op_diagonal, Jacobi-preconditioned CG).
//
// Per stored macro copy, d_i = sum over the micro elements e of the macro that
// contain carrier i of (A_e)_ii; the interface step then adds the copies
// (unsigned: (s_i)^2 = 1 for ND1 orientation signs), exactly as the assembled
// reference operator's diagonal (sum over all elements of all macros,
// forms.cpp:133-193 local_matrix).
//   P1  -Lap:  the centre weight of the point's stencil variant (tables.cpp)
//   P1K:       k_p1k_gather.cu (same incidence table, diagonal terms only)
//   N1:        per edge, the incident (orientation, local edge) pairs of its
//              class; (A_e)_ii = sa Kc_ii + B_aa g_bb + B_bb g_aa - 2 B_ab g_ab
//              (Gram form, tables.hpp N1GramTable)
// Deterministic: every carrier sums its own terms in a fixed order.
#include "device.hpp"
#include "runtime_check.hpp"

namespace tetmf {

namespace {

constexpr int kThreads = 256;

__device__ bool decode_pt(int n, i64 idx, int& x, int& y, int& z) {
  if (idx >= tet_count(n)) return false;
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (plane_offset(n, mid) <= idx) lo = mid; else hi = mid - 1;
  }
  z = lo;
  const i64 r = idx - plane_offset(n, z);
  lo = 0;
  hi = n - z;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (row_offset(n, z, mid) <= r) lo = mid; else hi = mid - 1;
  }
  y = lo;
  x = static_cast<int>(r - row_offset(n, z, y));
  return true;
}

// (orientation, local edge) pairs by edge class: the element anchored at
// (edge anchor - offset) with orientation o has the edge as local edge i
struct N1Incidence {
  int begin[8];                 // CSR over classes 0..6
  int o[36], i[36], ox[36], oy[36], oz[36];
};
constexpr N1Incidence make_n1_incidence() {
  N1Incidence t{};
  int k = 0;
  for (int c = 0; c < 7; ++c) {
    t.begin[c] = k;
    for (int o = 0; o < 6; ++o)
      for (int i = 0; i < 6; ++i) {
        const LocalEdgeRef r = local_edge_ref(o, i);
        if (r.cls != c) continue;
        t.o[k] = o;
        t.i[k] = i;
        t.ox[k] = r.ax;
        t.oy[k] = r.ay;
        t.oz[k] = r.az;
        ++k;
      }
  }
  t.begin[7] = k;
  return t;
}
__constant__ N1Incidence kN1Inc = make_n1_incidence();

__global__ void __launch_bounds__(kThreads)
p1_diagonal_kernel(double* __restrict__ d, const MacroDesc* __restrict__ macros, int nmacros, i64 stride, int n,
                   const P1DeviceTable* __restrict__ tabs) {
  const i64 tid = blockIdx.x * static_cast<i64>(kThreads) + threadIdx.x;
  if (tid >= stride * nmacros) return;
  const int li = static_cast<int>(tid / stride);
  int x, y, z;
  if (!decode_pt(n, tid - li * stride, x, y, z)) return;
  const int type = (x == 0 ? 1 : 0) | (y == 0 ? 2 : 0) | (z == 0 ? 4 : 0) | (x + y + z == n ? 8 : 0);
  d[tid] = tabs[macros[li].group].stencil[type][0];  // weight of the point itself
}

// N1 mass moments under quadrature(1) / quadrature(2) (tables.hpp
// n1_rule_moments): B_pq = sum_m beta_m R[m][pq] replaces S + beta_p + beta_q
__constant__ double kDiagRule[2][4][10];

template <int RULE>
__global__ void __launch_bounds__(kThreads)
n1_diagonal_kernel(double* __restrict__ d, const double* __restrict__ alpha, const double* __restrict__ beta,
                   const MacroDesc* __restrict__ macros, int nmacros, i64 stride, i64 cstride, i64 cf_stride, int n,
                   const N1GramTable* __restrict__ gram) {
  const i64 tid = blockIdx.x * static_cast<i64>(kThreads) + threadIdx.x;
  if (tid >= stride * nmacros) return;
  const int li = static_cast<int>(tid / stride);
  const i64 s = tid - li * stride;
  const int c = static_cast<int>(s / cstride);
  int ax, ay, az;
  if (c >= 7 || !decode_pt(n - 1, s - c * cstride, ax, ay, az)) return;
  const Off3 b = edge_base_from_anchor(c), dd = edge_dir(c);
  const int bx = ax + b.x, by = ay + b.y, bz = az + b.z;
  const int tx = bx + dd.x, ty = by + dd.y, tz = bz + dd.z;
  if (bx < 0 || by < 0 || bz < 0 || tx < 0 || ty < 0 || tz < 0 || bx + by + bz > n || tx + ty + tz > n) return;
  const double* __restrict__ A = alpha + static_cast<i64>(li) * cf_stride;
  const double* __restrict__ B = beta + static_cast<i64>(li) * cf_stride;
  const double* __restrict__ tb0 = &gram[macros[li].group].o[0][0];
  double acc = 0.0;
  for (int k = kN1Inc.begin[c]; k < kN1Inc.begin[c + 1]; ++k) {
    const int o = kN1Inc.o[k], i = kN1Inc.i[k];
    const int cx = ax - kN1Inc.ox[k], cy = ay - kN1Inc.oy[k], cz = az - kN1Inc.oz[k];  // element anchor
    if (cx < 0 || cy < 0 || cz < 0 || cx + cy + cz > orient_sum_limit(o, n)) continue;
    double al = 0.0, bv[4];
    for (int j = 0; j < 4; ++j) {
      const Off3 v = orient_offset(o, j);
      const i64 q = lattice_index(n, cx + v.x, cy + v.y, cz + v.z);
      al += __ldg(A + q);
      bv[j] = __ldg(B + q);
    }
    const int la = local_edge_vertex(i, 0), lb = local_edge_vertex(i, 1);
    double Baa, Bbb, Bab;
    if (RULE == 0) {
      const double S = (bv[0] + bv[1]) + (bv[2] + bv[3]);
      Baa = 2.0 * S + 4.0 * bv[la];
      Bbb = 2.0 * S + 4.0 * bv[lb];
      Bab = S + bv[la] + bv[lb];
    } else {
      Baa = Bbb = Bab = 0.0;
      for (int m = 0; m < 4; ++m) {
        Baa = fma(bv[m], kDiagRule[RULE - 1][m][sym4(la, la)], Baa);
        Bbb = fma(bv[m], kDiagRule[RULE - 1][m][sym4(lb, lb)], Bbb);
        Bab = fma(bv[m], kDiagRule[RULE - 1][m][sym4(la, lb)], Bab);
      }
    }
    const double* tb = tb0 + o * kGramRow;
    double m = Baa * tb[22 + sym4(lb, lb)];
    m = fma(Bbb, tb[22 + sym4(la, la)], m);
    m = fma(Bab, tb[32 + i], m);
    acc += fma(al, tb[sym6(i, i)], m);
  }
  d[tid] = acc;
}

unsigned grid_for(i64 count) {
  const i64 g = (count + kThreads - 1) / kThreads;
  return static_cast<unsigned>(g < 1 ? 1 : g);
}

} // namespace

void launch_p1_diagonal(double* d, const MacroDesc* d_macros, int nmacros, i64 macro_stride, int n,
                        const P1DeviceTable* d_tables, cudaStream_t s) {
  if (nmacros == 0) return;
  p1_diagonal_kernel<<<grid_for(macro_stride * nmacros), kThreads, 0, s>>>(d, d_macros, nmacros, macro_stride, n,
                                                                          d_tables);
  check_launch("p1_diagonal");
}

void launch_n1_diagonal(double* d, const double* alpha, const double* beta, const MacroDesc* d_macros, int nmacros,
                        i64 macro_stride, i64 class_stride, i64 coeff_stride, int n, const N1GramTable* d_gram,
                        int rule, cudaStream_t s) {
  if (nmacros == 0) return;
  static const bool ready = [] {
    double R[2][4][10];
    n1_rule_moments(1, R[0]);
    n1_rule_moments(2, R[1]);
    TETMF_CUDA(cudaMemcpyToSymbol(kDiagRule, R, sizeof(R)));
    return true;
  }();
  (void)ready;
  const unsigned grid = grid_for(macro_stride * nmacros);
  if (rule == 0)
    n1_diagonal_kernel<0><<<grid, kThreads, 0, s>>>(d, alpha, beta, d_macros, nmacros, macro_stride, class_stride,
                                                    coeff_stride, n, d_gram);
  else if (rule == 1)
    n1_diagonal_kernel<1><<<grid, kThreads, 0, s>>>(d, alpha, beta, d_macros, nmacros, macro_stride, class_stride,
                                                    coeff_stride, n, d_gram);
  else
    n1_diagonal_kernel<2><<<grid, kThreads, 0, s>>>(d, alpha, beta, d_macros, nmacros, macro_stride, class_stride,
                                                    coeff_stride, n, d_gram);
  check_launch("n1_diagonal");
}

} // namespace tetmf

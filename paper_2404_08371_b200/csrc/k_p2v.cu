// k_p2v.cu -- P2V apply: -div(k grad u), u and k in P2
// (forms.cpp:12), exact integration.
//
// First version (cf. k_apply_v1.cu): one thread per (macro, cube anchor); the
// up-to-six micro elements of the cube gather their ten P2 values (vertices
// at the four corners, edge midpoints at the six local edges; P2 edge DoFs
// are unsigned) and the ten coefficient values, form A_e = sum_m k_m T_m from
// the exact per-orientation tables (tables.cpp p2v_table; 55 packed entries x
// 10 coefficient terms) and scatter A_e x_e with FP64 atomics into a zeroed y.
// The interface step then sums the macro copies as for P1 / ND1.
#include "device.hpp"
#include "runtime_check.hpp"

namespace tetmf {

namespace {

constexpr int kThreads = 128;

__device__ bool decode_anchor(int n, i64 idx, int& x, int& y, int& z) {
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

__global__ void __launch_bounds__(kThreads)
p2v_cubes_kernel(const double* __restrict__ x, const double* __restrict__ kc, double* __restrict__ y,
                 const MacroDesc* __restrict__ macros, int nmacros, i64 stride, i64 cstride, int n,
                 const P2VTable* __restrict__ tabs) {
  const i64 anchors = tet_count(n - 1);
  const i64 tid = blockIdx.x * static_cast<i64>(kThreads) + threadIdx.x;
  if (tid >= anchors * nmacros) return;
  const int li = static_cast<int>(tid / anchors);
  int ax, ay, az;
  decode_anchor(n - 1, tid - li * anchors, ax, ay, az);
  const i64 vstride = (tet_count(n) + 31) / 32 * 32;
  const double* __restrict__ xm = x + static_cast<i64>(li) * stride;
  const double* __restrict__ km = kc + static_cast<i64>(li) * stride;
  double* __restrict__ ym = y + static_cast<i64>(li) * stride;
  const P2VTable& T = tabs[macros[li].group];
  const int s = ax + ay + az;
  for (int o = 0; o < 6; ++o) {
    if (s > orient_sum_limit(o, n)) continue;
    i64 idx[10];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const Off3 v = orient_offset(o, i);
      idx[i] = lattice_index(n, ax + v.x, ay + v.y, az + v.z);
    }
#pragma unroll
    for (int e = 0; e < 6; ++e) {
      const LocalEdgeRef r = local_edge_ref(o, e);
      idx[4 + e] = vstride + r.cls * cstride + lattice_index(n - 1, ax + r.ax, ay + r.ay, az + r.az);
    }
    double xe[10], ke[10];
#pragma unroll
    for (int i = 0; i < 10; ++i) {
      xe[i] = __ldg(xm + idx[i]);
      ke[i] = __ldg(km + idx[i]);
    }
    double ye[10];
#pragma unroll
    for (int i = 0; i < 10; ++i) ye[i] = 0.0;
#pragma unroll
    for (int i = 0; i < 10; ++i) {
#pragma unroll
      for (int j = i; j < 10; ++j) {
        const int q = sym10(i, j);
        double a = 0.0;
#pragma unroll
        for (int m = 0; m < 10; ++m) a = fma(ke[m], T.T[o][m][q], a);
        ye[i] = fma(a, xe[j], ye[i]);
        if (j != i) ye[j] = fma(a, xe[i], ye[j]);
      }
    }
#pragma unroll
    for (int i = 0; i < 10; ++i) atomicAdd(ym + idx[i], ye[i]);
  }
}

} // namespace

void launch_p2v_cubes(const double* x, const double* k, double* y, const MacroDesc* d_macros, int nmacros,
                      i64 macro_stride, i64 class_stride, int n, const P2VTable* d_tables, cudaStream_t s) {
  TETMF_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * macro_stride * nmacros, s));
  const i64 total = tet_count(n - 1) * nmacros;
  if (total == 0) return;
  p2v_cubes_kernel<<<static_cast<unsigned>((total + kThreads - 1) / kThreads), kThreads, 0, s>>>(
      x, k, y, d_macros, nmacros, macro_stride, class_stride, n, d_tables);
  check_launch("p2v_cubes");
}

} // namespace tetmf

// k_apply_v1.cu -- first (reference-structure) versions of K1-K3.
//
// K1 p1_stencil: one thread per lattice point, y(p) = sum_k w[type(p)][k]
//    x(p + off_k) with the macro's 15-point stencil variants.
// K2 p1k_cubes / K3 n1_cubes: one thread per cube anchor, the up-to-six
//    micro elements of the cube, local matvec, FP64 atomic scatter into a
//    zeroed y (Alg. 1 LocalApply, in cubes order,
//    PAPER.md:586-621).
#include "device.hpp"
#include "runtime_check.hpp"

namespace tetmf {

namespace {

constexpr int kThreads = 256;

inline unsigned grid_for(i64 count) {
  i64 g = (count + kThreads - 1) / kThreads;
  return static_cast<unsigned>(g < 1 ? 1 : g);
}

__device__ bool decode(int n, i64 idx, int& x, int& y, int& z) {
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

__global__ void p1_stencil_v1_kernel(const double* __restrict__ x, double* __restrict__ y,
                                     const MacroDesc* __restrict__ macros, int nmacros, i64 stride, int n,
                                     const P1DeviceTable* __restrict__ tabs) {
  const i64 tid = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (tid >= stride * nmacros) return;
  const int li = static_cast<int>(tid / stride);
  const i64 slot = tid - li * stride;
  int px, py, pz;
  if (!decode(n, slot, px, py, pz)) {
    y[tid] = 0.0;
    return;
  }
  const MacroDesc& m = macros[li];
  const double* xm = x + static_cast<i64>(li) * stride;
  const int type = (px == 0 ? 1 : 0) | (py == 0 ? 2 : 0) | (pz == 0 ? 4 : 0) | (px + py + pz == n ? 8 : 0);
  const double* w = tabs[m.group].stencil[type];
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < 15; ++k) {
    const Off3 o = stencil_offset(k);
    const int qx = px + o.x, qy = py + o.y, qz = pz + o.z;
    if (type != 0 && (qx < 0 || qy < 0 || qz < 0 || qx + qy + qz > n)) continue;
    acc += __ldg(w + k) * __ldg(xm + lattice_index(n, qx, qy, qz));
  }
  y[tid] = acc;
}

__global__ void p1k_cubes_v1_kernel(const double* __restrict__ x, const double* __restrict__ kc,
                                    double* __restrict__ y, const MacroDesc* __restrict__ macros, int nmacros,
                                    i64 stride, int n, const P1DeviceTable* __restrict__ tabs) {
  const i64 anchors = tet_count(n - 1);
  const i64 tid = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (tid >= anchors * nmacros) return;
  const int li = static_cast<int>(tid / anchors);
  const i64 a = tid - li * anchors;
  int ax, ay, az;
  decode(n - 1, a, ax, ay, az);
  const MacroDesc& m = macros[li];
  const double* K = tabs[m.group].K[0];
  const double* xm = x + static_cast<i64>(li) * stride;
  const double* km = kc + static_cast<i64>(li) * stride;
  double* ym = y + static_cast<i64>(li) * stride;
  const int s = ax + ay + az;
  for (int o = 0; o < 6; ++o) {
    if (s > orient_sum_limit(o, n)) continue;
    i64 idx[4];
    double xe[4], ks = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const Off3 v = orient_offset(o, i);
      idx[i] = lattice_index(n, ax + v.x, ay + v.y, az + v.z);
      xe[i] = __ldg(xm + idx[i]);
      ks += __ldg(km + idx[i]);
    }
    const double kb = 0.25 * ks;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      double r = 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) r += __ldg(K + o * 10 + sym4(i, j)) * xe[j];
      atomicAdd(ym + idx[i], kb * r);
    }
  }
}

__global__ void n1_cubes_v1_kernel(const double* __restrict__ x, const double* __restrict__ alpha,
                                   const double* __restrict__ beta, double* __restrict__ y,
                                   const MacroDesc* __restrict__ macros, int nmacros, i64 stride, i64 cstride,
                                   i64 coeff_stride, int n, const N1DeviceTable* __restrict__ tabs) {
  const i64 anchors = tet_count(n - 1);
  const i64 tid = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (tid >= anchors * nmacros) return;
  const int li = static_cast<int>(tid / anchors);
  const i64 a = tid - li * anchors;
  int ax, ay, az;
  decode(n - 1, a, ax, ay, az);
  const MacroDesc& m = macros[li];
  const double* tab = &tabs[m.group].e[0][0][0];
  const double* xm = x + static_cast<i64>(li) * stride;
  double* ym = y + static_cast<i64>(li) * stride;
  const double* am = alpha + static_cast<i64>(li) * coeff_stride;
  const double* bm = beta + static_cast<i64>(li) * coeff_stride;
  const int s = ax + ay + az;
  for (int o = 0; o < 6; ++o) {
    if (s > orient_sum_limit(o, n)) continue;
    double sa = 0.0, bt[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const Off3 v = orient_offset(o, i);
      const i64 vi = lattice_index(n, ax + v.x, ay + v.y, az + v.z);
      sa += __ldg(am + vi);
      bt[i] = __ldg(bm + vi);
    }
    i64 eidx[6];
    double xe[6];
#pragma unroll
    for (int le = 0; le < 6; ++le) {
      const LocalEdgeRef r = local_edge_ref(o, le);
      eidx[le] = r.cls * cstride + lattice_index(n - 1, ax + r.ax, ay + r.ay, az + r.az);
      xe[le] = __ldg(xm + eidx[le]);
    }
    const double* t = tab + o * 105;
    double A[21];
#pragma unroll
    for (int q = 0; q < 21; ++q)
      A[q] = sa * __ldg(t + q) + bt[0] * __ldg(t + 21 + q) + bt[1] * __ldg(t + 42 + q) +
             bt[2] * __ldg(t + 63 + q) + bt[3] * __ldg(t + 84 + q);
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      double r = 0.0;
#pragma unroll
      for (int j = 0; j < 6; ++j) r += A[sym6(i, j)] * xe[j];
      atomicAdd(ym + eidx[i], r);
    }
  }
}

} // namespace

void launch_p1_stencil(const double* x, double* y, const MacroDesc* d_macros, int nmacros, i64 macro_stride, int n,
                       const P1DeviceTable* d_tables, cudaStream_t s) {
  const i64 total = macro_stride * nmacros;
  p1_stencil_v1_kernel<<<grid_for(total), kThreads, 0, s>>>(x, y, d_macros, nmacros, macro_stride, n, d_tables);
  check_launch("p1_stencil");
}

void launch_p1k_cubes(const double* x, const double* k, double* y, const MacroDesc* d_macros, int nmacros,
                      i64 macro_stride, int n, const P1DeviceTable* d_tables, cudaStream_t s) {
  TETMF_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * macro_stride * nmacros, s));
  const i64 total = tet_count(n - 1) * nmacros;
  p1k_cubes_v1_kernel<<<grid_for(total), kThreads, 0, s>>>(x, k, y, d_macros, nmacros, macro_stride, n, d_tables);
  check_launch("p1k_cubes");
}

void launch_n1_cubes(const double* x, const double* alpha, const double* beta, double* y,
                     const MacroDesc* d_macros, int nmacros, i64 macro_stride, i64 class_stride,
                     i64 coeff_stride, int n, const N1DeviceTable* d_tables, cudaStream_t s) {
  TETMF_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * macro_stride * nmacros, s));
  const i64 total = tet_count(n - 1) * nmacros;
  n1_cubes_v1_kernel<<<grid_for(total), kThreads, 0, s>>>(x, alpha, beta, y, d_macros, nmacros, macro_stride,
                                                          class_stride, coeff_stride, n, d_tables);
  check_launch("n1_cubes");
}

} // namespace tetmf

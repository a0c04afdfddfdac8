// k_transfer.cu -- P1 <-> ND1 discrete gradient (the
// transfer of the hybrid (Hiptmair) smoother around the N1 apply).
//
//   G  : P1 -> ND1,  (G phi)_e = phi(tip) - phi(base)   (edge e = base -> tip in
//        this library's macro-local canonical orientation; equals the ND1
//        interpolant of grad phi: the line integral of grad phi . t)
//   G^T: ND1 -> P1,  (G^T u)_p = sum over edges e incident to p of
//        (+u_e if p is e's tip, -u_e if p is its base)
// G is local per stored copy (every copy of an edge sees the same endpoint
// values, stored in its own macro's orientation, so copies stay consistent).
// G^T sums over the edges incident to p in the copy's macro, counting only
// the OWNER copy of each edge (solver slot class, bit 1), then the P1
// interface step adds the partial sums of the macros sharing p -- each global
// edge contributes exactly once.
#include "device.hpp"
#include "runtime_check.hpp"

namespace tetmf {

namespace {

constexpr int kThreads = 256;

__device__ bool decode_pt2(int n, i64 idx, int& x, int& y, int& z) {
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

__device__ __forceinline__ bool in_lattice(int n, int x, int y, int z) {
  return x >= 0 && y >= 0 && z >= 0 && x + y + z <= n;
}
__device__ __forceinline__ unsigned pmask(int n, int x, int y, int z) {
  return (x + y + z < n ? 1u : 0u) | (x > 0 ? 2u : 0u) | (y > 0 ? 4u : 0u) | (z > 0 ? 8u : 0u);
}

__global__ void __launch_bounds__(kThreads)
gradient_kernel(const double* __restrict__ phi, double* __restrict__ u, int nmacros, i64 stride_nd1, i64 cstride,
                i64 stride_p1, int n) {
  const i64 tid = blockIdx.x * static_cast<i64>(kThreads) + threadIdx.x;
  if (tid >= stride_nd1 * nmacros) return;
  const int li = static_cast<int>(tid / stride_nd1);
  const i64 s = tid - li * stride_nd1;
  const int c = static_cast<int>(s / cstride);
  int ax, ay, az;
  if (c >= 7 || !decode_pt2(n - 1, s - c * cstride, ax, ay, az)) return;
  const Off3 b = edge_base_from_anchor(c), d = edge_dir(c);
  const int bx = ax + b.x, by = ay + b.y, bz = az + b.z;
  const int tx = bx + d.x, ty = by + d.y, tz = bz + d.z;
  if (!in_lattice(n, bx, by, bz) || !in_lattice(n, tx, ty, tz)) return;
  const double* __restrict__ P = phi + static_cast<i64>(li) * stride_p1;
  u[tid] = P[lattice_index(n, tx, ty, tz)] - P[lattice_index(n, bx, by, bz)];
}

// table: ND1 solver slot classes per local macro [16 * li + mask], bit 1 owner
__global__ void __launch_bounds__(kThreads)
gradient_t_kernel(const double* __restrict__ u, double* __restrict__ phi, int nmacros, i64 stride_nd1, i64 cstride,
                  i64 stride_p1, int n, const unsigned char* __restrict__ table) {
  const i64 tid = blockIdx.x * static_cast<i64>(kThreads) + threadIdx.x;
  if (tid >= stride_p1 * nmacros) return;
  const int li = static_cast<int>(tid / stride_p1);
  int px, py, pz;
  if (!decode_pt2(n, tid - li * stride_p1, px, py, pz)) return;
  const double* __restrict__ U = u + static_cast<i64>(li) * stride_nd1;
  const unsigned char* tb = table + 16 * li;
  const unsigned mp = pmask(n, px, py, pz);
  double acc = 0.0;
  for (int c = 0; c < 7; ++c) {
    const Off3 b = edge_base_from_anchor(c), d = edge_dir(c);
    // edge c with tip p (sign +1) and with base p (sign -1)
    for (int side = 0; side < 2; ++side) {
      const int sg = side == 0 ? 1 : -1;
      const int ox = px - sg * d.x, oy = py - sg * d.y, oz = pz - sg * d.z;  // the other endpoint
      if (!in_lattice(n, ox, oy, oz)) continue;
      const int bx = side == 0 ? ox : px, by = side == 0 ? oy : py, bz = side == 0 ? oz : pz;  // base
      const int ax = bx - b.x, ay = by - b.y, az = bz - b.z;  // anchor
      const unsigned mask = mp | pmask(n, ox, oy, oz);
      if (!(tb[mask] & 2u)) continue;  // another macro owns this edge
      const double v = U[c * cstride + lattice_index(n - 1, ax, ay, az)];
      acc += side == 0 ? v : -v;
    }
  }
  phi[tid] = acc;
}

unsigned grid_of(i64 count) {
  const i64 g = (count + kThreads - 1) / kThreads;
  return static_cast<unsigned>(g < 1 ? 1 : g);
}

} // namespace

void launch_gradient(const double* phi, double* u, int nmacros, i64 stride_nd1, i64 class_stride, i64 stride_p1,
                     int n, cudaStream_t s) {
  if (nmacros == 0) return;
  gradient_kernel<<<grid_of(stride_nd1 * nmacros), kThreads, 0, s>>>(phi, u, nmacros, stride_nd1, class_stride,
                                                                     stride_p1, n);
  check_launch("gradient");
}

void launch_gradient_t(const double* u, double* phi, int nmacros, i64 stride_nd1, i64 class_stride, i64 stride_p1,
                       int n, const unsigned char* d_nd1_slot_table, cudaStream_t s) {
  if (nmacros == 0) return;
  gradient_t_kernel<<<grid_of(stride_p1 * nmacros), kThreads, 0, s>>>(u, phi, nmacros, stride_nd1, class_stride,
                                                                       stride_p1, n, d_nd1_slot_table);
  check_launch("gradient_t");
}

} // namespace tetmf

// solver.cu -- Dirichlet-masked vector kernels of the matrix-free CG
// (the first caller of the apply).
//
// Functions store every macro's closure, so interface carriers have one copy
// per sharing macro (layout.hpp). The solver's vectors keep all copies equal
// (the apply's interface sum does, and the vector updates are elementwise),
// so an inner product must count each carrier once: weight 1 on the OWNER
// copy (lowest sharing macro id, the reference's owner rule fespace.cpp:
// 216-231) of an INTERIOR carrier (not in a domain-boundary face plane,
// fespace.cpp:207-214), 0 elsewhere (other copies, Dirichlet carriers,
// padding). Both bits depend only on the carrier's support mask in its macro
// (local vertices with nonzero barycentric weight), so each macro carries a
// 16-entry table [mask] -> {bit 0 interior, bit 1 owner} and the kernels
// derive the mask from the slot's lattice position:
//   P1 slot: point p, mask = {v : w_v(p) > 0}
//   ND1 slot (class c, anchor a): mask = mask(base) | mask(tip), base =
//     a + edge_base_from_anchor(c), tip = base + edge_dir(c)
// Reductions are deterministic: a fixed grid, fixed per-thread order, a
// fixed shuffle tree and one fixed-order final pass (independent of the
// GPU's SM count).
#include "device.hpp"
#include "runtime_check.hpp"
#include "solver.hpp"

namespace tetmf {

namespace {

constexpr int kThreads = 256;
constexpr int kBlocks = 1024;  // fixed reduction grid

__device__ __forceinline__ unsigned point_mask(int n, int x, int y, int z) {
  return (x + y + z < n ? 1u : 0u) | (x > 0 ? 2u : 0u) | (y > 0 ? 4u : 0u) | (z > 0 ? 8u : 0u);
}

__device__ bool decode_point(int n, i64 idx, int& x, int& y, int& z) {
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

// slot class {bit 0 interior, bit 1 owner} of storage entry i; 0 for padding
// and non-existent carriers
__device__ unsigned slot_class(const SlotSpace& sp, const unsigned char* __restrict__ table, i64 i) {
  const int li = static_cast<int>(i / sp.macro_stride);
  i64 s = i - static_cast<i64>(li) * sp.macro_stride;
  const int n = sp.n;
  unsigned mask;
  const i64 vstride = sp.nd1 == 2 ? (tet_count(n) + 31) / 32 * 32 : 0;  // P2: vertex block first
  if (sp.nd1 == 0 || (sp.nd1 == 2 && s < vstride)) {
    int x, y, z;
    if (!decode_point(n, s, x, y, z)) return 0;
    mask = point_mask(n, x, y, z);
  } else {
    s -= vstride;
    const int c = static_cast<int>(s / sp.class_stride);
    int ax, ay, az;
    if (c >= 7 || !decode_point(n - 1, s - c * sp.class_stride, ax, ay, az)) return 0;
    const Off3 b = edge_base_from_anchor(c), d = edge_dir(c);
    const int bx = ax + b.x, by = ay + b.y, bz = az + b.z;
    const int tx = bx + d.x, ty = by + d.y, tz = bz + d.z;
    if (bx < 0 || by < 0 || bz < 0 || tx < 0 || ty < 0 || tz < 0 || bx + by + bz > n || tx + ty + tz > n) return 0;
    mask = point_mask(n, bx, by, bz) | point_mask(n, tx, ty, tz);
  }
  return table[16 * li + mask];
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// partial[block] = sum over the block's grid-stride slots of w(i) a[i] b[i]
__global__ void __launch_bounds__(kThreads)
masked_dot_kernel(const double* __restrict__ a, const double* __restrict__ b, SlotSpace sp,
                  const unsigned char* __restrict__ table, i64 count, double* __restrict__ partial) {
  __shared__ double red[kThreads / 32];
  double acc = 0.0;
  for (i64 i = blockIdx.x * static_cast<i64>(kThreads) + threadIdx.x; i < count;
       i += static_cast<i64>(kThreads) * kBlocks) {
    if (slot_class(sp, table, i) == 3u) acc = fma(a[i], b[i], acc);
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < kThreads / 32 ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) partial[blockIdx.x] = v;
  }
}

// out[0] = sum of partial[0 .. nparts) in a fixed order (one block)
__global__ void __launch_bounds__(kThreads) sum_partials_kernel(const double* __restrict__ partial, int nparts,
                                                                double* __restrict__ out) {
  __shared__ double red[kThreads / 32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < nparts; i += kThreads) acc += partial[i];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < kThreads / 32 ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) out[0] = v;
  }
}

// zero every non-interior (Dirichlet) carrier
__global__ void __launch_bounds__(kThreads)
mask_dirichlet_kernel(double* __restrict__ y, SlotSpace sp, const unsigned char* __restrict__ table, i64 count) {
  for (i64 i = blockIdx.x * static_cast<i64>(kThreads) + threadIdx.x; i < count;
       i += static_cast<i64>(kThreads) * gridDim.x) {
    if ((slot_class(sp, table, i) & 1u) == 0) y[i] = 0.0;
  }
}

// y = x + beta y   (CG search direction update)
__global__ void __launch_bounds__(kThreads) xpby_kernel(double* __restrict__ y, const double* __restrict__ x,
                                                        double beta, i64 count) {
  for (i64 i = blockIdx.x * static_cast<i64>(kThreads) + threadIdx.x; i < count;
       i += static_cast<i64>(kThreads) * gridDim.x)
    y[i] = fma(beta, y[i], x[i]);
}

// z = r / d where d != 0 (Jacobi preconditioner; Dirichlet carriers have r = 0)
__global__ void __launch_bounds__(kThreads) jacobi_kernel(double* __restrict__ z, const double* __restrict__ r,
                                                          const double* __restrict__ d, i64 count) {
  for (i64 i = blockIdx.x * static_cast<i64>(kThreads) + threadIdx.x; i < count;
       i += static_cast<i64>(kThreads) * gridDim.x) {
    const double di = d[i];
    z[i] = di != 0.0 ? r[i] / di : 0.0;
  }
}

// y = a x + b y
__global__ void __launch_bounds__(kThreads) axpby_kernel(double* __restrict__ y, const double* __restrict__ x,
                                                         double a, double b, i64 count) {
  for (i64 i = blockIdx.x * static_cast<i64>(kThreads) + threadIdx.x; i < count;
       i += static_cast<i64>(kThreads) * gridDim.x)
    y[i] = fma(a, x[i], b * y[i]);
}

// y = a y
__global__ void __launch_bounds__(kThreads) scale_kernel(double* __restrict__ y, double a, i64 count) {
  for (i64 i = blockIdx.x * static_cast<i64>(kThreads) + threadIdx.x; i < count;
       i += static_cast<i64>(kThreads) * gridDim.x)
    y[i] *= a;
}

// z = x .* d
__global__ void __launch_bounds__(kThreads) mul_kernel(double* __restrict__ z, const double* __restrict__ x,
                                                       const double* __restrict__ d, i64 count) {
  for (i64 i = blockIdx.x * static_cast<i64>(kThreads) + threadIdx.x; i < count;
       i += static_cast<i64>(kThreads) * gridDim.x)
    z[i] = x[i] * d[i];
}

unsigned stream_grid(i64 count) {
  const i64 g = (count + kThreads - 1) / kThreads;
  return static_cast<unsigned>(g < 1 ? 1 : (g > 148 * 32 ? 148 * 32 : g));
}

} // namespace

int masked_dot_partials() { return kBlocks; }

void launch_masked_dot(const double* a, const double* b, const SlotSpace& sp, const unsigned char* d_table, i64 count,
                       double* d_partials, double* d_out, cudaStream_t s) {
  masked_dot_kernel<<<kBlocks, kThreads, 0, s>>>(a, b, sp, d_table, count, d_partials);
  check_launch("masked_dot");
  sum_partials_kernel<<<1, kThreads, 0, s>>>(d_partials, kBlocks, d_out);
  check_launch("sum_partials");
}

void launch_sum_ordered(const double* d_values, int count, double* d_out, cudaStream_t s) {
  sum_partials_kernel<<<1, kThreads, 0, s>>>(d_values, count, d_out);
  check_launch("sum_ordered");
}

void launch_mask_dirichlet(double* y, const SlotSpace& sp, const unsigned char* d_table, i64 count, cudaStream_t s) {
  mask_dirichlet_kernel<<<stream_grid(count), kThreads, 0, s>>>(y, sp, d_table, count);
  check_launch("mask_dirichlet");
}

void launch_jacobi(double* z, const double* r, const double* d, i64 count, cudaStream_t s) {
  jacobi_kernel<<<stream_grid(count), kThreads, 0, s>>>(z, r, d, count);
  check_launch("jacobi");
}

void launch_axpby(double* y, const double* x, double a, double b, i64 count, cudaStream_t s) {
  axpby_kernel<<<stream_grid(count), kThreads, 0, s>>>(y, x, a, b, count);
  check_launch("axpby");
}

void launch_scale(double* y, double a, i64 count, cudaStream_t s) {
  scale_kernel<<<stream_grid(count), kThreads, 0, s>>>(y, a, count);
  check_launch("scale");
}

void launch_mul(double* z, const double* x, const double* d, i64 count, cudaStream_t s) {
  mul_kernel<<<stream_grid(count), kThreads, 0, s>>>(z, x, d, count);
  check_launch("mul");
}

void launch_xpby(double* y, const double* x, double beta, i64 count, cudaStream_t s) {
  xpby_kernel<<<stream_grid(count), kThreads, 0, s>>>(y, x, beta, count);
  check_launch("xpby");
}

} // namespace tetmf

// k_common.cu -- fill, reference-numbering permutation, interface sum (K4).
#include <cmath>

#include "device.hpp"
#include "exchange.hpp"
#include "runtime_check.hpp"

namespace tetmf {

namespace {

constexpr int kThreads = 256;

inline unsigned grid_for(i64 count, int threads = kThreads) {
  i64 g = (count + threads - 1) / threads;
  if (g < 1) g = 1;
  return static_cast<unsigned>(g);
}

// inverse of lattice_index for extent n: returns false for padding slots
__device__ bool decode_lattice(int n, i64 idx, int& x, int& y, int& z) {
  if (idx >= tet_count(n)) return false;
  int lo = 0, hi = n;
  while (lo < hi) {  // largest z with plane_offset(n, z) <= idx
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

// integer world coordinates (scaled by n*D) of lattice point p
__device__ void world_int(const MacroDesc& m, int x, int y, int z, i64 W[3]) {
  for (int r = 0; r < 3; ++r) W[r] = m.V0[r] + x * m.E[0][r] + y * m.E[1][r] + z * m.E[2][r];
}

// world coordinates as the reference computes them (lattice_to_world,
// mesh.cpp:264-271): p0 + h * (x*e1 + y*e2 + z*e3)
__device__ void world_pos(const MacroDesc& m, int n, int x, int y, int z, double P[3]) {
  const double h = 1.0 / static_cast<double>(n);
  for (int r = 0; r < 3; ++r)
    P[r] = m.X0[r] + h * ((static_cast<double>(x) * m.dX[0][r] + static_cast<double>(y) * m.dX[1][r]) +
                          static_cast<double>(z) * m.dX[2][r]);
}

// Dirichlet carrier: its support simplex lies in a domain boundary face of
// some macro (Topology::dirichlet_mask; fespace.cpp:207-214, 226)
__device__ bool on_boundary_face(const MacroDesc& m, unsigned mask) { return (m.dmask >> (mask & 15u)) & 1; }

__device__ unsigned support_mask_dev(int n, int x, int y, int z) {
  return (n - x - y - z > 0 ? 1u : 0u) | (x > 0 ? 2u : 0u) | (y > 0 ? 4u : 0u) | (z > 0 ? 8u : 0u);
}

// region: entries per macro this fill covers (the P2 vertex block, or the
// whole P1 block); stride: entries per macro of the function
__global__ void fill_seeded_p1_kernel(double* out, const MacroDesc* macros, int nmacros, i64 stride, i64 region,
                                      int n, std::uint64_t seed, bool dirichlet) {
  const i64 tid = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (tid >= region * nmacros) return;
  const int li = static_cast<int>(tid / region);
  const i64 slot = tid - li * region;
  out += static_cast<i64>(li) * stride - static_cast<i64>(li) * region;  // out[tid] = macro li, slot
  const MacroDesc& m = macros[li];
  int x, y, z;
  if (!decode_lattice(n, slot, x, y, z)) {
    out[tid] = 0.0;
    return;
  }
  if (dirichlet && on_boundary_face(m, support_mask_dev(n, x, y, z))) {
    out[tid] = 0.0;
    return;
  }
  i64 W[3];
  world_int(m, x, y, z, W);
  out[tid] = seeded_uniform(seed, key_hash_vertex(W[0], W[1], W[2]));
}

// unsigned_edges (P2 midpoint DoFs): the value of the key-ascending edge,
// whatever the storage direction; ND1: signed along the storage direction
__global__ void fill_seeded_nd1_kernel(double* out, const MacroDesc* macros, int nmacros, i64 stride, i64 region,
                                       i64 cstride, int n, std::uint64_t seed, bool dirichlet, bool unsigned_edges) {
  const i64 tid = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (tid >= region * nmacros) return;
  const int li = static_cast<int>(tid / region);
  const i64 r = tid - li * region;
  out += static_cast<i64>(li) * stride - static_cast<i64>(li) * region;
  const int c = static_cast<int>(r / cstride);
  const i64 slot = r - c * cstride;
  const MacroDesc& m = macros[li];
  int ax, ay, az;
  if (!decode_lattice(n - 1, slot, ax, ay, az) || (c == 6 && ax + ay + az > n - 2)) {
    out[tid] = 0.0;
    return;
  }
  const Off3 bo = edge_base_from_anchor(c);
  const int bx = ax + bo.x, by = ay + bo.y, bz = az + bo.z;
  const Off3 dc = edge_dir(c);
  const int tx = bx + dc.x, ty = by + dc.y, tz = bz + dc.z;
  if (dirichlet &&
      on_boundary_face(m, support_mask_dev(n, bx, by, bz) | support_mask_dev(n, tx, ty, tz))) {
    out[tid] = 0.0;
    return;
  }
  i64 B[3], T[3];
  world_int(m, bx, by, bz, B);
  world_int(m, tx, ty, tz, T);
  double v;
  if (lex_less(B[0], B[1], B[2], T[0], T[1], T[2]))
    v = seeded_uniform(seed, key_hash_edge(B[0], B[1], B[2], T[0], T[1], T[2]));
  else
    v = seeded_uniform(seed, key_hash_edge(T[0], T[1], T[2], B[0], B[1], B[2])) * (unsigned_edges ? 1.0 : -1.0);
  out[tid] = v;
}

__device__ double coeff_value(int which, double c, const double P[3]) {
  switch (which) {
    case 0: return 1.0 + P[0] * P[0] + P[1] * P[1];
    case 1: return 2.0 + sin(M_PI * P[2]);
    case 2: return 1.0 + 0.5 * sin(2.0 * M_PI * P[0]) * cos(2.0 * M_PI * P[1]) * (1.0 + P[2]);
    default: return c;
  }
}

__global__ void fill_coeff_kernel(double* out, const MacroDesc* macros, int nmacros, i64 stride, i64 region, int n,
                                  CoeffSpec spec) {
  const i64 tid = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (tid >= region * nmacros) return;
  const int li = static_cast<int>(tid / region);
  const i64 slot = tid - li * region;
  out += static_cast<i64>(li) * stride - static_cast<i64>(li) * region;
  int x, y, z;
  if (!decode_lattice(n, slot, x, y, z)) {
    out[tid] = 0.0;
    return;
  }
  double P[3];
  world_pos(macros[li], n, x, y, z, P);
  out[tid] = coeff_value(spec.which, spec.value, P);
}

// P2 coefficient edge DoFs: nodal value at the edge midpoint (fespace.cpp:
// 494-506)
__global__ void fill_coeff_edges_kernel(double* out, const MacroDesc* macros, int nmacros, i64 stride, i64 region,
                                        i64 cstride, int n, CoeffSpec spec) {
  const i64 tid = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (tid >= region * nmacros) return;
  const int li = static_cast<int>(tid / region);
  const i64 r = tid - li * region;
  out += static_cast<i64>(li) * stride - static_cast<i64>(li) * region;
  const int c = static_cast<int>(r / cstride);
  int ax, ay, az;
  if (c >= 7 || !decode_lattice(n - 1, r - c * cstride, ax, ay, az) || (c == 6 && ax + ay + az > n - 2)) {
    out[tid] = 0.0;
    return;
  }
  const Off3 bo = edge_base_from_anchor(c), dc = edge_dir(c);
  const int bx = ax + bo.x, by = ay + bo.y, bz = az + bo.z;
  double PB[3], PT[3];
  world_pos(macros[li], n, bx, by, bz, PB);
  world_pos(macros[li], n, bx + dc.x, by + dc.y, bz + dc.z, PT);
  const double P[3] = {0.5 * (PB[0] + PT[0]), 0.5 * (PB[1] + PT[1]), 0.5 * (PB[2] + PT[2])};
  out[tid] = coeff_value(spec.which, spec.value, P);
}

__global__ void import_ref_kernel(double* lat, const i64* map, i64 total, const double* ref) {
  const i64 tid = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (tid >= total) return;
  const i64 e = map[tid];
  if (e < 0) {
    lat[tid] = 0.0;
    return;
  }
  const double v = ref[e >> 2];
  lat[tid] = (e & 2) ? -v : v;
}

__global__ void export_ref_kernel(const double* lat, const i64* map, i64 total, double* ref) {
  const i64 tid = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (tid >= total) return;
  const i64 e = map[tid];
  if (e < 0 || !(e & 1)) return;
  const double v = lat[tid];
  ref[e >> 2] = (e & 2) ? -v : v;
}

// Owned slice [lo, hi) of the reference numbering (one rank's share): import
// sets every local copy of an owned carrier (others are ghosts, filled by the
// owner broadcast below); export writes the owner copies.
__global__ void import_ref_range_kernel(double* lat, const i64* map, i64 total, const double* ref, i64 lo, i64 hi) {
  const i64 tid = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (tid >= total) return;
  const i64 e = map[tid];
  if (e < 0) {
    lat[tid] = 0.0;
    return;
  }
  const i64 id = e >> 2;
  if (id < lo || id >= hi) return;
  const double v = ref[id - lo];
  lat[tid] = (e & 2) ? -v : v;
}

__global__ void export_ref_range_kernel(const double* lat, const i64* map, i64 total, double* ref, i64 lo, i64 hi) {
  const i64 tid = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (tid >= total) return;
  const i64 e = map[tid];
  if (e < 0 || !(e & 1)) return;
  const i64 id = e >> 2;
  if (id < lo || id >= hi) return;
  const double v = lat[tid];
  ref[id - lo] = (e & 2) ? -v : v;
}

// Ghost update of rank-local interface groups: every copy takes the owner
// copy's value (the first copy: copies are sorted by macro id, the owner is
// the lowest), with its orientation sign.
__global__ void interface_owner_kernel(double* y, const i64* offsets, const i64* copies, i64 ngroups) {
  const i64 g = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (g >= ngroups) return;
  const i64 b = offsets[g], e = offsets[g + 1];
  const i64 c0 = copies[b];
  const double v0 = y[c0 >> 1];
  const double s = (c0 & 1) ? -v0 : v0;
  for (i64 k = b + 1; k < e; ++k) {
    const i64 c = copies[k];
    y[c >> 1] = (c & 1) ? -s : s;
  }
}

// K4: one thread per shared carrier; copies are summed in macro-id order so
// every copy receives a bitwise-identical total.
// SIGNED: ND1 copies carry their orientation sign relative to the owner;
// unsigned sums (operator diagonals: sign^2 = 1) ignore it
template <bool SIGNED>
__global__ void interface_sum_kernel(double* y, const i64* offsets, const i64* copies, i64 ngroups) {
  const i64 g = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (g >= ngroups) return;
  const i64 b = offsets[g], e = offsets[g + 1];
  double s = 0.0;
  for (i64 k = b; k < e; ++k) {
    const i64 c = copies[k];
    const double v = y[c >> 1];
    s += (SIGNED && (c & 1)) ? -v : v;
  }
  for (i64 k = b; k < e; ++k) {
    const i64 c = copies[k];
    y[c >> 1] = (SIGNED && (c & 1)) ? -s : s;
  }
}

template <bool SIGNED>
__global__ void interface_sum_packed_kernel(double* y, const uint2* __restrict__ pairs, i64 npairs,
                                            const i64* __restrict__ offsets, const i64* __restrict__ copies,
                                            i64 nrest) {
  const i64 g = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  // no early launch_dependents here: the next apply's K1 CTAs (56 KB of shared
  // memory each) would take the SMs from this latency-bound kernel (measured:
  // config 4 90.1 -> 92.3 us per apply with it)
  if (g < npairs) {
    // the CSR kernel's order: s = 0; s += copy 0; s += copy 1
    const uint2 p = pairs[g];  // static index data: loaded while the element kernel drains
    pdl_wait();
    const double va = y[p.x >> 1], vb = y[p.y >> 1];
    double s = 0.0;
    s += (SIGNED && (p.x & 1u)) ? -va : va;
    s += (SIGNED && (p.y & 1u)) ? -vb : vb;
    y[p.x >> 1] = (SIGNED && (p.x & 1u)) ? -s : s;
    y[p.y >> 1] = (SIGNED && (p.y & 1u)) ? -s : s;
    return;
  }
  const i64 r = g - npairs;
  if (r >= nrest) return;
  const i64 b = offsets[r], e = offsets[r + 1];
  pdl_wait();
  double s = 0.0;
  for (i64 k = b; k < e; ++k) {
    const i64 c = copies[k];
    const double v = y[c >> 1];
    s += (SIGNED && (c & 1)) ? -v : v;
  }
  for (i64 k = b; k < e; ++k) {
    const i64 c = copies[k];
    y[c >> 1] = (SIGNED && (c & 1)) ? -s : s;
  }
}

__global__ void axpy_kernel(double* y, const double* x, double a, i64 count) {
  const i64 tid = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (tid < count) y[tid] += a * x[tid];
}

__global__ void fp64_peak_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-7, a1 = a0 + 1.0, a2 = a0 + 2.0, a3 = a0 + 3.0;
  double a4 = a0 + 4.0, a5 = a0 + 5.0, a6 = a0 + 6.0, a7 = a0 + 7.0;
  const double b = 0.999999, c = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.6789) out[0] = s;  // keep the chain alive
}

} // namespace

// space: 0 P1, 1 P2 (vertex block + unsigned edge blocks), 2 ND1
void launch_fill_seeded(double* out, const MacroDesc* d_macros, int nmacros, i64 macro_stride, int n, int space,
                        i64 class_stride, std::uint64_t seed, bool dirichlet, cudaStream_t s) {
  const i64 vstride = space == 2 ? 0 : (space == 1 ? ((tet_count(n) + 31) / 32 * 32) : macro_stride);
  if (vstride > 0) {
    fill_seeded_p1_kernel<<<grid_for(vstride * nmacros), kThreads, 0, s>>>(out, d_macros, nmacros, macro_stride,
                                                                            vstride, n, seed, dirichlet);
    check_launch("fill_seeded");
  }
  if (space != 0) {
    const i64 region = 7 * class_stride;
    fill_seeded_nd1_kernel<<<grid_for(region * nmacros), kThreads, 0, s>>>(
        out + vstride, d_macros, nmacros, macro_stride, region, class_stride, n, seed, dirichlet, space == 1);
    check_launch("fill_seeded");
  }
}

// P1 (class_stride 0) or P2 coefficient functions
void launch_fill_coeff(double* out, const MacroDesc* d_macros, int nmacros, i64 macro_stride, int n,
                       CoeffSpec spec, cudaStream_t s, i64 class_stride) {
  const i64 vstride = class_stride > 0 ? ((tet_count(n) + 31) / 32 * 32) : macro_stride;
  fill_coeff_kernel<<<grid_for(vstride * nmacros), kThreads, 0, s>>>(out, d_macros, nmacros, macro_stride, vstride,
                                                                      n, spec);
  check_launch("fill_coeff");
  if (class_stride > 0) {
    const i64 region = 7 * class_stride;
    fill_coeff_edges_kernel<<<grid_for(region * nmacros), kThreads, 0, s>>>(out + vstride, d_macros, nmacros,
                                                                            macro_stride, region, class_stride, n,
                                                                            spec);
    check_launch("fill_coeff");
  }
}

void launch_import_ref(double* lat, const i64* map, i64 total, const double* ref, cudaStream_t s) {
  import_ref_kernel<<<grid_for(total), kThreads, 0, s>>>(lat, map, total, ref);
  check_launch("import_ref");
}

void launch_export_ref(const double* lat, const i64* map, i64 total, double* ref, cudaStream_t s) {
  export_ref_kernel<<<grid_for(total), kThreads, 0, s>>>(lat, map, total, ref);
  check_launch("export_ref");
}

void launch_import_ref_range(double* lat, const i64* map, i64 total, const double* ref, i64 lo, i64 hi,
                             cudaStream_t s) {
  import_ref_range_kernel<<<grid_for(total), kThreads, 0, s>>>(lat, map, total, ref, lo, hi);
  check_launch("import_ref_range");
}

void launch_export_ref_range(const double* lat, const i64* map, i64 total, double* ref, i64 lo, i64 hi,
                             cudaStream_t s) {
  export_ref_range_kernel<<<grid_for(total), kThreads, 0, s>>>(lat, map, total, ref, lo, hi);
  check_launch("export_ref_range");
}

void launch_interface_owner(double* y, const i64* offsets, const i64* copies, i64 ngroups, cudaStream_t s) {
  if (ngroups <= 0) return;
  interface_owner_kernel<<<grid_for(ngroups), kThreads, 0, s>>>(y, offsets, copies, ngroups);
  check_launch("interface_owner");
}

void launch_interface_sum(double* y, const i64* offsets, const i64* copies, i64 ngroups, cudaStream_t s,
                          bool signed_values) {
  if (ngroups <= 0) return;
  if (signed_values)
    interface_sum_kernel<true><<<grid_for(ngroups), kThreads, 0, s>>>(y, offsets, copies, ngroups);
  else
    interface_sum_kernel<false><<<grid_for(ngroups), kThreads, 0, s>>>(y, offsets, copies, ngroups);
  check_launch("interface_sum");
}

void launch_interface_sum_packed(double* y, const unsigned* pairs, i64 npairs, const i64* offsets, const i64* copies,
                                 i64 nrest, cudaStream_t s, bool signed_values) {
  const i64 total = npairs + nrest;
  if (total <= 0) return;
  const uint2* p = reinterpret_cast<const uint2*>(pairs);
  if (signed_values)
    TETMF_CUDA(launch_pdl(kPdlK4, interface_sum_packed_kernel<true>, grid_for(total), kThreads, 0, s, y, p, npairs, offsets,
                          copies, nrest));
  else
    TETMF_CUDA(launch_pdl(kPdlK4, interface_sum_packed_kernel<false>, grid_for(total), kThreads, 0, s, y, p, npairs, offsets,
                          copies, nrest));
  check_launch("interface_sum_packed");
}

void launch_axpy(double* y, const double* x, double a, i64 count, cudaStream_t s) {
  axpy_kernel<<<grid_for(count), kThreads, 0, s>>>(y, x, a, count);
  check_launch("axpy");
}

void launch_fp64_peak(double* out, int blocks, int threads, int iters, cudaStream_t s) {
  fp64_peak_kernel<<<blocks, threads, 0, s>>>(out, iters);
  check_launch("fp64_peak");
}

} // namespace tetmf

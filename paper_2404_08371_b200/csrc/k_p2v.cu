// k_p2v.cu -- P2V apply: -div(k grad u), u and k in P2
// (forms.cpp:12), exact integration.
//
// v1 (variant 1, cf. k_apply_v1.cu): one thread per (macro, cube anchor); the
// up-to-six micro elements of the cube gather their ten P2 values (vertices
// at the four corners, edge midpoints at the six local edges; P2 edge DoFs
// are unsigned) and the ten coefficient values, form A_e = sum_m k_m T_m from
// the exact per-orientation tables (tables.cpp p2v_table; 55 packed entries x
// 10 coefficient terms) and scatter A_e x_e with FP64 atomics into a zeroed y.
// The interface step then sums the macro copies as for P1 / ND1.
#include "device.hpp"
#include "p2v_common.cuh"
#include "n1_common.cuh"
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

// ---------------------------------------------------------------- v2
// Default. Factored element (tables.hpp P2VTable::G, p2v_moments): with the
// chain rule in barycentrics, du/dlambda_q = sum_r U_qr lambda_r (U_qq = 3 x_q,
// U_qr = 4 x_qr - x_q), K_rs = sum_m k_m C[m][rs] (= int k lambda_r lambda_s /
// vol), W_qr = sum_p G_pq U_pr, Z_qs = sum_r W_qr K_rs, and
//   y_vertex i = 3 Z_ii - sum_{s != i} Z_is,   y_edge (a,b) = 4 (Z_ab + Z_ba)
// (row by row: W_q and Z_q live only while row q is accumulated)
// -- 282 FP64 instructions (480 flop) per element instead of 650 FMA, 10
// table values per orientation. One thread per cube: the six elements
// accumulate into the cube's 27 P2 DoFs (8 vertices, 19 edges) in registers,
// then one atomic per nonzero DoF (27 per cube instead of 60). Indices are
// 32-bit offsets from four row bases per lattice, computed once per cube. The
// six orientations run as a runtime loop over constant-bank offset tables
// with the 27 accumulators in shared memory: unrolled, ptxas overlaps the
// elements and spills at any occupancy (one element alone needs ~54
// registers plus the accumulators), and the code outgrows the I-cache.

// [rule][m][sym4(r, s)]: 0 exact (p2v_moments), 1..3 quadrature(degree)
// (p2v_rule_moments; degrees >= 4 integrate P2V exactly)
__constant__ double kC[4][10][10];

// cube edge id (n1_common.cuh numbering) -> (owner offset, class)
struct CubeEdgeRef {
  int ox, oy, oz, c;
};
__host__ __device__ constexpr CubeEdgeRef cube_edge_ref(int id) {
  return id < 7    ? CubeEdgeRef{0, 0, 0, id}
         : id == 7  ? CubeEdgeRef{1, 0, 0, 1}
         : id == 8  ? CubeEdgeRef{1, 0, 0, 2}
         : id == 9  ? CubeEdgeRef{1, 0, 0, 5}
         : id == 10 ? CubeEdgeRef{0, 1, 0, 0}
         : id == 11 ? CubeEdgeRef{0, 1, 0, 2}
         : id == 12 ? CubeEdgeRef{0, 1, 0, 4}
         : id == 13 ? CubeEdgeRef{1, 1, 0, 2}
         : id == 14 ? CubeEdgeRef{0, 0, 1, 0}
         : id == 15 ? CubeEdgeRef{0, 0, 1, 1}
         : id == 16 ? CubeEdgeRef{0, 0, 1, 3}
         : id == 17 ? CubeEdgeRef{1, 0, 1, 1}
                    : CubeEdgeRef{0, 1, 1, 0};
}
__host__ __device__ constexpr int cube_edge_of(int o, int le) {
  return n1::cube_edge_id(local_edge_ref(o, le).ax, local_edge_ref(o, le).ay, local_edge_ref(o, le).az,
                          local_edge_ref(o, le).cls);
}
// local edge joining local vertices q != r
__host__ __device__ constexpr int local_edge_of(int q, int r) {
  int e = 0;
  for (int k = 0; k < 6; ++k)
    if ((local_edge_vertex(k, 0) == q && local_edge_vertex(k, 1) == r) ||
        (local_edge_vertex(k, 0) == r && local_edge_vertex(k, 1) == q))
      e = k;
  return e;
}

// Row bases of the cube at anchor (ax, ay, az), 32-bit (a macro's storage
// fits in int): Rv[dz][dy] = index of lattice point (0, ay+dy, az+dz) in the
// vertex block, Re[dz][dy] the same in the (n-1) edge-anchor lattice
struct CubeRows {
  int Rv[2][2], Re[2][2];
};
__device__ __forceinline__ CubeRows cube_rows(int n, int ay, int az) {
  CubeRows c;
#pragma unroll
  for (int dz = 0; dz < 2; ++dz) {
    const int Pv = static_cast<int>(plane_offset(n, az + dz));
    const int Pe = static_cast<int>(plane_offset(n - 1, az + dz));
#pragma unroll
    for (int dy = 0; dy < 2; ++dy) {
      const int y = ay + dy, mv = n - az - dz, me = n - 1 - az - dz;
      c.Rv[dz][dy] = Pv + y * (mv + 1) - y * (y - 1) / 2;
      c.Re[dz][dy] = Pe + y * (me + 1) - y * (y - 1) / 2;
    }
  }
  return c;
}

// per-orientation geometry for the runtime orientation loop (constant bank;
// the orientation is warp-uniform)
struct OrientConsts {
  int vx[6][4], vy[6][4], vz[6][4];         // local vertex -> cube offset
  int ecls[6][6], ex[6][6], ey[6][6], ez[6][6];  // local edge -> (class, anchor offset)
  int vslot[6][4], eslot[6][6];             // local DoF -> cube accumulator slot
};
constexpr OrientConsts make_orient_consts() {
  OrientConsts c{};
  for (int o = 0; o < 6; ++o) {
    for (int i = 0; i < 4; ++i) {
      c.vx[o][i] = orient_offset(o, i).x;
      c.vy[o][i] = orient_offset(o, i).y;
      c.vz[o][i] = orient_offset(o, i).z;
      c.vslot[o][i] = n1::cube_vertex(o, i);
    }
    for (int e = 0; e < 6; ++e) {
      c.ecls[o][e] = local_edge_ref(o, e).cls;
      c.ex[o][e] = local_edge_ref(o, e).ax;
      c.ey[o][e] = local_edge_ref(o, e).ay;
      c.ez[o][e] = local_edge_ref(o, e).az;
      c.eslot[o][e] = 8 + cube_edge_of(o, e);
    }
  }
  return c;
}
__constant__ OrientConsts kOc = make_orient_consts();

#ifndef TETMF_P2V_OUNROLL
#define TETMF_P2V_OUNROLL 1  // orientation loop unroll (full unroll overflows the instruction cache)
#endif
constexpr int kOUnroll = TETMF_P2V_OUNROLL;
#ifndef TETMF_P2V_MINB
#define TETMF_P2V_MINB 1
#endif
#ifndef TETMF_P2V_CLOSED
#define TETMF_P2V_CLOSED 1  // exact rule: the moment matrix K in closed form (p2v_exact_moments)
#endif
#ifndef TETMF_P2V_STAGE
#define TETMF_P2V_STAGE 0  // 1: the cube's 27 x and 27 k values staged in shared memory once per cube
#endif
constexpr bool kStage2 = TETMF_P2V_STAGE;
constexpr int kThreads2 = kStage2 ? 64 : kThreads;  // cubes per CTA (static shared memory <= 48 KB)

// cube slots (0..7 vertices, 8..26 edges) touched by the elements valid at
// anchor-sum class c (0: WU only, 1: + BU BD GU GD, 2: + WD), as bit masks
[[maybe_unused]] constexpr unsigned slot_mask(int cls) {  // TETMF_P2V_STAGE builds
  unsigned m = 0;
  for (int o = 0; o < 6; ++o) {
    const int need = o == WU ? 0 : o == WD ? 2 : 1;
    if (need > cls) continue;
    for (int i = 0; i < 4; ++i) m |= 1u << n1::cube_vertex(o, i);
    for (int e = 0; e < 6; ++e) m |= 1u << (8 + cube_edge_of(o, e));
  }
  return m;
}

template <int RULE>
__global__ void __launch_bounds__(kThreads2, TETMF_P2V_MINB)
p2v_cubes2_kernel(const double* __restrict__ x, const double* __restrict__ kc, double* __restrict__ y,
                  const MacroDesc* __restrict__ macros, int nmacros, i64 stride, i64 cstride, int n,
                  const P2VTable* __restrict__ tabs) {
  __shared__ double acc[27][kThreads2];  // the cube's accumulators, [slot][thread]
  const i64 anchors = tet_count(n - 1);
  const i64 tid = blockIdx.x * static_cast<i64>(kThreads2) + threadIdx.x;
  if (tid >= anchors * nmacros) return;
  const int li = static_cast<int>(tid / anchors);
  int ax, ay, az;
  decode_anchor(n - 1, tid - li * anchors, ax, ay, az);
  const int vstride = static_cast<int>((tet_count(n) + 31) / 32 * 32);
  const int cs = static_cast<int>(cstride);
  const double* __restrict__ xm = x + static_cast<i64>(li) * stride;
  const double* __restrict__ km = kc + static_cast<i64>(li) * stride;
  double* __restrict__ ym = y + static_cast<i64>(li) * stride;
  const P2VTable* __restrict__ T = tabs + macros[li].group;
  const int s = ax + ay + az;
  const CubeRows cr = cube_rows(n, ay, az);
  double* Y = &acc[0][threadIdx.x];
#pragma unroll
  for (int i = 0; i < 27; ++i) Y[i * kThreads2] = 0.0;
#if TETMF_P2V_STAGE
  // the cube's DoFs touched by a valid element, all loads issued at once
  __shared__ double xs[27][kThreads2], ks[27][kThreads2];
  {
    const unsigned need = s <= n - 3 ? slot_mask(2) : s <= n - 2 ? slot_mask(1) : slot_mask(0);
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const int gi = cr.Rv[v >> 2][(v >> 1) & 1] + ax + (v & 1);
      const bool on = (need >> v) & 1u;
      xs[v][threadIdx.x] = on ? __ldg(xm + gi) : 0.0;
      ks[v][threadIdx.x] = on ? __ldg(km + gi) : 0.0;
    }
#pragma unroll
    for (int e = 0; e < 19; ++e) {
      const CubeEdgeRef r = cube_edge_ref(e);
      const int gi = vstride + r.c * cs + cr.Re[r.oz][r.oy] + ax + r.ox;
      const bool on = (need >> (8 + e)) & 1u;
      xs[8 + e][threadIdx.x] = on ? __ldg(xm + gi) : 0.0;
      ks[8 + e][threadIdx.x] = on ? __ldg(km + gi) : 0.0;
    }
  }
#endif
  // orientations valid by anchor sum (orient_sum_limit): WU s <= n-1
  // (always), BU BD GU GD s <= n-2, WD s <= n-3
#pragma unroll kOUnroll
  for (int o = 0; o < 6; ++o) {
    if (s > (o == WU ? n - 1 : o == WD ? n - 3 : n - 2)) continue;
    double xv[10], kv[10], g[10];
#if TETMF_P2V_STAGE
#pragma unroll
    for (int i = 0; i < 10; ++i) {
      const int sl = i < 4 ? kOc.vslot[o][i] : kOc.eslot[o][i - 4];
      xv[i] = xs[sl][threadIdx.x];
      kv[i] = ks[sl][threadIdx.x];
      g[i] = __ldg(T->G[o] + i);
    }
#else
    int idx[10];
#pragma unroll
    for (int i = 0; i < 4; ++i) idx[i] = cr.Rv[kOc.vz[o][i]][kOc.vy[o][i]] + ax + kOc.vx[o][i];
#pragma unroll
    for (int e = 0; e < 6; ++e)
      idx[4 + e] = vstride + kOc.ecls[o][e] * cs + cr.Re[kOc.ez[o][e]][kOc.ey[o][e]] + ax + kOc.ex[o][e];
#pragma unroll
    for (int i = 0; i < 10; ++i) {
      xv[i] = __ldg(xm + idx[i]);
      kv[i] = __ldg(km + idx[i]);
      g[i] = __ldg(T->G[o] + i);
    }
#endif
    // K_rs = sum_m k_m C[m][rs]
    double K[10];
    if constexpr (RULE == 0 && TETMF_P2V_CLOSED) {
      p2v_exact_moments(kv, K);
    } else {
#pragma unroll
      for (int rs = 0; rs < 10; ++rs) {
        double a = kv[0] * kC[RULE][0][rs];
#pragma unroll
        for (int m = 1; m < 10; ++m) a = fma(kv[m], kC[RULE][m][rs], a);
        K[rs] = a;
      }
    }
    // U_qr: coefficients of du/dlambda_q
    double U[4][4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int r = 0; r < 4; ++r) U[q][r] = q == r ? 3.0 * xv[q] : fma(4.0, xv[4 + local_edge_of(q, r)], -xv[q]);
    // row q: W_q. = sum_p G_pq U_p., Z_q. = W_q. K, accumulated at once:
    //   y_vertex q += 3 Z_qq - sum_{s != q} Z_qs,  y_edge (q,s) += 4 Z_qs
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double W[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        double a = g[sym4(0, q)] * U[0][r];
#pragma unroll
        for (int p = 1; p < 4; ++p) a = fma(g[sym4(p, q)], U[p][r], a);
        W[r] = a;
      }
      double v = 0.0;
#pragma unroll
      for (int s2 = 0; s2 < 4; ++s2) {
        double z = W[0] * K[sym4(0, s2)];
#pragma unroll
        for (int r = 1; r < 4; ++r) z = fma(W[r], K[sym4(r, s2)], z);
        if (s2 == q) {
          v = fma(3.0, z, v);
        } else {
          v -= z;
          double& ye = Y[kOc.eslot[o][local_edge_of(q, s2)] * kThreads2];
          ye = fma(4.0, z, ye);
        }
      }
      Y[kOc.vslot[o][q] * kThreads2] += v;
    }
  }
  // scatter: DoFs no valid element touched hold exact zeros (skipped; their
  // indices may lie outside the lattice)
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    const double val = Y[v * kThreads2];
    if (val != 0.0) atomicAdd(ym + cr.Rv[v >> 2][(v >> 1) & 1] + ax + (v & 1), val);
  }
#pragma unroll
  for (int e = 0; e < 19; ++e) {
    const CubeEdgeRef r = cube_edge_ref(e);
    const double val = Y[(8 + e) * kThreads2];
    if (val != 0.0) atomicAdd(ym + vstride + r.c * cs + cr.Re[r.oz][r.oy] + ax + r.ox, val);
  }
}

// operator diagonal per stored macro copy, factored form (rule-aware like
// the apply): per element, with K from kC[RULE] and the orientation's G,
//   vertex i:   A_ii = G_ii sum_rs d_r d_s K_rs,  d = (3 at i, -1 elsewhere)
//   edge (a,b): A_ee = 16 (G_aa K_bb + G_bb K_aa + 2 G_ab K_ab)
template <int RULE>
__global__ void __launch_bounds__(kThreads)
p2v_diagonal_kernel(const double* __restrict__ kc, double* __restrict__ d, const MacroDesc* __restrict__ macros,
                    int nmacros, i64 stride, i64 cstride, int n, const P2VTable* __restrict__ tabs) {
  const i64 anchors = tet_count(n - 1);
  const i64 tid = blockIdx.x * static_cast<i64>(kThreads) + threadIdx.x;
  if (tid >= anchors * nmacros) return;
  const int li = static_cast<int>(tid / anchors);
  int ax, ay, az;
  decode_anchor(n - 1, tid - li * anchors, ax, ay, az);
  const int vstride = static_cast<int>((tet_count(n) + 31) / 32 * 32);
  const int cs = static_cast<int>(cstride);
  const double* __restrict__ km = kc + static_cast<i64>(li) * stride;
  double* __restrict__ dm = d + static_cast<i64>(li) * stride;
  const P2VTable* __restrict__ T = tabs + macros[li].group;
  const int s = ax + ay + az;
  const CubeRows cr = cube_rows(n, ay, az);
#pragma unroll 1
  for (int o = 0; o < 6; ++o) {
    if (s > (o == WU ? n - 1 : o == WD ? n - 3 : n - 2)) continue;
    int idx[10];
#pragma unroll
    for (int i = 0; i < 4; ++i) idx[i] = cr.Rv[kOc.vz[o][i]][kOc.vy[o][i]] + ax + kOc.vx[o][i];
#pragma unroll
    for (int e = 0; e < 6; ++e)
      idx[4 + e] = vstride + kOc.ecls[o][e] * cs + cr.Re[kOc.ez[o][e]][kOc.ey[o][e]] + ax + kOc.ex[o][e];
    double kv[10], g[10], K[10];
#pragma unroll
    for (int i = 0; i < 10; ++i) {
      kv[i] = __ldg(km + idx[i]);
      g[i] = __ldg(T->G[o] + i);
    }
#pragma unroll
    for (int rs = 0; rs < 10; ++rs) {
      double a = kv[0] * kC[RULE][0][rs];
#pragma unroll
      for (int m = 1; m < 10; ++m) a = fma(kv[m], kC[RULE][m][rs], a);
      K[rs] = a;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      double q = 0.0;
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int t = 0; t < 4; ++t) q = fma((r == i ? 3.0 : -1.0) * (t == i ? 3.0 : -1.0), K[sym4(r, t)], q);
      atomicAdd(dm + idx[i], g[sym4(i, i)] * q);
    }
#pragma unroll
    for (int e = 0; e < 6; ++e) {
      const int a = local_edge_vertex(e, 0), b = local_edge_vertex(e, 1);
      const double v = g[sym4(a, a)] * K[sym4(b, b)] + g[sym4(b, b)] * K[sym4(a, a)] +
                       2.0 * g[sym4(a, b)] * K[sym4(a, b)];
      atomicAdd(dm + idx[4 + e], 16.0 * v);
    }
  }
}

// exact and quadrature(1..3) moment tables into constant memory (once)
void load_p2v_moments() {
  static const bool ready = [] {
    double C[4][10][10];
    for (int r = 0; r < 4; ++r) p2v_rule_moments(r, C[r]);
    TETMF_CUDA(cudaMemcpyToSymbol(kC, C, sizeof(C)));
    return true;
  }();
  (void)ready;
}

} // namespace

void launch_p2v_diagonal(const double* k, double* d, const MacroDesc* d_macros, int nmacros, i64 macro_stride,
                         i64 class_stride, int n, const P2VTable* d_tables, int rule, cudaStream_t s) {
  load_p2v_moments();
  if (rule < 0 || rule > 3) fail_internal("p2v: rule index out of range");
  TETMF_CUDA(cudaMemsetAsync(d, 0, sizeof(double) * macro_stride * nmacros, s));
  const i64 total = tet_count(n - 1) * nmacros;
  if (total == 0) return;
  const unsigned grid = static_cast<unsigned>((total + kThreads - 1) / kThreads);
  switch (rule) {
    case 0:
      p2v_diagonal_kernel<0><<<grid, kThreads, 0, s>>>(k, d, d_macros, nmacros, macro_stride, class_stride, n, d_tables);
      break;
    case 1:
      p2v_diagonal_kernel<1><<<grid, kThreads, 0, s>>>(k, d, d_macros, nmacros, macro_stride, class_stride, n, d_tables);
      break;
    case 2:
      p2v_diagonal_kernel<2><<<grid, kThreads, 0, s>>>(k, d, d_macros, nmacros, macro_stride, class_stride, n, d_tables);
      break;
    default:
      p2v_diagonal_kernel<3><<<grid, kThreads, 0, s>>>(k, d, d_macros, nmacros, macro_stride, class_stride, n, d_tables);
  }
  check_launch("p2v_diagonal");
}

void launch_p2v_cubes2(const double* x, const double* k, double* y, const MacroDesc* d_macros, int nmacros,
                       i64 macro_stride, i64 class_stride, int n, const P2VTable* d_tables, int rule,
                       cudaStream_t s) {
  load_p2v_moments();
  if (rule < 0 || rule > 3) fail_internal("p2v: rule index out of range");
  TETMF_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * macro_stride * nmacros, s));
  const i64 total = tet_count(n - 1) * nmacros;
  if (total == 0) return;
  const unsigned grid = static_cast<unsigned>((total + kThreads2 - 1) / kThreads2);
  switch (rule) {
    case 0:
      p2v_cubes2_kernel<0><<<grid, kThreads2, 0, s>>>(x, k, y, d_macros, nmacros, macro_stride, class_stride, n, d_tables);
      break;
    case 1:
      p2v_cubes2_kernel<1><<<grid, kThreads2, 0, s>>>(x, k, y, d_macros, nmacros, macro_stride, class_stride, n, d_tables);
      break;
    case 2:
      p2v_cubes2_kernel<2><<<grid, kThreads2, 0, s>>>(x, k, y, d_macros, nmacros, macro_stride, class_stride, n, d_tables);
      break;
    default:
      p2v_cubes2_kernel<3><<<grid, kThreads2, 0, s>>>(x, k, y, d_macros, nmacros, macro_stride, class_stride, n, d_tables);
  }
  check_launch("p2v_cubes2");
}

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

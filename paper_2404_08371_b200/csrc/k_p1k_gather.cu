// k_p1k_gather.cu -- K2 (default): P1 -div(k grad) with k in P1, gather form.
//
//   y_p = sum over the micro elements e containing p of  kbar_e (A_e x_e)_p,
//   kbar_e = (k_a + k_b + k_c + k_d) / 4,  A_e = K_o (P1 stiffness of the
//   element's orientation, tables.cpp)
// i.e. the config-2 harness (forms.cpp:133-193 local_matrix
// with k in P1 and the degree-2 rule, exact for P1 k).
//
// Each lane owns one lattice point; a warp covers 32 consecutive x of one row
// (task = macro, z, y, x0). The 24 elements around p are the 6 orientations
// of the 8 cubes anchored at p - d, d in {0,1}^3, restricted to the (o, i)
// with vertex i of orientation o at cube corner d (6 elements share corners
// 0 and 7, two share each other corner). Their vertices are p + (offset - d),
// all within p's 15-point neighbourhood; x and k are read there (L1 / L2
// resident across the warp). Each lane sums its own contributions in a fixed
// order: deterministic, no atomics (the first version, k_apply_v1.cu,
// scatters with FP64 atomics).
#include "device.hpp"
#include "runtime_check.hpp"

namespace tetmf {

namespace {

constexpr int kWarps = 4;

struct RowTask {
  int macro, z, y, x0;
};

// The 24 (corner d, orientation o, local vertex i) with vertex i of o at
// cube corner d, and for each the neighbourhood slots q = (rx+1) + 3 (ry+1) +
// 9 (rz+1) of the element's four vertices relative to the point: a compile-
// time table, so every index below folds to a constant.
struct Incident {
  int d, o, i, q[4];
};
struct IncidentTable {
  Incident e[24];
  unsigned slots;  // bit q: slot q is a vertex of some incident element
};
constexpr IncidentTable make_incident() {
  IncidentTable t{};
  int k = 0;
  for (int d = 0; d < 8; ++d)
    for (int o = 0; o < 6; ++o)
      for (int i = 0; i < 4; ++i) {
        const Off3 c = orient_offset(o, i);
        if (c.x + 2 * c.y + 4 * c.z != d) continue;
        Incident& e = t.e[k++];
        e.d = d;
        e.o = o;
        e.i = i;
        for (int j = 0; j < 4; ++j) {
          const Off3 v = orient_offset(o, j);
          e.q[j] = (v.x - (d & 1) + 1) + 3 * (v.y - ((d >> 1) & 1) + 1) + 9 * (v.z - (d >> 2) + 1);
          t.slots |= 1u << e.q[j];
        }
      }
  return t;
}
constexpr IncidentTable kInc = make_incident();

// contribution of incident element K (template recursion: everything about the
// element is a compile-time constant)
template <int K, bool DIAG>
__device__ __forceinline__ void incident(const double (&xv)[27], const double (&kv)[27],
                                         const double* __restrict__ Kt, int px, int py, int pz, int n,
                                         double& acc) {
  constexpr int d = kInc.e[K].d, o = kInc.e[K].o, i = kInc.e[K].i;
  constexpr int dx = d & 1, dy = (d >> 1) & 1, dz = d >> 2;
  constexpr int q0 = kInc.e[K].q[0], q1 = kInc.e[K].q[1], q2 = kInc.e[K].q[2], q3 = kInc.e[K].q[3];
  // element (anchor p - d, orientation o) exists
  if (px >= dx && py >= dy && pz >= dz && px + py + pz - dx - dy - dz <= orient_sum_limit(o, n)) {
    const double ks = (kv[q0] + kv[q1]) + (kv[q2] + kv[q3]);
    if constexpr (DIAG) {  // operator diagonal: kbar_e (K_o)_ii
      acc = fma(0.25 * ks, __ldg(Kt + o * 10 + sym4(i, i)), acc);
    } else {
      double row = __ldg(Kt + o * 10 + sym4(i, 0)) * xv[q0];
      row = fma(__ldg(Kt + o * 10 + sym4(i, 1)), xv[q1], row);
      row = fma(__ldg(Kt + o * 10 + sym4(i, 2)), xv[q2], row);
      row = fma(__ldg(Kt + o * 10 + sym4(i, 3)), xv[q3], row);
      acc = fma(0.25 * ks, row, acc);
    }
  }
  if constexpr (K + 1 < 24) incident<K + 1, DIAG>(xv, kv, Kt, px, py, pz, n, acc);
}

template <int Q, bool DIAG>
__device__ __forceinline__ void neighbour(double (&xv)[27], double (&kv)[27], const double* __restrict__ xm,
                                          const double* __restrict__ km, const i64 (&rs)[3][3], int px, int py,
                                          int pz, int n) {
  constexpr int rx = Q % 3 - 1, ry = (Q / 3) % 3 - 1, rz = Q / 9 - 1;
  xv[Q] = kv[Q] = 0.0;
  if constexpr (((kInc.slots >> Q) & 1u) != 0) {
    if (px + rx >= 0 && py + ry >= 0 && pz + rz >= 0 && px + py + pz + rx + ry + rz <= n) {
      const i64 a = rs[rz + 1][ry + 1] + rx;
      if constexpr (!DIAG) xv[Q] = __ldg(xm + a);
      kv[Q] = __ldg(km + a);
    }
  }
  if constexpr (Q + 1 < 27) neighbour<Q + 1, DIAG>(xv, kv, xm, km, rs, px, py, pz, n);
}

template <bool DIAG>
__global__ void __launch_bounds__(32 * kWarps)
p1k_gather_kernel(const double* __restrict__ x, const double* __restrict__ kc, double* __restrict__ y,
                  const RowTask* __restrict__ tasks, int ntasks, i64 stride, int n,
                  const P1DeviceTable* __restrict__ tabs, const MacroDesc* __restrict__ macros) {
  const int warp = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (warp >= ntasks) return;
  const RowTask t = tasks[warp];
  const int pz = t.z, py = t.y, px = t.x0 + (threadIdx.x & 31);
  if (px > n - pz - py) return;  // past the row end
  const double* __restrict__ K = &tabs[macros[t.macro].group].K[0][0];
  const double* __restrict__ xm = x + static_cast<i64>(t.macro) * stride;
  const double* __restrict__ km = kc + static_cast<i64>(t.macro) * stride;
  // row starts of rows py-1 .. py+1 in planes pz-1 .. pz+1
  i64 rs[3][3];
#pragma unroll
  for (int dz = -1; dz <= 1; ++dz)
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy)
      rs[dz + 1][dy + 1] = plane_offset(n, pz + dz) + row_offset(n, pz + dz, py + dy) + px;
  // x and k on the 15-point neighbourhood (slot (rx+1) + 3 (ry+1) + 9 (rz+1)),
  // all loads issued up front; out-of-lattice neighbours read as 0 (they
  // only belong to elements that are skipped)
  double xv[27], kv[27];
  neighbour<0, DIAG>(xv, kv, xm, km, rs, px, py, pz, n);
  double acc = 0.0;
  incident<0, DIAG>(xv, kv, K, px, py, pz, n, acc);
  y[static_cast<i64>(t.macro) * stride + rs[1][1]] = acc;
}

// ------------------------------------------------------------------------
// K2 default: the same gather, walked along y with register windows.
//
// Edge form: A_e has zero row sums (sum_j grad lambda_j = 0), so
//   y_p = sum_{q in N(p)} W_q (x_q - x_p),  W_q = sum_{e contains p, q} kbar_e K_o[i][j]
// -- per incident element 3 DADD (kbar) + 3 DFMA into the edge weights, then
// 14 DADD + 14 DFMA: 172 FP64 instructions per point (the per-element row
// form above needs ~216 plus its per-point setup).
// A warp owns 32 consecutive x of plane z and walks kWalkRows rows upward;
// the 15-point neighbourhood (slots q = (dx+1) + 3 (dy+1) + 9 (dz+1)) lives in
// registers and shifts by one row per step: 7 new x and 7 new k values per
// point (rows y+1 of planes z-1 / z, row y of plane z+1, incl. the x+1 / x-1
// columns read directly -- L1 hits of the neighbouring lanes). The 36
// off-diagonal K_o[i][j] / 4 of the group sit in registers for the whole
// walk. Elements outside the macro get kbar = 0 (selects, no divergence);
// neighbours outside the lattice then carry W_q = 0 exactly and read finite
// values (guard regions / other rows). One store per point, deterministic.
#ifndef TETMF_P1K_SMEMK
#define TETMF_P1K_SMEMK 1  // 0: the 36 K entries in registers (230 registers, 8 warps/SM; measured slower)
#endif
#ifndef TETMF_P1K_PF2
#define TETMF_P1K_PF2 0  // 1: fresh window slots prefetched two steps ahead
#endif
#ifndef TETMF_P1K_MINB
#define TETMF_P1K_MINB 3  // CTAs per SM the register budget is sized for (168 registers)
#endif
#ifndef TETMF_P1K_ROWS
#define TETMF_P1K_ROWS 32
#endif
constexpr int kWalkRows = TETMF_P1K_ROWS;  // rows per walk task

// neighbourhood slots used by the incident elements (kInc.slots) by row
__host__ __device__ constexpr bool used(int q) { return (kInc.slots >> q) & 1u; }
__host__ __device__ constexpr int slot(int dx, int dy, int dz) { return (dx + 1) + 3 * (dy + 1) + 9 * (dz + 1); }

// off-diagonal entry index of (orientation o, local i, local j), i != j: 6 per orientation
__host__ __device__ constexpr int offdiag(int o, int i, int j) {
  return o * 6 + (sym4(i, j) - (i < j ? i + 1 : j + 1));  // drop the diagonal from the packed row
}

template <int KK, typename KT>
__device__ __forceinline__ void walk_incident(const double (&kv)[27], const KT& Kt, int px, int py, int pz,
                                              int s, int n, double (&W)[27]) {
  constexpr int d = kInc.e[KK].d, o = kInc.e[KK].o, i = kInc.e[KK].i;
  constexpr int dx = d & 1, dy = (d >> 1) & 1, dz = d >> 2;
  constexpr int q0 = kInc.e[KK].q[0], q1 = kInc.e[KK].q[1], q2 = kInc.e[KK].q[2], q3 = kInc.e[KK].q[3];
  const bool valid = (dx == 0 || px >= 1) && (dy == 0 || py >= 1) && (dz == 0 || pz >= 1) &&
                     s - (dx + dy + dz) <= orient_sum_limit(o, n);
  const double ks0 = (kv[q0] + kv[q1]) + (kv[q2] + kv[q3]);
  const double ks = valid ? ks0 : 0.0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (j == i) continue;
    constexpr int qarr[4] = {q0, q1, q2, q3};
    W[qarr[j]] = fma(ks, Kt[offdiag(o, i, j)], W[qarr[j]]);
  }
  if constexpr (KK + 1 < 24) walk_incident<KK + 1, KT>(kv, Kt, px, py, pz, s, n, W);
}

__global__ void __launch_bounds__(32 * kWarps, TETMF_P1K_MINB)
p1k_walk_kernel(const double* __restrict__ x, const double* __restrict__ kc, double* __restrict__ y,
                const RowTask* __restrict__ tasks, int ntasks, i64 stride, int n,
                const P1DeviceTable* __restrict__ tabs, const MacroDesc* __restrict__ macros) {
  const int warp = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (warp >= ntasks) return;
  const RowTask t = tasks[warp];
  const int pz = t.z, px = t.x0 + (threadIdx.x & 31);
  const int yend = min(t.y + kWalkRows, n - pz - px + 1);  // rows of this column in the chunk
#if TETMF_P1K_SMEMK
  // the group's 36 off-diagonal K_o[i][j] / 4 in this warp's shared slot (broadcast loads)
  __shared__ double skt[kWarps][36];
  double* Kt = skt[threadIdx.x >> 5];
  {
    const double* __restrict__ K = &tabs[macros[t.macro].group].K[0][0];
    const int lane = threadIdx.x & 31;
    for (int e = lane; e < 36; e += 32) {
      const int o = e / 6, r = e % 6;
      const int i = r < 3 ? 0 : r < 5 ? 1 : 2, j = r < 3 ? r + 1 : r < 5 ? r - 1 : 3;
      Kt[e] = 0.25 * __ldg(K + o * 10 + sym4(i, j));
    }
    __syncwarp();  // every lane of the warp took part (no lane has left yet)
  }
  if (t.y >= yend) return;  // this column has no row in the chunk
#else
  double Kt[36];
  {
    const double* __restrict__ K = &tabs[macros[t.macro].group].K[0][0];
#pragma unroll
    for (int o = 0; o < 6; ++o)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = i + 1; j < 4; ++j) Kt[offdiag(o, i, j)] = 0.25 * __ldg(K + o * 10 + sym4(i, j));
  }
  if (t.y >= yend) return;
#endif
  const double* __restrict__ xm = x + static_cast<i64>(t.macro) * stride;
  const double* __restrict__ km = kc + static_cast<i64>(t.macro) * stride;
  double* __restrict__ ym = y + static_cast<i64>(t.macro) * stride;
  // start of row r (x = 0) of plane zz; plane -1 maps to plane 0 (its
  // elements do not exist, its values only need to be finite)
  const int pb[3] = {static_cast<int>(plane_offset(n, pz > 0 ? pz - 1 : 0)), static_cast<int>(plane_offset(n, pz)),
                     static_cast<int>(plane_offset(n, pz + 1))};
  auto rowstart = [&](int zz, int r) -> int {
    const int dz = zz - pz, zc = zz < 0 ? 0 : zz;  // dz in {-1, 0, 1} (compile-time at every call)
    return pb[dz + 1] + r * (n - zc + 1) - (r * (r - 1) >> 1);
  };
  // slots refilled from memory when the window moves up one row (the rest
  // shift from the row above)
  auto fresh = [](int q) { return used(q) && !((q / 3) % 3 < 2 && used(q + 3)); };
  double xv[27], kv[27], nx[27], nk[27];
#if TETMF_P1K_PF2
  double mx[27], mk[27];  // second prefetch stage: fresh slots two steps ahead
#endif
#pragma unroll
  for (int q = 0; q < 27; ++q) {
    xv[q] = kv[q] = nx[q] = nk[q] = 0.0;
#if TETMF_P1K_PF2
    mx[q] = mk[q] = 0.0;
#endif
  }
  auto load = [&](double& xo, double& ko, int zz, int r, int dxo) {
    const int a = rowstart(zz, r) + px + dxo;
    xo = __ldg(xm + a);
    ko = __ldg(km + a);
  };
  // initial window for row t.y and the fresh slots of row t.y + 1 (loaded one
  // step ahead: their latency hides behind a whole step of FP64 work)
#pragma unroll
  for (int q = 0; q < 27; ++q)
    if (used(q)) load(xv[q], kv[q], pz + q / 9 - 1, t.y + (q / 3) % 3 - 1, q % 3 - 1);
  if (t.y + 1 < yend) {
#pragma unroll
    for (int q = 0; q < 27; ++q)
      if (fresh(q)) load(nx[q], nk[q], pz + q / 9 - 1, t.y + 1 + (q / 3) % 3 - 1, q % 3 - 1);
  }
#if TETMF_P1K_PF2
  if (t.y + 2 < yend) {
#pragma unroll
    for (int q = 0; q < 27; ++q)
      if (fresh(q)) load(mx[q], mk[q], pz + q / 9 - 1, t.y + 2 + (q / 3) % 3 - 1, q % 3 - 1);
  }
#endif
  for (int py = t.y; py < yend; ++py) {
    const int s = px + py + pz;
    double W[27];
#pragma unroll
    for (int q = 0; q < 27; ++q) W[q] = 0.0;
    walk_incident<0>(kv, Kt, px, py, pz, s, n, W);
    double acc = 0.0;
    const double xc = xv[slot(0, 0, 0)];
#pragma unroll
    for (int q = 0; q < 27; ++q)
      if (used(q) && q != slot(0, 0, 0)) acc = fma(W[q], xv[q] - xc, acc);
    ym[rowstart(pz, py) + px] = acc;
    // move the window up one row: dy = -1 <- 0, dy = 0 <- +1 where both are
    // used slots, the fresh slots from the prefetch; then prefetch ahead
#pragma unroll
    for (int q = 0; q < 27; ++q) {
      if (!used(q)) continue;
      if (fresh(q)) {
        xv[q] = nx[q];
        kv[q] = nk[q];
#if TETMF_P1K_PF2
        nx[q] = mx[q];
        nk[q] = mk[q];
#endif
      } else {
        xv[q] = xv[q + 3];
        kv[q] = kv[q + 3];
      }
    }
#if TETMF_P1K_PF2
    if (py + 3 < yend) {
#pragma unroll
      for (int q = 0; q < 27; ++q)
        if (fresh(q)) load(mx[q], mk[q], pz + q / 9 - 1, py + 3 + (q / 3) % 3 - 1, q % 3 - 1);
    }
#else
    if (py + 2 < yend) {
#pragma unroll
      for (int q = 0; q < 27; ++q)
        if (fresh(q)) load(nx[q], nk[q], pz + q / 9 - 1, py + 2 + (q / 3) % 3 - 1, q % 3 - 1);
    }
#endif
  }
}

} // namespace

// one task per (macro, plane z, row y, 32-wide x segment)
void build_p1k_tasks(int nmacros, int n, std::vector<int>& out) {
  out.clear();
  for (int li = 0; li < nmacros; ++li)
    for (int z = 0; z <= n; ++z)
      for (int yy = 0; yy <= n - z; ++yy)
        for (int x0 = 0; x0 <= n - z - yy; x0 += 32) {
          out.push_back(li);
          out.push_back(z);
          out.push_back(yy);
          out.push_back(x0);
        }
}

// one task per (macro, plane z, x segment of 32, chunk of kWalkRows rows)
void build_p1k_walk_tasks(int nmacros, int n, std::vector<int>& out) {
  out.clear();
  for (int li = 0; li < nmacros; ++li)
    for (int z = 0; z <= n; ++z)
      for (int x0 = 0; x0 <= n - z; x0 += 32)
        for (int y0 = 0; y0 <= n - z - x0; y0 += kWalkRows) {
          out.push_back(li);
          out.push_back(z);
          out.push_back(y0);
          out.push_back(x0);
        }
}

void launch_p1k_walk(const double* x, const double* k, double* y, const int* d_tasks, int ntasks, i64 macro_stride,
                     int n, const P1DeviceTable* d_tables, const MacroDesc* d_macros, cudaStream_t s) {
  if (ntasks == 0) return;
  const unsigned grid = static_cast<unsigned>((ntasks + kWarps - 1) / kWarps);
  p1k_walk_kernel<<<grid, 32 * kWarps, 0, s>>>(x, k, y, reinterpret_cast<const RowTask*>(d_tasks), ntasks,
                                               macro_stride, n, d_tables, d_macros);
  check_launch("p1k_walk");
}

void launch_p1k_gather(const double* x, const double* k, double* y, const int* d_tasks, int ntasks, i64 macro_stride,
                       int n, const P1DeviceTable* d_tables, const MacroDesc* d_macros, cudaStream_t s) {
  if (ntasks == 0) return;
  const unsigned grid = static_cast<unsigned>((ntasks + kWarps - 1) / kWarps);
  p1k_gather_kernel<false><<<grid, 32 * kWarps, 0, s>>>(x, k, y, reinterpret_cast<const RowTask*>(d_tasks), ntasks,
                                                        macro_stride, n, d_tables, d_macros);
  check_launch("p1k_gather");
}

// operator diagonal (per macro copy; interface copies are summed afterwards)
void launch_p1k_diagonal(const double* k, double* d, const int* d_tasks, int ntasks, i64 macro_stride, int n,
                         const P1DeviceTable* d_tables, const MacroDesc* d_macros, cudaStream_t s) {
  if (ntasks == 0) return;
  const unsigned grid = static_cast<unsigned>((ntasks + kWarps - 1) / kWarps);
  p1k_gather_kernel<true><<<grid, 32 * kWarps, 0, s>>>(k, k, d, reinterpret_cast<const RowTask*>(d_tasks), ntasks,
                                                       macro_stride, n, d_tables, d_macros);
  check_launch("p1k_diagonal");
}

} // namespace tetmf

// k_p1_stencil_tile.cu -- K1 (default): P1 -Laplace 15-point stencil,
// one warp per 32 x kR register tile.
//
// Task = (macro, plane z, 32-column segment x0, row block [y0, y0+kR)); lane
// = column x. The warp issues ALL window loads of its tile up front -- column
// x of plane z rows y0-1..y0+kR, of plane z-1 rows y0..y0+kR and of plane z+1
// rows y0-1..y0+kR-1, plus one "edge" load per row for the columns x0-1 and
// x0+32 (lanes 0 and 31) -- so a warp keeps ~3kR+4 independent 8-byte loads in
// flight (memory-level parallelism instead of a sequential row walk). The x-1
// and x+1 neighbours come from warp shuffles. Per point: ~(3kR+4)/kR coalesced
// loads, 15 DFMA, 1 store; HBM traffic stays the compulsory 16 B per point
// because the three planes a tile touches are shared through L1/L2 with the
// neighbouring tiles that run alongside it.
//
// No bounds predicates: level buffers carry zeroed guard regions and every
// out-of-lattice value meets a zero stencil weight. Tiles without a point on
// a macro face use the interior stencil held in registers; the others use
// the per-type variant (tables.cpp) per lane.
#include "device.hpp"
#include "runtime_check.hpp"

namespace tetmf {

namespace {

constexpr int kWarps = 4;
constexpr int kR = 4;  // rows per tile

struct TileTask {
  int macro, z, x0, y0;
};

__device__ __forceinline__ double shl(double v) { return __shfl_up_sync(0xffffffffu, v, 1); }   // value of x-1
__device__ __forceinline__ double shr(double v) { return __shfl_down_sync(0xffffffffu, v, 1); } // value of x+1

__global__ void __launch_bounds__(32 * kWarps)
p1_stencil_tile_kernel(const double* __restrict__ xin, double* __restrict__ yout, const TileTask* __restrict__ tasks,
                       int ntasks, i64 stride, int n, const P1DeviceTable* __restrict__ tabs,
                       const MacroDesc* __restrict__ macros) {
  const int warp = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (warp >= ntasks) return;
  const int lane = threadIdx.x & 31;
  const TileTask t = tasks[warp];
  const int z = t.z, x0 = t.x0, y0 = t.y0;
  const int px = x0 + lane;
  const double* __restrict__ X = xin + static_cast<i64>(t.macro) * stride;
  double* __restrict__ Y = yout + static_cast<i64>(t.macro) * stride;
  const double* __restrict__ tab = &tabs[macros[t.macro].group].stencil[0][0];
  // lanes 0 / 31 fetch the columns just outside the segment
  const int edge = lane == 0 ? x0 - 1 : x0 + 32;
  const bool edge_lane = lane == 0 || lane == 31;

  // row starts: plane z rows y0-1 .. y0+kR, plane z-1 rows y0 .. y0+kR,
  // plane z+1 rows y0-1 .. y0+kR-1 (a missing plane aliases plane z)
  const int rz0 = static_cast<int>(plane_offset(n, z) + row_offset(n, z, y0));
  const int rl0 = z > 0 ? static_cast<int>(plane_offset(n, z - 1) + row_offset(n, z - 1, y0)) : rz0;
  const int ru0 = z < n ? static_cast<int>(plane_offset(n, z + 1) + row_offset(n, z + 1, y0)) : rz0;
  const int lenz = n - z - y0 + 1;  // length of row y0 in plane z
  const int dl = z > 0 ? 1 : 0, du = z < n ? -1 : 0;

  double Z[kR + 2], Ze[kR + 2];  // plane z rows y0-1+r (centre, edge)
  double L[kR + 1], Le[kR + 1];  // plane z-1 rows y0+r
  double U[kR + 1], Ue[kR + 1];  // plane z+1 rows y0-1+r
  {
    int rz = rz0 - (lenz + 1);              // row y0-1 of plane z
    int ru = ru0 - (lenz + du + 1);         // row y0-1 of plane z+1
    int rl = rl0;
    int len = lenz + 1;                     // length of row y0-1 in plane z
#pragma unroll
    for (int r = 0; r < kR + 2; ++r) {
      Z[r] = __ldg(X + rz + px);
      Ze[r] = edge_lane ? __ldg(X + rz + edge) : 0.0;
      rz += len;
      --len;
    }
    len = lenz + dl;                        // length of row y0 in plane z-1
#pragma unroll
    for (int r = 0; r < kR + 1; ++r) {
      L[r] = __ldg(X + rl + px);
      Le[r] = edge_lane ? __ldg(X + rl + edge) : 0.0;
      rl += len;
      --len;
    }
    len = lenz + 1 + du;                    // length of row y0-1 in plane z+1
#pragma unroll
    for (int r = 0; r < kR + 1; ++r) {
      U[r] = __ldg(X + ru + px);
      Ue[r] = edge_lane ? __ldg(X + ru + edge) : 0.0;
      ru += len;
      --len;
    }
  }
  // x-1 / x+1 neighbours
  double Zl[kR + 2], Zr[kR + 2], Lr[kR + 1], Ul[kR + 1];
#pragma unroll
  for (int r = 0; r < kR + 2; ++r) {
    const double a = shl(Z[r]), b = shr(Z[r]);
    Zl[r] = lane == 0 ? Ze[r] : a;
    Zr[r] = lane == 31 ? Ze[r] : b;
  }
#pragma unroll
  for (int r = 0; r < kR + 1; ++r) {
    const double a = shr(L[r]);
    Lr[r] = lane == 31 ? Le[r] : a;
    const double b = shl(U[r]);
    Ul[r] = lane == 0 ? Ue[r] : b;
  }

  // warp-uniform: no point of the tile on a macro face
  const bool interior = z > 0 && y0 > 0 && x0 > 0 && x0 + 31 + y0 + kR - 1 + z < n;
  double w[15];
#pragma unroll
  for (int k = 0; k < 15; ++k) w[k] = __ldg(tab + k);
  int row = rz0;
  int len = lenz;
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    const int yy = y0 + r;
    // stencil neighbours of (x, yy, z): index r+1 is row yy in Z, r in L,
    // r+1 in U (see header)
    const double c00 = Z[r + 1], c01 = Zr[r + 1], c0m = Zl[r + 1];
    const double cm0 = Z[r], cm1 = Zr[r], cp0 = Z[r + 2], cpm = Zl[r + 2];
    const double l00 = L[r], l01 = Lr[r], lp0 = L[r + 1], lp1 = Lr[r + 1];
    const double u00 = U[r + 1], u0m = Ul[r + 1], um0 = U[r], umm = Ul[r];
    double acc;
    if (interior) {
      double a0 = w[0] * c00, a1 = w[1] * c01, a2 = w[2] * c0m, a3 = w[3] * cp0;
      a0 = fma(w[4], cm0, a0);
      a1 = fma(w[5], u00, a1);
      a2 = fma(w[6], l00, a2);
      a3 = fma(w[7], cm1, a3);
      a0 = fma(w[8], cpm, a0);
      a1 = fma(w[9], l01, a1);
      a2 = fma(w[10], u0m, a2);
      a3 = fma(w[11], lp0, a3);
      a0 = fma(w[12], um0, a0);
      a1 = fma(w[13], lp1, a1);
      a2 = fma(w[14], umm, a2);
      acc = (a0 + a1) + (a2 + a3);
    } else {
      const int s = px + yy + z;
      const int type = (px == 0 ? 1 : 0) | (yy == 0 ? 2 : 0) | (z == 0 ? 4 : 0) | (s == n ? 8 : 0);
      const double* __restrict__ wt = tab + 16 * type;
      double a0 = __ldg(wt + 0) * c00, a1 = __ldg(wt + 1) * c01, a2 = __ldg(wt + 2) * c0m,
             a3 = __ldg(wt + 3) * cp0;
      a0 = fma(__ldg(wt + 4), cm0, a0);
      a1 = fma(__ldg(wt + 5), u00, a1);
      a2 = fma(__ldg(wt + 6), l00, a2);
      a3 = fma(__ldg(wt + 7), cm1, a3);
      a0 = fma(__ldg(wt + 8), cpm, a0);
      a1 = fma(__ldg(wt + 9), l01, a1);
      a2 = fma(__ldg(wt + 10), u0m, a2);
      a3 = fma(__ldg(wt + 11), lp0, a3);
      a0 = fma(__ldg(wt + 12), um0, a0);
      a1 = fma(__ldg(wt + 13), lp1, a1);
      a2 = fma(__ldg(wt + 14), umm, a2);
      acc = (a0 + a1) + (a2 + a3);
    }
    if (yy <= n - z && px <= n - z - yy) Y[row + px] = acc;
    row += len;
    --len;
  }
}

} // namespace

void build_stencil_tile_tasks(int nmacros, int n, std::vector<int>& out) {
  out.clear();
  for (int li = 0; li < nmacros; ++li)
    for (int z = 0; z <= n; ++z)
      for (int y0 = 0; y0 <= n - z; y0 += kR)
        for (int x0 = 0; x0 <= n - z - y0; x0 += 32) {
          out.push_back(li);
          out.push_back(z);
          out.push_back(x0);
          out.push_back(y0);
        }
}

void launch_p1_stencil_tile(const double* x, double* y, const int* d_tasks, int ntasks, i64 macro_stride, int n,
                            const P1DeviceTable* d_tables, const MacroDesc* d_macros, cudaStream_t s) {
  if (ntasks == 0) return;
  const unsigned grid = static_cast<unsigned>((ntasks + kWarps - 1) / kWarps);
  p1_stencil_tile_kernel<<<grid, 32 * kWarps, 0, s>>>(x, y, reinterpret_cast<const TileTask*>(d_tasks), ntasks,
                                                      macro_stride, n, d_tables, d_macros);
  check_launch("p1_stencil_tile");
}

} // namespace tetmf

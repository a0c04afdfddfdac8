// k_p1_stencil.cu -- K1: P1 -Laplace apply via the assembled 15-point stencil,
// register-window row walk.
//
// Work decomposition: one warp per task (macro, row chunk [y0, y0+kChunk),
// 32-wide x segment x0, plane z); lane = x. The warp walks the rows of its
// chunk. All neighbours of the 15-point stencil lie in planes z-1, z, z+1 and
// rows y-1..y+1, so a rolling register window keeps every value loaded once
// per warp: per point 7 coalesced 8-byte loads (plane z: row y at x+1, row
// y+1 at x-1, x; plane z-1: row y+1 at x, x+1; plane z+1: row y at x-1, x),
// 15 DFMA, 1 store. The chunk loop is fully unrolled (static register
// renaming, no rotation copies) and branch-free.
//
// Task order puts z innermost: the four warps of a CTA compute the same
// (x0, y0) tile of four consecutive planes, so the planes they share (each
// plane is read by the tasks of planes z-1, z and z+1) are served from L1
// instead of three separate L2 reads.
//
// No bounds predicates on the window loads: the level buffers carry zeroed
// guard regions (runtime.cpp storage_guard) and every out-of-lattice value a
// window picks up meets a zero stencil weight. Interior steps (no point of
// the warp on a macro face) use the macro's interior stencil in registers;
// steps touching a face / edge / vertex of the macro take the per-lane
// variant of the point's face set (tables.cpp: 16 types) from the L1-cached
// table.
#include "device.hpp"
#include "runtime_check.hpp"

namespace tetmf {

namespace {

constexpr int kWarps = 4;
constexpr int kChunk = 8;  // rows per task

struct StencilTask {
  int macro, z, x0, y0;
};

__global__ void __launch_bounds__(32 * kWarps)
p1_stencil_kernel(const double* __restrict__ xin, double* __restrict__ yout, const StencilTask* __restrict__ tasks,
                  int ntasks, i64 stride, int n, const P1DeviceTable* __restrict__ tabs,
                  const MacroDesc* __restrict__ macros) {
  const int warp = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (warp >= ntasks) return;
  const int lane = threadIdx.x & 31;
  const StencilTask t = tasks[warp];
  const int z = t.z, x0 = t.x0, y0 = t.y0;
  const int px = x0 + lane;
  // per-lane base pointers; all row offsets below are 32-bit, relative to them
  const double* __restrict__ X = xin + static_cast<i64>(t.macro) * stride + px;
  double* __restrict__ Y = yout + static_cast<i64>(t.macro) * stride + px;
  const double* __restrict__ tab = &tabs[macros[t.macro].group].stencil[0][0];
  double w[15];
#pragma unroll
  for (int k = 0; k < 15; ++k) w[k] = __ldg(tab + k);

  // row starts (offset of x = 0) of row y0 in planes z, z-1, z+1; a missing
  // plane aliases plane z (its weights are zero)
  int rz = static_cast<int>(plane_offset(n, z) + row_offset(n, z, y0));
  int rl = z > 0 ? static_cast<int>(plane_offset(n, z - 1) + row_offset(n, z - 1, y0)) : rz;
  int ru = z < n ? static_cast<int>(plane_offset(n, z + 1) + row_offset(n, z + 1, y0)) : rz;
  const int dl = z > 0 ? 1 : 0;   // row-length delta of plane z-1 vs z
  const int du = z < n ? -1 : 0;  // and of plane z+1
  int lenz = n - z - y0 + 1;      // length of row y in plane z

  // window at row y0: rows y0-1 may lie in the front guard (zero weights)
  const int rzm = rz - (lenz + 1);
  const int rum = ru - (lenz + du + 1);
  double Zm0 = __ldg(X + rzm), Zm1 = __ldg(X + rzm + 1);
  double Umm = __ldg(X + rum - 1), Um0 = __ldg(X + rum);
  double Z0m = __ldg(X + rz - 1), Z00 = __ldg(X + rz);
  double L00 = __ldg(X + rl), L01 = __ldg(X + rl + 1);
  const bool face_free = z > 0 && x0 > 0;  // rows y >= 1 of this warp avoid x=0, z=0

#pragma unroll
  for (int r = 0; r < kChunk; ++r) {
    const int yy = y0 + r;
    const int rz1 = rz + lenz, rl1 = rl + lenz + dl;
    const double Z01 = __ldg(X + rz + 1);
    const double Zpm = __ldg(X + rz1 - 1), Zp0 = __ldg(X + rz1);
    const double Lp0 = __ldg(X + rl1), Lp1 = __ldg(X + rl1 + 1);
    const double U0m = __ldg(X + ru - 1), U00 = __ldg(X + ru);
    double acc;
    // warp-uniform: no lane of this row on a macro face (x=0, y=0, z=0 or
    // x+y+z=n) -> every lane is an interior point
    if (face_free && yy > 0 && x0 + 31 + yy + z < n) {
      double a0 = w[0] * Z00, a1 = w[1] * Z01, a2 = w[2] * Z0m, a3 = w[3] * Zp0;
      a0 = fma(w[4], Zm0, a0);
      a1 = fma(w[5], U00, a1);
      a2 = fma(w[6], L00, a2);
      a3 = fma(w[7], Zm1, a3);
      a0 = fma(w[8], Zpm, a0);
      a1 = fma(w[9], L01, a1);
      a2 = fma(w[10], U0m, a2);
      a3 = fma(w[11], Lp0, a3);
      a0 = fma(w[12], Um0, a0);
      a1 = fma(w[13], Lp1, a1);
      a2 = fma(w[14], Umm, a2);
      acc = (a0 + a1) + (a2 + a3);
      if (yy <= n - z) Y[rz] = acc;
    } else {
      const int s = px + yy + z;
      const int type = (px == 0 ? 1 : 0) | (yy == 0 ? 2 : 0) | (z == 0 ? 4 : 0) | (s == n ? 8 : 0);
      const double* __restrict__ wt = tab + 16 * type;
      double a0 = __ldg(wt + 0) * Z00, a1 = __ldg(wt + 1) * Z01, a2 = __ldg(wt + 2) * Z0m,
             a3 = __ldg(wt + 3) * Zp0;
      a0 = fma(__ldg(wt + 4), Zm0, a0);
      a1 = fma(__ldg(wt + 5), U00, a1);
      a2 = fma(__ldg(wt + 6), L00, a2);
      a3 = fma(__ldg(wt + 7), Zm1, a3);
      a0 = fma(__ldg(wt + 8), Zpm, a0);
      a1 = fma(__ldg(wt + 9), L01, a1);
      a2 = fma(__ldg(wt + 10), U0m, a2);
      a3 = fma(__ldg(wt + 11), Lp0, a3);
      a0 = fma(__ldg(wt + 12), Um0, a0);
      a1 = fma(__ldg(wt + 13), Lp1, a1);
      a2 = fma(__ldg(wt + 14), Umm, a2);
      acc = (a0 + a1) + (a2 + a3);
      if (s <= n) Y[rz] = acc;
    }
    // slide the window to row y+1 (static renaming after unrolling)
    Zm0 = Z00;
    Zm1 = Z01;
    Z0m = Zpm;
    Z00 = Zp0;
    L00 = Lp0;
    L01 = Lp1;
    Umm = U0m;
    Um0 = U00;
    ru += lenz + du;
    rz = rz1;
    rl = rl1;
    --lenz;
  }
}

} // namespace

// Task list of one level: (macro, z, x0, y0) for every row chunk, 32-wide x
// segment and plane, z innermost (L1 sharing of adjacent planes in a CTA).
void build_stencil_tasks(int nmacros, int n, std::vector<int>& out) {
  out.clear();
  for (int li = 0; li < nmacros; ++li)
    for (int y0 = 0; y0 <= n; y0 += kChunk)
      for (int x0 = 0; x0 <= n - y0; x0 += 32)
        for (int z = 0; z <= n - y0 - x0; ++z) {
          out.push_back(li);
          out.push_back(z);
          out.push_back(x0);
          out.push_back(y0);
        }
}

void launch_p1_stencil_v2(const double* x, double* y, const int* d_tasks, int ntasks, i64 macro_stride, int n,
                          const P1DeviceTable* d_tables, const MacroDesc* d_macros, cudaStream_t s) {
  if (ntasks == 0) return;
  const unsigned grid = static_cast<unsigned>((ntasks + kWarps - 1) / kWarps);
  p1_stencil_kernel<<<grid, 32 * kWarps, 0, s>>>(x, y, reinterpret_cast<const StencilTask*>(d_tasks), ntasks,
                                                 macro_stride, n, d_tables, d_macros);
  check_launch("p1_stencil");
}

} // namespace tetmf

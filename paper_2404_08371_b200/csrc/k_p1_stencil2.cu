// k_p1_stencil2.cu -- K1 (default): P1 -Laplace 15-point stencil, row walk
// over TWO planes per warp.
//
// Task = (macro, row chunk [y0, y0+kChunk), 32-column segment x0, plane pair
// (z, z+1)); lane = column x. Per row step the warp loads the new row of the
// four planes involved -- z-1 at {x, x+1}, z and z+1 at {x-1, x, x+1}, z+2
// at {x-1, x} -- i.e. 10 coalesced loads for 2 output points (5 per point;
// one plane per warp needs 7), keeps the older rows in a register window and
// computes both planes' points with 15 DFMA each. The chunk loop is fully
// unrolled; two independent point streams per warp double the memory-level
// parallelism of the single-plane walk (variant 2, removed in round 2).
//
// No bounds predicates on the window loads (guard-padded level buffers; all
// out-of-lattice values meet zero weights). Rows whose points of both planes
// are interior use the interior stencil in registers; others use per-lane
// stencil variants (tables.cpp).
#include "device.hpp"
#include "runtime_check.hpp"

namespace tetmf {

namespace {

constexpr int kWarps = 4;
#ifndef TETMF_P1S_CHUNK
#define TETMF_P1S_CHUNK 8
#endif
#ifndef TETMF_P1S_PREFETCH
#define TETMF_P1S_PREFETCH 0  // rows ahead warmed into L1 (measured: 2-8 rows ahead are 10-15 % slower)
#endif
constexpr int kChunk = TETMF_P1S_CHUNK;  // rows per task
constexpr int kAhead = TETMF_P1S_PREFETCH;

#ifndef TETMF_P1S_PREFETCH_L2
#define TETMF_P1S_PREFETCH_L2 0  // 1: prefetch into L2 only (no L1 allocation)
#endif
__device__ __forceinline__ void prefetch_l1(const double* p) {
  if (TETMF_P1S_PREFETCH_L2)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
  else
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

struct Task2 {
  int macro, z, x0, y0;
};

__device__ __forceinline__ double stencil_sum(const double* __restrict__ w, double c00, double c01, double c0m,
                                              double cp0, double cm0, double u00, double l00, double cm1,
                                              double cpm, double l01, double u0m, double lp0, double um0,
                                              double lp1, double umm) {
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
  return (a0 + a1) + (a2 + a3);
}

__device__ __forceinline__ double stencil_var(const double* __restrict__ wt, double c00, double c01, double c0m,
                                              double cp0, double cm0, double u00, double l00, double cm1,
                                              double cpm, double l01, double u0m, double lp0, double um0,
                                              double lp1, double umm) {
  double a0 = __ldg(wt + 0) * c00, a1 = __ldg(wt + 1) * c01, a2 = __ldg(wt + 2) * c0m, a3 = __ldg(wt + 3) * cp0;
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
  return (a0 + a1) + (a2 + a3);
}

// no minimum-blocks bound by default: ptxas then settles at 128 registers
// (an explicit minimum of 1 lets it take 190 and costs 55 % in occupancy)
#ifdef TETMF_P1S_MIN_BLOCKS
__global__ void __launch_bounds__(32 * kWarps, TETMF_P1S_MIN_BLOCKS)
#else
__global__ void __launch_bounds__(32 * kWarps)
#endif
p1_stencil2_kernel(const double* __restrict__ xin, double* __restrict__ yout, const Task2* __restrict__ tasks,
                   int ntasks, i64 stride, int n, const P1DeviceTable* __restrict__ tabs,
                   const MacroDesc* __restrict__ macros) {
  const int warp = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (warp >= ntasks) return;
  const int lane = threadIdx.x & 31;
  const Task2 t = tasks[warp];
  const int z = t.z, x0 = t.x0, y0 = t.y0;
  const int px = x0 + lane;
  const double* __restrict__ X = xin + static_cast<i64>(t.macro) * stride + px;
  double* __restrict__ Y = yout + static_cast<i64>(t.macro) * stride + px;
  const double* __restrict__ tab = &tabs[macros[t.macro].group].stencil[0][0];
  double w[15];
#pragma unroll
  for (int k = 0; k < 15; ++k) w[k] = __ldg(tab + k);

  // row y0 starts of planes L = z-1, A = z, B = z+1, U = z+2 (missing planes
  // alias plane A / B; their weights are zero) and their row lengths
  const bool hasL = z > 0, hasB = z + 1 <= n, hasU = z + 2 <= n;
  int ra = static_cast<int>(plane_offset(n, z) + row_offset(n, z, y0));
  int rl = hasL ? static_cast<int>(plane_offset(n, z - 1) + row_offset(n, z - 1, y0)) : ra;
  int rb = hasB ? static_cast<int>(plane_offset(n, z + 1) + row_offset(n, z + 1, y0)) : ra;
  int ru = hasU ? static_cast<int>(plane_offset(n, z + 2) + row_offset(n, z + 2, y0)) : rb;
  int la = n - z - y0 + 1;                  // row y0 length, plane A
  int ll = hasL ? la + 1 : la;              // plane L
  int lb = hasB ? la - 1 : la;              // plane B
  int lu = hasU ? la - 2 : lb;              // plane U

  // window at row y0 (row y0-1 may be in the front guard: zero weights)
  // plane A rows y0-1 {x, x+1}, y0 {x-1, x, x+1}; plane L row y0 {x, x+1};
  // plane B rows y0-1 {x-1, x, x+1}, y0 {x-1, x, x+1}; plane U row y0-1 {x-1, x}
  const int ram = ra - (la + 1), rbm = rb - (lb + 1), rum = ru - (lu + 1);
  double Am0 = __ldg(X + ram), Am1 = __ldg(X + ram + 1);
  double A0m = __ldg(X + ra - 1), A00 = __ldg(X + ra), A01 = __ldg(X + ra + 1);
  double L00 = __ldg(X + rl), L01 = __ldg(X + rl + 1);
  double Bmm = __ldg(X + rbm - 1), Bm0 = __ldg(X + rbm), Bm1 = __ldg(X + rbm + 1);
  double B0m = __ldg(X + rb - 1), B00 = __ldg(X + rb), B01 = __ldg(X + rb + 1);
  double Umm = __ldg(X + rum - 1), Um0 = __ldg(X + rum);
  const bool face_free = z > 0 && x0 > 0;

#pragma unroll
  for (int r = 0; r < kChunk; ++r) {
    const int yy = y0 + r;
    // new rows: L, A, B row y+1; U row y
    const int rl1 = rl + ll, ra1 = ra + la, rb1 = rb + lb;
    if (kAhead > 0) {
      // warm L1 with row y + 1 + kAhead of the four planes (no registers held)
      const int d = kAhead;
      const int tr = d * (d + 1) / 2;  // rows shrink by one per step
      prefetch_l1(X + rl1 + d * ll - tr);
      prefetch_l1(X + ra1 + d * la - tr);
      prefetch_l1(X + rb1 + d * lb - tr);
      prefetch_l1(X + ru + (d + 1) * lu - tr);
    }
    const double Lp0 = __ldg(X + rl1), Lp1 = __ldg(X + rl1 + 1);
    const double Apm = __ldg(X + ra1 - 1), Ap0 = __ldg(X + ra1), Ap1 = __ldg(X + ra1 + 1);
    const double Bpm = __ldg(X + rb1 - 1), Bp0 = __ldg(X + rb1), Bp1 = __ldg(X + rb1 + 1);
    const double U0m = __ldg(X + ru - 1), U00 = __ldg(X + ru);
    double fa, fb;
    if (face_free && yy > 0 && x0 + 31 + yy + z + 1 < n) {
      fa = stencil_sum(w, A00, A01, A0m, Ap0, Am0, B00, L00, Am1, Apm, L01, B0m, Lp0, Bm0, Lp1, Bmm);
      fb = stencil_sum(w, B00, B01, B0m, Bp0, Bm0, U00, A00, Bm1, Bpm, A01, U0m, Ap0, Um0, Ap1, Umm);
      Y[ra] = fa;
      Y[rb] = fb;
    } else {
      const int sa = px + yy + z;
      const int ta = (px == 0 ? 1 : 0) | (yy == 0 ? 2 : 0) | (z == 0 ? 4 : 0) | (sa == n ? 8 : 0);
      const int tb = (px == 0 ? 1 : 0) | (yy == 0 ? 2 : 0) | (sa + 1 == n ? 8 : 0);
      fa = stencil_var(tab + 16 * ta, A00, A01, A0m, Ap0, Am0, B00, L00, Am1, Apm, L01, B0m, Lp0, Bm0, Lp1, Bmm);
      fb = stencil_var(tab + 16 * tb, B00, B01, B0m, Bp0, Bm0, U00, A00, Bm1, Bpm, A01, U0m, Ap0, Um0, Ap1, Umm);
      if (sa <= n) Y[ra] = fa;
      if (sa + 1 <= n) Y[rb] = fb;
    }
    // slide to row y+1
    Am0 = A00; Am1 = A01;
    A0m = Apm; A00 = Ap0; A01 = Ap1;
    L00 = Lp0; L01 = Lp1;
    Bmm = B0m; Bm0 = B00; Bm1 = B01;
    B0m = Bpm; B00 = Bp0; B01 = Bp1;
    Umm = U0m; Um0 = U00;
    ru += lu;
    rl = rl1; ra = ra1; rb = rb1;
    --ll; --la; --lb; --lu;
  }
}

} // namespace

// Task list: (macro, z, x0, y0) for every row chunk, 32-wide x segment and
// plane pair (z even), plane pairs innermost (L1 sharing inside a CTA).
void build_stencil2_tasks(int nmacros, int n, std::vector<int>& out) {
  out.clear();
  for (int li = 0; li < nmacros; ++li)
    for (int y0 = 0; y0 <= n; y0 += kChunk)
      for (int x0 = 0; x0 <= n - y0; x0 += 32)
        for (int z = 0; z <= n - y0 - x0; z += 2) {
          out.push_back(li);
          out.push_back(z);
          out.push_back(x0);
          out.push_back(y0);
        }
}

void launch_p1_stencil2(const double* x, double* y, const int* d_tasks, int ntasks, i64 macro_stride, int n,
                        const P1DeviceTable* d_tables, const MacroDesc* d_macros, cudaStream_t s) {
  if (ntasks == 0) return;
  const unsigned grid = static_cast<unsigned>((ntasks + kWarps - 1) / kWarps);
  p1_stencil2_kernel<<<grid, 32 * kWarps, 0, s>>>(x, y, reinterpret_cast<const Task2*>(d_tasks), ntasks,
                                                  macro_stride, n, d_tables, d_macros);
  check_launch("p1_stencil2");
}

} // namespace tetmf

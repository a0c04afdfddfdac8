// k_p1_stencil5.cu -- K1 variant 5: P1 -Laplace, interior stencil only +
// separate face pass; CTA-wide L2 bulk prefetch of the block's plane slabs.
//
// Why (ncu of the two-plane row walk, profiles/r1_k1_v2_ncu_summary.txt):
// ~220 warp instructions per 32 points, because every 32-column segment that
// touches a macro face (x = 0, y = 0, z = 0 or the diagonal x+y+z = n) took
// the per-lane stencil-variant path (30 table loads per row step) -- with
// rows ~100 points long on average that is most segments. Here:
//   * main kernel: the interior 15-point stencil (weights uniform per geometry
//     group, in registers) for every point; stores are masked to interior
//     points (x, y, z >= 1, x+y+z <= n-1), where all 15 neighbours exist;
//   * face kernel: one thread per face point (4.6 % of the points at L8)
//     gathers its neighbours with the point-type variant (tables.cpp) in the
//     same summation order as the row walks (bitwise-equal results).
//   * memory-level parallelism: a CTA = (macro, row block [y0, y0+kChunk),
//     block of 2*kWarps planes); its planes' row slabs are contiguous stretches
//     of the plane-major storage, so one thread per plane issues ONE
//     cp.async.bulk.prefetch.L2 for the whole slab at CTA start: the CTA's
//     whole read set is requested from DRAM at once instead of one row step
//     (~2.5 KB per warp) at a time. The row walks then mostly hit L2.
//
// Warp w of a CTA walks the plane pair (z0 + 2w, z0 + 2w + 1) over all
// 32-column segments of the block (register window along y, 10 coalesced
// loads per row step for 2 points, 15 DFMA per point), as k_p1_stencil2.cu.
#include "device.hpp"
#include "runtime_check.hpp"

namespace tetmf {

namespace {

#ifndef TETMF_P1F_WARPS
#define TETMF_P1F_WARPS 4
#endif
#ifndef TETMF_P1F_CHUNK
#define TETMF_P1F_CHUNK 8
#endif
#ifndef TETMF_P1F_PREFETCH
#define TETMF_P1F_PREFETCH 1  // 0: no L2 bulk prefetch (A/B)
#endif
#ifndef TETMF_P1F_MINB
#define TETMF_P1F_MINB 0
#endif
constexpr int kWarps = TETMF_P1F_WARPS;
constexpr int kChunk = TETMF_P1F_CHUNK;
constexpr int kPlanes = 2 * kWarps;
#ifndef TETMF_P1F_AHEAD
#define TETMF_P1F_AHEAD 0  // prefetch the slabs of the CTA this many places later (0: own)
#endif
constexpr int kAhead = TETMF_P1F_AHEAD;
#ifndef TETMF_P1F_NEXTSEG
#define TETMF_P1F_NEXTSEG 0  // 1: warm L1 with the next 32-column segment's rows while walking this one
#endif

struct Task5 {
  int macro, z0, y0, pad;
};

__device__ __forceinline__ void bulk_prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// the same summation order as stencil_sum / stencil_var (k_p1_stencil2.cu)
__device__ __forceinline__ double sum15(const double* __restrict__ w, double c00, double c01, double c0m, double cp0,
                                        double cm0, double u00, double l00, double cm1, double cpm, double l01,
                                        double u0m, double lp0, double um0, double lp1, double umm) {
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

// One face point (x, y, z) of type `type` as a direct 15-point gather with
// the variant weights, in the summation order of sum15. 32-bit incremental
// indexing from the point's own index (neighbour offsets depend only on y
// and the plane side m = n - z). Neighbours outside the lattice have zero
// weights and are not read.
__device__ __forceinline__ double gather_point(const double* __restrict__ X, const double* __restrict__ wt, int n,
                                               int x, int y, int z) {
  const int m = n - z;
  const int i0 = static_cast<int>(plane_offset(n, z)) + y * (m + 1) - y * (y - 1) / 2 + x;
  const int lr = m + 1 - y;              // row y length, plane z
  const int tz = (m + 1) * (m + 2) / 2;  // points of plane z
  const int up = i0 + tz - y;            // (x, y, z+1)
  const int dn = i0 - (tz + m + 2) + y;  // (x, y, z-1): plane z-1 holds tz + m + 2 points
  const bool xm = x > 0, ym = y > 0, zm = z > 0, pp = x + y + z < n;
  // stencil_offset order (tables.hpp): centre, then +/- of the 7 edge directions
  double v[15];
  v[0] = __ldg(X + i0);
  v[1] = pp ? __ldg(X + i0 + 1) : 0.0;                // (+1, 0, 0)
  v[2] = xm ? __ldg(X + i0 - 1) : 0.0;                // (-1, 0, 0)
  v[3] = pp ? __ldg(X + i0 + lr) : 0.0;               // (0, +1, 0)
  v[4] = ym ? __ldg(X + i0 - lr - 1) : 0.0;           // (0, -1, 0): row y-1 holds lr + 1 points
  v[5] = pp ? __ldg(X + up) : 0.0;                    // (0, 0, +1)
  v[6] = zm ? __ldg(X + dn) : 0.0;                    // (0, 0, -1)
  v[7] = ym ? __ldg(X + i0 - lr) : 0.0;               // (+1, -1, 0)
  v[8] = xm ? __ldg(X + i0 + lr - 1) : 0.0;           // (-1, +1, 0)
  v[9] = zm ? __ldg(X + dn + 1) : 0.0;                // (+1, 0, -1)
  v[10] = xm ? __ldg(X + up - 1) : 0.0;               // (-1, 0, +1)
  v[11] = zm ? __ldg(X + dn + lr + 1) : 0.0;          // (0, +1, -1): row y of plane z-1 holds lr + 1 points
  v[12] = ym ? __ldg(X + up - lr) : 0.0;              // (0, -1, +1): row y-1 of plane z+1 holds lr points
  v[13] = zm ? __ldg(X + dn + lr + 2) : 0.0;          // (+1, +1, -1)
  v[14] = (xm && ym) ? __ldg(X + up - lr - 1) : 0.0;  // (-1, -1, +1)
  double w[15];
#pragma unroll
  for (int k = 0; k < 15; ++k) w[k] = __ldg(wt + k);
  return sum15(w, v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], v[8], v[9], v[10], v[11], v[12], v[13], v[14]);
}

// Fused exchange put (FusedPut, device.hpp): the value just stored at slot
// j of the level buffer also goes to every peer window entry it is sent to.
// Only storage slots on a macro face can be shared, so the callers test
// this at their face stores (x = 0 lanes, diagonal and face points).
__device__ __forceinline__ void put_slot(const FusedPut* fp, i64 j, double v) {
  if (!fp) return;
  for (int e = fp->first[j]; e >= 0; e = fp->chain[e]) {
    const i64 d = fp->dst[e];
    fp->win[d >> 48][d & ((i64(1) << 48) - 1)] = v;
  }
}

// Point q of face f (0: z = 0, 1: y = 0, the z = 0 edge excluded) of macro
// li: the triangle a + b <= n enumerated b-major (row b starts at
// S(b) = b(2n+3-b)/2); x = a, and y (f = 0) or z (f = 1) = b.
__device__ __forceinline__ void face_point(const double* __restrict__ xin, double* __restrict__ yout, i64 stride,
                                           int n, const P1DeviceTable* __restrict__ tabs,
                                           const MacroDesc* __restrict__ macros, int li, int f, int q,
                                           const int2* __restrict__ zrange = nullptr,
                                           const FusedPut* fp = nullptr) {
  const float c = 2.0f * n + 3.0f;
  int b = static_cast<int>((c - sqrtf(fmaxf(c * c - 8.0f * q, 0.0f))) * 0.5f);
  b = min(max(b, 0), n);
  while (b > 0 && b * (2 * n + 3 - b) / 2 > q) --b;
  while (b < n && (b + 1) * (2 * n + 2 - b) / 2 <= q) ++b;
  const int a = q - b * (2 * n + 3 - b) / 2;
  const int x = a, y = f == 0 ? b : 0, z = f == 0 ? 0 : b;
  if (f == 1 && z == 0) return;  // on the z = 0 face
  if (zrange && (z < zrange[li].x || z >= zrange[li].y)) return;  // slab partition: another rank's plane
  const int type = (x == 0 ? 1 : 0) | (y == 0 ? 2 : 0) | (z == 0 ? 4 : 0) | (x + y + z == n ? 8 : 0);
  const double* __restrict__ X = xin + static_cast<i64>(li) * stride;
  const double* __restrict__ wt = &tabs[macros[li].group].stencil[type][0];
  const i64 j = static_cast<i64>(li) * stride + lattice_index(n, x, y, z);
  const double v = gather_point(X, wt, n, x, y, z);
  yout[j] = v;
  put_slot(fp, j, v);
}

#if TETMF_P1F_MINB > 0
__global__ void __launch_bounds__(32 * kWarps, TETMF_P1F_MINB)
#else
__global__ void __launch_bounds__(32 * kWarps)
#endif
p1_interior_kernel(const double* __restrict__ xin, double* __restrict__ yout, const Task5* __restrict__ tasks,
                   int ntasks, i64 stride, int n, const P1DeviceTable* __restrict__ tabs, const MacroDesc* __restrict__ macros) {
  const Task5 t = tasks[blockIdx.x];
  const int y0 = t.y0;
  const double* __restrict__ Xm = xin + static_cast<i64>(t.macro) * stride;
  double* __restrict__ Ym = yout + static_cast<i64>(t.macro) * stride;
  if (TETMF_P1F_PREFETCH && threadIdx.x < kPlanes + 2) {
    // slabs of the CTA kAhead places later in the task list (a later wave:
    // its data lands in L2 while this CTA works), or this CTA's own (kAhead 0;
    // the first wave also takes its own): plane p rows max(y0-1, 0) ..
    // min(y0+kChunk, n-p), one contiguous stretch
    auto prefetch = [&](const Task5& u) {
      const int p = u.z0 - 1 + static_cast<int>(threadIdx.x);
      const int ya = u.y0 > 0 ? u.y0 - 1 : 0;
      if (p >= 0 && p <= n - ya) {
        const int yb = min(u.y0 + kChunk, n - p);
        const i64 P = plane_offset(n, p);
        const i64 g0 = (P + row_offset(n, p, ya)) & ~i64(1);
        const i64 g1 = (P + row_offset(n, p, yb + 1) + 1) & ~i64(1);
        bulk_prefetch_l2(xin + static_cast<i64>(u.macro) * stride + g0, static_cast<unsigned>((g1 - g0) * 8));
      }
    };
    if (kAhead == 0 || static_cast<int>(blockIdx.x) < kAhead) prefetch(t);
    if (kAhead > 0 && static_cast<int>(blockIdx.x) + kAhead < ntasks) prefetch(tasks[blockIdx.x + kAhead]);
  }
  const int lane = threadIdx.x & 31;
  const int z = t.z0 + 2 * static_cast<int>(threadIdx.x >> 5);
  if (z > n - y0) return;  // no rows of the block in this plane
  const double* __restrict__ tab = &tabs[macros[t.macro].group].stencil[0][0];

  const bool hasL = z > 0, hasB = z + 1 <= n, hasU = z + 2 <= n;
  const int ra00 = static_cast<int>(plane_offset(n, z) + row_offset(n, z, y0));
  const int rl00 = hasL ? static_cast<int>(plane_offset(n, z - 1) + row_offset(n, z - 1, y0)) : ra00;
  const int rb00 = hasB ? static_cast<int>(plane_offset(n, z + 1) + row_offset(n, z + 1, y0)) : ra00;
  const int ru00 = hasU ? static_cast<int>(plane_offset(n, z + 2) + row_offset(n, z + 2, y0)) : rb00;
  const int la00 = n - z - y0 + 1;
  const int ll00 = hasL ? la00 + 1 : la00;
  const int lb00 = hasB ? la00 - 1 : la00;
  const int lu00 = hasU ? la00 - 2 : lb00;
  // interior: x >= 1, y >= 1, z >= 1 and x + y + z <= n - 1
  const bool zA = z >= 1;

  for (int x0 = 0; x0 < la00; x0 += 32) {
    const int px = x0 + lane;
    const double* __restrict__ X = Xm + px;
    double* __restrict__ Y = Ym + px;
    if (TETMF_P1F_NEXTSEG && x0 + 32 < la00) {
      // rows y0-1 .. y0+kChunk of this warp's planes A, B (and L / U at the
      // CTA's plane-block edges; inner L / U planes are other warps' A / B)
      const double* Xn = X + 32;
      const int wid = static_cast<int>(threadIdx.x >> 5);
      int a = ra00 - (la00 + 1), b = rb00 - (lb00 + 1), l = rl00, u = ru00 - (lu00 + 1);
      int lna = la00 + 1, lnb = lb00 + 1, lnl = ll00, lnu = lu00 + 1;
#pragma unroll 1
      for (int r = 0; r < kChunk + 2; ++r) {
        asm volatile("prefetch.global.L1 [%0];" ::"l"(Xn + a));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(Xn + b));
        if (wid == 0 && r < kChunk + 1) asm volatile("prefetch.global.L1 [%0];" ::"l"(Xn + l));
        if (wid == kWarps - 1) asm volatile("prefetch.global.L1 [%0];" ::"l"(Xn + u));
        a += lna; b += lnb; l += lnl; u += lnu;
        --lna; --lnb; --lnl; --lnu;
      }
    }
    // per-lane weights: the x = 0 column (lane 0 of segment 0) walks with the
    // x = 0 face variant (type 1), every other column with the interior stencil
    double w[15];
    {
      const double* __restrict__ wt = tab + (px == 0 ? 16 : 0);
#pragma unroll
      for (int k = 0; k < 15; ++k) w[k] = __ldg(wt + k);
    }
    int ra = ra00, rl = rl00, rb = rb00, ru = ru00;
    int la = la00, ll = ll00, lb = lb00, lu = lu00;
    const int ram = ra - (la + 1), rbm = rb - (lb + 1), rum = ru - (lu + 1);
    double Am0 = __ldg(X + ram), Am1 = __ldg(X + ram + 1);
    double A0m = __ldg(X + ra - 1), A00 = __ldg(X + ra), A01 = __ldg(X + ra + 1);
    double L00 = __ldg(X + rl), L01 = __ldg(X + rl + 1);
    double Bmm = __ldg(X + rbm - 1), Bm0 = __ldg(X + rbm), Bm1 = __ldg(X + rbm + 1);
    double B0m = __ldg(X + rb - 1), B00 = __ldg(X + rb), B01 = __ldg(X + rb + 1);
    double Umm = __ldg(X + rum - 1), Um0 = __ldg(X + rum);
    // s = px + yy + z of plane A's point at row yy; the walk stores points of
    // type 0 and 1: y >= 1, z >= 1, x + y + z <= n - 1
    const int s0 = px + y0 + z;
#pragma unroll
    for (int r = 0; r < kChunk; ++r) {
      const int yy = y0 + r;
      const int rl1 = rl + ll, ra1 = ra + la, rb1 = rb + lb;
      const double Lp0 = __ldg(X + rl1), Lp1 = __ldg(X + rl1 + 1);
      const double Apm = __ldg(X + ra1 - 1), Ap0 = __ldg(X + ra1), Ap1 = __ldg(X + ra1 + 1);
      const double Bpm = __ldg(X + rb1 - 1), Bp0 = __ldg(X + rb1), Bp1 = __ldg(X + rb1 + 1);
      const double U0m = __ldg(X + ru - 1), U00 = __ldg(X + ru);
      const double fa = sum15(w, A00, A01, A0m, Ap0, Am0, B00, L00, Am1, Apm, L01, B0m, Lp0, Bm0, Lp1, Bmm);
      const double fb = sum15(w, B00, B01, B0m, Bp0, Bm0, U00, A00, Bm1, Bpm, A01, U0m, Ap0, Um0, Ap1, Umm);
      if (yy >= 1 && zA && s0 + r <= n - 1) Y[ra] = fa;
      if (yy >= 1 && s0 + r + 1 <= n - 1) Y[rb] = fb;
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
  // diagonal points (x + y + z = n) of the block's rows: lanes 0..kChunk-1
  // plane A (z), lanes 16..16+kChunk-1 plane B (z+1); y = 0 and z = 0 belong
  // to the face kernel
  {
    const int zz = z + (lane >> 4), yy = y0 + (lane & 15);
    if ((lane & 15) < kChunk && zz >= 1 && yy >= 1 && yy <= n - zz) {
      const int xx = n - zz - yy;
      Ym[lattice_index(n, xx, yy, zz)] = gather_point(Xm, tab + 16 * (8 | (xx == 0 ? 1 : 0)), n, xx, yy, zz);
    }
  }
}

// ---------------------------------------------------------------------------
// Variant 6: the same two-plane walk, fed from shared memory. A CTA owns the
// box (macro, planes [z0, z0 + 2*kWarps6), rows [y0, y0 + kRows6), columns
// [x0, x0 + kCols6)); at start one thread per (plane, row) of the box plus
// halo (planes z0-1 .. z0+2*kWarps6, rows y0-1 .. y0+kRows6) issues ONE 1-D
// TMA bulk copy (cp.async.bulk) of the row piece [x0-1, x0+kCols6+1) into its
// own shared-memory row, all completing on one mbarrier. The whole read set
// of the CTA is thus in flight at once (no registers held, no per-step
// latency), and the walk reads shared memory only. Several CTAs per SM
// overlap one CTA's copies with the others' walks.
// Shared-memory row i holds global indices [base_i, base_i + kPitch6) with
// base_i = (start_i + x0 - 2) & ~1 (16-byte aligned copies); column x of the
// row that starts at global index g sits at (g + x0) & 1 ... see srow().
// Copied pieces are real lattice data or finite neighbours (the previous /
// next row, the guard regions): every read of a stored point is in-lattice,
// and lanes that do not store may read anything finite or not.
#ifndef TETMF_P1S_COLS
#define TETMF_P1S_COLS 64
#endif
#ifndef TETMF_P1S_ROWS
#define TETMF_P1S_ROWS 8   // cube6 L8: 8 rows x 4 warps 94 us, x 2 warps 118 us, 4 rows x 4 warps 108 us
#endif
#ifndef TETMF_P1S_WARPS
#define TETMF_P1S_WARPS 4
#endif
#ifndef TETMF_P1S_COPYONLY
#define TETMF_P1S_COPYONLY 0
#endif
#ifndef TETMF_P1S_NOSTORE
#define TETMF_P1S_NOSTORE 0
#endif
#ifndef TETMF_P1S_MINB
#define TETMF_P1S_MINB 0
#endif
constexpr int kCols6 = TETMF_P1S_COLS;
constexpr int kRows6 = TETMF_P1S_ROWS;
constexpr int kWarps6 = TETMF_P1S_WARPS;
constexpr int kSegs6 = kCols6 / 32;
#ifndef TETMF_P1S_SINGLE
#define TETMF_P1S_SINGLE 0  // 1: one plane per warp (7 shared loads per point, fewer registers)
#endif
constexpr bool kSingle6 = TETMF_P1S_SINGLE;
constexpr int kBoxPlanes6 = kSingle6 ? kWarps6 : 2 * kWarps6;  // planes computed per box
constexpr int kPlanes6 = kBoxPlanes6 + 2;        // with the halo planes
constexpr int kRowsH6 = kRows6 + 2;              // with the halo rows
constexpr int kCopies6 = kPlanes6 * kRowsH6;
constexpr int kPitch6 = kCols6 + 6;              // doubles per shared-memory row
static_assert(kCols6 % 32 == 0 && kRows6 <= 16 && kCopies6 <= 32 * kWarps6, "p1 smem tiling");

// 32-bit lattice offsets: a macro's storage (tet_count(n) points) fits in
// int up to level 11 (the launchers check); the product is formed in 64 bits
__device__ __forceinline__ int tet32(int k) {
  return static_cast<int>(static_cast<long long>((k + 1) * (k + 2)) * (k + 3) / 6);
}
__device__ __forceinline__ int rstart32(int n, int p, int y) {
  return tet32(n) - tet32(n - p) + y * (n - p + 1) - y * (y - 1) / 2;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// shared-memory load at byte address a + IMM (the immediate folds into the LDS)
template <int IMM>
__device__ __forceinline__ double lds_at(unsigned a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(a), "n"(IMM));
  return v;
}

__device__ __forceinline__ void mbar_wait_parity(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "W7_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra W7_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680u)
      : "memory");
}

// Box copies (thread tid < kCopies6 of the CTA): box u into stage S (row
// address table rowtab), completing on barp.
__device__ __forceinline__ void box_issue6(const Task5& u, int tid, double* S, unsigned* rowtab,
                                           unsigned long long* barp, const double* __restrict__ xin, i64 stride,
                                           int n) {
  const int y0 = u.y0, z0 = u.z0, x0 = u.pad;
  const double* __restrict__ Xm = xin + static_cast<i64>(u.macro) * stride;
    const int pi = tid / kRowsH6, ri = tid - pi * kRowsH6;
    const int p = min(max(z0 - 1 + pi, 0), n);  // missing planes alias the nearest (zero weights)
    const int y = y0 - 1 + ri;                  // -1 for the halo of block 0: the formula's finite neighbours
    const int m = n - p;
    const int rs = rstart32(n, p, y);
    // Slab mode: when the box starts at x0 = 0 and the plane's box rows
    // (y0-1 .. yb) are short, their whole contiguous stretch [start(y0-1) - 1,
    // start(yb+1) + 1) fits the plane's shared-memory region and is ONE copy
    // (issued by the plane's row-0 thread); rows then sit at their natural
    // offsets inside the stretch. Otherwise one copy per row, as below.
    const int yb = min(y0 + kRows6, m);
    const int rsa = rstart32(n, p, y0 - 1), rse = rstart32(n, p, yb + 1);
    const int sbase = (rsa - 1) & ~1;
    const int send = (rse + 2) & ~1;
    const bool slab = x0 == 0 && y0 - 1 <= m && send - sbase <= kRowsH6 * kPitch6;
    unsigned bytes = 0;
    if (slab) {
      const unsigned reg = smem_u32(S + pi * kRowsH6 * kPitch6);
      rowtab[tid] = reg + 8u * static_cast<unsigned>(y <= yb + 1 ? rs - sbase : 0);
      if (ri == 0) {
        bytes = static_cast<unsigned>(send - sbase) * 8u;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(barp)), "r"(bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(reg),
            "l"(Xm + sbase), "r"(bytes), "r"(smem_u32(barp))
            : "memory");
      }
    } else {
      const int base = (rs + x0 - 2) & ~1;
      rowtab[tid] = smem_u32(S) + 8u * static_cast<unsigned>(tid * kPitch6 + 2 + ((rs + x0) & 1) - x0);
      if (y <= m) {
        const int g0 = (rs + x0 - 1) & ~1;
        const int g1 = (rs + min(x0 + kCols6 + 1, m + 2 - y) + 1) & ~1;  // row end + 1 at most
        if (g1 > g0) {
          bytes = static_cast<unsigned>(g1 - g0) * 8u;
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(barp)), "r"(bytes)
                       : "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(S + tid * kPitch6 + (g0 - base))),
              "l"(Xm + g0), "r"(bytes), "r"(smem_u32(barp))
              : "memory");
        }
      }
    }
    if (bytes == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(barp)) : "memory");
}

#ifndef TETMF_P1S_DIAG_EARLY
#define TETMF_P1S_DIAG_EARLY 1  // diagonal gathers while the box copies land (0: after the walk)
#endif
constexpr bool kDiagInWalk = !TETMF_P1S_DIAG_EARLY;

// Diagonal points (x + y + z = n) of the warp's plane pair in the box rows,
// by the CTA whose column range holds them: lanes 0..kRows6-1 plane z,
// lanes 16.. plane z+1; direct gathers (global / L2), independent of the box
// copies.
__device__ __forceinline__ void box_diag6(const Task5& t, int wid, int lane, const double* __restrict__ xin,
                                          double* __restrict__ yout, i64 stride, int n,
                                          const double* __restrict__ tab, const FusedPut* fp) {
  const int y0 = t.y0, x0 = t.pad;
  const int z = t.z0 + 2 * wid;
  const double* __restrict__ Xm = xin + static_cast<i64>(t.macro) * stride;
  double* __restrict__ Ym = yout + static_cast<i64>(t.macro) * stride;
  const int zz = z + (lane >> 4), yy = y0 + (lane & 15);
  if ((lane & 15) < kRows6 && zz >= 1 && zz <= n && yy >= 1 && yy <= n - zz) {
    const int xx = n - zz - yy;
    if (xx >= x0 && xx < x0 + kCols6) {
      const double v = gather_point(Xm, tab + 16 * (8 | (xx == 0 ? 1 : 0)), n, xx, yy, zz);
      Ym[lattice_index(n, xx, yy, zz)] = v;
      put_slot(fp, static_cast<i64>(t.macro) * stride + lattice_index(n, xx, yy, zz), v);
    }
  }
}

#ifndef TETMF_P1S_DIAG_SMEM
#define TETMF_P1S_DIAG_SMEM 1  // diagonal points from the landed box (0: global gathers)
#endif

// The same diagonal points as box_diag6, read from the box in shared memory
// (row address table rowtab) after the copies landed: the same 15 values
// (positions past the face read the same global words the gather reads, or
// 0 where the gather uses 0) and the same sum15 order -- bitwise equal.
__device__ __forceinline__ void box_diag6_smem(const Task5& t, const unsigned* __restrict__ rowtab, int wid,
                                               int lane, double* __restrict__ yout, i64 stride, int n,
                                               const double* __restrict__ tab, const FusedPut* fp) {
  const int y0 = t.y0, x0 = t.pad;
  const int z = t.z0 + 2 * wid;
  const int zz = z + (lane >> 4), yy = y0 + (lane & 15);
  if ((lane & 15) < kRows6 && zz >= 1 && zz <= n && yy >= 1 && yy <= n - zz) {
    const int xx = n - zz - yy;
    if (xx >= x0 && xx < x0 + kCols6) {
      const unsigned* R = rowtab + (2 * wid + 1 + (lane >> 4)) * kRowsH6 + (lane & 15) + 1;  // (zz, yy)
      const unsigned bx = 8u * static_cast<unsigned>(xx);
      const unsigned c = R[0] + bx, cm = R[-1] + bx, cp = R[1] + bx;            // rows yy, yy-1, yy+1
      const unsigned d = R[-kRowsH6] + bx, dp = R[-kRowsH6 + 1] + bx;          // plane zz-1: rows yy, yy+1
      const unsigned u = R[kRowsH6] + bx, um = R[kRowsH6 - 1] + bx;            // plane zz+1: rows yy, yy-1
      const bool xm = xx > 0, ym = yy > 0, zm = zz > 0;
      double v[15];
      v[0] = lds_at<0>(c);
      v[1] = 0.0;                           // (+1, 0, 0): past the face
      v[2] = xm ? lds_at<-8>(c) : 0.0;      // (-1, 0, 0)
      v[3] = 0.0;                           // (0, +1, 0)
      v[4] = ym ? lds_at<0>(cm) : 0.0;      // (0, -1, 0)
      v[5] = 0.0;                           // (0, 0, +1)
      v[6] = zm ? lds_at<0>(d) : 0.0;       // (0, 0, -1)
      v[7] = ym ? lds_at<8>(cm) : 0.0;      // (+1, -1, 0)
      v[8] = xm ? lds_at<-8>(cp) : 0.0;     // (-1, +1, 0)
      v[9] = zm ? lds_at<8>(d) : 0.0;       // (+1, 0, -1)
      v[10] = xm ? lds_at<-8>(u) : 0.0;     // (-1, 0, +1)
      v[11] = zm ? lds_at<0>(dp) : 0.0;     // (0, +1, -1)
      v[12] = ym ? lds_at<0>(um) : 0.0;     // (0, -1, +1)
      v[13] = zm ? lds_at<8>(dp) : 0.0;     // (+1, +1, -1): the word after the row, as the gather
      v[14] = (xm && ym) ? lds_at<-8>(um) : 0.0;  // (-1, -1, +1)
      const double* __restrict__ wt = tab + 16 * (8 | (xx == 0 ? 1 : 0));
      double w[15];
#pragma unroll
      for (int k = 0; k < 15; ++k) w[k] = __ldg(wt + k);
      double* __restrict__ Ym = yout + static_cast<i64>(t.macro) * stride;
      const double f =
          sum15(w, v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], v[8], v[9], v[10], v[11], v[12], v[13], v[14]);
      Ym[lattice_index(n, xx, yy, zz)] = f;
      put_slot(fp, static_cast<i64>(t.macro) * stride + lattice_index(n, xx, yy, zz), f);
    }
  }
}

// Fused put of the walk's x = 0 column (the only shared slots the walk
// stores): after the walk, lane l < planes * kRows6 takes row l % kRows6 of
// plane z + l / kRows6 -- the slots lane 0 stored (the walk's store
// conditions), read back after __syncwarp, so the index loads of all rows
// are in flight at once instead of one per row inside the walk.
__device__ __forceinline__ void x0_column_puts(const Task5& t, const FusedPut* fp, int lane, int z, int planes,
                                               double* __restrict__ yout, i64 stride, int n) {
  static_assert(2 * kRows6 <= 32, "one lane per row of the plane pair");
  __syncwarp();  // lane 0's stores are visible to the warp
  const int pl = lane / kRows6, r = lane - pl * kRows6;
  const int ystart = t.y0 == 0 ? 1 : 0;
  const int rlast = pl == 0 ? (z >= 1 ? n - 1 - (t.y0 + z) : -1) : n - 2 - (t.y0 + z);
  if (pl < planes && r >= ystart && r <= rlast) {
    const i64 j = static_cast<i64>(t.macro) * stride + lattice_index(n, 0, t.y0 + r, z + pl);
    put_slot(fp, j, yout[j]);
  }
}

// The warp's walk of box t (plane pair z = z0 + 2*wid) out of the stage whose
// row address table is rowtab; w holds the interior weights on entry.
__device__ __forceinline__ void box_walk6(const Task5& t, const unsigned* __restrict__ rowtab, double (&w)[15],
                                          int wid, int lane, const double* __restrict__ xin,
                                          double* __restrict__ yout, i64 stride, int n,
                                          const double* __restrict__ tab, const FusedPut* fp) {
  const int y0 = t.y0, x0 = t.pad;
  const int z = t.z0 + 2 * wid;
  double* __restrict__ Ym = yout + static_cast<i64>(t.macro) * stride;
  // planes L = z-1, A = z, B = z+1, U = z+2 = box planes 2w .. 2w+3
  const unsigned* __restrict__ RL = rowtab + (2 * wid) * kRowsH6;
  const unsigned* __restrict__ RA = RL + kRowsH6;
  const unsigned* __restrict__ RB = RA + kRowsH6;
  const unsigned* __restrict__ RU = RB + kRowsH6;
  const int la0 = n - z - y0 + 1;  // row y0 length, plane A
  const int ystart = y0 == 0 ? 1 : 0;  // first stored row of the block (y = 0 is the face pass's)
#pragma unroll 1
  for (int sg = 0; sg < kSegs6; ++sg) {
    const int px = x0 + 32 * sg + lane;
    if (x0 + 32 * sg >= la0) break;  // segment past the row ends of both planes
    if (x0 + 32 * sg <= 32) {
      // the lane at x = 0 (segment 0 of an x0 = 0 box) walks with the x = 0
      // face variant (type 1); the next segment's lane 0 is interior again
      const double* __restrict__ wt = tab + (px == 0 ? 16 : 0);
#pragma unroll
      for (int k = 0; k < 15; ++k) w[k] = __ldg(wt + k);
    }
    // last stored row offsets: A stores rows r with s0 + r <= n-1 (z >= 1), B with s0 + r + 1 <= n-1
    const int s0 = px + y0 + z;
    const int rlastA = z >= 1 ? n - 1 - s0 : -1, rlastB = n - 2 - s0;
    double* __restrict__ Ya = Ym + (rstart32(n, z, y0) + px);
    double* __restrict__ Yb = Ym + (rstart32(n, min(z + 1, n), y0) + px);
    int la = la0;
    const unsigned bx = 8u * static_cast<unsigned>(px);  // byte offset of the lane's column
    double Am0 = lds_at<0>(RA[0] + bx), Am1 = lds_at<8>(RA[0] + bx);
    double A0m = lds_at<-8>(RA[1] + bx), A00 = lds_at<0>(RA[1] + bx), A01 = lds_at<8>(RA[1] + bx);
    double L00 = lds_at<0>(RL[1] + bx), L01 = lds_at<8>(RL[1] + bx);
    double Bmm = lds_at<-8>(RB[0] + bx), Bm0 = lds_at<0>(RB[0] + bx), Bm1 = lds_at<8>(RB[0] + bx);
    double B0m = lds_at<-8>(RB[1] + bx), B00 = lds_at<0>(RB[1] + bx), B01 = lds_at<8>(RB[1] + bx);
    double Umm = lds_at<-8>(RU[0] + bx), Um0 = lds_at<0>(RU[0] + bx);
#pragma unroll
    for (int r = 0; r < kRows6; ++r) {
      const unsigned il = RL[r + 2] + bx, ia = RA[r + 2] + bx, ib = RB[r + 2] + bx, iu = RU[r + 1] + bx;
      const double Lp0 = lds_at<0>(il), Lp1 = lds_at<8>(il);
      const double Apm = lds_at<-8>(ia), Ap0 = lds_at<0>(ia), Ap1 = lds_at<8>(ia);
      const double Bpm = lds_at<-8>(ib), Bp0 = lds_at<0>(ib), Bp1 = lds_at<8>(ib);
      const double U0m = lds_at<-8>(iu), U00 = lds_at<0>(iu);
      const double fa = sum15(w, A00, A01, A0m, Ap0, Am0, B00, L00, Am1, Apm, L01, B0m, Lp0, Bm0, Lp1, Bmm);
      const double fb = sum15(w, B00, B01, B0m, Bp0, Bm0, U00, A00, Bm1, Bpm, A01, U0m, Ap0, Um0, Ap1, Umm);
#if TETMF_P1S_NOSTORE  // A/B: the loads and arithmetic without the stores
      if (fa == 12345.678 && fb == 0.5) *Ya = fa;
#else
      if (r >= ystart && r <= rlastA) *Ya = fa;
      if (r >= ystart && r <= rlastB) *Yb = fb;
#endif
      Ya += la;       // row y -> y+1: + row y length (plane A)
      Yb += la - 1;   // plane B rows are one shorter
      --la;
      Am0 = A00; Am1 = A01;
      A0m = Apm; A00 = Ap0; A01 = Ap1;
      L00 = Lp0; L01 = Lp1;
      Bmm = B0m; Bm0 = B00; Bm1 = B01;
      B0m = Bpm; B00 = Bp0; B01 = Bp1;
      Umm = U0m; Um0 = U00;
    }
  }
  if (fp && x0 == 0) x0_column_puts(t, fp, lane, z, 2, yout, stride, n);
  if (TETMF_P1S_DIAG_SMEM)
    box_diag6_smem(t, rowtab, wid, lane, yout, stride, n, tab, fp);
  else if (kDiagInWalk)
    box_diag6(t, wid, lane, xin, yout, stride, n, tab, fp);
}


// Single-plane walk (TETMF_P1S_SINGLE): warp wid walks plane z = z0 + wid
// (box planes wid .. wid+2 = z-1, z, z+1) over the box's segments; 7 shared
// loads per point, the same sums in the same order as the pair walk.
__device__ __forceinline__ void box_walk6_single(const Task5& t, const unsigned* __restrict__ rowtab,
                                                 double (&w)[15], int wid, int lane, const double* __restrict__ xin,
                                                 double* __restrict__ yout, i64 stride, int n,
                                                 const double* __restrict__ tab, const FusedPut* fp) {
  const int y0 = t.y0, x0 = t.pad;
  const int z = t.z0 + wid;
  const double* __restrict__ Xm = xin + static_cast<i64>(t.macro) * stride;
  double* __restrict__ Ym = yout + static_cast<i64>(t.macro) * stride;
  const unsigned* __restrict__ RL = rowtab + wid * kRowsH6;
  const unsigned* __restrict__ RZ = RL + kRowsH6;
  const unsigned* __restrict__ RU = RZ + kRowsH6;
  const int la0 = n - z - y0 + 1;
  const int ystart = y0 == 0 ? 1 : 0;
#pragma unroll 1
  for (int sg = 0; sg < kSegs6; ++sg) {
    const int px = x0 + 32 * sg + lane;
    if (x0 + 32 * sg >= la0) break;
    if (x0 + 32 * sg <= 32) {
      const double* __restrict__ wt = tab + (px == 0 ? 16 : 0);
#pragma unroll
      for (int k = 0; k < 15; ++k) w[k] = __ldg(wt + k);
    }
    const int s0 = px + y0 + z;
    const int rlast = z >= 1 ? n - 1 - s0 : -1;
    double* __restrict__ Yz = Ym + (rstart32(n, z, y0) + px);
    int la = la0;
    const unsigned bx = 8u * static_cast<unsigned>(px);
    double Zm0 = lds_at<0>(RZ[0] + bx), Zm1 = lds_at<8>(RZ[0] + bx);
    double Z0m = lds_at<-8>(RZ[1] + bx), Z00 = lds_at<0>(RZ[1] + bx);
    double L00 = lds_at<0>(RL[1] + bx), L01 = lds_at<8>(RL[1] + bx);
    double Umm = lds_at<-8>(RU[0] + bx), Um0 = lds_at<0>(RU[0] + bx);
#pragma unroll
    for (int r = 0; r < kRows6; ++r) {
      const unsigned iz0 = RZ[r + 1] + bx, iz = RZ[r + 2] + bx, il = RL[r + 2] + bx, iu = RU[r + 1] + bx;
      const double Z01 = lds_at<8>(iz0);
      const double Zpm = lds_at<-8>(iz), Zp0 = lds_at<0>(iz);
      const double Lp0 = lds_at<0>(il), Lp1 = lds_at<8>(il);
      const double U0m = lds_at<-8>(iu), U00 = lds_at<0>(iu);
      const double f = sum15(w, Z00, Z01, Z0m, Zp0, Zm0, U00, L00, Zm1, Zpm, L01, U0m, Lp0, Um0, Lp1, Umm);
      if (r >= ystart && r <= rlast) *Yz = f;
      Yz += la;
      --la;
      Zm0 = Z00; Zm1 = Z01;
      Z0m = Zpm; Z00 = Zp0;
      L00 = Lp0; L01 = Lp1;
      Umm = U0m; Um0 = U00;
    }
  }
  if (fp && x0 == 0) x0_column_puts(t, fp, lane, z, 1, yout, stride, n);
  const int yy = y0 + lane;
  if (lane < kRows6 && z >= 1 && yy >= 1 && yy <= n - z) {
    const int xx = n - z - yy;
    if (xx >= x0 && xx < x0 + kCols6) {
      const double v = gather_point(Xm, tab + 16 * (8 | (xx == 0 ? 1 : 0)), n, xx, yy, z);
      Ym[lattice_index(n, xx, yy, z)] = v;
      put_slot(fp, static_cast<i64>(t.macro) * stride + lattice_index(n, xx, yy, z), v);
    }
  }
}

// kPersistent = false (variant 6, the default): one box per CTA, copy -> wait
// -> walk; several CTAs per SM overlap. kPersistent = true (variant 10): a
// persistent CTA double-buffers two boxes (full / empty mbarrier per stage):
// the copies of box k+1 land while the warps walk box k. Face CTAs (faces
// z = 0, y = 0) follow the boxes in the same launch.
template <bool kPersistent, bool kFused>
#if TETMF_P1S_MINB > 0
__global__ void __launch_bounds__(32 * kWarps6, TETMF_P1S_MINB)
#else
__global__ void __launch_bounds__(32 * kWarps6)
#endif
p1_box_kernel(const double* __restrict__ xin, double* __restrict__ yout, const Task5* __restrict__ tasks, int ntasks,
              int nboxctas, int nmacros, i64 stride, int n, const P1DeviceTable* __restrict__ tabs,
              const MacroDesc* __restrict__ macros, const int2* __restrict__ zrange, const FusedPut fput) {
  const FusedPut* fp = kFused ? &fput : nullptr;  // kFused: the exchange's puts from the store sites
  // Early trigger only where the next kernel on the stream is another K1 (one
  // macro: no K4), whose CTAs then set up their barriers during this grid's
  // tail (config 1: 6.2 -> 4.5 us per apply). With K4 next it is left to the
  // grid's end: K4 CTAs made resident early and parked in pdl_wait() measured
  // slower (config 4: 90.1 -> 94.6 us per apply).
  if (nmacros == 1) pdl_launch_dependents();
  if (static_cast<int>(blockIdx.x) >= nboxctas) {
    pdl_wait();
    // face CTAs after the boxes (same launch, they fill the tail): faces z = 0
    // and y = 0 of every macro, one point per thread
    const int T = (n + 1) * (n + 2) / 2;
    const int gid = (static_cast<int>(blockIdx.x) - nboxctas) * static_cast<int>(blockDim.x) + static_cast<int>(threadIdx.x);
    const int li = gid / (2 * T), rem = gid - li * 2 * T;
    if (li < nmacros)
      face_point(xin, yout, stride, n, tabs, macros, li, rem >= T ? 1 : 0, rem >= T ? rem - T : rem, zrange, fp);
    return;
  }
  extern __shared__ __align__(128) double sm[];
  // row address tables: column x of box row j is at shared byte address
  // rowaddr[stage][j] + 8x (per-row copies: row j holds global [base_j,
  // base_j + kPitch6), base_j = (start_j + x0 - 2) & ~1; slab mode: the
  // plane's rows at their natural offsets in one stretch)
  __shared__ unsigned rowaddr[kPersistent ? 2 : 1][kCopies6];
  __shared__ __align__(8) unsigned long long full[2], empty[2];
  const int tid = static_cast<int>(threadIdx.x), lane = tid & 31, wid = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < (kPersistent ? 2 : 1); ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[i])), "r"(kCopies6));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[i])), "r"(kWarps6));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  pdl_wait();  // x and y are the previous grid's (K4 of the last apply, a solver kernel): barriers set up meanwhile
  __syncthreads();
  constexpr int kStage6 = kCopies6 * kPitch6 + 96;  // doubles per stage (+ slab-mode overread margin)
  if (!kPersistent) {
    const Task5 t = tasks[blockIdx.x];
    if (tid < kCopies6) box_issue6(t, tid, sm, rowaddr[0], &full[0], xin, stride, n);
    __syncthreads();  // rowaddr visible
    const int z = t.z0 + (kSingle6 ? wid : 2 * wid);
    if (!(z <= n - t.y0 && t.pad <= n - t.y0 - z)) return;  // (warp 0 always works: it keeps the CTA alive)
    const double* __restrict__ tab = &tabs[macros[t.macro].group].stencil[0][0];
    double w[15];  // interior weights, loaded while the copies land
#pragma unroll
    for (int k = 0; k < 15; ++k) w[k] = __ldg(tab + k);
    if (!kDiagInWalk && !kSingle6 && !TETMF_P1S_DIAG_SMEM) box_diag6(t, wid, lane, xin, yout, stride, n, tab, fp);
    mbar_wait_parity(&full[0], 0u);
    if (TETMF_P1S_COPYONLY) return;  // A/B: the box copies alone
    if (kSingle6)
      box_walk6_single(t, rowaddr[0], w, wid, lane, xin, yout, stride, n, tab, fp);
    else
      box_walk6(t, rowaddr[0], w, wid, lane, xin, yout, stride, n, tab, fp);
    return;
  }
  const int G = nboxctas;
  if (tid < kCopies6 && static_cast<int>(blockIdx.x) < ntasks)
    box_issue6(tasks[blockIdx.x], tid, sm, rowaddr[0], &full[0], xin, stride, n);
  int k = 0;
  for (int ti = static_cast<int>(blockIdx.x); ti < ntasks; ti += G, ++k) {
    const int st = k & 1;
    if (tid < kCopies6 && ti + G < ntasks) {
      // the other stage is free once every warp released box k-1
      if (k >= 1) mbar_wait_parity(&empty[st ^ 1], static_cast<unsigned>((k - 1) >> 1) & 1u);
      box_issue6(tasks[ti + G], tid, sm + (st ^ 1) * kStage6, rowaddr[st ^ 1], &full[st ^ 1], xin, stride, n);
    }
    const Task5 t = tasks[ti];
    const double* __restrict__ tab = &tabs[macros[t.macro].group].stencil[0][0];
    double w[15];
#pragma unroll
    for (int q = 0; q < 15; ++q) w[q] = __ldg(tab + q);
    if (!kDiagInWalk && !kSingle6 && !TETMF_P1S_DIAG_SMEM && t.z0 + 2 * wid <= n - t.y0)
      box_diag6(t, wid, lane, xin, yout, stride, n, tab, fp);
    // every warp observes the box before releasing it (a released,
    // unobserved phase would alias the stage's next phase)
    mbar_wait_parity(&full[st], static_cast<unsigned>(k >> 1) & 1u);
    const int z = t.z0 + (kSingle6 ? wid : 2 * wid);
    if (z <= n - t.y0 && t.pad <= n - t.y0 - z) {
      if (kSingle6)
        box_walk6_single(t, rowaddr[st], w, wid, lane, xin, yout, stride, n, tab, fp);
      else
        box_walk6(t, rowaddr[st], w, wid, lane, xin, yout, stride, n, tab, fp);
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[st])) : "memory");
  }
}

// Faces z = 0 and y = 0 (coalesced along x): thread per (macro, face f, point
// of the face triangle); a point on both is computed by f = 0 (z = 0). Grid:
// x = points of a face triangle, y = macro * 2 + f. The x = 0 face is walked
// by the interior kernel's lane 0 with its variant weights, the diagonal
// face by its per-block gathers.
__global__ void __launch_bounds__(256) p1_face_kernel(const double* __restrict__ xin, double* __restrict__ yout,
                                                      i64 stride, int n, const P1DeviceTable* __restrict__ tabs,
                                                      const MacroDesc* __restrict__ macros) {
  const int T = (n + 1) * (n + 2) / 2;
  const int q = static_cast<int>(blockIdx.x * blockDim.x + threadIdx.x);
  if (q >= T) return;
  face_point(xin, yout, stride, n, tabs, macros, static_cast<int>(blockIdx.y >> 1), static_cast<int>(blockIdx.y & 1), q);
}

} // namespace

// CTA tasks (macro, z0, y0): row block [y0, y0+kChunk) x planes [z0, z0+2*kWarps)
// with rows in the block (z0 <= n - y0); order macro, y0, z0.
void build_stencil5_tasks(int nmacros, int n, std::vector<int>& out) {
  out.clear();
  for (int li = 0; li < nmacros; ++li)
    for (int y0 = 0; y0 <= n; y0 += kChunk)
      for (int z0 = 0; z0 <= n - y0; z0 += kPlanes) {
        out.push_back(li);
        out.push_back(z0);
        out.push_back(y0);
        out.push_back(0);
      }
}

// CTA boxes of variant 6 (macro, z0, y0, x0): x0 < row length of (y0, z0)
void build_stencil6_tasks(int nmacros, int n, std::vector<int>& out) {
  out.clear();
  for (int li = 0; li < nmacros; ++li)
    for (int y0 = 0; y0 <= n; y0 += kRows6)
      for (int z0 = 0; z0 <= n - y0; z0 += kBoxPlanes6)
        for (int x0 = 0; x0 <= n - y0 - z0; x0 += kCols6) {
          out.push_back(li);
          out.push_back(z0);
          out.push_back(y0);
          out.push_back(x0);
        }
}

template <bool kPersistent, bool kFused>
static void launch_p1_box(const double* x, double* y, const int* d_tasks, int ntasks, i64 macro_stride, int n,
                          int nmacros, const P1DeviceTable* d_tables, const MacroDesc* d_macros, cudaStream_t s,
                          const int* zrange = nullptr, const FusedPut& fp = FusedPut{}) {
  if (ntasks == 0 && !zrange) return;
  if (tet_count(n) + n + 96 >= (i64(1) << 31)) fail_arg("p1 box kernel: level too large for 32-bit lattice offsets");
  // per stage: the box rows + a margin (in slab mode lanes past the short rows
  // read up to a segment beyond the last plane's stretch; never stored)
  const std::size_t smem = (kPersistent ? 2 : 1) * (static_cast<std::size_t>(kCopies6) * kPitch6 + 96) * sizeof(double);
  static int box_ctas = 0;
  if (box_ctas == 0) {
    TETMF_CUDA(cudaFuncSetAttribute(p1_box_kernel<kPersistent, kFused>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
    int dev = 0, sms = 0, per_sm = 0;
    TETMF_CUDA(cudaGetDevice(&dev));
    TETMF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    TETMF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, p1_box_kernel<kPersistent, kFused>, 32 * kWarps6, smem));
    box_ctas = sms * (per_sm > 0 ? per_sm : 1);
  }
  const int nbox = kPersistent ? (ntasks < box_ctas ? ntasks : box_ctas) : ntasks;
  // boxes, then the face CTAs (faces z = 0 and y = 0) in the same launch
  const int T = (n + 1) * (n + 2) / 2;
  const int face_ctas = (2 * T * nmacros + 32 * kWarps6 - 1) / (32 * kWarps6);
  TETMF_CUDA(launch_pdl(kPdlK1, p1_box_kernel<kPersistent, kFused>, dim3(static_cast<unsigned>(nbox + face_ctas)),
                        dim3(32 * kWarps6), smem, s, x, y, reinterpret_cast<const Task5*>(d_tasks), ntasks, nbox,
                        nmacros, macro_stride, n, d_tables, d_macros, reinterpret_cast<const int2*>(zrange), fp));
  check_launch("p1_box");
}

void launch_p1_stencil6(const double* x, double* y, const int* d_tasks, int ntasks, i64 macro_stride, int n,
                        int nmacros, const P1DeviceTable* d_tables, const MacroDesc* d_macros, cudaStream_t s,
                        const int* zrange, const FusedPut& fp) {
  if (fp.first)
    launch_p1_box<false, true>(x, y, d_tasks, ntasks, macro_stride, n, nmacros, d_tables, d_macros, s, zrange, fp);
  else
    launch_p1_box<false, false>(x, y, d_tasks, ntasks, macro_stride, n, nmacros, d_tables, d_macros, s, zrange);
}

void launch_p1_stencil10(const double* x, double* y, const int* d_tasks, int ntasks, i64 macro_stride, int n,
                         int nmacros, const P1DeviceTable* d_tables, const MacroDesc* d_macros, cudaStream_t s) {
  launch_p1_box<true, false>(x, y, d_tasks, ntasks, macro_stride, n, nmacros, d_tables, d_macros, s);
}

void launch_p1_stencil5(const double* x, double* y, const int* d_tasks, int ntasks, i64 macro_stride, int n,
                        int nmacros, const P1DeviceTable* d_tables, const MacroDesc* d_macros, cudaStream_t s) {
  if (ntasks == 0) return;
  p1_interior_kernel<<<static_cast<unsigned>(ntasks), 32 * kWarps, 0, s>>>(
      x, y, reinterpret_cast<const Task5*>(d_tasks), ntasks, macro_stride, n, d_tables, d_macros);
  check_launch("p1_interior");
  const int T = (n + 1) * (n + 2) / 2;
  p1_face_kernel<<<dim3(static_cast<unsigned>((T + 255) / 256), static_cast<unsigned>(2 * nmacros)), 256, 0, s>>>(
      x, y, macro_stride, n, d_tables, d_macros);
  check_launch("p1_face");
}

} // namespace tetmf

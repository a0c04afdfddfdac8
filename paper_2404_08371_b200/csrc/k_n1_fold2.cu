// k_n1_fold2.cu -- K3 (default since round 2): N1 alpha curl curl + beta
// apply, folded cube walk over LAYER PAIRS.
//
// The walk, the fold of near / far columns, the lane roles, the input ring
// and the delayed writes of phase 2 are those of k_n1_fold.cu (read its
// header first). What changes: a task covers the layer pair (z, z+1) of a
// segment pair, and every step processes two cubes per lane, A = (x, y, z)
// and B = (x, y, z+1) (the ZW element, n1_common.cuh), sharing:
//  * the input rows: planes z, z+1, z+2 of x, alpha, beta are copied once
//    for both cubes (23 arrays per row for two cubes instead of 2 x 14);
//  * the row address math, the table-base selection, the loop control;
//  * plane z+1: A's top-face contributions (cube edges 14..18) are the
//    first terms of B's bottom-face accumulators (B's edges 0, 1, 3, 7, 10),
//    so the in-plane edges of plane z+1 are complete inside the step and
//    are stored once, with no read-modify-write.
// Parity passes now alternate layer PAIRS: pass 0 walks the pairs starting at
// z = 0, 4, 8, ..., pass 1 those at z = 2, 6, 10, ... Only the in-plane
// edges of the planes between pairs (A's bottom, B's top) are stored by
// pass 0 and read-modify-written by pass 1, so each plane of x, alpha and
// beta moves 1.5 times per apply instead of 2, and half as many partial sums.
// The last layer of an odd count walks as a pair whose B layer is empty (its
// cubes read the zero table; its stores are guarded by the lattice limits).
//
// Ring arrays (per row): 0..6 x plane z classes 0..6; 7..13 x plane z+1
// classes 0..6; 14, 15, 16 x plane z+2 classes 0, 1, 3; 17, 18, 19 alpha
// planes z, z+1, z+2; 20, 21, 22 beta planes z, z+1, z+2.
#include <cstdlib>

#include "device.hpp"
#include "n1_common.cuh"
#include "runtime_check.hpp"

namespace tetmf {

namespace {

using namespace n1;

#ifndef TETMF_N1F2_WARPS
#define TETMF_N1F2_WARPS 4  // warps per CTA
#endif
constexpr int kWarps = TETMF_N1F2_WARPS;
#ifndef TETMF_N1F2_MIN_BLOCKS
#define TETMF_N1F2_MIN_BLOCKS 2
#endif
#ifndef TETMF_N1F2_CHUNK
#define TETMF_N1F2_CHUNK 32
#endif
constexpr int kChunk = TETMF_N1F2_CHUNK;  // steps per task (+1 halo step)
constexpr int kSeg = 31;                  // owner columns per segment
constexpr int kArrays = 23;               // input arrays per row
constexpr int kRow = 34;                  // positions per array row
constexpr int kSlot = kArrays * kRow;     // doubles per ring slot
constexpr int kRing = 3 * kSlot;          // input ring, doubles per warp
constexpr int kRmw = 2 * 6 * 32;          // pass-1 staging, two slots (step parity), doubles per warp
constexpr int kWarpSmem = kRing + kRmw;
constexpr int kZeroTab = 6 * kGramRow + 8;         // doubles: zero table offset (+64 B bank phase)
constexpr int kTabs = kZeroTab + 6 * kGramRow + 8;  // doubles before the warps' rings

struct FoldTask {
  int macro, z, k, t0;  // first layer of the pair, near segment, first step of the chunk
};

// cube edge K -> (class, offset in {0,1}^3) as in n1_common.cuh cube_edge_id
__host__ __device__ constexpr int edge_cls(int k) {
  return k <= 6 ? k : k == 7 ? 1 : k == 8 ? 2 : k == 9 ? 5 : k == 10 ? 0 : k == 11 ? 2 : k == 12 ? 4
       : k == 13 ? 2 : k == 14 ? 0 : k == 15 ? 1 : k == 16 ? 3 : k == 17 ? 1 : 0;
}
__host__ __device__ constexpr bool edge_up(int k) { return k >= 14; }  // anchor in the upper plane
__host__ __device__ constexpr bool edge_row1(int k) { return (k >= 10 && k <= 13) || k == 18; }
__host__ __device__ constexpr bool edge_plus1(int k) { return k == 7 || k == 8 || k == 9 || k == 13 || k == 17; }
// ring array of cube edge K for the cube of layer offset B (0: A, 1: B)
template <int B>
__host__ __device__ constexpr int ring_array(int k) {
  return !edge_up(k) ? 7 * B + edge_cls(k)
         : B == 0    ? 7 + edge_cls(k)
                     : 14 + (edge_cls(k) == 0 ? 0 : edge_cls(k) == 1 ? 1 : 2);
}

template <int B>
struct FoldIn2 {
  const double* r0;  // own position, row y
  const double* r1;  // own position, row y + 1
  const double* q0;  // x+1 neighbour position, row y
  const double* q1;  // x+1 neighbour position, row y + 1
  template <int K>
  __device__ __forceinline__ double x() const {
    const double* p = edge_plus1(K) ? (edge_row1(K) ? q1 : q0) : (edge_row1(K) ? r1 : r0);
    return lds(p + ring_array<B>(K) * kRow);
  }
  template <int V, int W>
  __device__ __forceinline__ double c() const {
    constexpr int a = 17 + 3 * W + B + (V >> 2);
    const double* p = (V & 1) ? (((V >> 1) & 1) ? q1 : q0) : (((V >> 1) & 1) ? r1 : r0);
    return lds(p + a * kRow);
  }
};

#ifdef TETMF_N1F2_MAXNREG
#define TETMF_N1F2_BOUNDS __maxnreg__(TETMF_N1F2_MAXNREG)
#else
#define TETMF_N1F2_BOUNDS __launch_bounds__(32 * kWarps, TETMF_N1F2_MIN_BLOCKS)
#endif
template <int PASS, int RULE>
__global__ void TETMF_N1F2_BOUNDS
n1_fold2_kernel(const N1GramTable* __restrict__ gram,
                const MacroDesc* __restrict__ macros,
                const double* __restrict__ xin, const double* __restrict__ alpha, const double* __restrict__ beta,
                double* __restrict__ yout, const FoldTask* __restrict__ tasks, int ntasks, i64 stride, i64 cstride,
                i64 cf_stride, int n, int chunk) {
  extern __shared__ __align__(16) double dsm[];
  {
    const N1GramTable* gt = gram + macros[tasks[blockIdx.x * kWarps].macro].group;
    for (int i = threadIdx.x; i < 6 * kGramRow; i += blockDim.x) dsm[i] = __ldg(&gt->o[0][0] + i);
  }
  double* ztab = dsm + kZeroTab;
  for (int i = threadIdx.x; i < 6 * kGramRow; i += blockDim.x) ztab[i] = 0.0;
  const unsigned tab_a = static_cast<unsigned>(__cvta_generic_to_shared(dsm));
  const unsigned zero_a = static_cast<unsigned>(__cvta_generic_to_shared(ztab));
  const int lane = threadIdx.x & 31;
  double* ring = dsm + kTabs + (threadIdx.x >> 5) * kWarpSmem;
  for (int i = lane; i < kRing; i += 32) ring[i] = 0.0;  // unfilled positions must read finite
  double* rmw = ring + kRing + lane;                     // [2][6][32]
  __syncthreads();
  const int warp = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (warp >= ntasks) return;
  const FoldTask tk = tasks[warp];
  if (tk.macro < 0) return;  // padding task
  const int z = tk.z, m = n - 1, L = n - 1 - z;
  const int K = (L + 1) / kSeg;
  const int kn = tk.k, kf = K - 1 - kn;
  const bool paired = kn < K && kf > kn;
  const int x0 = kSeg * kn;
  const int D = 2 * L + 4 - kSeg * K;
  const int Xn = x0 - 1 + lane;
  const int P1 = lane == 0 ? L - x0 + 1 : L - Xn + 1;
  const int Xf = lane < 31 ? kSeg * kf + 30 - lane : kSeg * kf - 1;
  const bool far_ok = paired && Xf <= L;
  const int ytop = L - Xf - (lane == 31 ? 1 : 0);
  const int nsteps = paired ? D + 2 : L - x0 + 1;
  const int t0 = tk.t0;
  const int ts = t0 > 0 ? t0 - 1 : 0;
  const int te = min(t0 + chunk, nsteps);

  const int cs = static_cast<int>(cstride);
  const double* __restrict__ Xm = xin + static_cast<i64>(tk.macro) * stride;
  double* __restrict__ Ym = yout + static_cast<i64>(tk.macro) * stride;
  const double* __restrict__ Am = alpha + static_cast<i64>(tk.macro) * cf_stride;
  const double* __restrict__ Bm = beta + static_cast<i64>(tk.macro) * cf_stride;
  // planes z, z+1, z+2 of the edge (extent m) and vertex (extent n) lattices;
  // planes past the lattice (the B layer of the top pair) are clamped to the
  // top plane: their values only reach zero-table elements and guarded stores
  const int pe0 = static_cast<int>(plane_offset(m, z));
  const int pe1 = static_cast<int>(plane_offset(m, min(z + 1, m)));
  const int pe2 = static_cast<int>(plane_offset(m, min(z + 2, m)));
  const int pv0 = static_cast<int>(plane_offset(n, z));
  const int pv1 = static_cast<int>(plane_offset(n, min(z + 1, n)));
  const int pv2 = static_cast<int>(plane_offset(n, min(z + 2, n)));
  const int le0 = m - z + 1, le1 = max(le0 - 1, 1), le2 = max(le0 - 2, 1);  // row-0 lengths
  const int lv0 = n - z + 1, lv1 = max(lv0 - 1, 1), lv2 = max(lv0 - 2, 1);
  auto tri = [](int r) { return r * (r - 1) / 2; };
  auto e0_of = [&](int r) { return pe0 + r * le0 - tri(r); };
  auto e1_of = [&](int r) { return pe1 + r * le1 - tri(r); };
  auto e2_of = [&](int r) { return pe2 + r * le2 - tri(r); };

  auto copy_for = [&](int tc, int slot) {
    int row = -1, col = 0;
    bool far = false;
    if (tc + 1 < P1) {
      row = tc + 2;
      col = Xn;
    } else if (far_ok) {
      const int yp = D - tc - 1;
      if (yp >= 0 && yp <= ytop + 1) {
        row = yp;
        col = Xf;
        far = true;
      }
    }
    if (row >= 0) {
      double* d = ring + slot * kSlot;
      const int tr = tri(row);
      const double* x0p = Xm + (pe0 + row * le0 - tr + col);
      const double* x1p = Xm + (pe1 + row * le1 - tr + col);
      const double* x2p = Xm + (pe2 + row * le2 - tr + col);
      const int v0 = pv0 + row * lv0 - tr + col, v1 = pv1 + row * lv1 - tr + col, v2 = pv2 + row * lv2 - tr + col;
      double* o = d + lane + 1;
#pragma unroll
      for (int c = 0; c < 7; ++c) cp_async8(o + c * kRow, x0p + c * cs);
#pragma unroll
      for (int c = 0; c < 7; ++c) cp_async8(o + (7 + c) * kRow, x1p + c * cs);
      cp_async8(o + 14 * kRow, x2p);
      cp_async8(o + 15 * kRow, x2p + cs);
      cp_async8(o + 16 * kRow, x2p + 3 * cs);
      cp_async8(o + 17 * kRow, Am + v0);
      cp_async8(o + 18 * kRow, Am + v1);
      cp_async8(o + 19 * kRow, Am + v2);
      cp_async8(o + 20 * kRow, Bm + v0);
      cp_async8(o + 21 * kRow, Bm + v1);
      cp_async8(o + 22 * kRow, Bm + v2);
      if (far ? lane == 0 : lane == 31) {  // column + 1 of the phase's boundary lane
        double* e = d + (far ? 0 : 33);
        cp_async8(e + 1 * kRow, x0p + cs + 1);
        cp_async8(e + 2 * kRow, x0p + 2 * cs + 1);
        cp_async8(e + 5 * kRow, x0p + 5 * cs + 1);
        cp_async8(e + 8 * kRow, x1p + cs + 1);
        cp_async8(e + 9 * kRow, x1p + 2 * cs + 1);
        cp_async8(e + 12 * kRow, x1p + 5 * cs + 1);
        cp_async8(e + 15 * kRow, x2p + cs + 1);
        cp_async8(e + 17 * kRow, Am + v0 + 1);
        cp_async8(e + 18 * kRow, Am + v1 + 1);
        cp_async8(e + 19 * kRow, Am + v2 + 1);
        cp_async8(e + 20 * kRow, Bm + v0 + 1);
        cp_async8(e + 21 * kRow, Bm + v1 + 1);
        cp_async8(e + 22 * kRow, Bm + v2 + 1);
      }
    }
    cp_async_commit();
  };
  // pass 1: the partial sums step tn adds to -- [0..2] plane z classes 0, 1,
  // 3 (A's bottom); [3..5] plane z+2 classes 0, 1, 3 (B's top); class 0 at the
  // delayed row in phase 2
  auto stage_rmw = [&](int tn) {
    double* r = rmw + (tn & 1) * 192;
    if (tn < P1) {
      if (tn >= 0 && lane > 0) {
        const double* a = Ym + e0_of(tn) + Xn;
        const double* b = Ym + e2_of(tn) + Xn;
        cp_async8(r, a);
        cp_async8(r + 32, a + cs);
        cp_async8(r + 64, a + 3 * cs);
        cp_async8(r + 96, b);
        cp_async8(r + 128, b + cs);
        cp_async8(r + 160, b + 3 * cs);
      }
    } else if (far_ok && lane < 31) {
      const int yn = D - tn;
      if (yn >= 0 && yn <= ytop) {
        const double* a = Ym + e0_of(yn) + Xf;
        const double* b = Ym + e2_of(yn) + Xf;
        cp_async8(r + 32, a + cs);
        cp_async8(r + 64, a + 3 * cs);
        cp_async8(r + 128, b + cs);
        cp_async8(r + 160, b + 3 * cs);
      }
      if (yn + 1 >= 0 && yn + 1 <= ytop) {
        cp_async8(r, Ym + e0_of(yn + 1) + Xf);
        cp_async8(r + 96, Ym + e2_of(yn + 1) + Xf);
      }
    }
    cp_async_commit();
  };

  int slot = ts % 3;
  copy_for(ts - 2, slot == 0 ? 1 : slot == 1 ? 2 : 0);
  copy_for(ts - 1, slot == 0 ? 2 : slot - 1);
  if (PASS == 1) {  // the first writing step's partial sums (an empty group before a halo step)
    if (t0 == 0)
      stage_rmw(0);
    else
      cp_async_commit();
  }

  // carried sums: A plane z (0, 2, 4), B plane z+1 (0, 2, 4), B plane z+2 (0)
  double a0 = 0.0, a2 = 0.0, a4 = 0.0, b0 = 0.0, b2 = 0.0, b4 = 0.0, bT = 0.0;
  for (int tt = ts; tt < te; ++tt) {
    asm volatile("" ::: "memory");
    copy_for(tt, slot);
    if constexpr (PASS == 1) {
      // staging two slots deep: the partial sums step tt + 1 adds to are
      // requested now and land while this step computes
      if (tt + 1 < te)
        stage_rmw(tt + 1);
      else
        cp_async_commit();
      asm volatile("cp.async.wait_group 2;" ::: "memory");  // this step's inputs and staged sums
    } else {
      cp_async_wait1();
    }
    __syncwarp();
    const int sA = slot == 2 ? 0 : slot + 1;
    const int sB = sA == 2 ? 0 : sA + 1;
    slot = sA;
    const bool p1 = tt < P1;
    const int yf = D - tt;
    const int y = p1 ? tt : yf;
    const int X = p1 ? Xn : Xf;
    const bool cube = p1 ? Xn >= 0 : far_ok && yf >= 0 && yf <= ytop;
    const double* r0 = ring + (p1 ? sA : sB) * kSlot + lane + 1;
    const double* r1 = ring + (p1 ? sB : sA) * kSlot + lane + 1;
    const int dq = p1 ? 1 : -1;
    const int s = X + y + z;  // anchor sum of A; B's is s + 1

    const bool wrt = tt >= t0;  // the halo step only restores the carried sums
    const double* st = rmw + (tt & 1) * 192;  // pass 1: staged partial sums (requested at step tt - 1)
    auto wr = [&](double* p, int k, double v) {
      if (PASS == 0)
        *p = v;
      else
        *p = st[32 * k] + v;
    };
    const int src = (p1 ? lane - 1 : lane + 1) & 31;

    // ---- cube A = (x, y, z): plane z stores; its top face seeds B
    double YB[19];
    {
      double YA[19];
      cube_elements_zw<RULE>(SmemTabs3{opaque_u32(cube && s <= n - 1 ? tab_a : zero_a),
                                       opaque_u32(cube && s <= n - 2 ? tab_a : zero_a),
                                       opaque_u32(cube && s <= n - 3 ? tab_a : zero_a)},
                             FoldIn2<0>{r0, r1, r0 + dq, r1 + dq}, YA);
      const double r7 = __shfl_sync(0xffffffffu, YA[7], src);
      const double r8 = __shfl_sync(0xffffffffu, YA[8], src);
      const double r9 = __shfl_sync(0xffffffffu, YA[9], src);
      const double r13 = __shfl_sync(0xffffffffu, YA[13], src);
      if (wrt) {
        if (p1) {
          if (lane > 0 && cube && s <= n - 1) {  // all owned edges of row y
            double* __restrict__ ya = Ym + e0_of(y) + X;
            ya[2 * cs] = YA[2] + a2 + r8;
            ya[4 * cs] = YA[4] + a4;
            ya[5 * cs] = YA[5] + r9;
            wr(ya, 0, YA[0] + a0);
            wr(ya + cs, 1, YA[1] + r7);
            wr(ya + 3 * cs, 2, YA[3]);
            if (s <= n - 2) ya[6 * cs] = YA[6];
          }
        } else if (lane < 31 && far_ok) {
          if (cube) {  // owned edges of row y with no share from row y-1
            double* __restrict__ ya = Ym + e0_of(y) + X;
            ya[5 * cs] = YA[5] + r9;
            wr(ya + cs, 1, YA[1] + r7);
            wr(ya + 3 * cs, 2, YA[3]);
            if (s <= n - 2) ya[6 * cs] = YA[6];
          }
          if (y + 1 >= 0 && y + 1 <= ytop) {  // delayed edges of row y+1
            double* __restrict__ ya = Ym + e0_of(y + 1) + X;
            ya[2 * cs] = YA[11] + a2 + r13;
            ya[4 * cs] = YA[12] + a4;
            wr(ya, 0, YA[10] + a0);
          }
        }
      }
      if (p1) {
        a0 = YA[10];
        a2 = YA[11] + r13;
        a4 = YA[12];
      } else {
        a0 = YA[0];
        a2 = YA[2] + r8;
        a4 = YA[4];
      }
      // B's bottom face starts from A's top face (plane z+1 in-plane edges)
      YB[0] = YA[14];
      YB[1] = YA[15];
      YB[3] = YA[16];
      YB[7] = YA[17];
      YB[10] = YA[18];
    }

    // ---- cube B = (x, y, z+1): plane z+1 (complete) and plane z+2 stores
    cube_elements_zw<RULE, true>(SmemTabs3{opaque_u32(cube && s <= n - 2 ? tab_a : zero_a),
                                           opaque_u32(cube && s <= n - 3 ? tab_a : zero_a),
                                           opaque_u32(cube && s <= n - 4 ? tab_a : zero_a)},
                                 FoldIn2<1>{r0, r1, r0 + dq, r1 + dq}, YB);
    __syncwarp();  // ring slot tt mod 3 is refilled by the next step's copies
    {
      const double r7 = __shfl_sync(0xffffffffu, YB[7], src);
      const double r8 = __shfl_sync(0xffffffffu, YB[8], src);
      const double r9 = __shfl_sync(0xffffffffu, YB[9], src);
      const double r13 = __shfl_sync(0xffffffffu, YB[13], src);
      const double r17 = __shfl_sync(0xffffffffu, YB[17], src);
      if (wrt) {
        if (p1) {
          if (lane > 0 && cube && s <= n - 2) {
            double* __restrict__ yb = Ym + e1_of(y) + X;
            yb[2 * cs] = YB[2] + b2 + r8;
            yb[4 * cs] = YB[4] + b4;
            yb[5 * cs] = YB[5] + r9;
            yb[0] = YB[0] + b0;
            yb[cs] = YB[1] + r7;
            yb[3 * cs] = YB[3];
            if (s <= n - 3) {
              yb[6 * cs] = YB[6];
              double* __restrict__ yc = Ym + e2_of(y) + X;
              wr(yc, 3, YB[14] + bT);
              wr(yc + cs, 4, YB[15] + r17);
              wr(yc + 3 * cs, 5, YB[16]);
            }
          }
        } else if (lane < 31 && far_ok) {
          if (cube && s <= n - 2) {
            double* __restrict__ yb = Ym + e1_of(y) + X;
            yb[5 * cs] = YB[5] + r9;
            yb[cs] = YB[1] + r7;
            yb[3 * cs] = YB[3];
            if (s <= n - 3) {
              yb[6 * cs] = YB[6];
              double* __restrict__ yc = Ym + e2_of(y) + X;
              wr(yc + cs, 4, YB[15] + r17);
              wr(yc + 3 * cs, 5, YB[16]);
            }
          }
          if (y + 1 >= 0 && y + 1 <= ytop && s + 1 <= n - 2) {
            double* __restrict__ yb = Ym + e1_of(y + 1) + X;
            yb[2 * cs] = YB[11] + b2 + r13;
            yb[4 * cs] = YB[12] + b4;
            yb[0] = YB[10] + b0;
            if (s + 1 <= n - 3) wr(Ym + e2_of(y + 1) + X, 3, YB[18] + bT);
          }
        }
      }
      if (p1) {
        b0 = YB[10];
        b2 = YB[11] + r13;
        b4 = YB[12];
        bT = YB[18];
      } else {
        b0 = YB[0];
        b2 = YB[2] + r8;
        b4 = YB[4];
        bT = YB[14];
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

} // namespace

// Task list of one level and parity pass: (macro, z, k, t0) per layer pair
// (z, z+1) with z = 4j + 2 * parity, segment pair or unpaired segment of
// layer z, and chunk of `chunk` steps.
void build_n1_fold2_tasks(const std::vector<int>& local_macros, int n, int parity, std::vector<int>& out,
                          int chunk) {
  out.clear();
  for (int z = 2 * parity; z <= n - 1; z += 4) {
    const int L = n - 1 - z, K = (L + 1) / kSeg;
    const int klast = (L + 1) % kSeg ? K : K - 1;
    for (int k = 0; k <= klast; ++k) {
      if (k < K && K - 1 - k < k) continue;
      const bool paired = k < K && K - 1 - k > k;
      const int nsteps = paired ? 2 * L + 6 - kSeg * K : L - kSeg * k + 1;
      for (int t0 = 0; t0 < nsteps; t0 += chunk)
        for (int li : local_macros) {
          out.push_back(li);
          out.push_back(z);
          out.push_back(k);
          out.push_back(t0);
        }
    }
  }
}

void pad_n1_fold2_tasks(std::vector<int>& tasks) {
  while ((tasks.size() / 4) % kWarps) {
    tasks.push_back(-1);
    tasks.push_back(0);
    tasks.push_back(0);
    tasks.push_back(0);
  }
}

int n1_fold2_chunk(const std::vector<int>& local_macros, int n, int sms) {
  if (const char* e = std::getenv("TETMF_N1F2_CHUNK_STEPS")) {  // tuning sweeps (tools/k3_chunk.py)
    const int c = std::atoi(e);
    if (c >= 1) return c;
  }
  // 32 steps per task while that leaves every resident warp (8 per SM) five
  // tasks; on small lattices shorter tasks (each pays one halo step) down to
  // 2 steps: a task is a serial walk and the kernel ends with its longest one.
  // Measured (tools/k3_chunk.py, profiles/r2_k3_chunk_sweep.txt; bitwise equal
  // for every length): config 3 (one macro at L6) 72 us at 8 steps, 46 at 4,
  // 33 at 2; cube6 L6 75 / 70 / 77; 48 macros at L5 102 / 94 / 108.
  std::vector<int> t;
  auto count = [&](int c) {
    build_n1_fold2_tasks(local_macros, n, 0, t, c);
    return static_cast<long long>(t.size() / 4);
  };
  int chunk = kChunk;
  while (chunk > 8 && count(chunk) < 4LL * 10 * sms) chunk /= 2;
  if (chunk == 8 && count(8) < 2LL * 8 * sms) chunk = 4;
  if (chunk == 4 && count(4) < 4LL * sms) chunk = 2;
  return chunk;
}

void launch_n1_fold2(const N1GramTable* gram, const MacroDesc* macros, int pass, const double* x, const double* alpha,
                     const double* beta, double* y, const int* d_tasks, int ntasks, i64 macro_stride,
                     i64 class_stride, i64 coeff_stride, int n, int rule, cudaStream_t s, int chunk) {
  if (ntasks == 0) return;
  if (rule < 0 || rule > 2) fail_internal("n1_fold2: rule index out of range");
  if (chunk < 1) fail_internal("n1_fold2: chunk < 1");
  constexpr int smem = static_cast<int>(sizeof(double) * (kTabs + kWarpSmem * kWarps));
  using Kf = decltype(&n1_fold2_kernel<0, 0>);
  static const Kf kerns[2][3] = {{n1_fold2_kernel<0, 0>, n1_fold2_kernel<0, 1>, n1_fold2_kernel<0, 2>},
                                 {n1_fold2_kernel<1, 0>, n1_fold2_kernel<1, 1>, n1_fold2_kernel<1, 2>}};
  static const bool attr = [] {
    for (int p = 0; p < 2; ++p)
      for (int r = 0; r < 3; ++r) cudaFuncSetAttribute(kerns[p][r], cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    double R[2][4][10];
    n1_rule_moments(1, R[0]);
    n1_rule_moments(2, R[1]);
    cudaMemcpyToSymbol(n1::kN1Rule, R, sizeof(R));
    return true;
  }();
  (void)attr;
  const unsigned grid = static_cast<unsigned>((ntasks + kWarps - 1) / kWarps);
  kerns[pass][rule]<<<grid, 32 * kWarps, smem, s>>>(gram, macros, x, alpha, beta, y,
                                                     reinterpret_cast<const FoldTask*>(d_tasks), ntasks, macro_stride,
                                                     class_stride, coeff_stride, n, chunk);
  check_launch("n1_fold2");
}

} // namespace tetmf

// k_p2v_fold.cu -- P2V (-div(k grad u), u and k in P2; forms.cpp:12) as the
// folded cube walk of K3 (k_n1_fold.cu, one layer per task), default for the
// exact rule since round 2, session 2.
//
// Why: the cube kernel (k_p2v.cu, one thread per cube) spends two thirds of
// its instructions outside the FP64 work -- index arithmetic through
// constant-bank tables for a runtime orientation loop, 20 dependent global
// loads per element, shared-memory accumulators, 27 FP64 atomics per cube.
// Here the six elements of a cube are compile-time code fed from a per-warp
// shared-memory row ring, the cube's 27 accumulators live in registers, and
// every DoF is stored once, in a fixed order, with no atomics.
//
// Element: the factored P2V form of k_p2v.cu (W = G U, Z = W K, y_vertex q
// = 3 Z_qq - sum_{s != q} Z_qs, y_edge (q,s) = 4 (Z_qs + Z_sq)) with the
// moment matrix K in closed form (p2v_exact_moments). Validity by table:
// elements outside the macro read an all-zero G (W = Z = 0).
//
// Walk: K3's fold -- a warp owns a pair of 31-column segments of layer z;
// each lane walks its near column upward, then the mirrored far column
// downward (every lane the same step count). The fold runs over the POINT
// columns of plane z (x + y <= n - z), one more than the cube columns, so
// every vertex of plane z is some lane's own corner; the extra cubes read
// the zero table. Ownership:
//  * edges: exactly K3's (seven owned classes at the cube's anchor, x+1
//    owners by shuffle, y neighbours carried, phase-2 edges shared with the
//    row below written one step late);
//  * vertices: corner 0 is the lane's own point; corners 1 / 3 (x+1) come
//    from the x-1 lane by shuffle, corners 2 / 3 (y+1) are carried to the
//    next row step (upward) or complete the row above one step late
//    (downward); planes z and z+1 alike.
// Layers alternate parity passes: pass 0 (even z) stores the in-plane edges
// and the vertices of planes z and z+1, pass 1 (odd z) adds its sums
// (staged two slots deep by cp.async); the apex plane z + 1 = n, which only
// layer n - 1 touches, is stored plainly.
//
// Ring arrays (per row): 0..6 x edges plane z classes 0..6; 7, 8, 9 x edges
// plane z+1 classes 0, 1, 3; 10, 11 x vertices planes z, z+1; 12..23 the same
// for k.
#include <cstdlib>

#include "device.hpp"
#include "n1_common.cuh"
#include "p2v_common.cuh"
#include "runtime_check.hpp"

namespace tetmf {

namespace {

using namespace n1;

#ifndef TETMF_P2VF_WARPS
#define TETMF_P2VF_WARPS 4
#endif
constexpr int kWarps = TETMF_P2VF_WARPS;
#ifndef TETMF_P2VF_MINB
#define TETMF_P2VF_MINB 2
#endif
#ifndef TETMF_P2VF_CHUNK
#define TETMF_P2VF_CHUNK 32
#endif
constexpr int kChunk = TETMF_P2VF_CHUNK;
constexpr int kSeg = 31;
constexpr int kArrays = 24;
constexpr int kRow = 34;
constexpr int kSlot = kArrays * kRow;
constexpr int kRing = 3 * kSlot;
constexpr int kStageW = 8 * 32;             // pass-1 staging: 8 partial sums x 32 lanes
constexpr int kWarpSmem = kRing + 2 * kStageW;
constexpr int kTabRow = 12;                 // G row (10 values) padded to 16 bytes
constexpr int kTab = 6 * kTabRow;           // doubles of one table
constexpr int kZeroOff = kTab + 8;          // zero table, 64 bytes off the real one's bank phase
constexpr int kTabs = kZeroOff + kTab + 8;  // doubles before the warps' rings (multiple of 2)

struct FoldTask {
  int macro, z, k, t0;
};

// cube edge K -> ring array / row / x+1 position (as k_n1_fold.cu)
__host__ __device__ constexpr int edge_array(int k) {
  return k <= 6 ? k : k == 7 ? 1 : k == 8 ? 2 : k == 9 ? 5 : k == 10 ? 0 : k == 11 ? 2 : k == 12 ? 4
       : k == 13 ? 2 : k == 14 ? 7 : k == 15 ? 8 : k == 16 ? 9 : k == 17 ? 8 : 7;
}
__host__ __device__ constexpr bool edge_row1(int k) { return (k >= 10 && k <= 13) || k == 18; }
__host__ __device__ constexpr bool edge_plus1(int k) { return k == 7 || k == 8 || k == 9 || k == 13 || k == 17; }
__host__ __device__ constexpr int local_edge_of(int q, int r) {  // local edge joining local vertices q != r
  return q < r ? edge_of_pair(q, r) : edge_of_pair(r, q);
}

struct FoldInP2 {
  const double* r0;  // own position, row y
  const double* r1;  // own position, row y + 1
  const double* q0;  // x+1 neighbour position, row y
  const double* q1;  // x+1 neighbour position, row y + 1
  template <int K, int F>  // F = 0: x, 1: k
  __device__ __forceinline__ double e() const {
    const double* p = edge_plus1(K) ? (edge_row1(K) ? q1 : q0) : (edge_row1(K) ? r1 : r0);
    return lds(p + (12 * F + edge_array(K)) * kRow);
  }
  template <int V, int F>
  __device__ __forceinline__ double v() const {
    const double* p = (V & 1) ? (((V >> 1) & 1) ? q1 : q0) : (((V >> 1) & 1) ? r1 : r0);
    return lds(p + (12 * F + 10 + (V >> 2)) * kRow);
  }
};

// one orientation's G row at a 32-bit shared address (pure pair loads)
template <int O>
struct GTab {
  unsigned a;
  template <int I>
  __device__ __forceinline__ double get() const {
    double lo, hi;
    asm("ld.shared.v2.f64 {%0, %1}, [%2+%3];" : "=d"(lo), "=d"(hi) : "r"(a), "n"((O * kTabRow + (I & ~1)) * 8));
    return (I & 1) ? hi : lo;
  }
};

template <int O, int V, int F>
__device__ __forceinline__ double vload(const FoldInP2& in) {
  return in.template v<cube_vertex(O, V), F>();
}
template <int O, int E, int F>
__device__ __forceinline__ double eload(const FoldInP2& in) {
  return in.template e<cube_edge(O, E), F>();
}

// Y[0..7] cube vertices (x + 2y + 4z), Y[8 + K] cube edge K
template <int O>
__device__ __forceinline__ void p2v_element(const GTab<O>& tb, const FoldInP2& in, double (&Y)[27]) {
  double xv[10], kv[10];
  xv[0] = vload<O, 0, 0>(in), xv[1] = vload<O, 1, 0>(in), xv[2] = vload<O, 2, 0>(in), xv[3] = vload<O, 3, 0>(in);
  kv[0] = vload<O, 0, 1>(in), kv[1] = vload<O, 1, 1>(in), kv[2] = vload<O, 2, 1>(in), kv[3] = vload<O, 3, 1>(in);
  xv[4] = eload<O, 0, 0>(in), xv[5] = eload<O, 1, 0>(in), xv[6] = eload<O, 2, 0>(in);
  xv[7] = eload<O, 3, 0>(in), xv[8] = eload<O, 4, 0>(in), xv[9] = eload<O, 5, 0>(in);
  kv[4] = eload<O, 0, 1>(in), kv[5] = eload<O, 1, 1>(in), kv[6] = eload<O, 2, 1>(in);
  kv[7] = eload<O, 3, 1>(in), kv[8] = eload<O, 4, 1>(in), kv[9] = eload<O, 5, 1>(in);
  double K[10];
  p2v_exact_moments(kv, K);
  double U[4][4];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int r = 0; r < 4; ++r) U[q][r] = q == r ? 3.0 * xv[q] : fma(4.0, xv[4 + local_edge_of(q, r)], -xv[q]);
  double g[10];
  g[0] = tb.template get<0>(), g[1] = tb.template get<1>(), g[2] = tb.template get<2>();
  g[3] = tb.template get<3>(), g[4] = tb.template get<4>(), g[5] = tb.template get<5>();
  g[6] = tb.template get<6>(), g[7] = tb.template get<7>(), g[8] = tb.template get<8>();
  g[9] = tb.template get<9>();
  // G has zero row and column sums (sum_p grad lambda_p = 0), so
  //   W_qr = sum_{p<3} G_qp (U_pr - U_3r)   and   Z_3s = -(Z_0s + Z_1s + Z_2s):
  // rows 0..2 of W and Z are formed, row 3 of Z is the negated running sum
  // (104 FP64 instead of 128 for W and Z)
  double V[3][4];
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int r = 0; r < 4; ++r) V[p][r] = U[p][r] - U[3][r];
  double Zs[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double Zq[4];
    if (q < 3) {
      double W[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        double a = g[sym4(0, q)] * V[0][r];
        a = fma(g[sym4(1, q)], V[1][r], a);
        W[r] = fma(g[sym4(2, q)], V[2][r], a);
      }
#pragma unroll
      for (int s2 = 0; s2 < 4; ++s2) {
        double zz = W[0] * K[sym4(0, s2)];
#pragma unroll
        for (int r = 1; r < 4; ++r) zz = fma(W[r], K[sym4(r, s2)], zz);
        Zq[s2] = zz;
        Zs[s2] = q == 0 ? zz : Zs[s2] + zz;
      }
    } else {
#pragma unroll
      for (int s2 = 0; s2 < 4; ++s2) Zq[s2] = -Zs[s2];
    }
    double v = 0.0;
#pragma unroll
    for (int s2 = 0; s2 < 4; ++s2) {
      if (s2 == q) {
        v = fma(3.0, Zq[s2], v);
      } else {
        v -= Zq[s2];
        double& ye = Y[8 + cube_edge(O, local_edge_of(q, s2))];
        ye = fma(4.0, Zq[s2], ye);
      }
    }
    Y[cube_vertex(O, q)] += v;
  }
}

template <int PASS>
__global__ void __launch_bounds__(32 * kWarps, TETMF_P2VF_MINB)
p2v_fold_kernel(const P2VTable* __restrict__ tabs, const MacroDesc* __restrict__ macros,
                const double* __restrict__ xin, const double* __restrict__ kin, double* __restrict__ yout,
                const FoldTask* __restrict__ tasks, int ntasks, i64 stride, i64 cstride, int n, int chunk) {
  extern __shared__ __align__(16) double dsm[];
  {
    const P2VTable* gt = tabs + macros[tasks[blockIdx.x * kWarps].macro].group;
    for (int i = threadIdx.x; i < kTab; i += blockDim.x) {
      const int o = i / kTabRow, j = i - o * kTabRow;
      dsm[i] = j < 10 ? __ldg(&gt->G[o][j]) : 0.0;
      dsm[kZeroOff + i] = 0.0;
    }
  }
  const unsigned tab_a = static_cast<unsigned>(__cvta_generic_to_shared(dsm));
  const unsigned zero_a = static_cast<unsigned>(__cvta_generic_to_shared(dsm + kZeroOff));
  const int lane = threadIdx.x & 31;
  double* ring = dsm + kTabs + (threadIdx.x >> 5) * kWarpSmem;
  for (int i = lane; i < kRing; i += 32) ring[i] = 0.0;
  double* stg = ring + kRing + lane;  // [2][8][32]
  __syncthreads();
  const int warp = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (warp >= ntasks) return;
  const FoldTask tk = tasks[warp];
  if (tk.macro < 0) return;  // padding task
  const int z = tk.z, m = n - 1, L = n - z;  // plane z's POINT columns: x + y <= L
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
  const int vstride = static_cast<int>((tet_count(n) + 31) / 32 * 32);  // edge blocks follow the vertex block
  const double* __restrict__ Xm = xin + static_cast<i64>(tk.macro) * stride;
  const double* __restrict__ Km = kin + static_cast<i64>(tk.macro) * stride;
  double* __restrict__ Ym = yout + static_cast<i64>(tk.macro) * stride;
  const double* __restrict__ Xe = Xm + vstride;
  const double* __restrict__ Ke = Km + vstride;
  double* __restrict__ Ye = Ym + vstride;
  // edge planes z, z+1 (extent m) and vertex planes z, z+1 (extent n);
  // planes past the lattice are clamped (only zero-table elements and
  // guarded stores see them)
  const int pez = static_cast<int>(plane_offset(m, min(z, m))), peu = static_cast<int>(plane_offset(m, min(z + 1, m)));
  const int pvz = static_cast<int>(plane_offset(n, z)), pvu = static_cast<int>(plane_offset(n, min(z + 1, n)));
  const int lez = max(m - z + 1, 1), leu = max(m - z, 1);  // row-0 lengths
  const int lvz = n - z + 1, lvu = max(n - z, 1);
  auto tri = [](int r) { return r * (r - 1) / 2; };
  auto ez_of = [&](int r) { return pez + r * lez - tri(r); };
  auto eu_of = [&](int r) { return peu + r * leu - tri(r); };
  auto vz_of = [&](int r) { return pvz + r * lvz - tri(r); };
  auto vu_of = [&](int r) { return pvu + r * lvu - tri(r); };
  // pass 1 adds to what pass 0 stored; the apex plane (z + 1 = n) has no
  // other layer
  const bool add_up = PASS == 1 && z + 1 <= n - 1;

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
      const int oz = pez + row * lez - tr + col, ou = peu + row * leu - tr + col;
      const int vz = pvz + row * lvz - tr + col, vu = pvu + row * lvu - tr + col;
      double* o = d + lane + 1;
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        const double* E = f ? Ke : Xe;
        const double* V = f ? Km : Xm;
        double* of = o + 12 * f * kRow;
#pragma unroll
        for (int c = 0; c < 7; ++c) cp_async8(of + c * kRow, E + oz + c * cs);
        cp_async8(of + 7 * kRow, E + ou);
        cp_async8(of + 8 * kRow, E + ou + cs);
        cp_async8(of + 9 * kRow, E + ou + 3 * cs);
        cp_async8(of + 10 * kRow, V + vz);
        cp_async8(of + 11 * kRow, V + vu);
      }
      if (far ? lane == 0 : lane == 31) {  // column + 1 of the phase's boundary lane
        double* e = d + (far ? 0 : 33);
#pragma unroll
        for (int f = 0; f < 2; ++f) {
          const double* E = f ? Ke : Xe;
          const double* V = f ? Km : Xm;
          double* ef = e + 12 * f * kRow;
          cp_async8(ef + 1 * kRow, E + oz + cs + 1);
          cp_async8(ef + 2 * kRow, E + oz + 2 * cs + 1);
          cp_async8(ef + 5 * kRow, E + oz + 5 * cs + 1);
          cp_async8(ef + 8 * kRow, E + ou + cs + 1);
          cp_async8(ef + 10 * kRow, V + vz + 1);
          cp_async8(ef + 11 * kRow, V + vu + 1);
        }
      }
    }
    cp_async_commit();
  };
  // pass 1: the partial sums step tn adds to, into slot tn & 1: [0..2] edges
  // plane z classes 0, 1, 3; [3..5] plane z+1 classes 0, 1, 3 (class 0 at
  // the delayed row in phase 2); [6], [7] the vertex of planes z, z+1 (the
  // delayed row in phase 2)
  auto stage = [&](int tn) {
    double* r = stg + (tn & 1) * kStageW;
    if (tn < P1) {
      if (tn >= 0 && lane > 0) {
        const double* a = Ye + ez_of(tn) + Xn;
        const double* b = Ye + eu_of(tn) + Xn;
        cp_async8(r, a);
        cp_async8(r + 32, a + cs);
        cp_async8(r + 64, a + 3 * cs);
        cp_async8(r + 96, b);
        cp_async8(r + 128, b + cs);
        cp_async8(r + 160, b + 3 * cs);
        cp_async8(r + 192, Ym + vz_of(tn) + Xn);
        cp_async8(r + 224, Ym + vu_of(tn) + Xn);
      }
    } else if (far_ok && lane < 31) {
      const int yn = D - tn;
      if (yn >= 0 && yn <= ytop) {
        const double* a = Ye + ez_of(yn) + Xf;
        const double* b = Ye + eu_of(yn) + Xf;
        cp_async8(r + 32, a + cs);
        cp_async8(r + 64, a + 3 * cs);
        cp_async8(r + 128, b + cs);
        cp_async8(r + 160, b + 3 * cs);
      }
      if (yn + 1 >= 0 && yn + 1 <= ytop) {
        cp_async8(r, Ye + ez_of(yn + 1) + Xf);
        cp_async8(r + 96, Ye + eu_of(yn + 1) + Xf);
        cp_async8(r + 192, Ym + vz_of(yn + 1) + Xf);
        cp_async8(r + 224, Ym + vu_of(yn + 1) + Xf);
      }
    }
    cp_async_commit();
  };

  int slot = ts % 3;
  copy_for(ts - 2, slot == 0 ? 1 : slot == 1 ? 2 : 0);
  copy_for(ts - 1, slot == 0 ? 2 : slot - 1);
  if (PASS == 1) {
    if (t0 == 0)
      stage(0);
    else
      cp_async_commit();
  }

  // carried sums: edges (c0, c2, c4 plane z; cT0 plane z+1 class 0), vertices
  // (cv0 plane z, cv1 plane z+1)
  double c0 = 0.0, c2 = 0.0, c4 = 0.0, cT0 = 0.0, cv0 = 0.0, cv1 = 0.0;
  for (int tt = ts; tt < te; ++tt) {
    asm volatile("" ::: "memory");
    copy_for(tt, slot);
    if constexpr (PASS == 1) {
      if (tt + 1 < te)
        stage(tt + 1);
      else
        cp_async_commit();
      asm volatile("cp.async.wait_group 2;" ::: "memory");
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
    const int s = X + y + z;

    double Y[27];
#pragma unroll
    for (int k = 0; k < 27; ++k) Y[k] = 0.0;
    {
      const unsigned bWU = opaque_u32(cube && s <= n - 1 ? tab_a : zero_a);
      const unsigned bMid = opaque_u32(cube && s <= n - 2 ? tab_a : zero_a);
      const unsigned bWD = opaque_u32(cube && s <= n - 3 ? tab_a : zero_a);
      const FoldInP2 in{r0, r1, r0 + dq, r1 + dq};
      p2v_element<WU>(GTab<WU>{bWU}, in, Y);
      p2v_element<BU>(GTab<BU>{bMid}, in, Y);
      p2v_element<BD>(GTab<BD>{bMid}, in, Y);
      p2v_element<GU>(GTab<GU>{bMid}, in, Y);
      p2v_element<GD>(GTab<GD>{bMid}, in, Y);
      p2v_element<WD>(GTab<WD>{bWD}, in, Y);
    }
    __syncwarp();  // ring slot tt mod 3 is refilled by the next step's copies

    const int src = (p1 ? lane - 1 : lane + 1) & 31;
    // edges of the x-1 neighbour cube (K3 numbering, + 8)
    const double r7 = __shfl_sync(0xffffffffu, Y[8 + 7], src);
    const double r8 = __shfl_sync(0xffffffffu, Y[8 + 8], src);
    const double r9 = __shfl_sync(0xffffffffu, Y[8 + 9], src);
    const double r13 = __shfl_sync(0xffffffffu, Y[8 + 13], src);
    const double r17 = __shfl_sync(0xffffffffu, Y[8 + 17], src);
    // x+1 corners of the x-1 neighbour cube
    const double v1 = __shfl_sync(0xffffffffu, Y[1], src);
    const double v3 = __shfl_sync(0xffffffffu, Y[3], src);
    const double v5 = __shfl_sync(0xffffffffu, Y[5], src);
    const double v7 = __shfl_sync(0xffffffffu, Y[7], src);
    const double* E = Y + 8;

    if (tt >= t0) {
      const double* st = stg + (tt & 1) * kStageW;
      auto wr = [&](double* p, int k, double v) {  // in-plane partial sums / vertices
        if (PASS == 0)
          *p = v;
        else
          *p = st[32 * k] + v;
      };
      if (p1) {
        if (lane > 0) {
          // vertices (X, y) of planes z and z+1
          if (s <= n) wr(Ym + vz_of(y) + X, 6, Y[0] + v1 + cv0);
          if (s + 1 <= n) {
            double* p = Ym + vu_of(y) + X;
            const double v = Y[4] + v5 + cv1;
            *p = add_up ? st[32 * 7] + v : v;
          }
          if (cube && s <= n - 1) {  // all owned edges of row y
            double* __restrict__ yz = Ye + ez_of(y) + X;
            yz[2 * cs] = E[2] + c2 + r8;
            yz[4 * cs] = E[4] + c4;
            yz[5 * cs] = E[5] + r9;
            wr(yz, 0, E[0] + c0);
            wr(yz + cs, 1, E[1] + r7);
            wr(yz + 3 * cs, 2, E[3]);
            if (s <= n - 2) {
              yz[6 * cs] = E[6];
              double* __restrict__ yu = Ye + eu_of(y) + X;
              wr(yu, 3, E[14] + cT0);
              wr(yu + cs, 4, E[15] + r17);
              wr(yu + 3 * cs, 5, E[16]);
            }
          }
        }
      } else if (lane < 31 && far_ok) {
        if (cube && s <= n - 1) {  // owned edges of row y with no share from row y-1
          double* __restrict__ yz = Ye + ez_of(y) + X;
          yz[5 * cs] = E[5] + r9;
          wr(yz + cs, 1, E[1] + r7);
          wr(yz + 3 * cs, 2, E[3]);
          if (s <= n - 2) {
            yz[6 * cs] = E[6];
            double* __restrict__ yu = Ye + eu_of(y) + X;
            wr(yu + cs, 4, E[15] + r17);
            wr(yu + 3 * cs, 5, E[16]);
          }
        }
        if (y + 1 >= 0 && y + 1 <= ytop) {  // the delayed row y+1
          if (s + 1 <= n) wr(Ym + vz_of(y + 1) + X, 6, cv0 + Y[2] + v3);
          if (s + 2 <= n) {
            double* p = Ym + vu_of(y + 1) + X;
            const double v = cv1 + Y[6] + v7;
            *p = add_up ? st[32 * 7] + v : v;
          }
          if (s + 1 <= n - 1) {
            double* __restrict__ yz = Ye + ez_of(y + 1) + X;
            yz[2 * cs] = E[11] + c2 + r13;
            yz[4 * cs] = E[12] + c4;
            wr(yz, 0, E[10] + c0);
            if (s + 1 <= n - 2) wr(Ye + eu_of(y + 1) + X, 3, E[18] + cT0);
          }
        }
      }
    }
    if (p1) {
      c0 = E[10];
      c2 = E[11] + r13;
      c4 = E[12];
      cT0 = E[18];
      cv0 = Y[2] + v3;
      cv1 = Y[6] + v7;
    } else {
      c0 = E[0];
      c2 = E[2] + r8;
      c4 = E[4];
      cT0 = E[14];
      cv0 = Y[0] + v1;
      cv1 = Y[4] + v5;
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

} // namespace

// one layer per task, parity = z mod 2; the fold over plane z's point columns
void build_p2v_fold_tasks(const std::vector<int>& local_macros, int n, int parity, std::vector<int>& out, int chunk) {
  out.clear();
  for (int z = parity; z <= n - 1; z += 2) {
    const int L = n - z, K = (L + 1) / kSeg;
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

void pad_p2v_fold_tasks(std::vector<int>& tasks) {
  while ((tasks.size() / 4) % kWarps) {
    tasks.push_back(-1);
    tasks.push_back(0);
    tasks.push_back(0);
    tasks.push_back(0);
  }
}

int p2v_fold_chunk(const std::vector<int>& local_macros, int n, int sms) {
  if (const char* e = std::getenv("TETMF_P2VF_CHUNK_STEPS")) {  // tuning sweeps (tools/k3_chunk.py --p2v)
    const int c = std::atoi(e);
    if (c >= 1) return c;
  }
  // as n1_fold2_chunk: shorter tasks on small lattices, down to 2 steps
  // (tools/k3_chunk.py --p2v, profiles/r2_p2v_chunk_sweep.txt; bitwise equal
  // for every length): one macro at L6 58 us at 8 steps, 39 at 4, 37 at 2;
  // cube6 L4 51 / 36 / 28; one macro at L7 88 / 88 / 92
  std::vector<int> t;
  auto count = [&](int c) {
    build_p2v_fold_tasks(local_macros, n, 0, t, c);
    return static_cast<long long>(t.size() / 4);
  };
  int chunk = kChunk;
  while (chunk > 8 && count(chunk) < 4LL * 8 * sms) chunk /= 2;
  if (chunk == 8 && count(8) < 6LL * sms) chunk = 4;
  if (chunk == 4 && count(4) < 3LL * sms) chunk = 2;
  return chunk;
}

void launch_p2v_fold(const P2VTable* tabs, const MacroDesc* macros, int pass, const double* x, const double* k,
                     double* y, const int* d_tasks, int ntasks, i64 macro_stride, i64 class_stride, int n,
                     cudaStream_t s, int chunk) {
  if (ntasks == 0) return;
  if (chunk < 1) fail_internal("p2v_fold: chunk < 1");
  constexpr int smem = static_cast<int>(sizeof(double) * (kTabs + kWarpSmem * kWarps));
  static const bool attr = [] {
    cudaFuncSetAttribute(p2v_fold_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(p2v_fold_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return true;
  }();
  (void)attr;
  const unsigned grid = static_cast<unsigned>((ntasks + kWarps - 1) / kWarps);
  const auto* t = reinterpret_cast<const FoldTask*>(d_tasks);
  if (pass == 0)
    p2v_fold_kernel<0><<<grid, 32 * kWarps, smem, s>>>(tabs, macros, x, k, y, t, ntasks, macro_stride, class_stride, n,
                                                       chunk);
  else
    p2v_fold_kernel<1><<<grid, 32 * kWarps, smem, s>>>(tabs, macros, x, k, y, t, ntasks, macro_stride, class_stride, n,
                                                       chunk);
  check_launch("p2v_fold");
}

} // namespace tetmf

// k_p1k_cube.cu -- K2 default: P1 -div(k grad u), k in P1, as a cube walk.
//
//   y = sum over the micro elements e of  kbar_e K_o(e) x_e,
//   kbar_e = (k_a + k_b + k_c + k_d) / 4
// (the config-2 harness; forms.cpp:133-193 local_matrix with
// k in P1, exact for P1 k). Same operator as k_p1k_gather.cu, organised by
// cubes instead of points.
//
// Element work per cube. The six orientations anchored at lattice point a
// tile the cube [a, a+1]^3 (lattice.hpp orient_offset) and together have 19
// distinct edges (36 element-edge incidences). K_o has zero row sums, so
//   (K_o x)_i = sum_{j != i} K_o[i][j] (x_j - x_i)
// and the cube's contribution to its 8 corners is, per cube edge (a, b),
//   w_ab = sum_{e contains a, b} kbar_e K_o[i][j],  d = x_b - x_a,
//   c_a += w_ab d,  c_b -= w_ab d.
// That is 13 DADD (the six kbar, sharing pair sums) + 36 DMUL/DFMA (w) +
// 19 DADD (d) + 38 DFMA + 4 DADD (merging the x+1 corners of the left
// neighbour): 110 FP64 instructions per cube, one cube per lattice point,
// against 172 per point for the gather (each element's kbar recomputed at
// its four vertices, each edge weight at both ends).
//
// Walk. A warp runs tasks (macro, x0, y0, z0): lanes l = 0..31 hold the
// columns x = x0 - 1 + l (lane 0 is the halo column: its cubes only feed the
// x0 corners of lane 1); the warp walks layers z = z0 - 1 .. z0 + Z - 1 and,
// in each layer, the cube rows y = y0 - 1 .. y0 + C - 1 (row y0 - 1 and layer
// z0 - 1 are halos). Every corner sum is carried in registers or in the
// lane's own shared-memory column, never re-read from HBM:
//   x + 1 corners (c1, c3, c5, c7)   -> lane + 1 by one shuffle each;
//   y + 1 corners of plane z (c2, c3) -> the next row step (register R);
//   plane z + 1 corners (c4 .. c7)    -> the next layer (the lane's column
//                                       P[0 .. C-1] in shared memory).
// A vertex is final when its row step of its layer has run: stored once, by
// exactly one task, with a fixed summation order (deterministic, no atomics).
// Inputs: each lane copies the x and x + 1 values of x and k in planes z and
// z + 1 of a row (8 eight-byte cp.async) into its own column of a 3-slot ring
// two rows ahead and reads them back one step ahead. (Register-destination
// loads one step ahead measured 445 us on c2l: their scoreboard is shared
// with the table's shared loads, so every step waited for HBM; 1-D bulk
// copies by one lane: 468 us, the per-copy issue code costs more than it saves.)
// Elements outside the macro get kbar = 0 (selects): their w are exactly 0,
// and the positions read for them are finite values (the guard regions or
// neighbouring rows / planes of the same buffer).
// Tasks are taken dynamically by the warps of one resident wave, heaviest
// first (the list is sorted by step count).
#include <cstdlib>

#include "device.hpp"
#include "runtime_check.hpp"

#include <algorithm>
#include <cstdint>
#include <type_traits>

namespace tetmf {

namespace {

#ifndef TETMF_P1KC_WARPS
#define TETMF_P1KC_WARPS 2  // warps per CTA
#endif
constexpr int kCWarps = TETMF_P1KC_WARPS;
#ifndef TETMF_P1KC_ROWS
#define TETMF_P1KC_ROWS 16  // C: cube rows per task (one halo row per task)
#endif
#ifndef TETMF_P1KC_LAYERS
#define TETMF_P1KC_LAYERS 16  // Z: layers per task (one halo layer per task)
#endif
#ifndef TETMF_P1KC_MINB
#define TETMF_P1KC_MINB 4  // CTAs per SM the register budget is sized for (8 warps)
#endif
#ifndef TETMF_P1KC_PAIR
#define TETMF_P1KC_PAIR 1  // 1: two layers per step (cubes z and z + 1 share the table loads)
#endif
#ifndef TETMF_P1KC_SPLIT
#define TETMF_P1KC_SPLIT 1  // 1: separate accumulators for the upper cube of a pair
#endif
constexpr int kRows = TETMF_P1KC_ROWS;
constexpr bool kPair = TETMF_P1KC_PAIR != 0;
constexpr int kPl = kPair ? 3 : 2;  // planes per staged row
constexpr int kWin = 4 * kPl;       // row window: x then k, (plane, x / x + 1) pairs
constexpr int kLayers = TETMF_P1KC_LAYERS;
constexpr int kSeg = 31;   // stored columns per task (lane 0 is the halo)
constexpr int kSlots = 3;  // ring slots per warp (row issued two steps ahead)

struct CubeTask {
  int macro, x0, y0, z0;
};

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

// cube corner of local vertex i of orientation o: bit 0 x, bit 1 y, bit 2 z
__host__ __device__ constexpr int corner_of(int o, int i) {
  return orient_offset(o, i).x + 2 * orient_offset(o, i).y + 4 * orient_offset(o, i).z;
}

// The 19 cube edges (corners a < b) and, grouped by edge, the 36 incidences
// (orientation o, local vertices i, j): table entry q = K_o[i][j] / 4.
struct CubeEdgeTable {
  int ne;
  int a[19], b[19];
  int first[20];
  int o[36], i[36], j[36];
};
constexpr CubeEdgeTable make_cube_edges() {
  CubeEdgeTable t{};
  for (int o = 0; o < 6; ++o)
    for (int le = 0; le < 6; ++le) {
      const int ca = corner_of(o, local_edge_vertex(le, 0)), cb = corner_of(o, local_edge_vertex(le, 1));
      const int lo = ca < cb ? ca : cb, hi = ca < cb ? cb : ca;
      bool found = false;
      for (int e = 0; e < t.ne; ++e) found = found || (t.a[e] == lo && t.b[e] == hi);
      if (!found && t.ne < 19) {
        t.a[t.ne] = lo;
        t.b[t.ne] = hi;
        ++t.ne;
      }
    }
  int k = 0;
  for (int e = 0; e < t.ne; ++e) {
    t.first[e] = k;
    for (int o = 0; o < 6; ++o)
      for (int le = 0; le < 6; ++le) {
        const int i = local_edge_vertex(le, 0), j = local_edge_vertex(le, 1);
        const int ca = corner_of(o, i), cb = corner_of(o, j);
        if ((ca == t.a[e] && cb == t.b[e]) || (ca == t.b[e] && cb == t.a[e])) {
          // orient the incidence so that local i sits at corner a
          t.o[k] = o;
          t.i[k] = ca == t.a[e] ? i : j;
          t.j[k] = ca == t.a[e] ? j : i;
          ++k;
        }
      }
  }
  t.first[t.ne] = k;
  return t;
}
constexpr CubeEdgeTable kCE = make_cube_edges();
static_assert(kCE.ne == 19 && kCE.first[19] == 36, "the six orientations tile the cube with 19 edges");

// the kbar pair-sharing below assumes these corner sets
constexpr bool corners_are(int o, int c0, int c1, int c2, int c3) {
  int m = 0;
  for (int i = 0; i < 4; ++i) m |= 1 << corner_of(o, i);
  return m == ((1 << c0) | (1 << c1) | (1 << c2) | (1 << c3));
}
static_assert(corners_are(WU, 0, 1, 2, 4) && corners_are(WD, 3, 5, 6, 7) && corners_are(BU, 1, 2, 3, 4) &&
                  corners_are(BD, 2, 3, 4, 6) && corners_are(GU, 1, 3, 4, 5) && corners_are(GD, 3, 4, 5, 6),
              "orientation corner sets (lattice.hpp)");

__constant__ CubeEdgeTable dCE = make_cube_edges();

// table entry Q from the warp's shared copy (16-byte broadcast loads of pairs)
template <int Q>
__device__ __forceinline__ double tab_at(const double2* __restrict__ T2) {
  const double2 v = T2[Q >> 1];
  return (Q & 1) ? v.y : v.x;
}

// w of edge E's incidences Q .. L-1 (template recursion: every index is a
// compile-time constant)
template <int Q, int L>
__device__ __forceinline__ double edge_weight(const double (&kb)[6], const double2* __restrict__ T, double w) {
  constexpr int o = kCE.o[Q];
  w = fma(kb[o], tab_at<Q>(T), w);
  if constexpr (Q + 1 < L) return edge_weight<Q + 1, L>(kb, T, w);
  return w;
}

// the cube's 19 edges into its corner sums c[CO + 0 .. CO + 7]
template <int E, int CO, int NC>
__device__ __forceinline__ void cube_edges(const double (&xv)[NC], const double (&kb)[6],
                                           const double2* __restrict__ T, double (&c)[NC]) {
  constexpr int a = kCE.a[E] + CO, b = kCE.b[E] + CO, f = kCE.first[E], l = kCE.first[E + 1], of = kCE.o[f];
  double w = kb[of] * tab_at<f>(T);
  if constexpr (f + 1 < l) w = edge_weight<f + 1, l>(kb, T, w);
  const double d = xv[b] - xv[a];
  c[a] = fma(w, d, c[a]);
  c[b] = fma(-w, d, c[b]);
  if constexpr (E + 1 < 19) cube_edges<E + 1, CO, NC>(xv, kb, T, c);
}

// the six kbar of the cube with corner k values kv[CO + 0 .. CO + 7], 0 for
// the orientations outside the macro (cube coordinate sum s)
template <int CO, int NC>
__device__ __forceinline__ void cube_kbar(const double (&kv)[NC], int s, int n, double (&kb)[6]) {
  const double s34 = kv[CO + 3] + kv[CO + 4], s12 = kv[CO + 1] + kv[CO + 2], s56 = kv[CO + 5] + kv[CO + 6];
  kb[WU] = s12 + (kv[CO + 0] + kv[CO + 4]);
  kb[BU] = s34 + s12;
  kb[BD] = s34 + (kv[CO + 2] + kv[CO + 6]);
  kb[GU] = s34 + (kv[CO + 1] + kv[CO + 5]);
  kb[GD] = s34 + s56;
  kb[WD] = s56 + (kv[CO + 3] + kv[CO + 7]);
  kb[WU] = s <= n - 1 ? kb[WU] : 0.0;
  kb[BU] = s <= n - 2 ? kb[BU] : 0.0;
  kb[BD] = s <= n - 2 ? kb[BD] : 0.0;
  kb[GU] = s <= n - 2 ? kb[GU] : 0.0;
  kb[GD] = s <= n - 2 ? kb[GD] : 0.0;
  kb[WD] = s <= n - 3 ? kb[WD] : 0.0;
}

// A row window w[kWin] of one lane: x at (x, y, z), (x + 1, y, z), (x, y,
// z + 1), (x + 1, y, z + 1) [, (x, y, z + 2), (x + 1, y, z + 2)], then k at
// the same positions.
__global__ void __launch_bounds__(32 * kCWarps, TETMF_P1KC_MINB)
p1k_cube_kernel(const double* __restrict__ x, const double* __restrict__ kc, double* __restrict__ y,
                const CubeTask* __restrict__ tasks, int ntasks, i64 stride, int n,
                const P1DeviceTable* __restrict__ tabs, const MacroDesc* __restrict__ macros, int chunk) {
  __shared__ __align__(16) double sT[kCWarps][36];
  __shared__ double sP[kCWarps][kRows][32];
  __shared__ double sRing[kCWarps][kSlots][kWin][32];  // [warp][slot][window entry][lane]
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* __restrict__ P = &sP[wib][0][lane];  // this lane's column, stride 32
  const double2* __restrict__ T2 = reinterpret_cast<const double2*>(sT[wib]);
  const unsigned ring0 = su32(&sRing[wib][0][0][lane]);
  int* ctr = const_cast<int*>(reinterpret_cast<const int*>(tasks + ntasks));  // [0] next task, [1] warps done
  int slot_i = 0, slot_t = 0;  // ring slots (warp-uniform), continued across tasks
  for (;;) {
    int ti = 0;
    if (lane == 0) ti = atomicAdd(&ctr[0], 1);
    ti = __shfl_sync(0xffffffffu, ti, 0);
    if (ti >= ntasks) break;
    __syncwarp();  // the previous task's table reads are done
    const CubeTask t = tasks[ti];
    {
      const double* __restrict__ K = &tabs[macros[t.macro].group].K[0][0];
      for (int q = lane; q < 36; q += 32) sT[wib][q] = 0.25 * __ldg(K + dCE.o[q] * 10 + sym4(dCE.i[q], dCE.j[q]));
    }
#pragma unroll
    for (int r = 0; r < kRows; ++r) P[32 * r] = 0.0;
    __syncwarp();

    const int px = t.x0 - 1 + lane;
    // this lane's column in x, k and y, kept in registers (opaque to the
    // compiler, so it is not recomputed from macro * stride every step)
    const double* xl = x + static_cast<i64>(t.macro) * stride + px;
    const double* kl = kc + static_cast<i64>(t.macro) * stride + px;
    double* yl = y + static_cast<i64>(t.macro) * stride + px;
    asm volatile("" : "+l"(xl), "+l"(kl), "+l"(yl));
    const int r0 = t.y0 == 0 ? 0 : -1;  // halo row unless the chunk starts at y = 0
    const int zs = t.z0 > 0 ? t.z0 - 1 : 0, ze = min(t.z0 + chunk - 1, n);
    for (int z = zs; z <= ze;) {
      const bool two = kPair && z + 1 <= ze;
      const int rend = min(chunk - 1, n - z - t.x0 - t.y0);  // last row with a stored vertex
      if (rend < 0) break;                                  // and none in the layers above
      const bool store0 = z >= t.z0, store1 = z + 1 >= t.z0;
      int len[kPl];  // row-0 lengths of planes z, z + 1 (, z + 2)
#pragma unroll
      for (int j = 0; j < kPl; ++j) len[j] = n - z + 1 - j;
      int yy = t.y0 + r0;
      // row r of plane zz starts at plane_offset + r len - r (r - 1) / 2, so
      // row r + 1 starts len - r further
      int gi[kPl], rho_i = yy;  // next row to issue
#pragma unroll
      for (int j = 0; j < kPl; ++j)
        gi[j] = static_cast<int>(plane_offset(n, z + j)) + yy * len[j] - ((yy * (yy - 1)) >> 1);
      int a0 = gi[0], a1 = gi[1];  // (px, yy, z), (px, yy, z + 1) relative to this lane's column
      const int last = t.y0 + rend + 1;  // last row the layer reads
      // one commit group per row (empty once the layer's rows are issued):
      // the row taken is complete when at most kSlots - 2 younger groups pend
      auto issue_next = [&]() {
        if (rho_i <= last) {
          const unsigned d = ring0 + static_cast<unsigned>(slot_i) * (kWin * 32 * 8);
#pragma unroll
          for (int j = 0; j < kPl; ++j) {
            const double* sx = xl + gi[j];
            const double* sk = kl + gi[j];
            asm volatile(
                "cp.async.ca.shared.global [%0], [%2], 8;\n"
                "cp.async.ca.shared.global [%0+256], [%2+8], 8;\n"
                "cp.async.ca.shared.global [%1], [%3], 8;\n"
                "cp.async.ca.shared.global [%1+256], [%3+8], 8;\n" ::"r"(d + 512u * j),
                "r"(d + 512u * (kPl + j)), "l"(sx), "l"(sk)
                : "memory");
            gi[j] += len[j] - rho_i;
          }
          ++rho_i;
          slot_i = slot_i == kSlots - 1 ? 0 : slot_i + 1;
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
      auto take = [&](double (&w)[kWin]) {
#pragma unroll
        for (int q = 0; q < kWin; ++q) w[q] = sRing[wib][slot_t][q][lane];
        slot_t = slot_t == kSlots - 1 ? 0 : slot_t + 1;
      };
      double A[kWin], B[kWin];
#pragma unroll
      for (int q = 0; q < kSlots; ++q) issue_next();
      asm volatile("cp.async.wait_group %0;" ::"n"(kSlots - 1) : "memory");
      take(A);  // row yy
      asm volatile("cp.async.wait_group %0;" ::"n"(kSlots - 2) : "memory");
      take(B);  // row yy + 1
      // running sums of (x, y0, z) (layer z - 1 only, without a halo row no
      // step adds it) and of (x, y0, z + 1)
      double R0 = r0 == 0 ? P[0] : 0.0, R1 = 0.0, Pn = 0.0;
      // one cube row (one or two layers): lo = row yy, hi = row yy + 1; lo
      // then receives row yy + 2
      auto step = [&](auto two_c, double (&lo)[kWin], double(&hi)[kWin], int r) {
        constexpr bool TWO = decltype(two_c)::value;
        constexpr int NC = TWO ? 12 : 8;  // corners dx + 2 dy + 4 dz
        issue_next();
        double xv[NC], kv[NC];
#pragma unroll
        for (int dz = 0; dz < NC / 4; ++dz)
#pragma unroll
          for (int dx = 0; dx < 2; ++dx) {
            xv[dx + 4 * dz] = lo[2 * dz + dx], xv[dx + 2 + 4 * dz] = hi[2 * dz + dx];
            kv[dx + 4 * dz] = lo[2 * kPl + 2 * dz + dx], kv[dx + 2 + 4 * dz] = hi[2 * kPl + 2 * dz + dx];
          }
        const int s = px < 0 ? (1 << 29) : px + yy + z;  // coordinate sum of cube (px, yy, z)
        double c[NC];
#pragma unroll
        for (int q = 0; q < NC; ++q) c[q] = 0.0;
        c[0] = R0;                                     // (x, y, z): layer z - 1 and row y - 1 so far
        c[2] = r + 1 < chunk ? P[32 * (r + 1)] : 0.0;  // (x, y + 1, z): layer z - 1
        if constexpr (TWO) {
          c[4] = R1;  // (x, y, z + 1): row y - 1 so far
          c[8] = Pn;  // (x, y, z + 2): row y - 1
        } else {
          c[4] = Pn;  // (x, y, z + 1): row y - 1 of this layer
        }
        {
          double kb[6];
          cube_kbar<0>(kv, s, n, kb);
          cube_edges<0, 0>(xv, kb, T2, c);
        }
        if constexpr (TWO) {
          double kb[6];
          cube_kbar<4>(kv, s + 1, n, kb);
#if TETMF_P1KC_SPLIT
          // own accumulators for the upper cube: its plane z + 1 sums do not
          // wait for the lower cube's (two independent FMA chains per corner)
          double xu[8], u[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) xu[q] = xv[q + 4], u[q] = 0.0;
          u[4] = c[8];
          cube_edges<0, 0>(xu, kb, T2, u);
#pragma unroll
          for (int q = 0; q < 4; ++q) c[4 + q] += u[q], c[8 + q] = u[4 + q];
#else
          cube_edges<0, 4>(xv, kb, T2, c);
#endif
        }
        // x + 1 corners come from the left neighbour's cubes
        const bool mine = r >= 0 && lane >= 1;
        const double l1 = __shfl_up_sync(0xffffffffu, c[1], 1), l3 = __shfl_up_sync(0xffffffffu, c[3], 1);
        const double l5 = __shfl_up_sync(0xffffffffu, c[5], 1), l7 = __shfl_up_sync(0xffffffffu, c[7], 1);
        const double out0 = c[0] + l1;
        R0 = c[2] + l3;
        if (mine && store0 && s <= n) yl[a0] = out0;
        if constexpr (TWO) {
          const double l9 = __shfl_up_sync(0xffffffffu, c[9], 1), l11 = __shfl_up_sync(0xffffffffu, c[11], 1);
          const double out1 = c[4] + l5;
          R1 = c[6] + l7;
          if (mine && store1 && s + 1 <= n) yl[a1] = out1;
          if (r >= 0) P[32 * r] = c[8] + l9;
          Pn = c[10] + l11;
        } else {
          if (r >= 0) P[32 * r] = c[4] + l5;
          Pn = c[6] + l7;
        }
        a0 += len[0] - yy;
        a1 += len[1] - yy;
        ++yy;
        if (r < rend) {
          asm volatile("cp.async.wait_group %0;" ::"n"(kSlots - 2) : "memory");
          take(lo);  // row yy + 1 of the next step
        }
      };
      if (two) {
        for (int r = r0;;) {
          step(std::true_type{}, A, B, r);
          if (++r > rend) break;
          step(std::true_type{}, B, A, r);
          if (++r > rend) break;
        }
        z += 2;
      } else {
        for (int r = r0;;) {
          step(std::false_type{}, A, B, r);
          if (++r > rend) break;
          step(std::false_type{}, B, A, r);
          if (++r > rend) break;
        }
        z += 1;
      }
    }
  }
  if (lane == 0 && atomicAdd(&ctr[1], 1) == static_cast<int>(gridDim.x) * kCWarps - 1) {
    atomicExch(&ctr[0], 0);  // every warp has left the task loop: reset for the next launch
    atomicExch(&ctr[1], 0);
  }
}

// rows of layer z the task walks (0 if none)
int task_steps(int n, int x0, int y0, int z, int chunk) {
  const int rend = std::min(chunk - 1, n - z - x0 - y0);
  return rend < 0 ? 0 : rend - (y0 == 0 ? 0 : -1) + 1;
}

} // namespace

// one task per (macro, layer chunk, row chunk, 31-column segment) with a
// stored vertex; heaviest first (the grid's tail then holds the short tasks)
void build_p1k_cube_tasks(int nmacros, int n, std::vector<int>& out, int chunk) {
  if (chunk < 1 || chunk > kRows || chunk > kLayers) fail_internal("p1k_cube: chunk out of range");
  struct T {
    int m, x0, y0, z0;
    long cost;
  };
  std::vector<T> ts;
  for (int m = 0; m < nmacros; ++m)
    for (int z0 = 0; z0 <= n; z0 += chunk)
      for (int y0 = 0; y0 <= n - z0; y0 += chunk)
        for (int x0 = 0; x0 <= n - z0 - y0; x0 += kSeg) {
          long cost = 0;
          for (int z = z0 > 0 ? z0 - 1 : 0; z <= std::min(z0 + chunk - 1, n); ++z) cost += task_steps(n, x0, y0, z, chunk);
          ts.push_back({m, x0, y0, z0, cost});
        }
  std::stable_sort(ts.begin(), ts.end(), [](const T& a, const T& b) { return a.cost > b.cost; });
  out.clear();
  out.reserve(4 * ts.size());
  for (const T& t : ts) out.insert(out.end(), {t.m, t.x0, t.y0, t.z0});
  out.insert(out.end(), {0, 0});  // the kernel's task counters (reset by the kernel after each launch)
}

// rows = layers per task: 16 when that gives every resident warp (8 per SM)
// two tasks, 8 when that gives it one, else 4. On a small lattice the 16 x 16
// tasks are fewer than the warps of one wave and each is a serial walk of
// ~140 steps: config 2 (one macro at L7, 95 / 305 / 1087 tasks) runs 73 /
// 29 / 21 us with 16 / 8 / 4; cube6 L7 76 / 57 / 70 us; cube6 L8 265 / 306 /
// 423 us (tools/k2_chunk.py). Results differ by rounding between task sizes
// (the order a vertex's cube contributions are summed in follows the tasks).
int p1k_cube_chunk(int nmacros, int n, int sms) {
  if (const char* e = std::getenv("TETMF_P1KC_CHUNK")) {  // tuning sweeps (tools/k2_chunk.py)
    const int c = std::atoi(e);
    if (c >= 1 && c <= std::min(kRows, kLayers)) return c;
  }
  std::vector<int> t;
  int chunk = std::min(kRows, kLayers);
  while (chunk > 4) {
    build_p1k_cube_tasks(nmacros, n, t, chunk);
    if (static_cast<long long>(t.size() / 4) >= static_cast<long long>(chunk) * sms) break;
    chunk /= 2;
  }
  return chunk;
}

void launch_p1k_cube(const double* x, const double* k, double* y, const int* d_tasks, int ntasks, i64 macro_stride,
                     int n, const P1DeviceTable* d_tables, const MacroDesc* d_macros, cudaStream_t s, int chunk) {
  if (ntasks == 0) return;
  if (chunk < 1 || chunk > kRows || chunk > kLayers) fail_internal("p1k_cube: chunk out of range");
  // one wave of resident CTAs (the warps take the tasks dynamically)
  static int resident = 0;
  if (resident == 0) {
    int dev = 0, sms = 0, per_sm = 0;
    TETMF_CUDA(cudaGetDevice(&dev));
    TETMF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // registers, not the L1 / shared split, should bound the resident warps
    TETMF_CUDA(cudaFuncSetAttribute(p1k_cube_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    cudaSharedmemCarveoutMaxShared));
    TETMF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, p1k_cube_kernel, 32 * kCWarps, 0));
    resident = std::max(1, sms * per_sm);
  }
  const unsigned grid = static_cast<unsigned>(std::min((ntasks + kCWarps - 1) / kCWarps, resident));
  p1k_cube_kernel<<<grid, 32 * kCWarps, 0, s>>>(x, k, y, reinterpret_cast<const CubeTask*>(d_tasks), ntasks,
                                                macro_stride, n, d_tables, d_macros, chunk);
  check_launch("p1k_cube");
}

} // namespace tetmf

// k_n1_cubes.cu -- K3: N1 alpha curl curl + beta mass apply, cube walk.
//
// Formulation (tables.cpp): per micro element e of orientation o
//   A_e = (sum_m alpha_m) Kc_o + sum_m beta_m T_o[m]     (21 packed entries)
//   y_e = A_e x_e                                         (symmetric 6x6)
// with the ND1 signs folded into the per-orientation tables, i.e. exact
// integration of alpha, beta in P1 (264 flop / element).
//
// Work decomposition. The six micro elements anchored at a lattice point
// tile the unit cube at that point ("cubes" loop); a cube
// touches 19 edges and 8 vertices. One warp per task (macro, layer z,
// x segment): lane l processes cube x = x0 - 1 + l and the warp walks the
// rows y = 0, 1, ... of layer z. Edges are owned by the cube whose anchor is
// their componentwise minimum (lattice.hpp), so a cube contributes to the
// edges of cubes at offsets {0,1}^3:
//   * x+1 owners: warp shuffle to the next lane (lane 0 is a halo cube that
//     only feeds lane 1; it owns nothing),
//   * y+1 owners: carried in registers to the next row step,
//   * z+1 owners (the edges lying in plane z+1): written to memory.
// In-plane edges (classes 0,1,3) of plane p get contributions from layers
// p-1 and p. Layers are processed in two launches: even layers store their
// partial sums, odd layers read-modify-write them -- deterministic, no
// atomics. Vertical edges (classes 2,4,5,6) are final after their layer.
//
// Tables: the launch covers the macros of ONE geometry group; each CTA
// copies that group's N1DeviceTable (5 KB) into shared memory once. Table
// reads are warp-uniform broadcasts with compile-time offsets, kept inside
// the row loop (a compiler memory barrier per step) so the 630 invariants are
// not hoisted into -- and spilled from -- registers. (A __grid_constant__
// table was tried first: ptxas hoisted the constants and spilled them.)
// Window loads are unpredicated: level buffers carry zeroed guard regions and
// values of non-existent edges only reach elements that are skipped.
#include <cstdlib>

#include "device.hpp"
#include "runtime_check.hpp"

namespace tetmf {

namespace {

constexpr int kWarps = 4;
#ifndef TETMF_N1_MIN_BLOCKS
#define TETMF_N1_MIN_BLOCKS 3  // 3 x 4 warps per SM -> <= 170 registers
#endif
constexpr int kMinBlocks = TETMF_N1_MIN_BLOCKS;
#ifndef TETMF_N1_CHUNK
#define TETMF_N1_CHUNK 32
#endif
constexpr int kChunk = TETMF_N1_CHUNK;  // rows per task
#ifndef TETMF_N1_PREFETCH
#define TETMF_N1_PREFETCH 1
#endif
constexpr bool kPrefetch = TETMF_N1_PREFETCH != 0;

__device__ __forceinline__ void prefetch_l1(const double* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

struct N1Task {
  int macro, z, x0, y0;
};

// per-orientation tables in shared memory: [o][term][22] (16-byte aligned
// rows: K, T0..T3 of the 21 packed entries)
struct SmemTable {
  double e[6][5][22];
};

// cube edge numbering: (owner offset, class)
//  0..6: (000, c)   7: (100,1)  8: (100,2)  9: (100,5)
// 10: (010,0) 11: (010,2) 12: (010,4) 13: (110,2)
// 14: (001,0) 15: (001,1) 16: (001,3) 17: (101,1) 18: (011,0)
__host__ __device__ constexpr int cube_edge_id(int ox, int oy, int oz, int c) {
  return (ox == 0 && oy == 0 && oz == 0) ? c
         : (ox == 1 && oy == 0 && oz == 0) ? (c == 1 ? 7 : c == 2 ? 8 : 9)
         : (ox == 0 && oy == 1 && oz == 0) ? (c == 0 ? 10 : c == 2 ? 11 : 12)
         : (ox == 1 && oy == 1 && oz == 0) ? 13
         : (ox == 0 && oy == 0 && oz == 1) ? (c == 0 ? 14 : c == 1 ? 15 : 16)
         : (ox == 1 && oy == 0 && oz == 1) ? 17
                                           : 18;
}

__host__ __device__ constexpr int cube_edge(int o, int le) {
  // local edge (a,b) of orientation o -> cube edge id (lattice.hpp conventions)
  return cube_edge_id(local_edge_ref(o, le).ax, local_edge_ref(o, le).ay, local_edge_ref(o, le).az,
                      local_edge_ref(o, le).cls);
}

__host__ __device__ constexpr int cube_vertex(int o, int i) {
  return orient_offset(o, i).x + 2 * orient_offset(o, i).y + 4 * orient_offset(o, i).z;
}

// one element: Y[cube edges] += A_e x_e
template <int O, typename TB>
__device__ __forceinline__ void element(const TB& tb, const double (&X)[19], const double (&al)[8],
                                        const double (&be)[8], double (&Y)[19]) {
  constexpr int v0 = cube_vertex(O, 0), v1 = cube_vertex(O, 1), v2 = cube_vertex(O, 2), v3 = cube_vertex(O, 3);
  const double sa = (al[v0] + al[v1]) + (al[v2] + al[v3]);
  const double b0 = be[v0], b1 = be[v1], b2 = be[v2], b3 = be[v3];
  double xe[6], ye[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) xe[i] = X[cube_edge(O, i)];
  const double* __restrict__ K = tb.e[O][0];
  const double* __restrict__ T0 = tb.e[O][1];
  const double* __restrict__ T1 = tb.e[O][2];
  const double* __restrict__ T2 = tb.e[O][3];
  const double* __restrict__ T3 = tb.e[O][4];
#pragma unroll
  for (int i = 0; i < 6; ++i) ye[i] = 0.0;
#pragma unroll
  for (int i = 0; i < 6; ++i) {
#pragma unroll
    for (int j = i; j < 6; ++j) {
      const int q = sym6(i, j);
      double a = sa * K[q];
      a = fma(b0, T0[q], a);
      a = fma(b1, T1[q], a);
      a = fma(b2, T2[q], a);
      a = fma(b3, T3[q], a);
      ye[i] = fma(a, xe[j], ye[i]);
      if (j != i) ye[j] = fma(a, xe[i], ye[j]);
    }
  }
#pragma unroll
  for (int i = 0; i < 6; ++i) Y[cube_edge(O, i)] += ye[i];
}

// Gram-form element (tables.hpp N1GramTable): 31 table values instead of 105
template <int O>
__device__ __forceinline__ void element_gram(const double* __restrict__ tb, const double (&X)[19],
                                             const double (&al)[8], const double (&be)[8], double (&Y)[19],
                                             bool valid) {
  constexpr int v0 = cube_vertex(O, 0), v1 = cube_vertex(O, 1), v2 = cube_vertex(O, 2), v3 = cube_vertex(O, 3);
  // invalid element: all coefficients 0 -> A_e = 0 (inputs are finite)
  const double sa = valid ? (al[v0] + al[v1]) + (al[v2] + al[v3]) : 0.0;
  const double bv[4] = {valid ? be[v0] : 0.0, valid ? be[v1] : 0.0, valid ? be[v2] : 0.0, valid ? be[v3] : 0.0};
  const double S = (bv[0] + bv[1]) + (bv[2] + bv[3]);
  const double S2 = S + S;
  double Bt[4][4];
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const double u = S + bv[p];
#pragma unroll
    for (int q = p + 1; q < 4; ++q) Bt[p][q] = Bt[q][p] = u + bv[q];
    Bt[p][p] = fma(4.0, bv[p], S2);
  }
  // A_e x_e accumulated straight into the cube accumulators Y
#pragma unroll
  for (int i = 0; i < 6; ++i) {
#pragma unroll
    for (int j = i; j < 6; ++j) {
      const int a = local_edge_vertex(i, 0), b = local_edge_vertex(i, 1);
      const int c = local_edge_vertex(j, 0), d = local_edge_vertex(j, 1);
      const bool neg = local_edge_ref(O, i).flipped != local_edge_ref(O, j).flipped;
      double m = Bt[a][c] * tb[22 + sym4(b, d)];
      m = fma(-Bt[a][d], tb[22 + sym4(b, c)], m);
      m = fma(-Bt[b][c], tb[22 + sym4(a, d)], m);
      m = fma(Bt[b][d], tb[22 + sym4(a, c)], m);
      const double aij = fma(sa, tb[sym6(i, j)], neg ? -m : m);
      Y[cube_edge(O, i)] = fma(aij, X[cube_edge(O, j)], Y[cube_edge(O, i)]);
      if (j != i) Y[cube_edge(O, j)] = fma(aij, X[cube_edge(O, i)], Y[cube_edge(O, j)]);
    }
  }
}

template <int PASS, int MODE>
__global__ void __launch_bounds__(32 * kWarps, kMinBlocks)
n1_cubes_kernel(const N1GramTable* __restrict__ gram, const N1DeviceTable* __restrict__ table,
                const double* __restrict__ xin,
                const double* __restrict__ alpha, const double* __restrict__ beta, double* __restrict__ yout,
                const N1Task* __restrict__ tasks, int ntasks, i64 stride, i64 cstride, i64 cf_stride, int n) {
  __shared__ __align__(16) SmemTable st;
  __shared__ __align__(16) N1GramTable sg;
  if (MODE == 0) {
    for (int i = threadIdx.x; i < 6 * 5 * 21; i += blockDim.x)
      st.e[i / 105][(i / 21) % 5][i % 21] = __ldg(&table->e[0][0][0] + i);
  } else {
    for (int i = threadIdx.x; i < 6 * 32; i += blockDim.x) sg.o[i / 32][i % 32] = __ldg(&gram->o[0][0] + i);
  }
  __syncthreads();
  const int warp = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (warp >= ntasks) return;
  const int lane = threadIdx.x & 31;
  const N1Task t = tasks[warp];
  const int z = t.z;
  const int cx = t.x0 - 1 + lane;  // cube anchor x of this lane (lane 0: halo)
  const bool owner = lane > 0;
  const int m = n - 1;             // extent of the edge-anchor lattice
  const double* __restrict__ X = xin + static_cast<i64>(t.macro) * stride + cx;
  double* __restrict__ Yo = yout + static_cast<i64>(t.macro) * stride + cx;
  const double* __restrict__ A = alpha + static_cast<i64>(t.macro) * cf_stride + cx;
  const double* __restrict__ B = beta + static_cast<i64>(t.macro) * cf_stride + cx;
  const int cs = static_cast<int>(cstride);

  // The task covers rows [y0, y0 + kChunk) of the layer; a task with y0 > 0
  // first recomputes cube row y0 - 1 (halo step, no stores) to obtain the
  // partial sums its row-y0 owners receive from that row.
  const int y0 = t.y0;
  const int ys = y0 > 0 ? y0 - 1 : 0;
  const int ymax = min(n - 1 - z - t.x0, y0 + kChunk - 1);  // lane 1 (x = x0) has a cube
  // row starts (offset of x = 0) of row ys in the edge lattice (planes z,
  // z+1) and in the vertex lattice (coefficients, planes z, z+1)
  int ez = static_cast<int>(plane_offset(m, z) + row_offset(m, z, ys));
  int eu = static_cast<int>(plane_offset(m, z + 1) + row_offset(m, z + 1, ys));
  int vz = static_cast<int>(plane_offset(n, z) + row_offset(n, z, ys));
  int vu = static_cast<int>(plane_offset(n, z + 1) + row_offset(n, z + 1, ys));
  int elen = m - z + 1 - ys;  // edge-lattice row length in plane z
  int vlen = n - z + 1 - ys;  // vertex-lattice row length in plane z

  // carried state: layer-z partial sums for row-y owners from cube row y-1
  // (the edge / coefficient windows are re-read each step; the values of
  // row y+1 are L1 hits by then and the kernel is FP64-bound)
  double c0 = 0.0, c2 = 0.0, c4 = 0.0, cT0 = 0.0;

  for (int yy = ys; yy <= ymax; ++yy) {
    // keep the table reads inside the loop (no hoisting of 630 invariants
    // into registers): they are warp-uniform shared-memory broadcasts
    asm volatile("" ::: "memory");
    const int ez1 = ez + elen, eu1 = eu + elen - 1;   // edge rows y+1 (plane z), y+1 (plane z+1)
    const int vz1 = vz + vlen, vu1 = vu + vlen - 1;   // vertex rows y+1
    if (kPrefetch && yy < ymax) {
      // warm L1 with the rows the next step loads first (y+2 rows of planes
      // z, z+1): no registers, no scoreboard, the lines land during this
      // step's arithmetic
      const int ez2 = ez1 + elen - 1, eu2 = eu1 + elen - 2;
      const int vz2 = vz1 + vlen - 1, vu2 = vu1 + vlen - 2;
      prefetch_l1(X + ez1);
      prefetch_l1(X + cs + ez1);
      prefetch_l1(X + 3 * cs + ez1);
      prefetch_l1(X + 5 * cs + ez1);
      prefetch_l1(X + 6 * cs + ez1);
      prefetch_l1(X + ez2);
      prefetch_l1(X + 2 * cs + ez2);
      prefetch_l1(X + 4 * cs + ez2);
      prefetch_l1(X + cs + eu1);
      prefetch_l1(X + 3 * cs + eu1);
      prefetch_l1(X + eu2);
      prefetch_l1(A + vz2);
      prefetch_l1(A + vu2);
      prefetch_l1(B + vz2);
      prefetch_l1(B + vu2);
      if (PASS == 1) {  // the in-plane partial sums the next step updates
        prefetch_l1(Yo + ez1);
        prefetch_l1(Yo + cs + ez1);
        prefetch_l1(Yo + 3 * cs + ez1);
        prefetch_l1(Yo + eu1);
        prefetch_l1(Yo + cs + eu1);
        prefetch_l1(Yo + 3 * cs + eu1);
      }
    }
    double Xc[19];
    Xc[0] = __ldg(X + ez);
    Xc[1] = __ldg(X + cs + ez);
    Xc[2] = __ldg(X + 2 * cs + ez);
    Xc[3] = __ldg(X + 3 * cs + ez);
    Xc[4] = __ldg(X + 4 * cs + ez);
    Xc[5] = __ldg(X + 5 * cs + ez);
    Xc[6] = __ldg(X + 6 * cs + ez);
    Xc[7] = __ldg(X + cs + ez + 1);
    Xc[8] = __ldg(X + 2 * cs + ez + 1);
    Xc[9] = __ldg(X + 5 * cs + ez + 1);
    Xc[10] = __ldg(X + ez1);
    Xc[11] = __ldg(X + 2 * cs + ez1);
    Xc[12] = __ldg(X + 4 * cs + ez1);
    Xc[13] = __ldg(X + 2 * cs + ez1 + 1);
    Xc[14] = __ldg(X + eu);
    Xc[15] = __ldg(X + cs + eu);
    Xc[16] = __ldg(X + 3 * cs + eu);
    Xc[17] = __ldg(X + cs + eu + 1);
    Xc[18] = __ldg(X + eu1);
    double al[8], be[8];
    al[0] = __ldg(A + vz); al[1] = __ldg(A + vz + 1); al[4] = __ldg(A + vu); al[5] = __ldg(A + vu + 1);
    be[0] = __ldg(B + vz); be[1] = __ldg(B + vz + 1); be[4] = __ldg(B + vu); be[5] = __ldg(B + vu + 1);
    al[2] = __ldg(A + vz1); al[3] = __ldg(A + vz1 + 1); al[6] = __ldg(A + vu1); al[7] = __ldg(A + vu1 + 1);
    be[2] = __ldg(B + vz1); be[3] = __ldg(B + vz1 + 1); be[6] = __ldg(B + vu1); be[7] = __ldg(B + vu1 + 1);

    double Y[19];
#pragma unroll
    for (int k = 0; k < 19; ++k) Y[k] = 0.0;
    const int s = cx + yy + z;
    if (MODE == 1) {
      // one branch-free path: an element outside the macro (partial cubes at
      // the row end, the halo cube x = -1 of an x0 = 0 task) gets zero
      // coefficients, so its (finite, guard-region) inputs contribute 0
      const bool in = cx >= 0;
      const bool vWU = in && s <= n - 1, vMid = in && s <= n - 2, vWD = in && s <= n - 3;
      element_gram<WU>(sg.o[WU], Xc, al, be, Y, vWU);
      element_gram<BU>(sg.o[BU], Xc, al, be, Y, vMid);
      element_gram<BD>(sg.o[BD], Xc, al, be, Y, vMid);
      element_gram<GU>(sg.o[GU], Xc, al, be, Y, vMid);
      element_gram<GD>(sg.o[GD], Xc, al, be, Y, vMid);
      element_gram<WD>(sg.o[WD], Xc, al, be, Y, vWD);
    } else if (cx >= 0) {
      if (MODE == 0) {
        if (s <= n - 1) element<WU>(st, Xc, al, be, Y);
        if (s <= n - 2) {
          element<BU>(st, Xc, al, be, Y);
          element<BD>(st, Xc, al, be, Y);
          element<GU>(st, Xc, al, be, Y);
          element<GD>(st, Xc, al, be, Y);
        }
        if (s <= n - 3) element<WD>(st, Xc, al, be, Y);
      }
    }
    // x+1 owners: from lane l to lane l+1
    double r7 = __shfl_up_sync(0xffffffffu, Y[7], 1);
    double r8 = __shfl_up_sync(0xffffffffu, Y[8], 1);
    double r9 = __shfl_up_sync(0xffffffffu, Y[9], 1);
    double r13 = __shfl_up_sync(0xffffffffu, Y[13], 1);
    double r17 = __shfl_up_sync(0xffffffffu, Y[17], 1);
    if (!owner) r7 = r8 = r9 = r13 = r17 = 0.0;

    // owners of row y: plane z (all classes) and plane z+1 (in-plane classes)
    if (owner && s <= n - 1 && yy >= y0) {
      double* __restrict__ yz = Yo + ez;
      yz[2 * cs] = Y[2] + c2 + r8;
      yz[4 * cs] = Y[4] + c4;
      yz[5 * cs] = Y[5] + r9;
      if (s <= n - 2) yz[6 * cs] = Y[6];
      const double f0 = Y[0] + c0, f1 = Y[1] + r7, f3 = Y[3];
      if (PASS == 0) {
        yz[0] = f0;
        yz[cs] = f1;
        yz[3 * cs] = f3;
      } else {
        yz[0] += f0;
        yz[cs] += f1;
        yz[3 * cs] += f3;
      }
      if (s <= n - 2) {
        double* __restrict__ yu = Yo + eu;
        const double g0 = Y[14] + cT0, g1 = Y[15] + r17, g3 = Y[16];
        if (PASS == 0) {
          yu[0] = g0;
          yu[cs] = g1;
          yu[3 * cs] = g3;
        } else {
          yu[0] += g0;
          yu[cs] += g1;
          yu[3 * cs] += g3;
        }
      }
    }
    // carry the partial sums of row y+1 owners
    c0 = Y[10];
    c2 = Y[11] + r13;
    c4 = Y[12];
    cT0 = Y[18];
    ez = ez1;
    eu = eu1;
    vz = vz1;
    vu = vu1;
    --elen;
    --vlen;
  }
}

} // namespace

// Task lists of one level, per parity pass: (macro, z, x0, y0) with x0
// stepping by 31 (lane 0 of every warp is a halo cube) and row chunks of
// kChunk rows (bounded critical path: the longest task is kChunk + 1 steps).
void build_n1_tasks(const std::vector<int>& local_macros, int n, int parity, std::vector<int>& out) {
  out.clear();
  for (int z = parity; z <= n - 1; z += 2)
    for (int x0 = 0; x0 <= n - 1 - z; x0 += 31)
      for (int y0 = 0; y0 <= n - 1 - z - x0; y0 += kChunk)
        for (int li : local_macros) {
          out.push_back(li);
          out.push_back(z);
          out.push_back(x0);
          out.push_back(y0);
        }
}

void launch_n1_cubes_v2(const N1DeviceTable* table, const N1GramTable* gram, int pass, const double* x,
                        const double* alpha, const double* beta, double* y, const int* d_tasks, int ntasks,
                        i64 macro_stride, i64 class_stride, i64 coeff_stride, int n, cudaStream_t s) {
  if (ntasks == 0) return;
  const unsigned grid = static_cast<unsigned>((ntasks + kWarps - 1) / kWarps);
  const auto* tk = reinterpret_cast<const N1Task*>(d_tasks);
  // table form: 1 = Gram (default, 31 shared-memory values per element);
  // 0 = assembled T tables (105 values per element; saturates L1 at 87%).
  // A kernel-parameter constant-bank variant measured 3.3x slower (ptxas
  // either hoists and spills the constants or emits an indexed LDC each).
  static const int mode = [] {
    const char* e = std::getenv("TETMF_N1_TABLE");
    return e ? std::atoi(e) : 1;
  }();
  auto go = [&](auto kern) {
    kern<<<grid, 32 * kWarps, 0, s>>>(gram, table, x, alpha, beta, y, tk, ntasks, macro_stride, class_stride,
                                      coeff_stride, n);
  };
  if (mode == 1)
    pass == 0 ? go(n1_cubes_kernel<0, 1>) : go(n1_cubes_kernel<1, 1>);
  else
    pass == 0 ? go(n1_cubes_kernel<0, 0>) : go(n1_cubes_kernel<1, 0>);
  check_launch("n1_cubes");
}

} // namespace tetmf

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
#include "n1_common.cuh"
#include "runtime_check.hpp"

namespace tetmf {

namespace {

using namespace n1;

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

struct N1Task {
  int macro, z, x0, y0;
};

// per-orientation tables in shared memory: [o][term][22] (16-byte aligned
// rows: K, T0..T3 of the 21 packed entries)
struct SmemTable {
  double e[6][5][22];
};

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

// MODE 1 input accessor: the cube's inputs loaded into registers
struct RegIn {
  const double (&X)[19];
  const double (&al)[8];
  const double (&be)[8];
  template <int K>
  __device__ __forceinline__ double x() const { return X[K]; }
  template <int V, int W>
  __device__ __forceinline__ double c() const { return W ? be[V] : al[V]; }
};

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
    for (int i = threadIdx.x; i < 6 * kGramRow; i += blockDim.x) (&sg.o[0][0])[i] = __ldg(&gram->o[0][0] + i);
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
      cube_elements(SmemTabs{sg}, RegIn{Xc, al, be}, Y, vWU, vMid, vWD);
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

// ---------------------------------------------------------------------------
// MODE 2: shared-memory row ring. Same tasks, traversal, element formula and
// write-back as n1_cubes_kernel<PASS, 1>; only the input path differs. Each
// warp keeps the rows y, y+1, y+2 of the 14 input arrays it reads
//   0..6  X plane z, classes 0..6        7..9  X plane z+1, classes 0, 1, 3
//   10/11 alpha planes z / z+1           12/13 beta planes z / z+1
// in a 3-slot ring (33 values per row: the warp's 32 columns + 1). At step y
// the warp issues cp.async copies of row y+2 and waits for row y+1: no global
// load latency on the arithmetic path, and the element code reads its inputs
// from shared memory where it uses them (lower register pressure -> 4 CTAs
// per SM). Only rows <= ymax + 1 are copied -- the rows MODE 1 reads -- so
// every address is one MODE 1 reads and the results are bit-identical.
constexpr int kRingArrays = 14;
constexpr int kRingRow = 34;                            // doubles per ring row
constexpr int kRingSlot = kRingArrays * kRingRow;       // one row of all arrays
constexpr int kRingWarp = 3 * kRingSlot;                // doubles per warp
#ifndef TETMF_N1R_MIN_BLOCKS
#define TETMF_N1R_MIN_BLOCKS 3  // 168 registers, no spills (4 -> 128 + spills: slower)
#endif

// ring position (array, row +0/+1, column +0/+1) of cube edge k
__host__ __device__ constexpr int ring_edge_array(int k) {
  return k <= 6 ? k : k == 7 ? 1 : k == 8 ? 2 : k == 9 ? 5 : k == 10 ? 0 : k == 11 ? 2 : k == 12 ? 4
       : k == 13 ? 2 : k == 14 ? 7 : k == 15 ? 8 : k == 16 ? 9 : k == 17 ? 8 : 7;
}
__host__ __device__ constexpr int ring_edge_row(int k) { return (k >= 10 && k <= 13) || k == 18 ? 1 : 0; }
__host__ __device__ constexpr int ring_edge_col(int k) {
  return k == 7 || k == 8 || k == 9 || k == 13 || k == 17 ? 1 : 0;
}

// MODE 2 input accessor: rows y (r0) and y+1 (r1) of the warp's ring
struct RingIn {
  const double* r0;
  const double* r1;
  template <int K>
  __device__ __forceinline__ double x() const {
    return lds((ring_edge_row(K) ? r1 : r0) + ring_edge_array(K) * kRingRow + ring_edge_col(K));
  }
  // coefficient at cube vertex v (bit 0 x, bit 1 y, bit 2 z); W 0 alpha, 1 beta
  template <int V, int W>
  __device__ __forceinline__ double c() const {
    return lds((((V >> 1) & 1) ? r1 : r0) + (10 + 2 * W + (V >> 2)) * kRingRow + (V & 1));
  }
};

template <int PASS>
__global__ void __launch_bounds__(32 * kWarps, TETMF_N1R_MIN_BLOCKS)
n1_ring_kernel(const N1GramTable* __restrict__ gram, const double* __restrict__ xin,
               const double* __restrict__ alpha, const double* __restrict__ beta, double* __restrict__ yout,
               const N1Task* __restrict__ tasks, int ntasks, i64 stride, i64 cstride, i64 cf_stride, int n) {
  extern __shared__ __align__(16) double dsm[];
  N1GramTable& sg = *reinterpret_cast<N1GramTable*>(dsm);
  for (int i = threadIdx.x; i < 6 * kGramRow; i += blockDim.x) (&sg.o[0][0])[i] = __ldg(&gram->o[0][0] + i);
  __syncthreads();
  const int warp = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (warp >= ntasks) return;
  const int lane = threadIdx.x & 31;
  double* ring = dsm + sizeof(N1GramTable) / sizeof(double) + (threadIdx.x >> 5) * kRingWarp;
  const N1Task t = tasks[warp];
  const int z = t.z;
  const int cx = t.x0 - 1 + lane;
  const bool owner = lane > 0;
  const int m = n - 1;
  const double* __restrict__ X = xin + static_cast<i64>(t.macro) * stride + cx;
  double* __restrict__ Yo = yout + static_cast<i64>(t.macro) * stride + cx;
  const double* __restrict__ A = alpha + static_cast<i64>(t.macro) * cf_stride + cx;
  const double* __restrict__ B = beta + static_cast<i64>(t.macro) * cf_stride + cx;
  const int cs = static_cast<int>(cstride);

  const int y0 = t.y0;
  const int ys = y0 > 0 ? y0 - 1 : 0;
  const int ymax = min(n - 1 - z - t.x0, y0 + kChunk - 1);
  int ez = static_cast<int>(plane_offset(m, z) + row_offset(m, z, ys));
  int eu = static_cast<int>(plane_offset(m, z + 1) + row_offset(m, z + 1, ys));
  int elen = m - z + 1 - ys;

  // copy cursor: row rc of every array into ring slot rc % 3
  int rc = ys, cslot = 0;
  int cez = ez, ceu = eu, celen = elen;
  int cvz = static_cast<int>(plane_offset(n, z) + row_offset(n, z, ys));
  int cvu = static_cast<int>(plane_offset(n, z + 1) + row_offset(n, z + 1, ys));
  int cvlen = n - z + 1 - ys;
  auto copy_row = [&]() {
    double* d = ring + cslot * kRingSlot + lane;
#pragma unroll
    for (int c = 0; c < 7; ++c) cp_async8(d + c * kRingRow, X + c * cs + cez);
    cp_async8(d + 7 * kRingRow, X + ceu);
    cp_async8(d + 8 * kRingRow, X + cs + ceu);
    cp_async8(d + 9 * kRingRow, X + 3 * cs + ceu);
    cp_async8(d + 10 * kRingRow, A + cvz);
    cp_async8(d + 11 * kRingRow, A + cvu);
    cp_async8(d + 12 * kRingRow, B + cvz);
    cp_async8(d + 13 * kRingRow, B + cvu);
    if (lane == 31) {  // column +1 of the arrays read at x+1
      cp_async8(d + 1 * kRingRow + 1, X + cs + cez + 1);
      cp_async8(d + 2 * kRingRow + 1, X + 2 * cs + cez + 1);
      cp_async8(d + 5 * kRingRow + 1, X + 5 * cs + cez + 1);
      cp_async8(d + 8 * kRingRow + 1, X + cs + ceu + 1);
      cp_async8(d + 10 * kRingRow + 1, A + cvz + 1);
      cp_async8(d + 11 * kRingRow + 1, A + cvu + 1);
      cp_async8(d + 12 * kRingRow + 1, B + cvz + 1);
      cp_async8(d + 13 * kRingRow + 1, B + cvu + 1);
    }
    ++rc;
    cslot = cslot == 2 ? 0 : cslot + 1;
    cez += celen;
    ceu += celen - 1;
    cvz += cvlen;
    cvu += cvlen - 1;
    --celen;
    --cvlen;
  };
  copy_row();  // row ys
  cp_async_commit();
  copy_row();  // row ys + 1 (<= ymax + 1)
  cp_async_commit();

  double c0 = 0.0, c2 = 0.0, c4 = 0.0, cT0 = 0.0;
  int sy = 0;  // ring slot of row yy
  for (int yy = ys; yy <= ymax; ++yy) {
    asm volatile("" ::: "memory");
    if (rc <= ymax + 1) copy_row();  // row yy + 2
    cp_async_commit();
    if (PASS == 1 && yy < ymax) {  // the in-plane partial sums the next step updates
      const int ez1 = ez + elen, eu1 = eu + elen - 1;
      prefetch_l1(Yo + ez1);
      prefetch_l1(Yo + cs + ez1);
      prefetch_l1(Yo + 3 * cs + ez1);
      prefetch_l1(Yo + eu1);
      prefetch_l1(Yo + cs + eu1);
      prefetch_l1(Yo + 3 * cs + eu1);
    }
    cp_async_wait1();  // rows yy, yy + 1 have landed (this lane's copies)
    __syncwarp();      // ... and every lane's
    const double* r0 = ring + sy * kRingSlot + lane;
    const double* r1 = ring + (sy == 2 ? 0 : sy + 1) * kRingSlot + lane;

    double Y[19];
#pragma unroll
    for (int k = 0; k < 19; ++k) Y[k] = 0.0;
    const int s = cx + yy + z;
    const bool in = cx >= 0;
    const bool vWU = in && s <= n - 1, vMid = in && s <= n - 2, vWD = in && s <= n - 3;
    cube_elements(SmemTabs{sg}, RingIn{r0, r1}, Y, vWU, vMid, vWD);
    __syncwarp();  // ring slot sy is refilled by the next step's copies

    double r7 = __shfl_up_sync(0xffffffffu, Y[7], 1);
    double r8 = __shfl_up_sync(0xffffffffu, Y[8], 1);
    double r9 = __shfl_up_sync(0xffffffffu, Y[9], 1);
    double r13 = __shfl_up_sync(0xffffffffu, Y[13], 1);
    double r17 = __shfl_up_sync(0xffffffffu, Y[17], 1);
    if (!owner) r7 = r8 = r9 = r13 = r17 = 0.0;

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
    c0 = Y[10];
    c2 = Y[11] + r13;
    c4 = Y[12];
    cT0 = Y[18];
    ez += elen;
    eu += elen - 1;
    --elen;
    sy = sy == 2 ? 0 : sy + 1;
  }
}

} // namespace

// Task lists of one level, per parity pass: (macro, z, x0, y0) with x0
// stepping by 31 (lane 0 of every warp is a halo cube) and row chunks of
// kChunk rows (bounded critical path: the longest task is kChunk + 1 steps).
int n1_kernel_mode() {
  static const int mode = [] {
    const char* e = std::getenv("TETMF_N1_TABLE");
    return e ? std::atoi(e) : 3;
  }();
  return mode;
}

void build_n1_tasks(const std::vector<int>& local_macros, int n, int parity, std::vector<int>& out) {
  if (n1_kernel_mode() == 3) return build_n1_fold_tasks(local_macros, n, parity, out);
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
  const int mode = n1_kernel_mode();
  if (mode == 3) fail_internal("n1 fold kernel: launched per pass by the runtime (launch_n1_fold)");
  auto go = [&](auto kern) {
    kern<<<grid, 32 * kWarps, 0, s>>>(gram, table, x, alpha, beta, y, tk, ntasks, macro_stride, class_stride,
                                      coeff_stride, n);
  };
  if (mode == 2) {
    constexpr int smem = static_cast<int>(sizeof(N1GramTable) + sizeof(double) * kRingWarp * kWarps);
    static const bool attr = [] {
      cudaFuncSetAttribute(n1_ring_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(n1_ring_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      return true;
    }();
    (void)attr;
    auto kern = pass == 0 ? n1_ring_kernel<0> : n1_ring_kernel<1>;
    kern<<<grid, 32 * kWarps, smem, s>>>(gram, x, alpha, beta, y, tk, ntasks, macro_stride, class_stride,
                                         coeff_stride, n);
  } else if (mode == 1)
    pass == 0 ? go(n1_cubes_kernel<0, 1>) : go(n1_cubes_kernel<1, 1>);
  else
    pass == 0 ? go(n1_cubes_kernel<0, 0>) : go(n1_cubes_kernel<1, 0>);
  check_launch("n1_cubes");
}

} // namespace tetmf

// k_n1_fold.cu -- K3 (default): N1 alpha curl curl + beta apply, cube walk
// with folded lane columns.
//
// Same element formula (n1_common.cuh element_gram), edge ownership, parity
// passes and write-back rules as the round-1 segment walk (removed in round 2,
// git history: k_n1_cubes.cu); what changes is which cube a
// lane processes at each step, so that no lane idles at the row ends.
//
// Layer z holds the cubes x + y <= L = n-1-z. In the segment walk a warp owns a
// 31-column segment and walks y upward; column x ends at y = L - x, so the
// lanes of a segment go idle one by one (a 31x31/2 triangle per segment, 16 %
// of all lane-steps at L8). Here the layer's K full segments S_k = [31k,
// 31k+30] are paired, S_k with S_{K-1-k}, and lane l walks
//   phase 1: near column x0-1+l of S_k upward (rows 0 .. L-x),
//   one bubble step,
//   phase 2: far column 31(K-1-k)+30-l of S_{K-1-k} DOWNWARD (reversed lane
//            order), from its top row to row 0, then one flush step.
// Near and far column lengths add up to the same number for every lane, so
// the pair finishes in 2L + 6 - 31K steps with every lane busy; all phase-1
// lanes sit on row t and all phase-2 lanes on row D - t (D = 2L + 4 - 31K),
// so loads stay coalesced per phase group. Lane 0 is the halo column of the
// near segment, lane 31 the halo column of the far one. The middle segment of
// an odd K and the partial last segment are walked alone. 89 % of lane-steps
// are useful at L8 (80 % before; chunk halos and halo lanes are the rest).
//
// Phase 2 walks rows downward, so the edges a cube owns that also receive
// contributions from the cube BELOW it -- classes 0, 2, 4 of plane z and
// class 0 of plane z+1 -- are written one step late (after the next cube of
// the column has added its share); the other six owned edges are final when
// the cube is done. x-1 neighbours are lane-1 in phase 1 and lane+1 in
// phase 2 (shuffle source per lane).
//
// Inputs: a per-warp shared-memory ring of 3 row slots x 14 arrays x 34
// positions, filled with cp.async one step ahead. Lane l copies its column
// into position l+1; its x+1 values are its neighbour's position -- l+2 in
// phase 1, l in phase 2 -- and the boundary lane of each phase (31 / 0) also
// copies column + 1 into position 33 / 0. The copy made at step t goes to
// slot t mod 3 for every lane, so phase 1 reads rows y, y+1 from slots t+1,
// t+2 and phase 2 from t+2, t+1. At a lane's phase switch its neighbour's
// slot may hold the other phase's row; that only happens for values the top
// cube of a column (one element, WU) does not use, and stale slots hold
// zeros or older finite values, which only reach zero-coefficient elements.
// Copied addresses are the ones the segment walk read.
//
// Pass 1 (odd layers) adds to in-plane partial sums written by pass 0; those
// six values per cube are staged by cp.async one step ahead as well (one slot
// per lane, filled at the end of the previous step), so the read-modify-write
// costs no load latency.
#include <cstdlib>

#include "device.hpp"
#include "n1_common.cuh"
#include "runtime_check.hpp"

namespace tetmf {

namespace {

using namespace n1;

#ifndef TETMF_N1F_WARPS
#define TETMF_N1F_WARPS 4  // warps per CTA
#endif
constexpr int kWarps = TETMF_N1F_WARPS;
#ifndef TETMF_N1F_MIN_BLOCKS
#define TETMF_N1F_MIN_BLOCKS 3
#endif
#ifndef TETMF_N1F_STAGE_RMW
#define TETMF_N1F_STAGE_RMW 1  // pass 1: stage the partial sums by cp.async (0: read-modify-write)
#endif
// measurement builds only (results are wrong): no input copies / no stores
#ifndef TETMF_N1F_NOCOPY
#define TETMF_N1F_NOCOPY 0
#endif
#ifndef TETMF_N1F_NOSTORE
#define TETMF_N1F_NOSTORE 0
#endif
#ifndef TETMF_N1F_CHUNK
#define TETMF_N1F_CHUNK 32
#endif
constexpr int kChunk = TETMF_N1F_CHUNK;  // steps per task (+1 halo step)
constexpr int kSeg = 31;                 // owner columns per segment
constexpr int kArrays = 14;              // input arrays per row
constexpr int kRow = 34;                 // positions per array row
constexpr int kSlot = kArrays * kRow;    // doubles per ring slot
constexpr int kRing = 3 * kSlot;         // input ring, doubles per warp
constexpr int kRmw = 6 * 32;             // pass-1 staging slot, doubles per warp
constexpr int kWarpSmem = kRing + kRmw;
constexpr int kZeroTab = 6 * kGramRow + 8;         // doubles: zero table offset (+64 B bank phase)
constexpr int kTabs = kZeroTab + 6 * kGramRow + 8;  // doubles before the warps' rings
static_assert(sizeof(N1GramTable) == 6 * kGramRow * sizeof(double), "table layout");

struct FoldTask {
  int macro, z, k, t0;  // layer, near segment, first step of the chunk
};

// ring arrays: 0..6 X plane z classes 0..6; 7, 8, 9 X plane z+1 classes
// 0, 1, 3; 10, 11 alpha planes z, z+1; 12, 13 beta planes z, z+1
__host__ __device__ constexpr int edge_array(int k) {
  return k <= 6 ? k : k == 7 ? 1 : k == 8 ? 2 : k == 9 ? 5 : k == 10 ? 0 : k == 11 ? 2 : k == 12 ? 4
       : k == 13 ? 2 : k == 14 ? 7 : k == 15 ? 8 : k == 16 ? 9 : k == 17 ? 8 : 7;
}
__host__ __device__ constexpr bool edge_row1(int k) { return (k >= 10 && k <= 13) || k == 18; }
__host__ __device__ constexpr bool edge_plus1(int k) { return k == 7 || k == 8 || k == 9 || k == 13 || k == 17; }

struct FoldIn {
  const double* r0;  // own position, row y
  const double* r1;  // own position, row y + 1
  const double* q0;  // x+1 neighbour position, row y
  const double* q1;  // x+1 neighbour position, row y + 1
  template <int K>
  __device__ __forceinline__ double x() const {
    const double* p = edge_plus1(K) ? (edge_row1(K) ? q1 : q0) : (edge_row1(K) ? r1 : r0);
    return lds(p + edge_array(K) * kRow);
  }
  template <int V, int W>
  __device__ __forceinline__ double c() const {
    constexpr int a = 10 + 2 * W + (V >> 2);
    const double* p = (V & 1) ? (((V >> 1) & 1) ? q1 : q0) : (((V >> 1) & 1) ? r1 : r0);
    return lds(p + a * kRow);
  }
};

// The group's Gram table is staged in shared memory; one launch per pass
// covers all geometry groups.
template <int PASS, int RULE>
__global__ void __launch_bounds__(32 * kWarps, TETMF_N1F_MIN_BLOCKS)
n1_fold_kernel(const N1GramTable* __restrict__ gram,
               const MacroDesc* __restrict__ macros,
               const double* __restrict__ xin, const double* __restrict__ alpha, const double* __restrict__ beta,
               double* __restrict__ yout, const FoldTask* __restrict__ tasks, int ntasks, i64 stride, i64 cstride,
               i64 cf_stride, int n, int chunk) {
  extern __shared__ __align__(16) double dsm[];
  N1GramTable& sg = *reinterpret_cast<N1GramTable*>(dsm);
  // one launch covers every geometry group of a pass; task lists are padded
  // per group to whole CTAs, so the CTA's first task (always real) names
  // the group of all its warps
  {
    const N1GramTable* gt = gram + macros[tasks[blockIdx.x * kWarps].macro].group;
    for (int i = threadIdx.x; i < 6 * kGramRow; i += blockDim.x) (&sg.o[0][0])[i] = __ldg(&gt->o[0][0] + i);
  }
  // all-zero table for elements outside the macro, 64 bytes off the real
  // table's bank phase (a warp reading both stays conflict-free)
  double* ztab = dsm + kZeroTab;
  for (int i = threadIdx.x; i < 6 * kGramRow; i += blockDim.x) ztab[i] = 0.0;
  const unsigned tab_a = static_cast<unsigned>(__cvta_generic_to_shared(dsm));
  const unsigned zero_a = static_cast<unsigned>(__cvta_generic_to_shared(ztab));
  const int lane = threadIdx.x & 31;
  double* ring = dsm + kTabs + (threadIdx.x >> 5) * kWarpSmem;
  for (int i = lane; i < kRing; i += 32) ring[i] = 0.0;  // unfilled positions must read finite
  double* rmw = ring + kRing + lane;                     // [6][32]
  __syncthreads();
  const int warp = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (warp >= ntasks) return;
  const FoldTask tk = tasks[warp];
  if (tk.macro < 0) return;  // padding task
  const int z = tk.z, m = n - 1, L = n - 1 - z;
  const int K = (L + 1) / kSeg;  // full segments of the layer (a partial one walks alone)
  const int kn = tk.k, kf = K - 1 - kn;
  const bool paired = kn < K && kf > kn;
  const int x0 = kSeg * kn;
  const int D = 2 * L + 4 - kSeg * K;
  // phase 1: near column Xn, rows 0 .. P1-1 (lane 0: halo column x0 - 1,
  // needed only while lane 1 runs)
  const int Xn = x0 - 1 + lane;
  const int P1 = lane == 0 ? L - x0 + 1 : L - Xn + 1;
  // phase 2: far column Xf, rows ytop .. 0 (lane 31: halo column, whose top
  // row is not needed by lane 30)
  const int Xf = lane < 31 ? kSeg * kf + 30 - lane : kSeg * kf - 1;
  const bool far_ok = paired && Xf <= L;
  const int ytop = L - Xf - (lane == 31 ? 1 : 0);
  const int nsteps = paired ? D + 2 : L - x0 + 1;
  const int t0 = tk.t0;
  const int ts = t0 > 0 ? t0 - 1 : 0;  // halo step: restores the carried sums
  const int te = min(t0 + chunk, nsteps);

  const int cs = static_cast<int>(cstride);
  const double* __restrict__ Xm = xin + static_cast<i64>(tk.macro) * stride;
  double* __restrict__ Ym = yout + static_cast<i64>(tk.macro) * stride;
  const double* __restrict__ Am = alpha + static_cast<i64>(tk.macro) * cf_stride;
  const double* __restrict__ Bm = beta + static_cast<i64>(tk.macro) * cf_stride;
  const int pez = static_cast<int>(plane_offset(m, z)), peu = static_cast<int>(plane_offset(m, z + 1));
  const int pvz = static_cast<int>(plane_offset(n, z)), pvu = static_cast<int>(plane_offset(n, z + 1));
  const int lez = m - z + 1, lvz = n - z + 1;  // row-0 lengths of plane z (edges, vertices)
  // row r starts (x = 0) in plane z / z+1 of the edge lattice
  auto tri = [](int r) { return r * (r - 1) / 2; };
  auto ez_of = [&](int r) { return pez + r * lez - tri(r); };
  auto eu_of = [&](int r) { return peu + r * (lez - 1) - tri(r); };

  // the copies made at step tc, for step tc + 1: input row (phase-1 row
  // tc + 2, or the far row step tc + 1 reads first) into ring slot `slot`
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
    if (row >= 0 && !TETMF_N1F_NOCOPY) {
      double* d = ring + slot * kSlot;
      const int tr = tri(row);
      const double* xz = Xm + (pez + row * lez - tr + col);
      const double* xu = Xm + (peu + row * (lez - 1) - tr + col);
      const int vz = pvz + row * lvz - tr + col, vu = pvu + row * (lvz - 1) - tr + col;
      double* o = d + lane + 1;
#pragma unroll
      for (int c = 0; c < 7; ++c) cp_async8(o + c * kRow, xz + c * cs);
      cp_async8(o + 7 * kRow, xu);
      cp_async8(o + 8 * kRow, xu + cs);
      cp_async8(o + 9 * kRow, xu + 3 * cs);
      cp_async8(o + 10 * kRow, Am + vz);
      cp_async8(o + 11 * kRow, Am + vu);
      cp_async8(o + 12 * kRow, Bm + vz);
      cp_async8(o + 13 * kRow, Bm + vu);
      if (far ? lane == 0 : lane == 31) {  // column + 1 of the phase's boundary lane
        double* e = d + (far ? 0 : 33);
        cp_async8(e + 1 * kRow, xz + cs + 1);
        cp_async8(e + 2 * kRow, xz + 2 * cs + 1);
        cp_async8(e + 5 * kRow, xz + 5 * cs + 1);
        cp_async8(e + 8 * kRow, xu + cs + 1);
        cp_async8(e + 10 * kRow, Am + vz + 1);
        cp_async8(e + 11 * kRow, Am + vu + 1);
        cp_async8(e + 12 * kRow, Bm + vz + 1);
        cp_async8(e + 13 * kRow, Bm + vu + 1);
      }
    }
    cp_async_commit();
  };
  // pass 1: the in-plane partial sums step tn adds to -- [0..2] plane z
  // classes 0, 1, 3; [3..5] plane z+1 classes 0, 1, 3 (class 0 at the delayed
  // row in phase 2) -- staged into the warp's single staging slot at the end
  // of step tn - 1 (after that step's writes consumed the slot); the next
  // step's cp.async.wait_group 1 covers it
  auto stage_rmw = [&](int tn) {
    double* r = rmw;
    if (tn < P1) {
      if (tn >= 0 && lane > 0) {
        const double* a = Ym + ez_of(tn) + Xn;
        const double* b = Ym + eu_of(tn) + Xn;
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
        const double* a = Ym + ez_of(yn) + Xf;
        const double* b = Ym + eu_of(yn) + Xf;
        cp_async8(r + 32, a + cs);
        cp_async8(r + 64, a + 3 * cs);
        cp_async8(r + 128, b + cs);
        cp_async8(r + 160, b + 3 * cs);
      }
      if (yn + 1 >= 0 && yn + 1 <= ytop) {
        cp_async8(r, Ym + ez_of(yn + 1) + Xf);
        cp_async8(r + 96, Ym + eu_of(yn + 1) + Xf);
      }
    }
    cp_async_commit();
  };
  constexpr bool kStage = PASS == 1 && TETMF_N1F_STAGE_RMW != 0;

  int slot = ts % 3;  // ring slot of the copy made at step tt
  copy_for(ts - 2, slot == 0 ? 1 : slot == 1 ? 2 : 0);
  copy_for(ts - 1, slot == 0 ? 2 : slot - 1);
  if (kStage && t0 == 0) stage_rmw(0);  // the first step writes (no halo step)

  double c0 = 0.0, c2 = 0.0, c4 = 0.0, cT0 = 0.0;
#if TETMF_N1F_NOSTORE
  double sink = 0.0;
#endif
  for (int tt = ts; tt < te; ++tt) {
    asm volatile("" ::: "memory");  // table reads stay in the loop (no hoisting)
    copy_for(tt, slot);
    cp_async_wait1();  // all but this step's input copy landed (this lane's)
    __syncwarp();      // ... and every lane's
    const int sA = slot == 2 ? 0 : slot + 1;  // (tt + 1) mod 3
    const int sB = sA == 2 ? 0 : sA + 1;      // (tt + 2) mod 3
    slot = sA;
    const bool p1 = tt < P1;
    const int yf = D - tt;
    const int y = p1 ? tt : yf;
    const int X = p1 ? Xn : Xf;
    const bool cube = p1 ? Xn >= 0 : far_ok && yf >= 0 && yf <= ytop;
    const double* r0 = ring + (p1 ? sA : sB) * kSlot + lane + 1;
    const double* r1 = ring + (p1 ? sB : sA) * kSlot + lane + 1;
    const int dq = p1 ? 1 : -1;  // x+1 neighbour position

    double Y[19];
    const int s = X + y + z;
#if TETMF_N1_ZW
    cube_elements_zw<RULE>(SmemTabs3{opaque_u32(cube && s <= n - 1 ? tab_a : zero_a),
                                     opaque_u32(cube && s <= n - 2 ? tab_a : zero_a),
                                     opaque_u32(cube && s <= n - 3 ? tab_a : zero_a)},
                           FoldIn{r0, r1, r0 + dq, r1 + dq}, Y);
#else
#pragma unroll
    for (int k = 0; k < 19; ++k) Y[k] = 0.0;
    cube_elements<RULE>(SmemTabs{sg}, FoldIn{r0, r1, r0 + dq, r1 + dq}, Y, cube && s <= n - 1, cube && s <= n - 2,
                        cube && s <= n - 3);
#endif
    __syncwarp();  // ring slot tt mod 3 is refilled by the next step's copies

    // contributions of the x-1 neighbour cube (same row)
    const int src = (p1 ? lane - 1 : lane + 1) & 31;
    const double r7 = __shfl_sync(0xffffffffu, Y[7], src);
    const double r8 = __shfl_sync(0xffffffffu, Y[8], src);
    const double r9 = __shfl_sync(0xffffffffu, Y[9], src);
    const double r13 = __shfl_sync(0xffffffffu, Y[13], src);
    const double r17 = __shfl_sync(0xffffffffu, Y[17], src);

#if TETMF_N1F_NOSTORE
    if (tt >= t0) {  // measurement build: keep every stored value alive, store nothing
#pragma unroll
      for (int k = 0; k < 19; ++k) sink += Y[k];
      sink += r7 + r8 + r9 + r13 + r17 + c0 + c2 + c4 + cT0;
    }
    if (false) {
#else
    if (tt >= t0) {
#endif
      // pass 1: the staged partial sums (copied at the end of step tt - 1)
      const double* st = rmw;
      // in-plane partial sums: pass 0 stores, pass 1 adds (staged operand k)
      auto wr = [&](double* p, int k, double v) {
        if (PASS == 0)
          *p = v;
        else if (TETMF_N1F_STAGE_RMW)
          *p = st[32 * k] + v;
        else
          *p += v;
      };
      if (p1) {
        if (lane > 0 && cube && s <= n - 1) {  // all owned edges of row y
          double* __restrict__ yz = Ym + ez_of(y) + X;
          yz[2 * cs] = Y[2] + c2 + r8;
          yz[4 * cs] = Y[4] + c4;
          yz[5 * cs] = Y[5] + r9;
          wr(yz, 0, (Y[0] + c0));
          wr(yz + cs, 1, (Y[1] + r7));
          wr(yz + 3 * cs, 2, Y[3]);
          if (s <= n - 2) {
            yz[6 * cs] = Y[6];
            double* __restrict__ yu = Ym + eu_of(y) + X;
            wr(yu, 3, (Y[14] + cT0));
            wr(yu + cs, 4, (Y[15] + r17));
            wr(yu + 3 * cs, 5, Y[16]);
          }
        }
      } else if (lane < 31 && far_ok) {
        if (cube) {  // owned edges of row y with no share from row y-1
          double* __restrict__ yz = Ym + ez_of(y) + X;
          yz[5 * cs] = Y[5] + r9;
          wr(yz + cs, 1, (Y[1] + r7));
          wr(yz + 3 * cs, 2, Y[3]);
          if (s <= n - 2) {
            yz[6 * cs] = Y[6];
            double* __restrict__ yu = Ym + eu_of(y) + X;
            wr(yu + cs, 4, (Y[15] + r17));
            wr(yu + 3 * cs, 5, Y[16]);
          }
        }
        if (y + 1 >= 0 && y + 1 <= ytop) {  // delayed edges of row y+1
          double* __restrict__ yz = Ym + ez_of(y + 1) + X;
          yz[2 * cs] = Y[11] + c2 + r13;
          yz[4 * cs] = Y[12] + c4;
          wr(yz, 0, (Y[10] + c0));
          if (s + 1 <= n - 2) wr(Ym + eu_of(y + 1) + X, 3, Y[18] + cT0);
        }
      }
    }
    if (kStage && tt + 1 < te) stage_rmw(tt + 1);  // tt + 1 >= t0 always (tt >= t0 - 1)
    // carried partial sums: phase 1 -> owners of row y+1, phase 2 -> this
    // row's delayed edges
    if (p1) {
      c0 = Y[10];
      c2 = Y[11] + r13;
      c4 = Y[12];
      cT0 = Y[18];
    } else {
      c0 = Y[0];
      c2 = Y[2] + r8;
      c4 = Y[4];
      cT0 = Y[14];
    }
  }
#if TETMF_N1F_NOSTORE
  if (sink == 1.2345) Ym[0] = sink;
#endif
  asm volatile("cp.async.wait_all;" ::: "memory");
}

} // namespace

// the layer-pair walk (k_n1_fold2.cu, default) and this file's one-layer walk
void build_n1_fold2_tasks(const std::vector<int>& local_macros, int n, int parity, std::vector<int>& out, int chunk);
void pad_n1_fold2_tasks(std::vector<int>& tasks);
int n1_fold2_chunk(const std::vector<int>& local_macros, int n, int sms);
void launch_n1_fold2(const N1GramTable* gram, const MacroDesc* macros, int pass, const double* x, const double* alpha,
                     const double* beta, double* y, const int* d_tasks, int ntasks, i64 macro_stride,
                     i64 class_stride, i64 coeff_stride, int n, int rule, cudaStream_t s, int chunk);
// TETMF_N1_WALK (read once): 2 = layer pairs (default), 1 = one layer per step
int n1_walk_layers() {
  static const int v = [] {
    const char* e = std::getenv("TETMF_N1_WALK");
    return e && e[0] == '1' ? 1 : 2;
  }();
  return v;
}

// Task list of one level and parity pass: (macro, z, k, t0) per layer z of
// the parity, segment pair (k, K-1-k) or unpaired segment, and chunk of
// `chunk` steps (kChunk by default; fewer for small levels, where the
// chunks are the parallelism).
void build_n1_fold_tasks(const std::vector<int>& local_macros, int n, int parity, std::vector<int>& out,
                         int chunk) {
  out.clear();
  for (int z = parity; z <= n - 1; z += 2) {
    const int L = n - 1 - z, K = (L + 1) / kSeg;  // full segments
    const int klast = (L + 1) % kSeg ? K : K - 1;  // + the partial one, unpaired
    for (int k = 0; k <= klast; ++k) {
      if (k < K && K - 1 - k < k) continue;        // far half of a pair
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

// Padding of one group's task list to whole CTAs (dummy tasks macro = -1).
void pad_n1_fold_tasks(std::vector<int>& tasks) {
  if (n1_walk_layers() == 2) return pad_n1_fold2_tasks(tasks);
  while ((tasks.size() / 4) % kWarps) {
    tasks.push_back(-1);
    tasks.push_back(0);
    tasks.push_back(0);
    tasks.push_back(0);
  }
}

// gram: tables of all geometry groups; macros: local macro descriptors
void launch_n1_fold(const N1GramTable* gram, const MacroDesc* macros, int pass, const double* x, const double* alpha,
                    const double* beta, double* y, const int* d_tasks, int ntasks, i64 macro_stride,
                    i64 class_stride, i64 coeff_stride, int n, int rule, cudaStream_t s, int chunk) {
  if (n1_walk_layers() == 2)
    return launch_n1_fold2(gram, macros, pass, x, alpha, beta, y, d_tasks, ntasks, macro_stride, class_stride,
                           coeff_stride, n, rule, s, chunk);
  if (ntasks == 0) return;
  if (rule < 0 || rule > 2) fail_internal("n1_fold: rule index out of range");
  if (chunk < 1) fail_internal("n1_fold: chunk < 1");
  constexpr int smem = static_cast<int>(sizeof(double) * (kTabs + kWarpSmem * kWarps));
  using K = decltype(&n1_fold_kernel<0, 0>);
  static const K kerns[2][3] = {{n1_fold_kernel<0, 0>, n1_fold_kernel<0, 1>, n1_fold_kernel<0, 2>},
                                {n1_fold_kernel<1, 0>, n1_fold_kernel<1, 1>, n1_fold_kernel<1, 2>}};
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
  check_launch("n1_fold");
}

// the N1 apply is the fold kernel; task lists per geometry group and pass
int n1_kernel_mode() { return 3; }

void build_n1_tasks(const std::vector<int>& local_macros, int n, int parity, std::vector<int>& out, int chunk) {
  if (n1_walk_layers() == 2) return build_n1_fold2_tasks(local_macros, n, parity, out, chunk);
  build_n1_fold_tasks(local_macros, n, parity, out, chunk);
}

// Steps per fold task for a level: kChunk, halved while one pass would not
// give every SM several waves of warps (small meshes / small per-GPU shares
// under strong scaling); each halving adds a halo step per 8-32 steps but
// multiplies the tasks.
int n1_fold_chunk(const std::vector<int>& local_macros, int n, int sms) {
  if (n1_walk_layers() == 2) return n1_fold2_chunk(local_macros, n, sms);
  std::vector<int> t;
  int chunk = kChunk;
  while (chunk > 8) {
    build_n1_fold_tasks(local_macros, n, 0, t, chunk);
    if (static_cast<long long>(t.size() / 4) >= 4LL * 12 * sms) break;
    chunk /= 2;
  }
  return chunk;
}

} // namespace tetmf

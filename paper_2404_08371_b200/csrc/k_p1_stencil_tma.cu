// k_p1_stencil_tma.cu -- K1 variant 3 ("stream"): P1 -Laplace 15-point
// stencil, persistent warp-specialised plane streaming through shared memory.
//
// Why: the row-walk kernels (k_p1_stencil2.cu) keep only ~1 KB of loads in
// flight per warp and stall on memory latency at ~2 TB/s. HBM needs ~40-60 KB
// in flight per SM; TMA bulk copies of >= 16 KB reach 7.2 TB/s with 2-4
// copies in flight per SM (tools/tma_probe.cu).
//
// Layout fact used: the rows y0-1 .. y0+kRows of one plane are ONE contiguous
// range of the lattice storage (plane-major, row-major), so the "slab" a row
// block needs from a plane is a single cp.async.bulk (1-D TMA, no tensor map).
//
// Task = (macro, row block [y0, y0+kRows), planes [za, zb]); it reads the
// slabs of planes za-1 .. zb+1 (those that exist). The grid is persistent
// (CTA c takes tasks c, c+G, ...; tasks ordered (macro, plane range, y0) so the
// CTAs running at the same time work on neighbouring row blocks and the two
// halo rows of a slab are L2 hits). Per CTA:
//   * producer warp (lane 0): walks the CTA's slab sequence; slab k takes
//     barrier descriptor k % kDesc and a contiguous stretch of a byte ring
//     (slabs are sized to their plane, ~1/3 of the worst case on average), and
//     is issued once the consumers released what it overwrites (empty
//     barriers), completing on its full barrier (expect_tx);
//   * consumer warps: per plane z (or plane pair, TETMF_P1T_PAIRS) observe
//     the slabs z-1 .. z+1, walk columns (32-column segments rotating over the
//     warps from plane to plane) with a register window along y -- 7 shared-
//     memory loads + 15 DFMA per point, fully unrolled rows, per-lane weights
//     (interior / x = 0 face) from a per-warp copy of the table, stores masked
//     before the diagonal point, which follows as one 15-point gather -- and
//     release slab z-1. No CTA-wide barrier in the loop.
//
// Measured (cube6 L8, C4): 155-166 us vs 152 us for the row walk; 12-macro
// Kuhn mesh L7: 175-178 us vs 203 us. ncu: latency / issue bound (~14 warps
// per SM at 128 registers, issue active ~50 %, DRAM ~17 %); deeper rings
// (1 CTA / SM, 10 slabs) and plane pairs were slower. DESIGN.md section 4.
//
// Boundaries: out-of-lattice neighbours always meet zero stencil weights (face
// points use the per-type stencil variant, tables.cpp) or belong to lanes that
// do not store; their reads land on finite data inside the slab's own
// margins (never on a stretch a TMA copy may be writing); row y0-1 of block 0
// is not read; a missing plane (z-1 < 0, z+1 > n) aliases plane z.
#include <cstdint>

#include "device.hpp"
#include "runtime_check.hpp"

namespace tetmf {

namespace {

#ifndef TETMF_P1T_WARPS
#define TETMF_P1T_WARPS 7
#endif
#ifndef TETMF_P1T_ROWS
#define TETMF_P1T_ROWS 8
#endif
#ifndef TETMF_P1T_DESC
#define TETMF_P1T_DESC 16
#endif
#ifndef TETMF_P1T_RING_KB
#define TETMF_P1T_RING_KB 106
#endif
#ifndef TETMF_P1T_PLANES
#define TETMF_P1T_PLANES 32
#endif
#ifndef TETMF_P1T_MINB
#define TETMF_P1T_MINB 2
#endif
constexpr int kConsumers = TETMF_P1T_WARPS;        // consumer warps per CTA
constexpr int kThreads = 32 * (kConsumers + 1);    // + one producer warp
constexpr int kRows = TETMF_P1T_ROWS;              // rows per block
constexpr int kDesc = TETMF_P1T_DESC;              // slabs resident at most (barrier pairs)
constexpr int kPlanes = TETMF_P1T_PLANES;          // planes per task
constexpr int kFront = 16;                         // margin before a slab's data (doubles)
constexpr int kBack = kRows + 64 + 16;
#ifndef TETMF_P1T_PAIRS
#define TETMF_P1T_PAIRS 0  // pairs measured slower (174 vs 166 us, C4)
#endif
constexpr bool kPairs = TETMF_P1T_PAIRS;           // plane pairs per column walk             // margin after it (reads past a row end)

struct TmaTask {
  int macro, y0, za, zb;
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(std::uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(std::uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// waiting threads sleep in try_wait (suspend-time hint) instead of spinning:
// idle consumer warps must not steal issue slots from the working ones
__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680u)
      : "memory");
}
__device__ __forceinline__ double lds(unsigned addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, std::uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// first / last plane whose slab task t reads; row range of a slab: ya .. yb
__device__ __forceinline__ int slab_ya(int y0) { return y0 > 0 ? y0 - 1 : 0; }
__device__ __forceinline__ int first_plane(const TmaTask& t) { return t.za > 0 ? t.za - 1 : 0; }
__device__ __forceinline__ int last_plane(const TmaTask& t, int n) { return min(t.zb + 1, n - slab_ya(t.y0)); }

// 32-bit lattice arithmetic (a level's storage fits in int): points of plane
// p = tri(n - p), row y of plane p starts at P(p) + rowoff(n - p, y)
__device__ __forceinline__ int tri(int m) { return (m + 1) * (m + 2) / 2; }
__device__ __forceinline__ int rowoff(int m, int y) { return y * (m + 1) - y * (y - 1) / 2; }
__device__ __forceinline__ int plane_start(int n, int p) { return static_cast<int>(plane_offset(n, p)); }

// slab of plane p (start P) for block y0: rows ya .. min(y0 + kRows, n - p),
// global [g0, g1), 128-byte aligned (macro blocks are 256-byte aligned)
__device__ __forceinline__ int slab_g0(int n, int P, int p, int y0) { return (P + rowoff(n - p, slab_ya(y0))) & ~15; }
__device__ __forceinline__ int slab_g1(int n, int P, int p, int y0) {
  return (P + rowoff(n - p, min(y0 + kRows, n - p) + 1) + 15) & ~15;
}

// shared-memory footprint of a slab: margins + data, 128-byte multiple
__device__ __forceinline__ int slab_len(int g0, int g1) { return (kFront + (g1 - g0) + kBack + 15) & ~15; }

__global__ void __launch_bounds__(kThreads, TETMF_P1T_MINB)
p1_stream_kernel(const double* __restrict__ xin, double* __restrict__ yout, const TmaTask* __restrict__ tasks,
                 int ntasks, i64 stride, int n, int ring_len, const P1DeviceTable* __restrict__ tabs,
                 const MacroDesc* __restrict__ macros) {
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) std::uint64_t full[kDesc], empty[kDesc];
  __shared__ int slab_off[kDesc];  // ring offset (doubles) of the slab held by each descriptor
  // per consumer warp: stencil rows of types 0, 1 (x = 0), 8 (diagonal), 9
  // of the current task's group (the L1 is small next to the ring)
  __shared__ __align__(16) double wtab[kConsumers][4][16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // zero the ring once: every read outside a slab's copied range (inside its
  // margins) then sees finite data (zeros or an older slab)
  for (int i = threadIdx.x; i < ring_len; i += kThreads) smem[i] = 0.0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kDesc; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kConsumers) {  // ---------------- producer
    if (lane != 0) return;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the zero fill precedes the copies
    // Byte ring: slab k takes descriptor k % kDesc and a contiguous stretch
    // of the ring (wrapping to 0 when it does not fit before the end). tl =
    // oldest slab not yet known to be released; the resident slabs occupy
    // [off(tl), head) circularly.
    int k = 0, tl = 0, head = 0;
    for (int ti = blockIdx.x; ti < ntasks; ti += gridDim.x) {
      const TmaTask t = tasks[ti];
      const double* __restrict__ X = xin + static_cast<i64>(t.macro) * stride;
      const int pf = first_plane(t), pl = last_plane(t, n);
      int P = plane_start(n, pf);
      for (int p = pf; p <= pl; P += tri(n - p), ++p, ++k) {
        const int d = k % kDesc;
        const int g0 = slab_g0(n, P, p, t.y0), g1 = slab_g1(n, P, p, t.y0);
        const int len = slab_len(g0, g1);
        int start;
        for (;;) {
          if (tl == k) {  // nothing resident
            start = 0;
            break;
          }
          const int toff = slab_off[tl % kDesc];
          if (head > toff) {  // resident: [toff, head)
            if (head + len <= ring_len) { start = head; break; }
            if (len <= toff) { start = 0; break; }
          } else if (head + len <= toff) {  // resident: [toff, end) and [0, head)
            start = head;
            break;
          }
          mbar_wait(&empty[tl % kDesc], (tl / kDesc) & 1);  // free the oldest slab
          ++tl;
        }
        if (k - tl >= kDesc) {  // descriptor still held by slab k - kDesc
          mbar_wait(&empty[d], (tl / kDesc) & 1);
          ++tl;
        }
        slab_off[d] = start;
        head = start + len;
        const unsigned bytes = static_cast<unsigned>(g1 - g0) * 8u;
        mbar_expect_tx(&full[d], bytes);
        bulk_g2s(smem + start + kFront, X + g0, bytes, &full[d]);
      }
    }
    return;
  }

  // ---------------------------------------------- consumers
  int k = 0;  // slab index of the task's first plane (same sequence as the producer)
  for (int ti = blockIdx.x; ti < ntasks; ti += gridDim.x) {
    const TmaTask t = tasks[ti];
    const int y0 = t.y0;
    double* __restrict__ Y = yout + static_cast<i64>(t.macro) * stride;
    const double* __restrict__ tab = &tabs[macros[t.macro].group].stencil[0][0];
    const int pf = first_plane(t), pl = last_plane(t, n);
    {
      const int r = lane >> 3, c = (lane & 7) * 2;  // 4 rows x 16 doubles, 2 per lane
      const int type = (r & 1) | ((r >> 1) << 3);
      __syncwarp();
      wtab[warp][r][c] = __ldg(tab + 16 * type + c);
      wtab[warp][r][c + 1] = __ldg(tab + 16 * type + c + 1);
      __syncwarp();
    }
    const unsigned wsm = smem_u32(&wtab[warp][0][0]);
    // Barrier bookkeeping: hw = highest slab index this warp has observed
    // (full barrier passed; all lower slabs of the task too). A slab is only
    // released after it was observed: a warp that released an unobserved slab
    // could later query the slot's next phase while this one is still pending,
    // and try_wait.parity would answer for the previous phase (copies complete
    // out of order).
    int hw = k - 1;
    auto observe = [&](int idx) {
      while (hw < idx) {
        ++hw;
        mbar_wait(&full[hw % kDesc], (hw / kDesc) & 1);
      }
    };
    auto release = [&](int idx) {
      observe(idx);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[idx % kDesc]);
    };
    // (read after the slab was observed: the producer wrote it before its arrive)
    auto slot_u32 = [&](int idx) { return smem_u32(smem + slab_off[idx % kDesc] + kFront); };

    // diagonal point (x, yd = m - x) of plane z (side m, start Pz, shared base
    // bZ), planes below / above at bases bL / bU (starts Pl / Pu): rows yd-1,
    // yd, yd+1 of Z, yd and yd+1 of L, yd-1 and yd of U; wt = weights
    auto diag_point = [&](unsigned bZ, int Pz, int m, unsigned bL, int Pl, bool hasL, unsigned bU, int Pu,
                          bool hasU, int x, unsigned wt) {
      const int yd = m - x;
      const unsigned z0 = bZ + 8u * static_cast<unsigned>(Pz + rowoff(m, yd) + x);
      const unsigned zp = bZ + 8u * static_cast<unsigned>(Pz + rowoff(m, yd + 1) + x);
      const unsigned zm = bZ + 8u * static_cast<unsigned>(Pz + rowoff(m, yd - 1) + x);
      const unsigned l0 = hasL ? bL + 8u * static_cast<unsigned>(Pl + rowoff(m + 1, yd) + x) : z0;
      const unsigned lp = hasL ? bL + 8u * static_cast<unsigned>(Pl + rowoff(m + 1, yd + 1) + x) : zp;
      const unsigned u0 = hasU ? bU + 8u * static_cast<unsigned>(Pu + rowoff(m - 1, yd) + x) : z0;
      const unsigned um = hasU ? bU + 8u * static_cast<unsigned>(Pu + rowoff(m - 1, yd - 1) + x) : zm;
      double a0 = lds(wt + 0u) * lds(z0), a1 = lds(wt + 8u) * lds(z0 + 8);
      double a2 = lds(wt + 16u) * lds(z0 - 8), a3 = lds(wt + 24u) * lds(zp);
      a0 = fma(lds(wt + 32u), lds(zm), a0);
      a1 = fma(lds(wt + 40u), lds(u0), a1);
      a2 = fma(lds(wt + 48u), lds(l0), a2);
      a3 = fma(lds(wt + 56u), lds(zm + 8), a3);
      a0 = fma(lds(wt + 64u), lds(zp - 8), a0);
      a1 = fma(lds(wt + 72u), lds(l0 + 8), a1);
      a2 = fma(lds(wt + 80u), lds(u0 - 8), a2);
      a3 = fma(lds(wt + 88u), lds(lp), a3);
      a0 = fma(lds(wt + 96u), lds(um), a0);
      a1 = fma(lds(wt + 104u), lds(lp + 8), a1);
      a2 = fma(lds(wt + 112u), lds(um - 8), a2);
      Y[Pz + rowoff(m, yd) + x] = (a0 + a1) + (a2 + a3);
    };

    int Pz = plane_start(n, t.za);
    int ic = k + (t.za - pf);  // slab index of plane z
    int z = t.za;
    while (z <= t.zb) {
      const int m = n - z;  // plane z is a triangle of side m
      const int lz0 = m - y0 + 1;
      const int Pl = Pz - tri(m + 1), Pu = Pz + tri(m);
      if (kPairs && z > 0 && y0 > 0 && z + 1 <= t.zb) {
        // ------------------------------------------------ plane pair (z, z+1)
        // planes L = z-1, A = z, B = z+1, U = z+2 (all exist: y0 > 0, z+1 <= zb)
        const int rot = (warp + (z >> 1)) % kConsumers;
        if (32 * rot < lz0) {
          observe(ic + 2);
          const int Pb = Pu, Puu = Pu + tri(m - 1);
          const unsigned bA = slot_u32(ic) - 8u * static_cast<unsigned>(slab_g0(n, Pz, z, y0));
          const unsigned bL = slot_u32(ic - 1) - 8u * static_cast<unsigned>(slab_g0(n, Pl, z - 1, y0));
          const unsigned bB = slot_u32(ic + 1) - 8u * static_cast<unsigned>(slab_g0(n, Pb, z + 1, y0));
          const unsigned bU = slot_u32(ic + 2) - 8u * static_cast<unsigned>(slab_g0(n, Puu, z + 2, y0));
          const int ra0 = Pz + rowoff(m, y0), rl0 = Pl + rowoff(m + 1, y0);
          const int rb0 = Pb + rowoff(m - 1, y0), ru0 = Puu + rowoff(m - 2, y0);
          const int ylastA = min(y0 + kRows - 1, m), ylastB = min(y0 + kRows - 1, m - 1);
          for (int xs = 32 * rot; xs < lz0; xs += 32 * kConsumers) {
            const int x = xs + lane;
            const bool colA = x < lz0, colB = x < lz0 - 1;
            const int colbits = x == 0 ? 1 : 0;
            double w[15];
#pragma unroll
            for (int q = 0; q < 15; ++q) w[q] = lds(wsm + 128u * colbits + 8u * q);
            const int ystA = colA ? min(ylastA, m - x - 1) : -1;
            const int ystB = colB ? min(ylastB, m - 2 - x) : -1;
            int lz8 = 8 * lz0;  // 8 x row length of plane A at the current row
            unsigned aA = bA + 8u * static_cast<unsigned>(ra0 + x);
            unsigned aL = bL + 8u * static_cast<unsigned>(rl0 + x);
            unsigned aB = bB + 8u * static_cast<unsigned>(rb0 + x);
            unsigned aU = bU + 8u * static_cast<unsigned>(ru0 + x);
            unsigned yiA = static_cast<unsigned>(ra0 + x), yiB = static_cast<unsigned>(rb0 + x);
            double Am0 = lds(aA - lz8 - 8), Am1 = lds(aA - lz8);
            double A0m = lds(aA - 8), A00 = lds(aA), A01 = lds(aA + 8);
            double L00 = lds(aL), L01 = lds(aL + 8);
            double Bmm = lds(aB - lz8 - 8), Bm0 = lds(aB - lz8), Bm1 = lds(aB - lz8 + 8);
            double B0m = lds(aB - 8), B00 = lds(aB), B01 = lds(aB + 8);
            double Umm = lds(aU - lz8), Um0 = lds(aU - lz8 + 8);
#pragma unroll
            for (int r = 0; r < kRows; ++r) {
              const unsigned aLn = aL + lz8 + 8, aAn = aA + lz8, aBn = aB + lz8 - 8;
              const double Lp0 = lds(aLn), Lp1 = lds(aLn + 8);
              const double Apm = lds(aAn - 8), Ap0 = lds(aAn), Ap1 = lds(aAn + 8);
              const double Bpm = lds(aBn - 8), Bp0 = lds(aBn), Bp1 = lds(aBn + 8);
              const double U0m = lds(aU - 8), U00 = lds(aU);
              double a0 = w[0] * A00, a1 = w[1] * A01, a2 = w[2] * A0m, a3 = w[3] * Ap0;
              double b0 = w[0] * B00, b1 = w[1] * B01, b2 = w[2] * B0m, b3 = w[3] * Bp0;
              a0 = fma(w[4], Am0, a0);
              b0 = fma(w[4], Bm0, b0);
              a1 = fma(w[5], B00, a1);
              b1 = fma(w[5], U00, b1);
              a2 = fma(w[6], L00, a2);
              b2 = fma(w[6], A00, b2);
              a3 = fma(w[7], Am1, a3);
              b3 = fma(w[7], Bm1, b3);
              a0 = fma(w[8], Apm, a0);
              b0 = fma(w[8], Bpm, b0);
              a1 = fma(w[9], L01, a1);
              b1 = fma(w[9], A01, b1);
              a2 = fma(w[10], B0m, a2);
              b2 = fma(w[10], U0m, b2);
              a3 = fma(w[11], Lp0, a3);
              b3 = fma(w[11], Ap0, b3);
              a0 = fma(w[12], Bm0, a0);
              b0 = fma(w[12], Um0, b0);
              a1 = fma(w[13], Lp1, a1);
              b1 = fma(w[13], Ap1, b1);
              a2 = fma(w[14], Bmm, a2);
              b2 = fma(w[14], Umm, b2);
              if (y0 + r <= ystA) Y[yiA] = (a0 + a1) + (a2 + a3);
              if (y0 + r <= ystB) Y[yiB] = (b0 + b1) + (b2 + b3);
              yiA += static_cast<unsigned>(lz8) >> 3;
              yiB += (static_cast<unsigned>(lz8) >> 3) - 1u;
              Am0 = A00; Am1 = A01;
              A0m = Apm; A00 = Ap0; A01 = Ap1;
              L00 = Lp0; L01 = Lp1;
              Bmm = B0m; Bm0 = B00; Bm1 = B01;
              B0m = Bpm; B00 = Bp0; B01 = Bp1;
              Umm = U0m; Um0 = U00;
              aL = aLn; aA = aAn; aB = aBn;
              aU += lz8 - 16;
              lz8 -= 8;
            }
            // diagonal points of A (x + y = m) and B (x + y = m - 1) in the block
            if (colA && m - x <= ylastA)
              diag_point(bA, Pz, m, bL, Pl, true, bB, Pb, true, x, wsm + 128u * (colbits | 2));
            if (colB && m - 1 - x <= ylastB)
              diag_point(bB, Pb, m - 1, bA, Pz, true, bU, Puu, true, x, wsm + 128u * (colbits | 2));
          }
        }
        release(ic - 1);  // planes z-1 and z are not read by the next pair
        release(ic);
        Pz += tri(m) + tri(m - 1);
        z += 2;
        ic += 2;
        continue;
      }
      // -------------------------------------------------- single plane z
      const bool hasL = z - 1 >= pf, hasU = z + 1 <= pl;
      const int rot = (warp + z) % kConsumers;
      if (32 * rot < lz0) {
        observe(hasU ? ic + 1 : ic);
        const unsigned bZ = slot_u32(ic) - 8u * static_cast<unsigned>(slab_g0(n, Pz, z, y0));
        const unsigned bL = hasL ? slot_u32(ic - 1) - 8u * static_cast<unsigned>(slab_g0(n, Pl, z - 1, y0)) : bZ;
        const unsigned bU = hasU ? slot_u32(ic + 1) - 8u * static_cast<unsigned>(slab_g0(n, Pu, z + 1, y0)) : bZ;
        // row y0 of planes z, z-1, z+1 (missing planes alias plane z)
        const int rz0 = Pz + rowoff(m, y0);
        const int rl0 = hasL ? Pl + rowoff(m + 1, y0) : rz0;
        const int ru0 = hasU ? Pu + rowoff(m - 1, y0) : rz0;
        const int dl = hasL ? 1 : 0, du = hasU ? -1 : 0;  // row length of L / U minus plane z's
        const int ylast = min(y0 + kRows - 1, m);
        for (int xs = 32 * rot; xs < lz0; xs += 32 * kConsumers) {
          const int x = xs + lane;
          // fast path (warp-uniform: z > 0, block y0 > 0): every lane walks its
          // column for all kRows rows (fully unrolled, per-lane column weights:
          // interior or the x = 0 face) and stores the points before its
          // diagonal point; lanes past the row end or the diagonal compute on
          // finite in-slab data and do not store; the diagonal point follows as
          // one direct 15-point gather
          if (z > 0 && y0 > 0) {
            const bool col = x < lz0;
            const int colbits = x == 0 ? 1 : 0;
            double w[15];
#pragma unroll
            for (int q = 0; q < 15; ++q) w[q] = lds(wsm + 128u * colbits + 8u * q);
            const int yst = col ? min(ylast, m - x - 1) : -1;  // last row stored by the walk
            int lz8 = 8 * lz0;
            const int dl8 = 8 * dl, du8 = 8 * du;
            unsigned aZ = bZ + 8u * static_cast<unsigned>(rz0 + x);
            unsigned aL = bL + 8u * static_cast<unsigned>(rl0 + x);
            unsigned aU = bU + 8u * static_cast<unsigned>(ru0 + x);
            unsigned yi = static_cast<unsigned>(rz0 + x);
            double Zm0 = lds(aZ - lz8 - 8), Zm1 = lds(aZ - lz8);
            double Umm = lds(aU - lz8 - du8 - 16), Um0 = lds(aU - lz8 - du8 - 8);
            double Z0m = lds(aZ - 8), Z00 = lds(aZ);
            double L00 = lds(aL), L01 = lds(aL + 8);
#pragma unroll
            for (int r = 0; r < kRows; ++r) {
              const unsigned aZn = aZ + lz8, aLn = aL + lz8 + dl8, aUn = aU + lz8 + du8;
              const double Z01 = lds(aZ + 8);
              const double Zpm = lds(aZn - 8), Zp0 = lds(aZn);
              const double Lp0 = lds(aLn), Lp1 = lds(aLn + 8);
              const double U0m = lds(aU - 8), U00 = lds(aU);
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
              if (y0 + r <= yst) Y[yi] = (a0 + a1) + (a2 + a3);
              yi += static_cast<unsigned>(lz8) >> 3;
              Zm0 = Z00;
              Zm1 = Z01;
              Z0m = Zpm;
              Z00 = Zp0;
              L00 = Lp0;
              L01 = Lp1;
              Umm = U0m;
              Um0 = U00;
              aZ = aZn;
              aL = aLn;
              aU = aUn;
              lz8 -= 8;
            }
            if (col && m - x <= ylast) diag_point(bZ, Pz, m, bL, Pl, hasL, bU, Pu, hasU, x, wsm + 128u * (colbits | 2));
            continue;
          }
          if (x >= lz0) continue;
          // column weights: interior, x = 0 face and / or z = 0 face (tables.cpp)
          const int colbits = (x == 0 ? 1 : 0) | (z == 0 ? 4 : 0);
          double w[15];
#pragma unroll
          for (int q = 0; q < 15; ++q) w[q] = __ldg(tab + 16 * colbits + q);
          int lz = lz0;
          unsigned aZ = bZ + 8u * static_cast<unsigned>(rz0 + x);
          unsigned aL = bL + 8u * static_cast<unsigned>(rl0 + x);
          unsigned aU = bU + 8u * static_cast<unsigned>(ru0 + x);
          unsigned yi = static_cast<unsigned>(rz0 + x);
          // window at row y0 (row -1 does not exist: zeros)
          double Zm0 = 0.0, Zm1 = 0.0, Umm = 0.0, Um0 = 0.0;
          if (y0 > 0) {
            Zm0 = lds(aZ - 8u * (lz + 1));
            Zm1 = lds(aZ - 8u * lz);
            Umm = lds(aU - 8u * (lz + du + 2));
            Um0 = lds(aU - 8u * (lz + du + 1));
          }
          double Z0m = lds(aZ - 8), Z00 = lds(aZ);
          double L00 = lds(aL), L01 = lds(aL + 8);
          // one point: the row's new window values, 15 DFMA with weights wv
          // (registers) or the table row wt (face / diagonal variants), slide
          auto point = [&](const double* __restrict__ wt, bool table) {
            const unsigned aZn = aZ + 8u * lz, aLn = aL + 8u * (lz + dl);
            const double Z01 = lds(aZ + 8);
            const double Zpm = lds(aZn - 8), Zp0 = lds(aZn);
            const double Lp0 = lds(aLn), Lp1 = lds(aLn + 8);
            const double U0m = lds(aU - 8), U00 = lds(aU);
            double v[15];
            if (table) {
#pragma unroll
              for (int q = 0; q < 15; ++q) v[q] = __ldg(wt + q);
            } else {
#pragma unroll
              for (int q = 0; q < 15; ++q) v[q] = w[q];
            }
            double a0 = v[0] * Z00, a1 = v[1] * Z01, a2 = v[2] * Z0m, a3 = v[3] * Zp0;
            a0 = fma(v[4], Zm0, a0);
            a1 = fma(v[5], U00, a1);
            a2 = fma(v[6], L00, a2);
            a3 = fma(v[7], Zm1, a3);
            a0 = fma(v[8], Zpm, a0);
            a1 = fma(v[9], L01, a1);
            a2 = fma(v[10], U0m, a2);
            a3 = fma(v[11], Lp0, a3);
            a0 = fma(v[12], Um0, a0);
            a1 = fma(v[13], Lp1, a1);
            a2 = fma(v[14], Umm, a2);
            Y[yi] = (a0 + a1) + (a2 + a3);
            Zm0 = Z00;
            Zm1 = Z01;
            Z0m = Zpm;
            Z00 = Zp0;
            L00 = Lp0;
            L01 = Lp1;
            Umm = U0m;
            Um0 = U00;
            yi += lz;
            aZ = aZn;
            aL = aLn;
            aU += 8u * (lz + du);
            --lz;
          };
          // rows before the column's diagonal point (x + y = m): column
          // weights, except row 0 (y = 0 face, uniform over the warp)
          const int ydiag = m - x;
          const int yend = min(ylast, ydiag - 1);
          int yy = y0;
          if (yy == 0 && yy <= yend) {
            point(tab + 16 * (colbits | 2), true);
            ++yy;
          }
#pragma unroll
          for (int r = 0; r < kRows; ++r) {
            if (yy > yend) break;
            point(nullptr, false);
            ++yy;
          }
          // the diagonal point, when it lies in this block
          if (ydiag <= ylast) point(tab + 16 * (colbits | (ydiag == 0 ? 2 : 0) | 8), true);
        }
      }
      if (hasL) release(ic - 1);
      Pz += tri(m);
      ++z;
      ++ic;
    }
    // the task's last slabs (z-1 were released step by step)
    release(ic - 1);              // plane zb
    if (t.zb + 1 <= pl) release(ic);  // plane zb + 1
    k += pl - pf + 1;
  }
}

int g_grid_ctas = 0;

} // namespace

// Tasks (macro, y0, za, zb): kPlanes planes per task; plane z has rows in
// block y0 while z <= n - y0. Order: macro, plane range, row block.
void build_stencil_tma_tasks(int nmacros, int n, std::vector<int>& out) {
  out.clear();
  for (int li = 0; li < nmacros; ++li)
    for (int za = 0; za <= n; za += kPlanes)
      for (int y0 = 0; y0 <= n - za; y0 += kRows) {
        out.push_back(li);
        out.push_back(y0);
        out.push_back(za);
        out.push_back(min(za + kPlanes - 1, n - y0));
      }
}

void launch_p1_stencil_tma(const double* x, double* y, const int* d_tasks, int ntasks, i64 macro_stride, int n,
                           const P1DeviceTable* d_tables, const MacroDesc* d_macros, cudaStream_t s) {
  if (ntasks == 0) return;
  // byte ring: it must hold the slabs one step reads (4 for a plane pair, 3
  // for a plane), one more in flight and the stretch lost when a slab wraps
  const int max_len = (kFront + (kRows + 2) * (n + 1) + 30 + kBack + 15) & ~15;
  const int ring_len = (TETMF_P1T_RING_KB * 1024 / 8) & ~15;
  if (ring_len < (kPairs ? 6 : 5) * max_len) fail_internal("p1_stream: ring too small for this level (raise the ring or lower kRows)");
  const std::size_t smem = static_cast<std::size_t>(ring_len) * sizeof(double);
  static std::size_t configured = 0;
  if (smem > configured) {
    TETMF_CUDA(cudaFuncSetAttribute(p1_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
    configured = smem;
    int dev = 0, sms = 0, per_sm = 0;
    TETMF_CUDA(cudaGetDevice(&dev));
    TETMF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    TETMF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, p1_stream_kernel, kThreads, smem));
    g_grid_ctas = sms * (per_sm > 0 ? per_sm : 1);
  }
  const int grid = ntasks < g_grid_ctas ? ntasks : g_grid_ctas;
  p1_stream_kernel<<<grid, kThreads, smem, s>>>(x, y, reinterpret_cast<const TmaTask*>(d_tasks), ntasks,
                                                macro_stride, n, ring_len, d_tables, d_macros);
  check_launch("p1_stream");
}

} // namespace tetmf

// k_p1_stencil_tma.cu -- K1 (TMA version): P1 -Laplace 15-point stencil with
// plane streaming through shared memory.
//
// CTA task = (macro, row block [y0, y0 + kRows), plane range [za, zb]). The
// rows y0-1 .. y0+kRows of one plane are ONE contiguous range of the lattice
// storage (plane-major, row-major), so each plane "slab" is a single
// cp.async.bulk (TMA bulk copy) into shared memory, completing on an
// mbarrier. A ring of kSlabs slabs streams the planes: computing plane z needs
// slabs z-1, z, z+1 while slab z+2 is in flight, so every plane of the task
// is read from L2/HBM once (plus the two halo rows per block and the two warm
// up planes per task).
//
// Compute: thread t owns column x = t (and t + blockDim for the widest
// planes) and walks the block rows with a register window (7 shared-memory
// loads + 15 DFMA per point, as the row-walk kernel). Results go straight to
// global memory, coalesced along x.
//
// Boundaries: every out-of-lattice read lands in a zeroed pad of its slab
// (rows before / after the slab) or in a slab aliased for a missing plane, and
// always meets a zero stencil weight; points on macro faces use the per-type
// stencil variant (tables.cpp).
#include <cstdint>

#include "device.hpp"
#include "runtime_check.hpp"

namespace tetmf {

namespace {

constexpr int kThreads = 256;
#ifndef TETMF_TMA_ROWS
#define TETMF_TMA_ROWS 6
#endif
#ifndef TETMF_TMA_AHEAD
#define TETMF_TMA_AHEAD 2
#endif
constexpr int kRows = TETMF_TMA_ROWS;     // rows per block
constexpr int kPlanes = 16;               // planes per task
constexpr int kAhead = TETMF_TMA_AHEAD;   // planes in flight beyond z+1
constexpr int kSlabs = 3 + kAhead;        // ring depth: z-1, z, z+1 + kAhead in flight

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
__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, std::uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// slab geometry of plane p for the block [y0, y0+kRows): rows ya..yb
struct SlabRange {
  int ya, yb;      // yb < ya: plane has no rows in range
  int g0;          // global (macro-relative) index of row ya, rounded down to even
  int g1;          // end index (exclusive), rounded up to even
};

__device__ __forceinline__ SlabRange slab_range(int n, int p, int y0) {
  SlabRange r;
  r.ya = y0 > 0 ? y0 - 1 : 0;
  r.yb = min(y0 + kRows, n - p);
  if (p < 0 || p > n || r.yb < r.ya) {
    r.yb = r.ya - 1;
    r.g0 = r.g1 = 0;
    return r;
  }
  const int s = static_cast<int>(plane_offset(n, p) + row_offset(n, p, r.ya));
  const int e = static_cast<int>(plane_offset(n, p) + row_offset(n, p, r.yb + 1));
  r.g0 = s & ~15;  // 128-byte aligned bulk copies (macro blocks are 256-byte aligned)
  r.g1 = (e + 15) & ~15;
  return r;
}

__global__ void __launch_bounds__(kThreads, 2)
p1_stencil_tma_kernel(const double* __restrict__ xin, double* __restrict__ yout, const TmaTask* __restrict__ tasks,
                      i64 stride, int n, int slab_cap, int pad, const P1DeviceTable* __restrict__ tabs,
                      const MacroDesc* __restrict__ macros) {
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) std::uint64_t bars[kSlabs];
  const TmaTask t = tasks[blockIdx.x];
  const int y0 = t.y0;
  const double* __restrict__ X = xin + static_cast<i64>(t.macro) * stride;
  double* __restrict__ Y = yout + static_cast<i64>(t.macro) * stride;
  const double* __restrict__ tab = &tabs[macros[t.macro].group].stencil[0][0];
  const int slab_len = pad + slab_cap + pad;  // doubles per ring slot

  // zero the front pad of every slot (reads before a slab's first row)
  for (int s = 0; s < kSlabs; ++s) {
    double* base = smem + s * slab_len;
    for (int i = threadIdx.x; i < pad; i += blockDim.x) base[i] = 0.0;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlabs; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();

  // issue the bulk copy of plane p into ring slot p % kSlabs (thread 0) and
  // zero the stretch after the copied range (reads past the slab's last row)
  auto issue = [&](int p) {
    if (p > t.zb + 1) return;
    const SlabRange r = slab_range(n, p, y0);
    if (r.yb < r.ya) return;
    const int slot = ((p % kSlabs) + kSlabs) % kSlabs;
    const int len = r.g1 - r.g0;
    double* base = smem + slot * slab_len + pad;
    for (int i = threadIdx.x; i < pad; i += blockDim.x) base[len + i] = 0.0;
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const unsigned bytes = static_cast<unsigned>(len) * 8u;
      mbar_expect_tx(&bars[slot], bytes);
      bulk_g2s(base, X + r.g0, bytes, &bars[slot]);
    }
  };
  // phase parity of each slot: flips every time the slot is reused
  unsigned phase_bits = 0;
  auto wait_plane = [&](int p) {
    const SlabRange r = slab_range(n, p, y0);
    if (r.yb < r.ya) return;
    const int slot = ((p % kSlabs) + kSlabs) % kSlabs;
    mbar_wait(&bars[slot], (phase_bits >> slot) & 1u);
    phase_bits ^= 1u << slot;
  };

  double w[15];
#pragma unroll
  for (int k = 0; k < 15; ++k) w[k] = __ldg(tab + k);

  const int za = t.za, zb = t.zb;
  for (int p = za - 1; p <= za + kAhead; ++p) issue(p);
  __syncthreads();  // tail zeroing of the first slots is visible
  wait_plane(za - 1);
  wait_plane(za);
  for (int z = za; z <= zb; ++z) {
    issue(z + 1 + kAhead);  // slot of plane z-2 (read last in the previous plane)
    if (threadIdx.x < 32) wait_plane(z + 1);  // one warp polls the barrier ...
    __syncthreads();                          // ... and releases the others
    const SlabRange rc = slab_range(n, z, y0);
    const SlabRange rl = slab_range(n, z - 1, y0);
    const SlabRange ru = slab_range(n, z + 1, y0);
    const double* sc = smem + ((z % kSlabs) + kSlabs) % kSlabs * slab_len + pad;
    const double* sl = rl.yb >= rl.ya ? smem + (((z - 1) % kSlabs) + kSlabs) % kSlabs * slab_len + pad : sc;
    const double* su = ru.yb >= ru.ya ? smem + ((z + 1) % kSlabs) * slab_len + pad : sc;
    // slab-relative offset of row y0 of each plane
    const int gz0 = static_cast<int>(plane_offset(n, z) + row_offset(n, z, y0));
    const int oc = gz0 - rc.g0;
    const int ol = rl.yb >= rl.ya ? static_cast<int>(plane_offset(n, z - 1) + row_offset(n, z - 1, y0)) - rl.g0
                                  : oc;
    const int ou = ru.yb >= ru.ya ? static_cast<int>(plane_offset(n, z + 1) + row_offset(n, z + 1, y0)) - ru.g0
                                  : oc;
    const int dl = rl.yb >= rl.ya ? 1 : 0, du = ru.yb >= ru.ya ? -1 : 0;
    const int ylast = min(y0 + kRows - 1, n - z);
    for (int x = threadIdx.x; x <= n - z - y0; x += blockDim.x) {
      int lenz = n - z - y0 + 1;
      int rz = oc + x, rl0 = ol + x, ru0 = ou + x;
      // window at row y0 (row y0-1 may be the zero pad)
      double Zm0 = sc[rz - (lenz + 1)], Zm1 = sc[rz - (lenz + 1) + 1];
      double Umm = su[ru0 - (lenz + du + 1) - 1], Um0 = su[ru0 - (lenz + du + 1)];
      double Z0m = sc[rz - 1], Z00 = sc[rz];
      double L00 = sl[rl0], L01 = sl[rl0 + 1];
      const int yend = min(ylast, n - z - x);
      for (int yy = y0; yy <= yend; ++yy) {
        const double Z01 = sc[rz + 1];
        const double Zpm = sc[rz + lenz - 1], Zp0 = sc[rz + lenz];
        const double Lp0 = sl[rl0 + lenz + dl], Lp1 = sl[rl0 + lenz + dl + 1];
        const double U0m = su[ru0 - 1], U00 = su[ru0];
        const int s = x + yy + z;
        const int type = (x == 0 ? 1 : 0) | (yy == 0 ? 2 : 0) | (z == 0 ? 4 : 0) | (s == n ? 8 : 0);
        double acc;
        if (type == 0) {
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
        } else {
          const double* __restrict__ wt = tab + 16 * type;
          acc = __ldg(wt + 0) * Z00;
          acc = fma(__ldg(wt + 1), Z01, acc);
          acc = fma(__ldg(wt + 2), Z0m, acc);
          acc = fma(__ldg(wt + 3), Zp0, acc);
          acc = fma(__ldg(wt + 4), Zm0, acc);
          acc = fma(__ldg(wt + 5), U00, acc);
          acc = fma(__ldg(wt + 6), L00, acc);
          acc = fma(__ldg(wt + 7), Zm1, acc);
          acc = fma(__ldg(wt + 8), Zpm, acc);
          acc = fma(__ldg(wt + 9), L01, acc);
          acc = fma(__ldg(wt + 10), U0m, acc);
          acc = fma(__ldg(wt + 11), Lp0, acc);
          acc = fma(__ldg(wt + 12), Um0, acc);
          acc = fma(__ldg(wt + 13), Lp1, acc);
          acc = fma(__ldg(wt + 14), Umm, acc);
        }
        Y[gz0 + (rz - oc)] = acc;
        Zm0 = Z00;
        Zm1 = Z01;
        Z0m = Zpm;
        Z00 = Zp0;
        L00 = Lp0;
        L01 = Lp1;
        Umm = U0m;
        Um0 = U00;
        rz += lenz;
        rl0 += lenz + dl;
        ru0 += lenz + du;
        --lenz;
      }
    }
    __syncthreads();  // every thread is done with slot (z-1) before it is refilled
  }
}

} // namespace

// Tasks: (macro, y0, za, zb), kPlanes planes per task; planes of a block
// exist while z <= n - y0.
void build_stencil_tma_tasks(int nmacros, int n, std::vector<int>& out) {
  out.clear();
  for (int li = 0; li < nmacros; ++li)
    for (int y0 = 0; y0 <= n; y0 += kRows)
      for (int za = 0; za <= n - y0; za += kPlanes) {
        out.push_back(li);
        out.push_back(y0);
        out.push_back(za);
        out.push_back(min(za + kPlanes - 1, n - y0));
      }
}

void launch_p1_stencil_tma(const double* x, double* y, const int* d_tasks, int ntasks, i64 macro_stride, int n,
                           const P1DeviceTable* d_tables, const MacroDesc* d_macros, cudaStream_t s) {
  if (ntasks == 0) return;
  const int slab_cap = ((kRows + 2) * (n + 1) + 32 + 15) & ~15;  // rows ya..yb + alignment slack
  const int pad = ((n + 1) + 8 + 15) & ~15;                      // one row + slack before / after
  const std::size_t smem = static_cast<std::size_t>(kSlabs) * (2 * pad + slab_cap) * sizeof(double);
  static std::size_t configured = 0;
  if (smem > configured) {
    TETMF_CUDA(cudaFuncSetAttribute(p1_stencil_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
    configured = smem;
  }
  p1_stencil_tma_kernel<<<ntasks, kThreads, smem, s>>>(x, y, reinterpret_cast<const TmaTask*>(d_tasks),
                                                       macro_stride, n, slab_cap, pad, d_tables, d_macros);
  check_launch("p1_stencil_tma");
}

} // namespace tetmf

// tools/n1_element_probe.cu -- compute-only ceiling of the K3 cube body.
//
// Modes: 0 the production Gram-form element (n1_common.cuh), 1 the b'-form
// element (b'_p = beta_p + S/2 makes every mass entry linear in 2-4 b' values:
// 127 FP64 instructions per element instead of 155, but 81 table values
// instead of 38), 2 the b'-form with two cubes per lane sharing every table
// load. Measured (profiles/r2_k3_element_probe.txt): 24.2-24.6, 26.5 and 30.0
// TFLOP/s algorithmic; in the walk kernel the b'-form variants lost (13.5 and
// 14.8 ms vs 12.3 ms per C5 apply).
//
// Runs the production element code (n1_common.cuh cube_elements: six
// Gram-form elements, tables in shared memory, inputs read from a per-lane
// shared-memory row as in the fold kernel) in a loop with NO global traffic,
// NO ring copies, NO stores, NO walk logic. The FP64 rate it reaches bounds
// what any walk around this body can reach; the gap to the fold kernel is
// the walk's cost.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//        --expt-relaxed-constexpr -I../paper_2404_08371_b200/csrc -o n1_element_probe n1_element_probe.cu
#include <cstdio>

#include "n1_common.cuh"

// ---- the b'-form element (measured here, not shipped: DESIGN.md section 4, K3)
namespace tetmf {
namespace n1 {
// b'-form of the same element (K3 default, k_n1_fold.cu): with
//   b'_p = beta_p + S/2,   S = sum_m beta_m,
// the Gram form's Bt_pq = S + beta_p + beta_q = b'_p + b'_q and
// Bt_pp = 2 S + 4 beta_p = 4 b'_p, so every mass entry is LINEAR in the b' of
// the (2, 3 or 4) distinct vertices of its two edges:
//   A_ij = sa Kc_ij + sum_{p in V(i, j)} b'_p C_ij,p           (signs folded)
// 2 terms on the diagonal, 3 for edges sharing a vertex (12 pairs), 4 for
// opposite edges (3 pairs): 60 coefficients per orientation instead of the
// 4-product Gram sums plus the 10 Bt values -- 127 FP64 instructions per
// element instead of 155 (K3).
// Packed entry P (0..20) -> edges (i, j), i <= j (row-major upper triangle)
TM_HD constexpr int pk_i(int p) { return p < 6 ? 0 : p < 11 ? 1 : p < 15 ? 2 : p < 18 ? 3 : p < 20 ? 4 : 5; }
TM_HD constexpr int pk_j(int p) {
  return p < 6 ? p : p < 11 ? p - 5 : p < 15 ? p - 9 : p < 18 ? p - 12 : p < 20 ? p - 14 : 5;
}
// bit v set <=> local vertex v is an endpoint of edge pk_i(P) or pk_j(P)
TM_HD constexpr unsigned bp_vmask(int P) {
  return (1u << local_edge_vertex(pk_i(P), 0)) | (1u << local_edge_vertex(pk_i(P), 1)) |
         (1u << local_edge_vertex(pk_j(P), 0)) | (1u << local_edge_vertex(pk_j(P), 1));
}
TM_HD constexpr int bp_nv(int P) {
  return int(bp_vmask(P) & 1u) + int((bp_vmask(P) >> 1) & 1u) + int((bp_vmask(P) >> 2) & 1u) +
         int((bp_vmask(P) >> 3) & 1u);
}
// k-th distinct vertex of entry P (ascending)
TM_HD constexpr int bp_vert(int P, int k) {
  int seen = 0, v = 0;
  for (int q = 0; q < 4; ++q)
    if ((bp_vmask(P) >> q) & 1u) {
      if (seen == k) v = q;
      ++seen;
    }
  return v;
}
// offset of entry P's coefficients after the 21 Kc values
TM_HD constexpr int bp_off(int P) {
  int o = 0;
  for (int q = 0; q < P; ++q) o += bp_nv(q);
  return o;
}
constexpr int kBpRow = 21 + 60;  // Kc (21, signs folded) + C (60)
struct N1BpTable {
  double o[6][kBpRow];
};

// ---- b'-form element (tables.hpp N1BpTable): A_ij = sa Kc_ij + sum_p b'_p C_ij,p
template <int O, int P, typename Tab>
__device__ __forceinline__ void bp_pairs(const Tab& tb, const double (&bq)[4], double sa, const double (&xe)[6],
                                         double (&Y)[19]) {
  constexpr int i = pair_i(P), j = pair_j(P), nv = bp_nv(P), off = 21 + bp_off(P);
  double a = sa * tb.template get<P>();
  a = fma(bq[bp_vert(P, 0)], tb.template get<off>(), a);
  a = fma(bq[bp_vert(P, 1)], tb.template get<off + 1>(), a);
  if constexpr (nv > 2) a = fma(bq[bp_vert(P, 2)], tb.template get<off + 2>(), a);
  if constexpr (nv > 3) a = fma(bq[bp_vert(P, 3)], tb.template get<off + 3>(), a);
  constexpr int ei = cube_edge(O, i), ej = cube_edge(O, j);
  Y[ei] = fma(a, xe[j], Y[ei]);
  if constexpr (i != j) Y[ej] = fma(a, xe[i], Y[ej]);
  if constexpr (P + 1 < 21) bp_pairs<O, P + 1>(tb, bq, sa, xe, Y);
}

// two cubes per lane: every table value loaded once feeds both elements
template <int O, int P, typename Tab>
__device__ __forceinline__ void bp_pairs2(const Tab& tb, const double (&bqA)[4], double saA, const double (&xeA)[6],
                                          double (&YA)[19], const double (&bqB)[4], double saB,
                                          const double (&xeB)[6], double (&YB)[19]) {
  constexpr int i = pair_i(P), j = pair_j(P), nv = bp_nv(P), off = 21 + bp_off(P);
  const double kc = tb.template get<P>();
  double a = saA * kc, b = saB * kc;
  const double c0 = tb.template get<off>(), c1 = tb.template get<off + 1>();
  a = fma(bqA[bp_vert(P, 0)], c0, a);
  b = fma(bqB[bp_vert(P, 0)], c0, b);
  a = fma(bqA[bp_vert(P, 1)], c1, a);
  b = fma(bqB[bp_vert(P, 1)], c1, b);
  if constexpr (nv > 2) {
    const double c2 = tb.template get<off + 2>();
    a = fma(bqA[bp_vert(P, 2)], c2, a);
    b = fma(bqB[bp_vert(P, 2)], c2, b);
  }
  if constexpr (nv > 3) {
    const double c3 = tb.template get<off + 3>();
    a = fma(bqA[bp_vert(P, 3)], c3, a);
    b = fma(bqB[bp_vert(P, 3)], c3, b);
  }
  constexpr int ei = cube_edge(O, i), ej = cube_edge(O, j);
  YA[ei] = fma(a, xeA[j], YA[ei]);
  YB[ei] = fma(b, xeB[j], YB[ei]);
  if constexpr (i != j) {
    YA[ej] = fma(a, xeA[i], YA[ej]);
    YB[ej] = fma(b, xeB[i], YB[ej]);
  }
  if constexpr (P + 1 < 21) bp_pairs2<O, P + 1>(tb, bqA, saA, xeA, YA, bqB, saB, xeB, YB);
}

template <int O, typename In>
__device__ __forceinline__ void bp_setup(const In& in, bool valid, double& sa, double (&bq)[4], double (&xe)[6]) {
  constexpr int v0 = cube_vertex(O, 0), v1 = cube_vertex(O, 1), v2 = cube_vertex(O, 2), v3 = cube_vertex(O, 3);
  const double a4 = (in.template c<v0, 0>() + in.template c<v1, 0>()) +
                    (in.template c<v2, 0>() + in.template c<v3, 0>());
  sa = valid ? a4 : 0.0;
  const double b0 = valid ? in.template c<v0, 1>() : 0.0, b1 = valid ? in.template c<v1, 1>() : 0.0;
  const double b2 = valid ? in.template c<v2, 1>() : 0.0, b3 = valid ? in.template c<v3, 1>() : 0.0;
  const double S = (b0 + b1) + (b2 + b3);
  bq[0] = fma(S, 0.5, b0);
  bq[1] = fma(S, 0.5, b1);
  bq[2] = fma(S, 0.5, b2);
  bq[3] = fma(S, 0.5, b3);
#pragma unroll
  for (int e = 0; e < 6; ++e) xe[e] = 0.0;
  xe[0] = in.template x<cube_edge(O, 0)>();
  xe[1] = in.template x<cube_edge(O, 1)>();
  xe[2] = in.template x<cube_edge(O, 2)>();
  xe[3] = in.template x<cube_edge(O, 3)>();
  xe[4] = in.template x<cube_edge(O, 4)>();
  xe[5] = in.template x<cube_edge(O, 5)>();
}

template <int O, typename Tab, typename In>
__device__ __forceinline__ void element_bp2(const Tab& tb, const In& inA, double (&YA)[19], bool vA, const In& inB,
                                            double (&YB)[19], bool vB) {
  double saA, bqA[4], xeA[6], saB, bqB[4], xeB[6];
  bp_setup<O>(inA, vA, saA, bqA, xeA);
  bp_setup<O>(inB, vB, saB, bqB, xeB);
  bp_pairs2<O, 0>(tb, bqA, saA, xeA, YA, bqB, saB, xeB, YB);
}

// In: as element_gram. An invalid element gets zero coefficients -> A_e = 0.
template <int O, typename Tab, typename In>
__device__ __forceinline__ void element_bp(const Tab& tb, const In& in, double (&Y)[19], bool valid) {
  constexpr int v0 = cube_vertex(O, 0), v1 = cube_vertex(O, 1), v2 = cube_vertex(O, 2), v3 = cube_vertex(O, 3);
  const double a4 = (in.template c<v0, 0>() + in.template c<v1, 0>()) +
                    (in.template c<v2, 0>() + in.template c<v3, 0>());
  const double sa = valid ? a4 : 0.0;
  const double b0 = valid ? in.template c<v0, 1>() : 0.0, b1 = valid ? in.template c<v1, 1>() : 0.0;
  const double b2 = valid ? in.template c<v2, 1>() : 0.0, b3 = valid ? in.template c<v3, 1>() : 0.0;
  const double S = (b0 + b1) + (b2 + b3);
  const double bq[4] = {fma(S, 0.5, b0), fma(S, 0.5, b1), fma(S, 0.5, b2), fma(S, 0.5, b3)};
  double xe[6];
  xe[0] = in.template x<cube_edge(O, 0)>();
  xe[1] = in.template x<cube_edge(O, 1)>();
  xe[2] = in.template x<cube_edge(O, 2)>();
  xe[3] = in.template x<cube_edge(O, 3)>();
  xe[4] = in.template x<cube_edge(O, 4)>();
  xe[5] = in.template x<cube_edge(O, 5)>();
  bp_pairs<O, 0>(tb, bq, sa, xe, Y);
}

// Tabs: template <int O> tab() -> accessor of the orientation's N1BpTable row
template <typename Tabs, typename In>
__device__ __forceinline__ void cube_elements_bp(const Tabs& ts, const In& in, double (&Y)[19], bool vWU, bool vMid,
                                                 bool vWD) {
  element_bp<WU>(ts.template tab<WU>(), in, Y, vWU);
  element_bp<BU>(ts.template tab<BU>(), in, Y, vMid);
  element_bp<BD>(ts.template tab<BD>(), in, Y, vMid);
  element_bp<GU>(ts.template tab<GU>(), in, Y, vMid);
  element_bp<GD>(ts.template tab<GD>(), in, Y, vMid);
  element_bp<WD>(ts.template tab<WD>(), in, Y, vWD);
}

} // namespace n1
} // namespace tetmf

using namespace tetmf;
using namespace tetmf::n1;

namespace tetmf {
int n1_kernel_mode() { return 3; }
}

constexpr int kRow = 34;
constexpr int kRows = 14 + 16 + 1;
constexpr int kTabD = 6 * kBpRow;  // table area (doubles): the larger of the two forms

struct ProbeIn {
  const double* r;  // 14 arrays x kRow, this lane's column
  template <int K>
  __device__ __forceinline__ double x() const {
    return lds(r + (K % 14) * kRow + (K >= 10 ? 1 : 0));
  }
  template <int V, int W>
  __device__ __forceinline__ double c() const {
    return lds(r + (10 + 2 * W + (V >> 2)) * kRow + (V & 1));
  }
};

struct SmemBp {
  const double* p;
  template <int O>
  __device__ __forceinline__ SmemTab tab() const { return SmemTab{p + O * kBpRow}; }
};

// MODE 0: Gram form, 1 cube per lane; 1: b'-form, 1 cube; 2: b'-form, 2 cubes sharing table loads
template <int WARPS, int MINB, int MODE>
__global__ void __launch_bounds__(32 * WARPS, MINB) probe(const N1GramTable* g, double* out, int iters) {
  extern __shared__ __align__(16) double sm[];
  N1GramTable& sg = *reinterpret_cast<N1GramTable*>(sm);
  double* ring = sm + kTabD + (threadIdx.x >> 5) * kRows * kRow;
  for (int i = threadIdx.x; i < kTabD; i += blockDim.x) sm[i] = 0.01 * (1 + (i * 7) % 13);
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < kRows * kRow; i += 32) ring[i] = 1.0 + 1e-3 * (i % 17);
  __syncthreads();
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    asm volatile("" ::: "memory");
    const int off = (it & 15) * kRow;  // iteration-dependent rows: nothing can be hoisted
    double Y[19], Z[19];
#pragma unroll
    for (int k = 0; k < 19; ++k) Y[k] = Z[k] = 0.0;
    const ProbeIn in{ring + lane + off}, in2{ring + lane + off + kRow};
    if constexpr (MODE == 3) {
      const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(sm));
      cube_elements_zw(SmemTabs3{opaque_u32(a), opaque_u32(a), opaque_u32(a)}, in, Z);
    } else if constexpr (MODE == 0) {
      cube_elements(SmemTabs{sg}, in, Y, true, true, true);
    } else if constexpr (MODE == 1) {
      cube_elements_bp(SmemBp{sm}, in, Y, true, true, true);
    } else {
      const SmemBp t{sm};
      element_bp2<WU>(t.tab<WU>(), in, Y, true, in2, Z, true);
      element_bp2<BU>(t.tab<BU>(), in, Y, true, in2, Z, true);
      element_bp2<BD>(t.tab<BD>(), in, Y, true, in2, Z, true);
      element_bp2<GU>(t.tab<GU>(), in, Y, true, in2, Z, true);
      element_bp2<GD>(t.tab<GD>(), in, Y, true, in2, Z, true);
      element_bp2<WD>(t.tab<WD>(), in, Y, true, in2, Z, true);
    }
#pragma unroll
    for (int k = 0; k < 19; ++k) acc += Y[k] + Z[k];
  }
  if (acc == 1.2345) out[0] = acc;
}

template <int WARPS, int MINB, int MODE>
void run(const N1GramTable* g, double* out, int sms) {
  const int smem = kTabD * 8 + WARPS * kRows * kRow * 8;
  cudaFuncSetAttribute(probe<WARPS, MINB, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int blocks = sms * MINB, iters = 2000;
  probe<WARPS, MINB, MODE><<<blocks, 32 * WARPS, smem>>>(g, out, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<WARPS, MINB, MODE><<<blocks, 32 * WARPS, smem>>>(g, out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, probe<WARPS, MINB, MODE>);
  const double flop = 264.0 * 6 * (MODE == 2 ? 2 : 1) * iters * 32.0 * WARPS * blocks;  // SURVEY 8(d) count
  printf("mode %d (%s) warps/CTA %d CTAs/SM %d (%2d warps/SM, %3d regs, spill %zu): %6.2f TFLOP/s algorithmic (%s)\n",
         MODE, MODE == 3 ? "ZW, 1 cube" : MODE == 0 ? "Gram, 1 cube" : MODE == 1 ? "b', 1 cube" : "b', 2 cubes", WARPS,
         MINB, WARPS * MINB, fa.numRegs, fa.localSizeBytes, flop / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  N1GramTable h;
  for (int o = 0; o < 6; ++o)
    for (int i = 0; i < kGramRow; ++i) h.o[o][i] = 0.01 * (1 + (o * 7 + i) % 13);
  N1GramTable* g;
  double* out;
  cudaMalloc(&g, sizeof(h));
  cudaMalloc(&out, 8);
  cudaMemcpy(g, &h, sizeof(h), cudaMemcpyHostToDevice);
  run<4, 3, 3>(g, out, sms);
  run<4, 4, 3>(g, out, sms);
  run<4, 3, 0>(g, out, sms);
  run<4, 4, 0>(g, out, sms);
  run<4, 3, 1>(g, out, sms);
  run<4, 4, 1>(g, out, sms);
  run<4, 2, 2>(g, out, sms);
  run<2, 4, 2>(g, out, sms);
  run<4, 3, 2>(g, out, sms);
  return 0;
}

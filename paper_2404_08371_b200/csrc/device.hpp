// device.hpp -- device-side descriptors and kernel launchers (sm_100a).
//
// Kernels:
//   K1 p1_stencil     P1 -Laplace via the assembled 15-point stencil
//   K2 p1k_cubes      P1 -div(k grad), k in P1, cube-wise element loop
//   K3 n1_cubes       N1 alpha curl curl + beta, cube-wise element loop
//   K4 interface_sum  sum of macro copies of shared carriers, write-back
//   fill / permute    seeded inputs, coefficients, reference numbering I/O
#pragma once

#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

#include "lattice.hpp"
#include "tables.hpp"

namespace tetmf {

// One stored macro as the kernels see it.
struct MacroDesc {
  int group;         // geometry group (index into the table array)
  int dmask;         // bit k: carriers with support mask k are Dirichlet (Topology::dirichlet_mask)
  i64 V0[3];         // integer world coords (scaled by n * D) of local vertex 0
  i64 E[3][3];       // integer edge vectors v_{c+1} - v_0 (scaled by D), E[c][r]
  double X0[3];      // world coords of local vertex 0
  double dX[3][3];   // world edge vectors, dX[c][r]
};

// In-kernel exchange puts (Exchange::fused_begin, exchange.hpp): a kernel that
// stores y at storage slot j also stores it into every peer receive window
// entry the exchange would pack slot j into: entries e = first[j],
// chain[e], ... (-1 ends), each at win[dst[e] >> 48][dst[e] & (2^48 - 1)].
// The window bases travel in the kernel parameters (no dependent load).
// first == nullptr: no puts.
constexpr int kFusedMaxPeers = 16;
struct FusedPut {
  const int* first = nullptr;
  const int* chain = nullptr;
  const i64* dst = nullptr;
  double* win[kFusedMaxPeers] = {};
};

struct CoeffSpec {
  int which;         // 0 alpha = 1+x^2+y^2, 1 beta = 2+sin(pi z), 2 k, 3 constant
  double value;      // for which == 3
};

// space: 0 P1, 1 P2, 2 ND1 (Space enum values)
void launch_fill_seeded(double* out, const MacroDesc* d_macros, int nmacros, i64 macro_stride, int n,
                        int space, i64 class_stride, std::uint64_t seed, bool dirichlet, cudaStream_t s);
// P1 (class_stride 0) or P2 (class_stride > 0: vertex block + edge midpoints)
void launch_fill_coeff(double* out, const MacroDesc* d_macros, int nmacros, i64 macro_stride, int n,
                       CoeffSpec spec, cudaStream_t s, i64 class_stride = 0);
void launch_import_ref(double* lat, const i64* map, i64 total, const double* ref, cudaStream_t s);
void launch_export_ref(const double* lat, const i64* map, i64 total, double* ref, cudaStream_t s);
void launch_interface_sum(double* y, const i64* offsets, const i64* copies, i64 ngroups, cudaStream_t s,
                          bool signed_values = true);
// one rank's owned slice [lo, hi) of the reference numbering (multi-rank I/O)
void launch_import_ref_range(double* lat, const i64* map, i64 total, const double* ref, i64 lo, i64 hi,
                             cudaStream_t s);
void launch_export_ref_range(const double* lat, const i64* map, i64 total, double* ref, i64 lo, i64 hi,
                             cudaStream_t s);
// ghost update of rank-local interface groups: copies := owner copy (signed)
void launch_interface_owner(double* y, const i64* offsets, const i64* copies, i64 ngroups, cudaStream_t s);
// K4 with two-copy groups packed as 32-bit pairs (one thread per pair) and
// the remaining groups in CSR form, one launch; same sums as interface_sum
void launch_interface_sum_packed(double* y, const unsigned* pairs, i64 npairs, const i64* offsets, const i64* copies,
                                 i64 nrest, cudaStream_t s, bool signed_values = true);
void launch_axpy(double* y, const double* x, double a, i64 count, cudaStream_t s);

void launch_p1_stencil(const double* x, double* y, const MacroDesc* d_macros, int nmacros, i64 macro_stride,
                       int n, const P1DeviceTable* d_tables, cudaStream_t s);
// K1 default: two-plane row walk (k_p1_stencil2.cu)
void build_stencil2_tasks(int nmacros, int n, std::vector<int>& out);
void launch_p1_stencil2(const double* x, double* y, const int* d_tasks, int ntasks, i64 macro_stride, int n,
                        const P1DeviceTable* d_tables, const MacroDesc* d_macros, cudaStream_t s);
// K1 variant 5: interior-only row walk + face pass, L2 bulk prefetch (k_p1_stencil5.cu)
void build_stencil5_tasks(int nmacros, int n, std::vector<int>& out);
void launch_p1_stencil5(const double* x, double* y, const int* d_tasks, int ntasks, i64 macro_stride, int n,
                        int nmacros, const P1DeviceTable* d_tables, const MacroDesc* d_macros, cudaStream_t s);
// K1 variant 6: shared-memory boxes filled by per-row TMA bulk copies (k_p1_stencil5.cu)
void build_stencil6_tasks(int nmacros, int n, std::vector<int>& out);
// zrange (optional, slab partition): per local macro {za, zb}, the planes this
// rank computes (the task list holds only boxes of those planes); fp (optional,
// put-mode exchange): the kernel also issues the exchange's puts of the values it stores
void launch_p1_stencil6(const double* x, double* y, const int* d_tasks, int ntasks, i64 macro_stride, int n,
                        int nmacros, const P1DeviceTable* d_tables, const MacroDesc* d_macros, cudaStream_t s,
                        const int* zrange = nullptr, const FusedPut& fp = FusedPut{});
// K1 variant 10: variant 6's boxes in a persistent double-buffered CTA loop (k_p1_stencil5.cu)
void launch_p1_stencil10(const double* x, double* y, const int* d_tasks, int ntasks, i64 macro_stride, int n,
                         int nmacros, const P1DeviceTable* d_tables, const MacroDesc* d_macros, cudaStream_t s);
// K3 v2: cube walk, two layer-parity passes, one launch per geometry group
void build_n1_tasks(const std::vector<int>& local_macros, int n, int parity, std::vector<int>& out, int chunk);
// K3 default: folded cube walk (k_n1_fold.cu); same task-list / launch contract
void build_n1_fold_tasks(const std::vector<int>& local_macros, int n, int parity, std::vector<int>& out, int chunk);
int n1_fold_chunk(const std::vector<int>& local_macros, int n, int sms);
void pad_n1_fold_tasks(std::vector<int>& tasks);
void launch_n1_fold(const N1GramTable* gram, const MacroDesc* macros, int pass, const double* x, const double* alpha,
                    const double* beta, double* y, const int* d_tasks, int ntasks, i64 macro_stride,
                    i64 class_stride, i64 coeff_stride, int n, int rule, cudaStream_t s, int chunk);
int n1_kernel_mode();
// K2 default: cube walk with per-cube edge weights (k_p1k_cube.cu)
void build_p1k_cube_tasks(int nmacros, int n, std::vector<int>& out, int chunk);
int p1k_cube_chunk(int nmacros, int n, int sms);  // rows = layers per task (16, 8 or 4 by task count)
void launch_p1k_cube(const double* x, const double* k, double* y, const int* d_tasks, int ntasks, i64 macro_stride,
                     int n, const P1DeviceTable* d_tables, const MacroDesc* d_macros, cudaStream_t s, int chunk);
// K2 variant 3 (round-2 first kernel): the gather walked along y with register windows (k_p1k_gather.cu)
void build_p1k_walk_tasks(int nmacros, int n, std::vector<int>& out);
void launch_p1k_walk(const double* x, const double* k, double* y, const int* d_tasks, int ntasks, i64 macro_stride,
                     int n, const P1DeviceTable* d_tables, const MacroDesc* d_macros, cudaStream_t s);
// K2 round 1: per-point gather over the 24 incident elements (k_p1k_gather.cu)
void build_p1k_tasks(int nmacros, int n, std::vector<int>& out);
void launch_p1k_gather(const double* x, const double* k, double* y, const int* d_tasks, int ntasks, i64 macro_stride,
                       int n, const P1DeviceTable* d_tables, const MacroDesc* d_macros, cudaStream_t s);
void launch_p1k_cubes(const double* x, const double* k, double* y, const MacroDesc* d_macros, int nmacros,
                      i64 macro_stride, int n, const P1DeviceTable* d_tables, cudaStream_t s);
void launch_n1_cubes(const double* x, const double* alpha, const double* beta, double* y,
                     const MacroDesc* d_macros, int nmacros, i64 macro_stride, i64 class_stride,
                     i64 coeff_stride, int n, const N1DeviceTable* d_tables, cudaStream_t s);

// P2V apply, first version (k_p2v.cu): cube loop + FP64 atomics into a zeroed y
// P2V operator diagonal per stored macro copy (k_p2v.cu)
void launch_p2v_diagonal(const double* k, double* d, const MacroDesc* d_macros, int nmacros, i64 macro_stride,
                         i64 class_stride, int n, const P2VTable* d_tables, int rule, cudaStream_t s);
// P2V factored cube kernel (default; k_p2v.cu v2)
// rule: 0 exact, 1..3 quadrature(rule) (under-integration; forms.cpp:12 "U")
// P2V default (exact rule): folded cube walk (k_p2v_fold.cu), one layer per
// task, parity passes
void build_p2v_fold_tasks(const std::vector<int>& local_macros, int n, int parity, std::vector<int>& out, int chunk);
void pad_p2v_fold_tasks(std::vector<int>& tasks);
int p2v_fold_chunk(const std::vector<int>& local_macros, int n, int sms);
void launch_p2v_fold(const P2VTable* tabs, const MacroDesc* macros, int pass, const double* x, const double* k,
                     double* y, const int* d_tasks, int ntasks, i64 macro_stride, i64 class_stride, int n,
                     cudaStream_t s, int chunk);
void launch_p2v_cubes2(const double* x, const double* k, double* y, const MacroDesc* d_macros, int nmacros,
                       i64 macro_stride, i64 class_stride, int n, const P2VTable* d_tables, int rule,
                       cudaStream_t s);
void launch_p2v_cubes(const double* x, const double* k, double* y, const MacroDesc* d_macros, int nmacros,
                      i64 macro_stride, i64 class_stride, int n, const P2VTable* d_tables, cudaStream_t s);

// operator diagonals per stored macro copy (k_diagonal.cu, k_p1k_gather.cu)
void launch_p1_diagonal(double* d, const MacroDesc* d_macros, int nmacros, i64 macro_stride, int n,
                        const P1DeviceTable* d_tables, cudaStream_t s);
void launch_p1k_diagonal(const double* k, double* d, const int* d_tasks, int ntasks, i64 macro_stride, int n,
                         const P1DeviceTable* d_tables, const MacroDesc* d_macros, cudaStream_t s);
void launch_n1_diagonal(double* d, const double* alpha, const double* beta, const MacroDesc* d_macros, int nmacros,
                        i64 macro_stride, i64 class_stride, i64 coeff_stride, int n, const N1GramTable* d_gram,
                        int rule, cudaStream_t s);

// P1 <-> ND1 discrete gradient and its transpose (k_transfer.cu)
void launch_gradient(const double* phi, double* u, int nmacros, i64 stride_nd1, i64 class_stride, i64 stride_p1,
                     int n, cudaStream_t s);
void launch_gradient_t(const double* u, double* phi, int nmacros, i64 stride_nd1, i64 class_stride, i64 stride_p1,
                       int n, const unsigned char* d_nd1_slot_table, cudaStream_t s);

// FP64 DFMA-chain peak probe (used by bench.py to measure the FP64 roof).
void launch_fp64_peak(double* out, int blocks, int threads, int iters, cudaStream_t s);

} // namespace tetmf

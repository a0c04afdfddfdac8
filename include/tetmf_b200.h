/* tetmf_b200.h -- C ABI of the B200-native matrix-free operator apply.
 *
 * Drop-in boundary for the reference's hot path. Plain
 * pointers and sizes only; no C++ exceptions cross this boundary.
 *
 * Reference interfaces replaced:
 *   tetmf_ctx_create / tetmf_ctx_create_dist
 *       FormSystem(Form, const MacroMesh&, int level) inputs
 *       (forms.hpp:46; mesh_by_name mesh.cpp:177-181)
 *   tetmf_fn_*
 *       FieldVector (fespace.hpp:69-77) as level-indexed, per-macro lattice
 *       storage on the device; tetmf_fn_import_ref / _export_ref convert
 *       from / to the reference's global numbering with ND1 signs
 *       (DoFIndexer::build fespace.cpp:182-307, fill_map :320-376)
 *   tetmf_fn_fill_coefficient
 *       interpolate(indexer, f) for the BASELINE coefficients
 *       (fespace.cpp:494-506)
 *   tetmf_op_create
 *       FormSystem(Form, ...) + coefficient binding (forms.cpp:43-67)
 *   tetmf_apply (update = TETMF_REPLACE)
 *       FieldVector FormSystem::apply(v, coeffs, rule) const
 *       (forms.hpp:65-66, forms.cpp:195-255): w = A v, exact integration
 *   tetmf_apply (update = TETMF_ADD)
 *       generated kernel_apply(v, w, c0, c1, ..., jp, tab), w += A v
 *       (ir.cpp:732-734)
 *   tetmf_apply_ref_host
 *       FormSystem::apply with host FieldVectors in reference numbering
 *       (H2D, permute, apply, permute, D2H)
 *
 * Conventions: return 0 on success, else a TETMF_E* code with a message in
 * tetmf_last_error() (thread-local). The library owns device memory; host
 * pointers are borrowed for the duration of a call. Calls are ordered on the
 * context's CUDA stream; tetmf_apply does not synchronize. One host process
 * per GPU; multi-rank contexts exchange interface sums over NCCL.
 */
#ifndef TETMF_B200_H
#define TETMF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef struct tetmf_ctx tetmf_ctx;
typedef struct tetmf_fn tetmf_fn;
typedef struct tetmf_op tetmf_op;
typedef struct tetmf_loopback tetmf_loopback;

enum {
  TETMF_OK = 0,
  TETMF_EINVAL = 1,    /* std::invalid_argument class (forms.cpp:58-67) */
  TETMF_EINTERNAL = 2, /* std::logic_error class (fespace.cpp:330,400) */
  TETMF_EDEVICE = 3,   /* CUDA failure */
  TETMF_ECOMM = 4      /* NCCL failure */
};

/* spaces: reference enum Space (fespace.hpp:15) */
enum { TETMF_SPACE_P1 = 0, TETMF_SPACE_P2 = 1, TETMF_SPACE_ND1 = 2 };
/* forms: reference enum Form (forms.hpp:16) + config 2's P1 -div(k grad) */
enum { TETMF_FORM_P1 = 0, TETMF_FORM_P2V = 1, TETMF_FORM_N1 = 2, TETMF_FORM_P1K = 3 };
enum { TETMF_REPLACE = 0, TETMF_ADD = 1 };
/* coefficients of the BASELINE configs (nodal P1 interpolation) */
enum { TETMF_COEFF_ALPHA = 0, TETMF_COEFF_BETA = 1, TETMF_COEFF_K = 2, TETMF_COEFF_CONST = 3 };

const char* tetmf_last_error(void);
const char* tetmf_version(void);

/* mesh_desc: "single-tet", "cube6", "cubes<K>", "cubes<Kx>x<Ky>x<Kz>" or a
 * reference-format mesh file path. device < 0 creates a planning-only
 * context (host index machinery, no CUDA calls). */
int tetmf_ctx_create(const char* mesh_desc, int device, tetmf_ctx** out);
/* One rank of a multi-GPU context: macros are partitioned contiguously by
 * id; nccl_unique_id (128 bytes from tetmf_nccl_unique_id) may be NULL for
 * nranks == 1 or planning-only contexts. */
int tetmf_ctx_create_dist(const char* mesh_desc, int device, int rank, int nranks,
                          const void* nccl_unique_id, tetmf_ctx** out);
/* partitions of the macro mesh over ranks:
 * MACRO  whole macros, contiguous by id (every form);
 * SLAB   (macro, z-slab) units of the P1 lattice points, cuts on multiples of
 *        8 planes, balanced point counts, every rank stores every macro and
 *        computes y on its units only (x read on ghost planes from its own
 *        copy) -- the strong-scaling partition of config 4; P1 -Laplace
 *        apply only (TETMF_EINVAL for other forms, dot and solvers). */
enum { TETMF_PARTITION_MACRO = 0, TETMF_PARTITION_SLAB = 1 };
int tetmf_ctx_create_dist_part(const char* mesh_desc, int device, int rank, int nranks,
                               const void* nccl_unique_id, int partition, tetmf_ctx** out);
/* In-memory macro mesh: the MacroMesh of FormSystem(Form, const MacroMesh&,
 * int level) (forms.hpp:46; mesh.hpp:37-56): vertices[3 * num_vertices]
 * (x, y, z per vertex), tets[4 * num_tets] (vertex ids; the local vertex order
 * defines the lattice axes, as in the reference). Validated like
 * MacroMesh::validate (mesh.cpp:76-94: ids in range, positive volumes, faces
 * shared by at most two tets) -> TETMF_EINVAL. The arrays are copied. */
int tetmf_ctx_create_mesh(const double* vertices, int num_vertices, const int* tets, int num_tets, int device,
                          tetmf_ctx** out);
/* Loopback group: nranks "virtual ranks" of ONE process on ONE device, each
 * driven by its own host thread (collective calls -- apply, dot, solvers --
 * must be made by every rank of the group). The interface exchange and the
 * solver all-gather run as device-to-device copies between the virtual
 * ranks' buffers, ordered by CUDA events and host barriers; the pack /
 * combine / interface-sum kernels are the multi-GPU path's own. No kernel
 * waits on another, so this is safe on a single GPU. Replaces nothing in the
 * reference (its parallel layer is HyTeG MPI); it is the
 * single-device test mode of the multi-rank apply. */
int tetmf_loopback_create(int nranks, tetmf_loopback** out);
int tetmf_loopback_destroy(tetmf_loopback* group);
int tetmf_ctx_create_loopback(const char* mesh_desc, int device, tetmf_loopback* group, int rank, int partition,
                              tetmf_ctx** out);
/* one line describing the context's transport ("nccl rank r of N ...",
 * "loopback virtual rank r of N ...", "single rank") */
int tetmf_ctx_transport_info(const tetmf_ctx* ctx, char* buf, int buflen);
int tetmf_ctx_destroy(tetmf_ctx* ctx);
/* All later work of the context is ordered on cuda_stream; NULL selects the
 * context's own (non-blocking) stream again. Work queued on the previous
 * stream is ordered before the new stream's later work (event + wait), so a
 * switch never races with an apply still running. To use the legacy default
 * stream pass cudaStreamLegacy ((void*)1). */
int tetmf_ctx_set_stream(tetmf_ctx* ctx, void* cuda_stream);
/* Interface exchange of a partitioned context (no effect on one rank):
 * TETMF_EXCHANGE_SENDRECV (default) packs into a send buffer and moves it with
 * the transport (grouped ncclSend / ncclRecv, or loopback copies);
 * TETMF_EXCHANGE_PUT stores every value straight into the peer's receive
 * window from the pack kernel (NVLink stores through NCCL symmetric windows /
 * LSA pointers, NCCL device API; plain device pointers between loopback
 * virtual ranks) followed by a barrier (LSA barrier kernel / host barrier).
 * In the (macro, z-slab) partition the P1 -Laplace stencil kernel (the
 * default K1) issues those stores itself as it computes each shared value --
 * compute and transfer in one kernel, no pack launch (measured faster there;
 * with whole-macro ranks the pack kernel measured faster and is used).
 * TETMF_EXCHANGE_PUT_PACK: always the pack kernel; TETMF_EXCHANGE_PUT_FUSED:
 * the in-kernel puts in every partition (A/B).
 * Collective; set before the context's first level is used (TETMF_EINVAL
 * after). With NCCL the put windows are registered and deregistered
 * collectively: every rank creates its levels and destroys the context in
 * the same order. Replaces the halo-exchange transport of HyTeG's MPI layer
 * (PAPER.md:404-405), which the reference does not contain. */
#define TETMF_EXCHANGE_SENDRECV 0
#define TETMF_EXCHANGE_PUT 1
#define TETMF_EXCHANGE_PUT_PACK 2
#define TETMF_EXCHANGE_PUT_FUSED 3
int tetmf_ctx_set_exchange_mode(tetmf_ctx* ctx, int mode);
int tetmf_ctx_synchronize(tetmf_ctx* ctx);
int tetmf_ctx_num_macros(const tetmf_ctx* ctx, int* global_count, int* local_count);
int tetmf_ctx_local_macros(const tetmf_ctx* ctx, int* out /* local_count */);
int tetmf_nccl_unique_id(void* out128);

int tetmf_fn_create(tetmf_ctx* ctx, int space, tetmf_fn** out);
int tetmf_fn_destroy(tetmf_fn* fn);
/* storage entries on this rank at a level (allocates the level) */
int tetmf_fn_size(tetmf_fn* fn, int level, int64_t* entries);
int tetmf_fn_device_ptr(tetmf_fn* fn, int level, double** ptr);
/* layout-independent seeded values; dirichlet_zero zeroes
 * carriers on the domain boundary (interior() == 0, fespace.hpp:95-96) */
int tetmf_fn_fill_seeded(tetmf_fn* fn, int level, uint64_t seed, int dirichlet_zero);
int tetmf_fn_fill_coefficient(tetmf_fn* fn, int level, int which, double value);
/* raw storage (this library's layout) <-> host */
int tetmf_fn_upload(tetmf_fn* fn, int level, const double* host, int64_t entries);
int tetmf_fn_download(tetmf_fn* fn, int level, double* host, int64_t entries);
/* reference global numbering (FieldVector order, ND1 key-ascending signs) */
int tetmf_fn_num_ref_dofs(tetmf_fn* fn, int level, int64_t* count);
int tetmf_fn_import_ref(tetmf_fn* fn, int level, const double* host_ref);
int tetmf_fn_export_ref(tetmf_fn* fn, int level, double* host_ref);

/* Multi-rank I/O in reference numbering (macro partition): this rank's owned
 * slice [lo, hi) of the global FieldVector -- the carriers whose owner macro
 * (lowest sharing macro id, fespace.cpp:216-231) is local; contiguous because
 * the reference numbering sorts by owner macro first (fespace.cpp:283-295).
 * import_ref_owned sets every local copy of an owned carrier and then the
 * ghost copies (carriers owned elsewhere) from their owners: collective over
 * the ranks. export_ref_owned writes the owned slice. Together they are
 * FormSystem::apply's host I/O for one rank of a distributed vector. */
int tetmf_fn_ref_owned_range(tetmf_fn* fn, int level, int64_t* lo, int64_t* hi);
int tetmf_fn_import_ref_owned(tetmf_fn* fn, int level, const double* host_owned);
int tetmf_fn_export_ref_owned(tetmf_fn* fn, int level, double* host_owned);

int tetmf_op_create(tetmf_ctx* ctx, int form, tetmf_fn* const* coeffs, int ncoeffs, tetmf_op** out);
int tetmf_op_destroy(tetmf_op* op);
int tetmf_apply(tetmf_op* op, const tetmf_fn* src, tetmf_fn* dst, int level, int update);
/* Drop-in for FormSystem::apply: host vectors in reference numbering. src
 * and dst are scratch functions of the operator's space (contents
 * overwritten); synchronizes before returning. */
int tetmf_apply_ref_host(tetmf_op* op, tetmf_fn* src, tetmf_fn* dst, int level, const double* host_v,
                         double* host_w);
/* The same for a batch of nvec independent host vectors (FormSystem::apply
 * called nvec times): w_k = A v_k, all in reference numbering, pinned host
 * memory recommended. Pipelined over three streams: the host->device copy
 * of v_{k+1} and the device->host copy of w_{k-1} overlap the permute /
 * apply / permute of v_k (two device staging buffers each way). Every w_k is
 * complete when the call returns (synchronizes). */
int tetmf_apply_ref_host_batch(tetmf_op* op, tetmf_fn* src, tetmf_fn* dst, int level, int nvec,
                               const double* const* host_v, double* const* host_w);

/* Dirichlet-masked matrix-free CG (the reference's
 * cg_solve, which its sources do not contain). Homogeneous
 * Dirichlet conditions on the reference's boundary carriers (interior() == 0,
 * fespace.hpp:95-96). Inner products count every carrier once (owner copy)
 * and skip Dirichlet carriers; all ranks see identical scalars. */
/* *out = sum over interior carriers of a * b (collective over ranks) */
int tetmf_fn_dot(const tetmf_fn* a, const tetmf_fn* b, int level, double* out);
/* zero the Dirichlet (boundary) carriers of fn */
int tetmf_fn_mask_dirichlet(tetmf_fn* fn, int level);
/* solve P A P x = P b for x (initial guess in, solution out, Dirichlet
 * carriers 0); stops at ||r|| <= rtol ||r0|| or max_iter iterations.
 * iterations / rel_residual / converged may be NULL. */
int tetmf_cg_solve(tetmf_op* op, const tetmf_fn* b, tetmf_fn* x, int level, double rtol, int max_iter,
                   int* iterations, double* rel_residual, int* converged);

/* operator diagonal d_i = A_ii of the level (every interface copy holds the
 * full sum, the inverse-diagonal of Jacobi / Chebyshev
 * smoothing): the diagonal of the reference's assembled FormSystem operator */
int tetmf_op_diagonal(tetmf_op* op, tetmf_fn* diag, int level);
/* tetmf_cg_solve with Jacobi preconditioning by diag (from tetmf_op_diagonal;
 * NULL = unpreconditioned) */
int tetmf_pcg_solve(tetmf_op* op, const tetmf_fn* b, tetmf_fn* x, const tetmf_fn* diag, int level, double rtol,
                    int max_iter, int* iterations, double* rel_residual, int* converged);

/* P1 <-> ND1 discrete gradient (the transfer of the
 * hybrid smoother): nd1 = G p1 with (G p)_e = p(tip) - p(base) along the
 * edge (the ND1 interpolant of grad p); p1 = G^T nd1 (its transpose) */
int tetmf_gradient(const tetmf_fn* p1, tetmf_fn* nd1, int level);
int tetmf_gradient_transpose(const tetmf_fn* nd1, tetmf_fn* p1, int level);

/* Chebyshev-Jacobi smoothing (the smoother of the paper's
 * multigrid): *lambda_max = largest eigenvalue of D^-1 A
 * (power iteration); degree Chebyshev steps on [lambda_max / eig_ratio,
 * lambda_max] update x towards A x = b */
int tetmf_estimate_lambda_max(tetmf_op* op, const tetmf_fn* diag, int level, int iterations, double* lambda_max);
int tetmf_chebyshev_smooth(tetmf_op* op, const tetmf_fn* diag, const tetmf_fn* b, tetmf_fn* x, int level,
                           int degree, double lambda_max, double eig_ratio);

/* instrumentation: CUDA events around the element kernel of every apply on
 * the context stream (enable resets the totals); stats synchronize. */
int tetmf_op_profile(tetmf_op* op, int enable);
/* 0 = optimized kernels (default); 1 = first-version kernels (A/B tests);
 * P1 -Laplace also 5, 7, 8, 9, 10 = alternative K1 kernels kept for A/B runs
 * (bitwise equal to the default); P1K 2 = the round-1
 * per-point gather. Other values: TETMF_EINVAL at the next apply. */
int tetmf_op_set_variant(tetmf_op* op, int variant);

/* Integration rule of tetmf_apply / tetmf_op_diagonal: 0 = exact (default;
 * equals FormSystem::reference_apply, forms.cpp:257-260), d = 1..6 = the
 * reference's quadrature(d) (quadrature.cpp:135-147), i.e.
 * FormSystem::apply(v, coeffs, quadrature(d)) (forms.hpp:65-66). P1 and P1K
 * integrate exactly under every rule; N1 is under-integrated for d <= 2 and
 * P2V for d <= 3 (the paper's "U" optimization, forms.cpp:12). TETMF_EINVAL
 * for d outside 0..6. */
int tetmf_op_set_quadrature(tetmf_op* op, int degree);
int tetmf_op_kernel_stats(tetmf_op* op, double* total_ms, int64_t* launches);
/* Negative control ("deliberately corrupted table"): adds delta
 * to entry `index` (flat double index over all geometry groups) of the
 * level's per-orientation table image the element kernel reads. Test hook. */
int tetmf_op_debug_perturb_table(tetmf_op* op, int level, int64_t index, double delta);
/* kernels launched by this library so far (process-wide) */
int tetmf_launch_count(int64_t* count);

/* pinned host memory for the end-to-end path */
int tetmf_host_alloc(void** ptr, int64_t bytes);
int tetmf_host_free(void* ptr);

/* ---- host-side planning hooks (no GPU needed; used by CPU tests) ---- */
/* reference numbering map of the stored macros (layout entries) */
int tetmf_plan_ref_map(tetmf_ctx* ctx, int space, int level, int64_t* out, int64_t entries,
                       int64_t* num_ref_dofs);
int tetmf_plan_layout(tetmf_ctx* ctx, int space, int level, int64_t* macro_stride, int64_t* class_stride);
/* interior (non-Dirichlet) mask in reference numbering, as the solver and the
 * seeded Dirichlet fill use it (FieldVector interior(), fespace.hpp:95-96) */
int tetmf_plan_interior(tetmf_ctx* ctx, int space, int level, unsigned char* out, int64_t num_ref_dofs);
/* rank-local interface groups: sizes, then CSR arrays */
int tetmf_plan_local_groups(tetmf_ctx* ctx, int space, int level, int64_t* ngroups, int64_t* ncopies,
                            int64_t* offsets, int64_t* copies);
/* cross-rank exchange plan: sizes, then arrays (any pointer may be NULL) */
int tetmf_plan_exchange(tetmf_ctx* ctx, int space, int level, int* npeers, int64_t* nsend, int64_t* nrecv,
                        int64_t* ngroups, int64_t* nentries, int* peers, int64_t* send_offsets,
                        int64_t* recv_offsets, int64_t* send_index, int64_t* group_offsets,
                        int64_t* group_entries);
/* slab partition (TETMF_PARTITION_SLAB) of a mesh with num_macros macros at
 * a level: rank's units as (macro, za, zb) triples, planes za <= z < zb */
int tetmf_plan_slab_units(int num_macros, int level, int nranks, int rank, int* nunits, int* units);
/* the product's pack / combine / local-sum bodies run on host arrays */
int tetmf_host_local_sum(const int64_t* offsets, const int64_t* copies, int64_t ngroups, double* y);
int tetmf_host_pack(const double* y, const int64_t* send_index, int64_t nsend, double* send);
/* put mode (TETMF_EXCHANGE_PUT): where this rank's values start in each
 * peer's receive buffer, from the group's send-count matrix
 * counts[src * nranks + dst]; and, per send entry, the target peer slot and
 * position (the put kernel's addressing) */
int tetmf_host_put_offsets(int nranks, const int64_t* counts, int rank, int npeers, const int* peers,
                           int64_t* peer_off);
int tetmf_host_put_targets(int npeers, const int64_t* send_offsets, const int64_t* peer_off, int64_t* dst_off,
                           int* dst_peer);
/* one-GPU check of the NCCL device-API put channel: a 1-rank communicator on
 * `device`, symmetric window registration, device communicator, `rounds` LSA
 * barrier kernels (no peers); TETMF_ECOMM with NCCL's message on failure */
int tetmf_selftest_nccl_put(int device, int rounds);
int tetmf_host_combine(double* y, const double* recv, const int64_t* group_offsets,
                       const int64_t* group_entries, int64_t ngroups);

/* element matrix (nloc x nloc, local basis in reference orientation, row =
 * test) assembled from this library's per-orientation tables; coefficient
 * vertex values c0/c1 (alpha/beta for N1, k for P1K) -- checks the tables
 * against FormSystem::local_matrix (forms.cpp:133-177) */
int tetmf_plan_local_matrix(tetmf_ctx* ctx, int form, int level, int macro, int orientation,
                            const double* c0, const double* c1, double* out);

/* P1 15-point stencil variants of a macro: 16 point types x 15 weights */
int tetmf_plan_stencil(tetmf_ctx* ctx, int level, int macro, double* out);

/* FP64 DFMA-chain peak probe: returns the sustained FP64 TFLOP/s measured
 * on the context's device (bench.py roofline denominator). */
int tetmf_measure_fp64_peak(tetmf_ctx* ctx, double seconds, double* tflops);
/* the same, also returning the sustained rate: flops / time over the second
 * half of the window (clocks settled under the power cap) */
int tetmf_measure_fp64_peak2(tetmf_ctx* ctx, double seconds, double* burst_tflops, double* sustained_tflops);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif

#endif /* TETMF_B200_H */

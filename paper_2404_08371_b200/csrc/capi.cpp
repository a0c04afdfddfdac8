// capi.cpp -- extern "C" boundary (include/tetmf_b200.h).
//
// Exceptions never cross the ABI: std::invalid_argument -> TETMF_EINVAL,
// std::logic_error -> TETMF_EINTERNAL, DeviceError -> TETMF_EDEVICE,
// CommError -> TETMF_ECOMM, anything else -> TETMF_EINTERNAL.
#include "../../include/tetmf_b200.h"

#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "common.hpp"
#include "exchange.hpp"
#include "runtime.hpp"
#include "runtime_check.hpp"
#include "solver.hpp"

#include "transport.hpp"

using namespace tetmf;

struct tetmf_ctx {
  std::unique_ptr<Context> impl;
};
struct tetmf_fn {
  std::unique_ptr<Function> impl;
};
struct tetmf_op {
  std::unique_ptr<Operator> impl;
};
struct tetmf_loopback {
  std::shared_ptr<LoopbackHub> hub;
};

namespace {

thread_local std::string g_error;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return TETMF_OK;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return TETMF_EINVAL;
  } catch (const DeviceError& e) {
    g_error = e.what();
    return TETMF_EDEVICE;
  } catch (const CommError& e) {
    g_error = e.what();
    return TETMF_ECOMM;
  } catch (const std::exception& e) {
    g_error = e.what();
    return TETMF_EINTERNAL;
  } catch (...) {
    g_error = "unknown error";
    return TETMF_EINTERNAL;
  }
}

void need(const void* p, const char* what) {
  if (!p) fail_arg(std::string("null argument: ") + what);
}

Space space_of(int s) {
  if (s < 0 || s > 2) fail_arg("unknown space id " + std::to_string(s));
  return static_cast<Space>(s);
}

std::vector<int> rank_of(const Context& c) {
  std::vector<int> r(c.mesh().num_tets(), 0);
  for (int k = 0; k < c.nranks(); ++k)
    for (int m : partition_macros(c.mesh().num_tets(), k, c.nranks())) r[m] = k;
  return r;
}

} // namespace

extern "C" {

const char* tetmf_last_error(void) { return g_error.c_str(); }
const char* tetmf_version(void) { return "tetmf-b200 0.1 (sm_100a)"; }

int tetmf_ctx_create(const char* mesh_desc, int device, tetmf_ctx** out) {
  return tetmf_ctx_create_dist(mesh_desc, device, 0, 1, nullptr, out);
}

int tetmf_ctx_create_dist(const char* mesh_desc, int device, int rank, int nranks, const void* nccl_unique_id,
                          tetmf_ctx** out) {
  return tetmf_ctx_create_dist_part(mesh_desc, device, rank, nranks, nccl_unique_id, TETMF_PARTITION_MACRO, out);
}

int tetmf_ctx_create_dist_part(const char* mesh_desc, int device, int rank, int nranks, const void* nccl_unique_id,
                               int partition, tetmf_ctx** out) {
  return guard([&] {
    need(mesh_desc, "mesh_desc");
    need(out, "out");
    if (nranks < 1 || rank < 0 || rank >= nranks) fail_arg("bad rank / world size");
    auto c = std::make_unique<tetmf_ctx>();
    const int nm = mesh_by_name(mesh_desc).num_tets();
    c->impl = std::make_unique<Context>(mesh_desc, device, rank, nranks, partition_macros(nm, rank, nranks), partition);
    if (nranks > 1 && device >= 0) {
      need(nccl_unique_id, "nccl_unique_id");
      c->impl->attach_transport(make_nccl_transport(nranks, nccl_unique_id, rank));
    }
    *out = c.release();
  });
}

int tetmf_ctx_create_mesh(const double* vertices, int num_vertices, const int* tets, int num_tets, int device,
                          tetmf_ctx** out) {
  return guard([&] {
    need(vertices, "vertices");
    need(tets, "tets");
    need(out, "out");
    if (num_vertices < 4 || num_tets < 1) fail_arg("mesh needs at least 4 vertices and 1 tetrahedron");
    MacroMesh mesh;
    mesh.vertices.resize(num_vertices);
    for (int v = 0; v < num_vertices; ++v)
      for (int r = 0; r < 3; ++r) mesh.vertices[v][r] = vertices[3 * v + r];
    mesh.tets.resize(num_tets);
    for (int t = 0; t < num_tets; ++t)
      for (int i = 0; i < 4; ++i) mesh.tets[t][i] = tets[4 * t + i];
    auto c = std::make_unique<tetmf_ctx>();
    c->impl = std::make_unique<Context>(std::move(mesh), device, 0, 1, std::vector<int>{});
    *out = c.release();
  });
}

int tetmf_loopback_create(int nranks, tetmf_loopback** out) {
  return guard([&] {
    need(out, "out");
    if (nranks < 1) fail_arg("loopback: nranks must be >= 1");
    auto g = std::make_unique<tetmf_loopback>();
    g->hub = std::make_shared<LoopbackHub>(nranks);
    *out = g.release();
  });
}

int tetmf_loopback_destroy(tetmf_loopback* g) {
  return guard([&] { delete g; });
}

int tetmf_ctx_create_loopback(const char* mesh_desc, int device, tetmf_loopback* group, int rank, int partition,
                              tetmf_ctx** out) {
  return guard([&] {
    need(mesh_desc, "mesh_desc");
    need(group, "group");
    need(out, "out");
    if (device < 0) fail_arg("loopback: virtual ranks need a device");
    const int nranks = group->hub->nranks();
    if (rank < 0 || rank >= nranks) fail_arg("bad rank / world size");
    auto c = std::make_unique<tetmf_ctx>();
    const int nm = mesh_by_name(mesh_desc).num_tets();
    c->impl = std::make_unique<Context>(mesh_desc, device, rank, nranks, partition_macros(nm, rank, nranks), partition);
    if (nranks > 1) c->impl->attach_transport(make_loopback_transport(group->hub, rank));
    *out = c.release();
  });
}

int tetmf_ctx_transport_info(const tetmf_ctx* ctx, char* buf, int buflen) {
  return guard([&] {
    need(ctx, "ctx");
    need(buf, "buf");
    if (buflen <= 0) fail_arg("buflen must be positive");
    const std::string d = ctx->impl->transport() ? ctx->impl->transport()->describe() : std::string("single rank");
    std::snprintf(buf, static_cast<size_t>(buflen), "%s", d.c_str());
  });
}

int tetmf_ctx_destroy(tetmf_ctx* ctx) {
  return guard([&] { delete ctx; });
}

int tetmf_ctx_set_stream(tetmf_ctx* ctx, void* cuda_stream) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->impl->set_stream(static_cast<cudaStream_t>(cuda_stream));
  });
}

int tetmf_ctx_set_exchange_mode(tetmf_ctx* ctx, int mode) {
  return guard([&] {
    need(ctx, "ctx");
    if (mode < TETMF_EXCHANGE_SENDRECV || mode > TETMF_EXCHANGE_PUT_FUSED)
      fail_arg("exchange mode: 0 (send/recv), 1 (put), 2 (put, pack kernel) or 3 (put, in-kernel)");
    ctx->impl->set_exchange_put(mode != TETMF_EXCHANGE_SENDRECV,
                                mode == TETMF_EXCHANGE_PUT_PACK    ? Context::kFusedNever
                                : mode == TETMF_EXCHANGE_PUT_FUSED ? Context::kFusedAlways
                                                                   : Context::kFusedSlab);
  });
}

int tetmf_ctx_synchronize(tetmf_ctx* ctx) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->impl->synchronize();
  });
}

int tetmf_ctx_num_macros(const tetmf_ctx* ctx, int* global_count, int* local_count) {
  return guard([&] {
    need(ctx, "ctx");
    if (global_count) *global_count = ctx->impl->mesh().num_tets();
    if (local_count) *local_count = static_cast<int>(ctx->impl->macros().size());
  });
}

int tetmf_ctx_local_macros(const tetmf_ctx* ctx, int* out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "out");
    const auto& m = ctx->impl->macros();
    std::memcpy(out, m.data(), m.size() * sizeof(int));
  });
}

int tetmf_nccl_unique_id(void* out128) {
  return guard([&] {
    need(out128, "out");
    nccl_get_unique_id(out128);
  });
}

int tetmf_fn_create(tetmf_ctx* ctx, int space, tetmf_fn** out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "out");
    const Space s = space_of(space);

    auto f = std::make_unique<tetmf_fn>();
    f->impl = std::make_unique<Function>(*ctx->impl, s);
    *out = f.release();
  });
}

int tetmf_fn_destroy(tetmf_fn* fn) {
  return guard([&] { delete fn; });
}

int tetmf_fn_size(tetmf_fn* fn, int level, int64_t* entries) {
  return guard([&] {
    need(fn, "fn");
    need(entries, "entries");
    fn->impl->data(level);
    *entries = fn->impl->size(level);
  });
}

int tetmf_fn_device_ptr(tetmf_fn* fn, int level, double** ptr) {
  return guard([&] {
    need(fn, "fn");
    need(ptr, "ptr");
    *ptr = fn->impl->data(level);
  });
}

int tetmf_fn_fill_seeded(tetmf_fn* fn, int level, uint64_t seed, int dirichlet_zero) {
  return guard([&] {
    need(fn, "fn");
    fn->impl->fill_seeded(level, seed, dirichlet_zero != 0);
  });
}

int tetmf_fn_fill_coefficient(tetmf_fn* fn, int level, int which, double value) {
  return guard([&] {
    need(fn, "fn");
    fn->impl->fill_coefficient(level, CoeffSpec{which, value});
  });
}

int tetmf_fn_upload(tetmf_fn* fn, int level, const double* host, int64_t entries) {
  return guard([&] {
    need(fn, "fn");
    need(host, "host");
    double* d = fn->impl->data(level);
    if (entries != fn->impl->size(level)) fail_arg("upload: entry count does not match the layout");
    Context& c = fn->impl->ctx();
    TETMF_CUDA(cudaMemcpyAsync(d, host, entries * sizeof(double), cudaMemcpyHostToDevice, c.stream()));
    c.synchronize();
  });
}

int tetmf_fn_download(tetmf_fn* fn, int level, double* host, int64_t entries) {
  return guard([&] {
    need(fn, "fn");
    need(host, "host");
    double* d = fn->impl->data(level);
    if (entries != fn->impl->size(level)) fail_arg("download: entry count does not match the layout");
    Context& c = fn->impl->ctx();
    TETMF_CUDA(cudaMemcpyAsync(host, d, entries * sizeof(double), cudaMemcpyDeviceToHost, c.stream()));
    c.synchronize();
  });
}

int tetmf_fn_num_ref_dofs(tetmf_fn* fn, int level, int64_t* count) {
  return guard([&] {
    need(fn, "fn");
    need(count, "count");
    *count = fn->impl->num_ref_dofs(level);
  });
}

int tetmf_fn_import_ref(tetmf_fn* fn, int level, const double* host_ref) {
  return guard([&] {
    need(fn, "fn");
    need(host_ref, "host_ref");
    fn->impl->import_ref(level, host_ref);
  });
}

int tetmf_fn_export_ref(tetmf_fn* fn, int level, double* host_ref) {
  return guard([&] {
    need(fn, "fn");
    need(host_ref, "host_ref");
    fn->impl->export_ref(level, host_ref);
  });
}

int tetmf_fn_ref_owned_range(tetmf_fn* fn, int level, int64_t* lo, int64_t* hi) {
  return guard([&] {
    need(fn, "fn");
    need(lo, "lo");
    need(hi, "hi");
    i64 a = 0, b = 0;
    fn->impl->owned_ref_range(level, &a, &b);
    *lo = a;
    *hi = b;
  });
}

int tetmf_fn_import_ref_owned(tetmf_fn* fn, int level, const double* host_owned) {
  return guard([&] {
    need(fn, "fn");
    i64 a = 0, b = 0;
    fn->impl->owned_ref_range(level, &a, &b);
    if (b > a) need(host_owned, "host_owned");
    fn->impl->import_ref_owned(level, host_owned);
  });
}

int tetmf_fn_export_ref_owned(tetmf_fn* fn, int level, double* host_owned) {
  return guard([&] {
    need(fn, "fn");
    i64 a = 0, b = 0;
    fn->impl->owned_ref_range(level, &a, &b);
    if (b > a) need(host_owned, "host_owned");
    fn->impl->export_ref_owned(level, host_owned);
  });
}

int tetmf_op_create(tetmf_ctx* ctx, int form, tetmf_fn* const* coeffs, int ncoeffs, tetmf_op** out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "out");
    if (ncoeffs < 0 || (ncoeffs > 0 && !coeffs)) fail_arg("bad coefficient list");
    std::vector<const Function*> cf;
    for (int i = 0; i < ncoeffs; ++i) cf.push_back(coeffs[i] ? coeffs[i]->impl.get() : nullptr);
    if (form < 0 || form > 3) fail_arg("unknown form id " + std::to_string(form));
    auto o = std::make_unique<tetmf_op>();
    o->impl = std::make_unique<Operator>(*ctx->impl, static_cast<Form>(form), std::move(cf));
    *out = o.release();
  });
}

int tetmf_op_destroy(tetmf_op* op) {
  return guard([&] { delete op; });
}

int tetmf_apply(tetmf_op* op, const tetmf_fn* src, tetmf_fn* dst, int level, int update) {
  return guard([&] {
    need(op, "op");
    need(src, "src");
    need(dst, "dst");
    if (update != TETMF_REPLACE && update != TETMF_ADD) fail_arg("unknown update type");
    op->impl->apply(*src->impl, *dst->impl, level, static_cast<Update>(update));
  });
}

int tetmf_apply_ref_host(tetmf_op* op, tetmf_fn* src, tetmf_fn* dst, int level, const double* host_v,
                         double* host_w) {
  return guard([&] {
    need(op, "op");
    need(src, "src");
    need(dst, "dst");
    need(host_v, "host_v");
    need(host_w, "host_w");
    Function& s = *src->impl;
    Function& d = *dst->impl;
    Context& c = s.ctx();
    if (c.nranks() > 1) fail_arg("apply_ref_host: single-rank contexts only");
    const i64 nd = s.num_ref_dofs(level);
    if (d.num_ref_dofs(level) != nd) fail_arg("apply_ref_host: src/dst space mismatch");
    double* ref = op->impl->ref_scratch(nd);
    TETMF_CUDA(cudaMemcpyAsync(ref, host_v, nd * sizeof(double), cudaMemcpyHostToDevice, c.stream()));
    s.import_ref_device(level, ref);
    op->impl->apply(s, d, level, Update::Replace);
    d.export_ref_device(level, ref);
    TETMF_CUDA(cudaMemcpyAsync(host_w, ref, nd * sizeof(double), cudaMemcpyDeviceToHost, c.stream()));
    c.synchronize();
  });
}

int tetmf_apply_ref_host_batch(tetmf_op* op, tetmf_fn* src, tetmf_fn* dst, int level, int nvec,
                               const double* const* host_v, double* const* host_w) {
  return guard([&] {
    need(op, "op");
    need(src, "src");
    need(dst, "dst");
    if (nvec < 0) fail_arg("apply_ref_host_batch: nvec < 0");
    if (nvec == 0) return;
    need(host_v, "host_v");
    need(host_w, "host_w");
    for (int k = 0; k < nvec; ++k) {
      need(host_v[k], "host_v[k]");
      need(host_w[k], "host_w[k]");
    }
    Function& s = *src->impl;
    Function& d = *dst->impl;
    Context& c = s.ctx();
    if (c.nranks() > 1) fail_arg("apply_ref_host_batch: single-rank contexts only");
    const i64 nd = s.num_ref_dofs(level);
    if (d.num_ref_dofs(level) != nd) fail_arg("apply_ref_host_batch: src/dst space mismatch");
    // staging: in[0..1], out[0..1] (reference numbering, device)
    double* stage = op->impl->ref_scratch(4 * nd);
    double* in[2] = {stage, stage + nd};
    double* out[2] = {stage + 2 * nd, stage + 3 * nd};
    const cudaStream_t cs = c.stream();
    // streams / events released on every exit path (errors throw)
    struct Res {
      cudaStream_t h2d = nullptr, d2h = nullptr;
      std::vector<cudaEvent_t> ev;
      ~Res() {
        if (h2d) cudaStreamSynchronize(h2d);
        if (d2h) cudaStreamSynchronize(d2h);
        for (cudaEvent_t e : ev) cudaEventDestroy(e);
        if (h2d) cudaStreamDestroy(h2d);
        if (d2h) cudaStreamDestroy(d2h);
      }
    } res;
    TETMF_CUDA(cudaStreamCreateWithFlags(&res.h2d, cudaStreamNonBlocking));
    TETMF_CUDA(cudaStreamCreateWithFlags(&res.d2h, cudaStreamNonBlocking));
    const cudaStream_t h2d = res.h2d, d2h = res.d2h;
    res.ev.assign(4 * static_cast<std::size_t>(nvec), nullptr);
    for (auto& e : res.ev) TETMF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cudaEvent_t* ev_in = res.ev.data();
    cudaEvent_t* ev_imported = ev_in + nvec;
    cudaEvent_t* ev_exported = ev_imported + nvec;
    cudaEvent_t* ev_out = ev_exported + nvec;
    const std::size_t bytes = static_cast<std::size_t>(nd) * sizeof(double);
    auto issue_h2d = [&](int k) {
      if (k >= 2) TETMF_CUDA(cudaStreamWaitEvent(h2d, ev_imported[k - 2], 0));  // in[k % 2] consumed
      TETMF_CUDA(cudaMemcpyAsync(in[k & 1], host_v[k], bytes, cudaMemcpyHostToDevice, h2d));
      TETMF_CUDA(cudaEventRecord(ev_in[k], h2d));
    };
    issue_h2d(0);
    if (nvec > 1) issue_h2d(1);
    for (int k = 0; k < nvec; ++k) {
      // compute stream: import v_k, apply, export w_k
      TETMF_CUDA(cudaStreamWaitEvent(cs, ev_in[k], 0));
      s.import_ref_device(level, in[k & 1]);
      TETMF_CUDA(cudaEventRecord(ev_imported[k], cs));
      if (k + 2 < nvec) issue_h2d(k + 2);
      op->impl->apply(s, d, level, Update::Replace);
      if (k >= 2) TETMF_CUDA(cudaStreamWaitEvent(cs, ev_out[k - 2], 0));  // out[k % 2] drained
      d.export_ref_device(level, out[k & 1]);
      TETMF_CUDA(cudaEventRecord(ev_exported[k], cs));
      // copy-out stream: w_k
      TETMF_CUDA(cudaStreamWaitEvent(d2h, ev_exported[k], 0));
      TETMF_CUDA(cudaMemcpyAsync(host_w[k], out[k & 1], bytes, cudaMemcpyDeviceToHost, d2h));
      TETMF_CUDA(cudaEventRecord(ev_out[k], d2h));
    }
    TETMF_CUDA(cudaStreamSynchronize(d2h));
    TETMF_CUDA(cudaStreamSynchronize(h2d));
    c.synchronize();
  });
}

int tetmf_fn_dot(const tetmf_fn* a, const tetmf_fn* b, int level, double* out) {
  return guard([&] {
    need(a, "a");
    need(b, "b");
    need(out, "out");
    *out = masked_dot(*a->impl, *b->impl, level);
  });
}

int tetmf_fn_mask_dirichlet(tetmf_fn* fn, int level) {
  return guard([&] {
    need(fn, "fn");
    mask_dirichlet(*fn->impl, level);
  });
}

int tetmf_cg_solve(tetmf_op* op, const tetmf_fn* b, tetmf_fn* x, int level, double rtol, int max_iter,
                   int* iterations, double* rel_residual, int* converged) {
  return guard([&] {
    need(op, "op");
    need(b, "b");
    need(x, "x");
    const CgResult r = cg_solve(*op->impl, *b->impl, *x->impl, level, rtol, max_iter);
    if (iterations) *iterations = r.iterations;
    if (rel_residual) *rel_residual = r.rel_residual;
    if (converged) *converged = r.converged ? 1 : 0;
  });
}

int tetmf_op_diagonal(tetmf_op* op, tetmf_fn* diag, int level) {
  return guard([&] {
    need(op, "op");
    need(diag, "diag");
    op->impl->diagonal(*diag->impl, level);
  });
}

int tetmf_pcg_solve(tetmf_op* op, const tetmf_fn* b, tetmf_fn* x, const tetmf_fn* diag, int level, double rtol,
                    int max_iter, int* iterations, double* rel_residual, int* converged) {
  return guard([&] {
    need(op, "op");
    need(b, "b");
    need(x, "x");
    const CgResult r =
        cg_solve(*op->impl, *b->impl, *x->impl, level, rtol, max_iter, diag ? diag->impl.get() : nullptr);
    if (iterations) *iterations = r.iterations;
    if (rel_residual) *rel_residual = r.rel_residual;
    if (converged) *converged = r.converged ? 1 : 0;
  });
}

int tetmf_gradient(const tetmf_fn* p1, tetmf_fn* nd1, int level) {
  return guard([&] {
    need(p1, "p1");
    need(nd1, "nd1");
    gradient(*p1->impl, *nd1->impl, level);
  });
}

int tetmf_gradient_transpose(const tetmf_fn* nd1, tetmf_fn* p1, int level) {
  return guard([&] {
    need(nd1, "nd1");
    need(p1, "p1");
    gradient_transpose(*nd1->impl, *p1->impl, level);
  });
}

int tetmf_estimate_lambda_max(tetmf_op* op, const tetmf_fn* diag, int level, int iterations, double* lambda_max) {
  return guard([&] {
    need(op, "op");
    need(diag, "diag");
    need(lambda_max, "lambda_max");
    *lambda_max = estimate_lambda_max(*op->impl, *diag->impl, level, iterations);
  });
}

int tetmf_chebyshev_smooth(tetmf_op* op, const tetmf_fn* diag, const tetmf_fn* b, tetmf_fn* x, int level,
                           int degree, double lambda_max, double eig_ratio) {
  return guard([&] {
    need(op, "op");
    need(diag, "diag");
    need(b, "b");
    need(x, "x");
    chebyshev_smooth(*op->impl, *diag->impl, *b->impl, *x->impl, level, degree, lambda_max, eig_ratio);
  });
}

int tetmf_op_profile(tetmf_op* op, int enable) {
  return guard([&] {
    need(op, "op");
    op->impl->set_profiling(enable != 0);
  });
}

int tetmf_op_set_variant(tetmf_op* op, int variant) {
  return guard([&] {
    need(op, "op");
    if (variant < 0 || variant > 10) fail_arg("unknown kernel variant");
    op->impl->set_kernel_variant(variant);
  });
}

int tetmf_op_set_quadrature(tetmf_op* op, int degree) {
  return guard([&] {
    need(op, "op");
    op->impl->set_quadrature(degree);
  });
}

int tetmf_op_debug_perturb_table(tetmf_op* op, int level, int64_t index, double delta) {
  return guard([&] {
    need(op, "op");
    op->impl->debug_perturb_table(level, index, delta);
  });
}

int tetmf_op_kernel_stats(tetmf_op* op, double* total_ms, int64_t* launches) {
  return guard([&] {
    need(op, "op");
    i64 l = 0;
    op->impl->kernel_stats(total_ms, &l);
    if (launches) *launches = l;
  });
}

int tetmf_launch_count(int64_t* count) {
  return guard([&] {
    need(count, "count");
    *count = launch_count();
  });
}

int tetmf_host_alloc(void** ptr, int64_t bytes) {
  return guard([&] {
    need(ptr, "ptr");
    TETMF_CUDA(cudaMallocHost(ptr, static_cast<std::size_t>(bytes)));
  });
}

int tetmf_host_free(void* ptr) {
  return guard([&] { TETMF_CUDA(cudaFreeHost(ptr)); });
}

// ------------------------------------------------------------ planning hooks
int tetmf_plan_interior(tetmf_ctx* ctx, int space, int level, unsigned char* out, int64_t num_ref_dofs) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "out");
    const Context& c = *ctx->impl;
    const Space sp = space_of(space);
    const auto lay = LevelLayout::make(sp, level, c.mesh().num_tets(), c.macros());
    const auto rn = build_ref_numbering(c.mesh(), c.topo(), lay);
    if (num_ref_dofs != rn.num_dofs) fail_arg("plan_interior: output length does not match num_ref_dofs");
    std::memset(out, 1, static_cast<std::size_t>(num_ref_dofs));
    for (std::size_t li = 0; li < lay.macros.size(); ++li) {
      const int m = lay.macros[li];
      const i64 base = static_cast<i64>(li) * lay.macro_stride;
      for_each_carrier(sp, lay.n, [&](const Carrier& car) {
        const i64 e = rn.map[base + car.slot];
        if (e >= 0 && !carrier_interior(c.topo(), m, lay.n, car)) out[e >> 2] = 0;
      });
    }
  });
}

int tetmf_plan_layout(tetmf_ctx* ctx, int space, int level, int64_t* macro_stride, int64_t* class_stride) {
  return guard([&] {
    need(ctx, "ctx");
    const Context& c = *ctx->impl;
    const auto lay = LevelLayout::make(space_of(space), level, c.mesh().num_tets(), c.macros());
    if (macro_stride) *macro_stride = lay.macro_stride;
    if (class_stride) *class_stride = lay.class_stride;
  });
}

int tetmf_plan_ref_map(tetmf_ctx* ctx, int space, int level, int64_t* out, int64_t entries,
                       int64_t* num_ref_dofs) {
  return guard([&] {
    need(ctx, "ctx");
    const Context& c = *ctx->impl;
    const auto lay = LevelLayout::make(space_of(space), level, c.mesh().num_tets(), c.macros());
    if (out && entries != lay.total()) fail_arg("plan_ref_map: entry count does not match the layout");
    const auto rn = build_ref_numbering(c.mesh(), c.topo(), lay);
    if (out) std::memcpy(out, rn.map.data(), rn.map.size() * sizeof(int64_t));
    if (num_ref_dofs) *num_ref_dofs = rn.num_dofs;
  });
}

int tetmf_plan_local_groups(tetmf_ctx* ctx, int space, int level, int64_t* ngroups, int64_t* ncopies,
                            int64_t* offsets, int64_t* copies) {
  return guard([&] {
    need(ctx, "ctx");
    const Context& c = *ctx->impl;
    const auto lay = LevelLayout::make(space_of(space), level, c.mesh().num_tets(), c.macros());
    const auto g = c.partition() == Context::kPartitionSlab
                       ? local_groups_slab(c.mesh(), c.topo(), lay, slab_partition(c.mesh().num_tets(), lay.n,
                                                                                     c.nranks()), c.rank())
                       : local_groups_only(c.mesh(), c.topo(), lay, rank_of(c), c.rank());
    if (ngroups) *ngroups = g.num_groups();
    if (ncopies) *ncopies = static_cast<int64_t>(g.copies.size());
    if (offsets) std::memcpy(offsets, g.offsets.data(), g.offsets.size() * sizeof(int64_t));
    if (copies) std::memcpy(copies, g.copies.data(), g.copies.size() * sizeof(int64_t));
  });
}

int tetmf_plan_exchange(tetmf_ctx* ctx, int space, int level, int* npeers, int64_t* nsend, int64_t* nrecv,
                        int64_t* ngroups, int64_t* nentries, int* peers, int64_t* send_offsets,
                        int64_t* recv_offsets, int64_t* send_index, int64_t* group_offsets,
                        int64_t* group_entries) {
  return guard([&] {
    need(ctx, "ctx");
    const Context& c = *ctx->impl;
    const auto lay = LevelLayout::make(space_of(space), level, c.mesh().num_tets(), c.macros());
    const auto p = c.partition() == Context::kPartitionSlab
                       ? build_exchange_plan_slab(c.mesh(), c.topo(), lay,
                                                  slab_partition(c.mesh().num_tets(), lay.n, c.nranks()), c.rank())
                       : build_exchange_plan(c.mesh(), c.topo(), lay, rank_of(c), c.rank());
    if (npeers) *npeers = static_cast<int>(p.peers.size());
    if (nsend) *nsend = p.send_total();
    if (nrecv) *nrecv = p.recv_total();
    if (ngroups) *ngroups = p.num_groups();
    if (nentries) *nentries = static_cast<int64_t>(p.group_entries.size());
    auto cp = [](auto* dst, const auto& v) {
      if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
    };
    cp(peers, p.peers);
    cp(send_offsets, p.send_offsets);
    cp(recv_offsets, p.recv_offsets);
    cp(send_index, p.send_index);
    cp(group_offsets, p.group_offsets);
    cp(group_entries, p.group_entries);
  });
}

int tetmf_plan_slab_units(int num_macros, int level, int nranks, int rank, int* nunits, int* units) {
  return guard([&] {
    need(nunits, "nunits");
    if (level < 0 || level > 14) fail_arg("level out of range");
    const auto all = slab_partition(num_macros, 1 << level, nranks);
    if (rank < 0 || rank >= nranks) fail_arg("bad rank / world size");
    *nunits = static_cast<int>(all[rank].size());
    if (units)
      for (std::size_t i = 0; i < all[rank].size(); ++i) {
        units[3 * i] = all[rank][i].macro;
        units[3 * i + 1] = all[rank][i].za;
        units[3 * i + 2] = all[rank][i].zb;
      }
  });
}

int tetmf_host_local_sum(const int64_t* offsets, const int64_t* copies, int64_t ngroups, double* y) {
  return guard([&] {
    for (int64_t g = 0; g < ngroups; ++g) interface_sum_one(y, offsets, copies, g);
  });
}

int tetmf_host_pack(const double* y, const int64_t* send_index, int64_t nsend, double* send) {
  return guard([&] {
    for (int64_t i = 0; i < nsend; ++i) exchange_pack_one(y, send_index, send, i);
  });
}

int tetmf_host_put_offsets(int nranks, const int64_t* counts, int rank, int npeers, const int* peers,
                           int64_t* peer_off) {
  return guard([&] {
    if (nranks < 1 || rank < 0 || rank >= nranks || npeers < 0) fail_arg("put offsets: bad rank / sizes");
    need(counts, "counts");
    const std::vector<int> pv(peers, peers + npeers);
    const std::vector<i64> off = put_peer_offsets(nranks, counts, rank, pv);
    for (int k = 0; k < npeers; ++k) peer_off[k] = off[k];
  });
}

int tetmf_host_put_targets(int npeers, const int64_t* send_offsets, const int64_t* peer_off, int64_t* dst_off,
                           int* dst_peer) {
  return guard([&] {
    if (npeers < 0) fail_arg("put targets: npeers < 0");
    ExchangePlan plan;
    plan.peers.assign(npeers, 0);
    plan.send_offsets.assign(send_offsets, send_offsets + npeers + 1);
    std::vector<i64> off(peer_off, peer_off + npeers), d;
    std::vector<int> pp;
    exchange_put_targets(plan, off, d, pp);
    for (std::size_t i = 0; i < d.size(); ++i) {
      dst_off[i] = d[i];
      dst_peer[i] = pp[i];
    }
  });
}

int tetmf_selftest_nccl_put(int device, int rounds) {
  return guard([&] {
    TETMF_CUDA(cudaSetDevice(device));
    char uid[128];
    nccl_get_unique_id(uid);
    auto t = make_nccl_transport(1, uid, 0);
    const std::vector<int> peers;
    const std::vector<i64> send_off{0}, recv_off{0};
    auto ch = t->open_put(peers, send_off, recv_off);
    if (!ch) fail_internal("nccl put self-test: no channel");
    cudaStream_t s = nullptr;
    TETMF_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    for (int r = 0; r < rounds; ++r) ch->fence(s);
    TETMF_CUDA(cudaStreamSynchronize(s));
    TETMF_CUDA(cudaStreamDestroy(s));
  });
}

int tetmf_host_combine(double* y, const double* recv, const int64_t* group_offsets, const int64_t* group_entries,
                       int64_t ngroups) {
  return guard([&] {
    for (int64_t g = 0; g < ngroups; ++g) exchange_combine_one(y, recv, group_offsets, group_entries, g);
  });
}

int tetmf_plan_local_matrix(tetmf_ctx* ctx, int form, int level, int macro, int orientation, const double* c0,
                            const double* c1, double* out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "out");
    const Context& c = *ctx->impl;
    if (orientation < 0 || orientation > 5) fail_arg("orientation out of range");
    if (form == TETMF_FORM_N1) {
      need(c0, "alpha");
      need(c1, "beta");
      const N1DeviceTable t = pack_n1(n1_tables(c.mesh(), macro, level));
      double s[6];
      for (int e = 0; e < 6; ++e) s[e] = local_edge_ref(orientation, e).flipped ? -1.0 : 1.0;
      const double sa = c0[0] + c0[1] + c0[2] + c0[3];
      for (int j = 0; j < 6; ++j)
        for (int i = 0; i < 6; ++i) {
          const int q = sym6(i, j);
          double a = sa * t.e[orientation][0][q];
          for (int m = 0; m < 4; ++m) a += c1[m] * t.e[orientation][1 + m][q];
          out[j * 6 + i] = s[i] * s[j] * a;
        }
    } else if (form == TETMF_FORM_P1 || form == TETMF_FORM_P1K) {
      const P1DeviceTable t = pack_p1(p1_tables(c.mesh(), macro, level));
      double kb = 1.0;
      if (form == TETMF_FORM_P1K) {
        need(c0, "k");
        kb = 0.25 * (c0[0] + c0[1] + c0[2] + c0[3]);
      }
      for (int j = 0; j < 4; ++j)
        for (int i = 0; i < 4; ++i) out[j * 4 + i] = kb * t.K[orientation][sym4(i, j)];
    } else if (form == TETMF_FORM_P2V) {
      need(c0, "k");  // k at the element's 10 local P2 DoFs (vertices, then edges)
      const P2VTable t = p2v_table(c.mesh(), macro, level);
      for (int j = 0; j < 10; ++j)
        for (int i = 0; i < 10; ++i) {
          double a = 0.0;
          for (int m = 0; m < 10; ++m) a += c0[m] * t.T[orientation][m][sym10(i, j)];
          out[j * 10 + i] = a;
        }
    } else {
      fail_arg("plan_local_matrix: unsupported form");
    }
  });
}

int tetmf_plan_stencil(tetmf_ctx* ctx, int level, int macro, double* out /* 16 x 15 */) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "out");
    const P1Tables t = p1_tables(ctx->impl->mesh(), macro, level);
    std::memcpy(out, t.stencil, sizeof(t.stencil));
  });
}

int tetmf_measure_fp64_peak(tetmf_ctx* ctx, double seconds, double* tflops) {
  return tetmf_measure_fp64_peak2(ctx, seconds, tflops, nullptr);
}

int tetmf_measure_fp64_peak2(tetmf_ctx* ctx, double seconds, double* tflops, double* sustained) {
  return guard([&] {
    need(ctx, "ctx");
    need(tflops, "tflops");
    Context& c = *ctx->impl;
    if (c.device() < 0) fail_arg("measure_fp64_peak: planning-only context");
    int sms = 0;
    TETMF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device()));
    DeviceBuffer<double> out(1);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    cudaEvent_t e0, e1;
    TETMF_CUDA(cudaEventCreate(&e0));
    TETMF_CUDA(cudaEventCreate(&e1));
    launch_fp64_peak(out.get(), blocks, threads, 64, c.stream());  // warm-up
    double best = 0.0, late_flops = 0.0, late_ms = 0.0;
    const auto t0 = std::chrono::steady_clock::now();
    double elapsed = 0.0;
    do {
      TETMF_CUDA(cudaEventRecord(e0, c.stream()));
      launch_fp64_peak(out.get(), blocks, threads, iters, c.stream());
      TETMF_CUDA(cudaEventRecord(e1, c.stream()));
      TETMF_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      TETMF_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      const double flops = 2.0 * 8.0 * 16.0 * double(iters) * double(blocks) * double(threads);
      const double tf = flops / (ms * 1e-3) / 1e12;
      if (tf > best) best = tf;
      elapsed = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (elapsed >= 0.5 * seconds) {  // second half: the power / clock steady state
        late_flops += flops;
        late_ms += ms;
      }
    } while (elapsed < seconds);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *tflops = best;
    if (sustained) *sustained = late_ms > 0 ? late_flops / (late_ms * 1e-3) / 1e12 : best;
  });
}

} // extern "C"

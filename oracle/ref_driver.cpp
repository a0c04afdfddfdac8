// oracle/ref_driver.cpp -- C entry points around the REFERENCE's own apply.
//
// TEST INFRASTRUCTURE ONLY. Built by oracle/Makefile into
// oracle/_ref/libtetmf_ref.so from the reference sources where they lie
// (/root/reference/proj/src/{mesh,quadrature,fespace,loops}.cpp, compiled in
// place) plus this driver, which unity-includes forms.cpp because
// FormSystem's implicit destructor needs the complete StarTables type
// (forms.hpp:75,86). Only tests/, __graft_entry__.smoke() and bench.py's
// reference/cpu_baseline legs load the result, as the checker.
//
// What is exercised (all reference code, unmodified):
//   FormSystem::FormSystem        forms.cpp:43-56
//   FormSystem::apply             forms.cpp:195-255  (Replace semantics)
//   FormSystem::reference_apply   forms.cpp:257-260
//   FormSystem::local_matrix      forms.cpp:133-177
//   DoFIndexer::dof_geometry      fespace.cpp:432-451
//   DoFIndexer::interior          fespace.hpp:95-96
//   DoFIndexer::local_dofs        fespace.cpp:393-430
//   interpolate                   fespace.cpp:494-506
//   enumerate_elements            mesh.cpp:204-241
// plus the config-2 harness (P1 -div(k grad)) built only
// from that public API: A_e = FormSystem(P1).local_matrix(e, {}, rule),
// kbar_e = 6 * sum_q w_q * sum_m k_m lambda_m(xhat_q).
#include "forms.cpp"

#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>

namespace {

thread_local std::string g_err;

struct RefHandle {
  tetmf::MacroMesh mesh;
  std::unique_ptr<tetmf::FormSystem> sys;
  bool p1k = false;
};

template <typename F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

double alpha_fn(const tetmf::Vec3& p) { return 1.0 + p[0] * p[0] + p[1] * p[1]; }
double beta_fn(const tetmf::Vec3& p) { return 2.0 + std::sin(M_PI * p[2]); }
double k_fn(const tetmf::Vec3& p) {
  return 1.0 + 0.5 * std::sin(2.0 * M_PI * p[0]) * std::cos(2.0 * M_PI * p[1]) * (1.0 + p[2]);
}

} // namespace

#pragma GCC visibility push(default)
extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// form: "P1", "N1" or "P1K" (P1K = config-2 harness over the P1 system)
void* ref_create(const char* mesh, const char* form, int level) {
  RefHandle* h = nullptr;
  int rc = guarded([&] {
    auto hh = std::make_unique<RefHandle>();
    hh->mesh = tetmf::mesh_by_name(mesh);
    std::string f(form);
    tetmf::Form fid;
    if (f == "P1K") {
      fid = tetmf::Form::P1Diffusion;
      hh->p1k = true;
    } else {
      fid = tetmf::form_from_string(f);
    }
    hh->sys = std::make_unique<tetmf::FormSystem>(fid, hh->mesh, level);
    h = hh.release();
    return 0;
  });
  return rc == 0 ? h : nullptr;
}

void ref_destroy(void* p) { delete static_cast<RefHandle*>(p); }

long long ref_num_dofs(void* p) { return static_cast<RefHandle*>(p)->sys->num_dofs(); }

int ref_num_macros(void* p) { return static_cast<RefHandle*>(p)->mesh.num_tets(); }

// Geometry of every primary DoF: kind (0 vertex, 1 edge), a and b (3 doubles
// each; for ND1 the edge runs a -> b in the reference's global orientation).
int ref_dof_geometry(void* p, unsigned char* kind, double* a, double* b) {
  auto* h = static_cast<RefHandle*>(p);
  return guarded([&] {
    const auto& idx = h->sys->primary();
    for (std::int64_t id = 0; id < idx.num_dofs(); ++id) {
      const auto g = idx.dof_geometry(id);
      kind[id] = g.kind == tetmf::DoFKey::Kind::vertex ? 0 : 1;
      for (int c = 0; c < 3; ++c) {
        a[3 * id + c] = g.a[c];
        b[3 * id + c] = g.b[c];
      }
    }
    return 0;
  });
}

int ref_interior(void* p, unsigned char* out) {
  auto* h = static_cast<RefHandle*>(p);
  const auto& in = h->sys->primary().interior();
  std::memcpy(out, in.data(), in.size());
  return 0;
}

// Coefficient space (P1) of N1; for P1/P1K the primary P1 indexer.
static const tetmf::DoFIndexer& coeff_idx(RefHandle* h) {
  if (h->sys->form().coeffSpaces.empty()) return h->sys->primary();
  return h->sys->coeff_indexer(0);
}

long long ref_coeff_num_dofs(void* p) { return coeff_idx(static_cast<RefHandle*>(p)).num_dofs(); }

int ref_coeff_geometry(void* p, double* a) {
  auto* h = static_cast<RefHandle*>(p);
  return guarded([&] {
    const auto& idx = coeff_idx(h);
    for (std::int64_t id = 0; id < idx.num_dofs(); ++id) {
      const auto g = idx.dof_geometry(id);
      for (int c = 0; c < 3; ++c) a[3 * id + c] = g.a[c];
    }
    return 0;
  });
}

// which: 0 alpha, 1 beta, 2 k -- nodal interpolation into the P1 coefficient
// indexer with the reference's interpolate() (fespace.cpp:494-506).
int ref_interpolate(void* p, int which, double* out) {
  auto* h = static_cast<RefHandle*>(p);
  return guarded([&] {
    tetmf::ScalarFn f = which == 0 ? tetmf::ScalarFn(alpha_fn)
                        : which == 1 ? tetmf::ScalarFn(beta_fn)
                                     : tetmf::ScalarFn(k_fn);
    const auto v = tetmf::interpolate(coeff_idx(h), f);
    std::memcpy(out, v.data.data(), v.data.size() * sizeof(double));
    return 0;
  });
}

// y = A x. degree <= 0 selects reference_apply (exactDegree + 2); otherwise
// FormSystem::apply with quadrature(degree). c0/c1: alpha/beta for N1,
// k for P1K, ignored for P1. *seconds receives the wall time of the apply.
int ref_apply(void* p, const double* v, const double* c0, const double* c1, int degree,
              double* w, double* seconds) {
  auto* h = static_cast<RefHandle*>(p);
  return guarded([&] {
    const auto& sys = *h->sys;
    const std::int64_t n = sys.num_dofs();
    tetmf::FieldVector x{sys.form().trial, sys.level(), std::vector<double>(v, v + n)};

    if (h->p1k) {
      // config-2 harness: public API only
      const auto& kidx = sys.primary();
      const tetmf::QuadratureRule rule = tetmf::quadrature(degree > 0 ? degree : 2);
      std::vector<double> y(static_cast<std::size_t>(n), 0.0);
      const auto t0 = std::chrono::steady_clock::now();
      for (int m = 0; m < h->mesh.num_tets(); ++m) {
        const auto order = tetmf::enumerate_elements(tetmf::Strategy::sawtooth, m, sys.level());
        for (const auto& e : order.elements) {
          const auto a = sys.local_matrix(e, {}, rule);
          const auto dofs = kidx.local_dofs(e);
          double kbar = 0.0;
          for (int q = 0; q < rule.num_points(); ++q) {
            double kq = 0.0;
            for (int mm = 0; mm < 4; ++mm)
              kq += c0[dofs.ids[mm]] * tetmf::eval_basis(tetmf::Space::P1, mm, rule.points[q]);
            kbar += rule.weights[q] * kq;
          }
          kbar *= 6.0;
          for (int j = 0; j < 4; ++j) {
            double acc = 0.0;
            for (int i = 0; i < 4; ++i) acc += kbar * a.mat(j, i) * x.data[dofs.ids[i]];
            y[dofs.ids[j]] += acc;
          }
        }
      }
      const auto t1 = std::chrono::steady_clock::now();
      if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
      std::memcpy(w, y.data(), y.size() * sizeof(double));
      return 0;
    }

    std::vector<tetmf::FieldVector> cf;
    std::vector<const tetmf::FieldVector*> coeffs;
    const auto& spaces = sys.form().coeffSpaces;
    if (!spaces.empty()) {
      const std::int64_t nc = sys.coeff_indexer(0).num_dofs();
      cf.push_back({spaces[0], sys.level(), std::vector<double>(c0, c0 + nc)});
      if (spaces.size() > 1) cf.push_back({spaces[1], sys.level(), std::vector<double>(c1, c1 + nc)});
      for (auto& f : cf) coeffs.push_back(&f);
    }
    const auto t0 = std::chrono::steady_clock::now();
    const tetmf::FieldVector y =
        degree <= 0 ? sys.reference_apply(x, coeffs) : sys.apply(x, coeffs, tetmf::quadrature(degree));
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    std::memcpy(w, y.data.data(), y.data.size() * sizeof(double));
    return 0;
  });
}

// Local matrix of one micro element (row-major nloc x nloc, (j,i) = (test, trial)).
int ref_local_matrix(void* p, int macro, int orientation, int x, int y, int z, const double* c0,
                     const double* c1, int degree, double* out) {
  auto* h = static_cast<RefHandle*>(p);
  return guarded([&] {
    const auto& sys = *h->sys;
    tetmf::MicroElement e{static_cast<tetmf::Orientation>(orientation), x, y, z, sys.level(), macro};
    std::vector<tetmf::FieldVector> cf;
    std::vector<const tetmf::FieldVector*> coeffs;
    const auto& spaces = sys.form().coeffSpaces;
    if (!spaces.empty()) {
      const std::int64_t nc = sys.coeff_indexer(0).num_dofs();
      cf.push_back({spaces[0], sys.level(), std::vector<double>(c0, c0 + nc)});
      if (spaces.size() > 1) cf.push_back({spaces[1], sys.level(), std::vector<double>(c1, c1 + nc)});
      for (auto& f : cf) coeffs.push_back(&f);
    }
    const auto lm = sys.local_matrix(e, coeffs, tetmf::quadrature(degree));
    const int nloc = lm.mat.rows();
    for (int j = 0; j < nloc; ++j)
      for (int i = 0; i < nloc; ++i) out[j * nloc + i] = lm.mat(j, i);
    return nloc;
  });
}

// Global ids and signs of one element's local DoFs (fespace.cpp:393-430).
int ref_local_dofs(void* p, int macro, int orientation, int x, int y, int z, long long* ids,
                   double* signs) {
  auto* h = static_cast<RefHandle*>(p);
  return guarded([&] {
    tetmf::MicroElement e{static_cast<tetmf::Orientation>(orientation), x, y, z,
                          h->sys->level(), macro};
    const auto d = h->sys->primary().local_dofs(e);
    for (int i = 0; i < d.count; ++i) {
      ids[i] = d.ids[i];
      signs[i] = d.signs[i];
    }
    return d.count;
  });
}

// Element traversal (mesh.cpp:204-241): writes up to cap (o,x,y,z) quads.
long long ref_enumerate(int strategy, int level, int* out, long long cap) {
  long long count = -1;
  guarded([&] {
    const auto order =
        tetmf::enumerate_elements(strategy == 0 ? tetmf::Strategy::sawtooth : tetmf::Strategy::cubes, 0, level);
    count = static_cast<long long>(order.elements.size());
    for (long long i = 0; i < count && i < cap; ++i) {
      const auto& e = order.elements[i];
      out[4 * i + 0] = static_cast<int>(e.orientation);
      out[4 * i + 1] = e.x;
      out[4 * i + 2] = e.y;
      out[4 * i + 3] = e.z;
    }
    return 0;
  });
  return count;
}

// Quadrature rule of a degree: writes points (3*nq) and weights (nq).
int ref_quadrature(int degree, double* pts, double* wts, int cap) {
  int nq = -1;
  guarded([&] {
    const auto r = tetmf::quadrature(degree);
    nq = r.num_points();
    for (int q = 0; q < nq && q < cap; ++q) {
      for (int c = 0; c < 3; ++c) pts[3 * q + c] = r.points[q][c];
      wts[q] = r.weights[q];
    }
    return 0;
  });
  return nq;
}

} // extern "C"
#pragma GCC visibility pop

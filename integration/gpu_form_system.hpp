// integration/gpu_form_system.hpp -- the reference-side binding a maintainer
// of the reference (tetmf, C++20) adds to route FormSystem::apply to the
// B200 library through its C ABI (include/tetmf_b200.h). Header-only; needs
// the reference's headers (<tetmf/forms.hpp>) and links libtetmf_b200.so.
//
// Same constructor inputs as FormSystem(Form, const MacroMesh&, int level)
// (forms.hpp:46) -- the caller's in-memory MacroMesh, not a mesh name -- and
// the same apply contract (forms.hpp:65-66): v and the coefficient
// FieldVectors in the reference's global numbering, w returned by value,
// Replace semantics, std::invalid_argument for a wrong space / level /
// coefficient count (forms.cpp:58-67, 198-200), std::logic_error otherwise.
// The GPU integrates exactly (= reference_apply, forms.cpp:257-260).
// Compiled and checked against the reference's own apply by
// integration/adapter_check.cpp (oracle/Makefile target `adapter`).
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include <tetmf/forms.hpp>

#include "tetmf_b200.h"

namespace tetmf {

class GpuFormSystem {
public:
  GpuFormSystem(Form form, const MacroMesh& mesh, int level, int device = 0) : form_(form), level_(level) {
    std::vector<double> xyz;
    std::vector<int> ids;
    for (const auto& v : mesh.vertices) xyz.insert(xyz.end(), {v[0], v[1], v[2]});
    for (const auto& t : mesh.tets) ids.insert(ids.end(), t.begin(), t.end());
    check(tetmf_ctx_create_mesh(xyz.data(), static_cast<int>(mesh.vertices.size()), ids.data(), mesh.num_tets(),
                                device, &ctx_));
    // trial space and coefficient spaces of kForms (forms.cpp:10-14)
    const int space = form == Form::N1CurlCurlMass ? TETMF_SPACE_ND1
                      : form == Form::P2VDiffusion ? TETMF_SPACE_P2
                                                   : TETMF_SPACE_P1;
    check(tetmf_fn_create(ctx_, space, &src_));
    check(tetmf_fn_create(ctx_, space, &dst_));
    if (form == Form::N1CurlCurlMass) {
      nc_ = 2;  // alpha, beta in P1
      check(tetmf_fn_create(ctx_, TETMF_SPACE_P1, &c_[0]));
      check(tetmf_fn_create(ctx_, TETMF_SPACE_P1, &c_[1]));
    } else if (form == Form::P2VDiffusion) {
      nc_ = 1;  // k in P2
      check(tetmf_fn_create(ctx_, TETMF_SPACE_P2, &c_[0]));
    }
    // the reference Form ids coincide with TETMF_FORM_{P1, P2V, N1}
    check(tetmf_op_create(ctx_, static_cast<int>(form), c_, nc_, &op_));
  }
  GpuFormSystem(const GpuFormSystem&) = delete;
  GpuFormSystem& operator=(const GpuFormSystem&) = delete;
  ~GpuFormSystem() {
    if (op_) tetmf_op_destroy(op_);
    for (tetmf_fn* f : {src_, dst_, c_[0], c_[1]})
      if (f) tetmf_fn_destroy(f);
    if (ctx_) tetmf_ctx_destroy(ctx_);
  }

  int level() const { return level_; }

  // FormSystem::apply(v, coeffs) with the exact rule (forms.hpp:65-66)
  FieldVector apply(const FieldVector& v, const std::vector<const FieldVector*>& coeffs) {
    if (v.level != level_) throw std::invalid_argument("field level does not match the system level");
    if (static_cast<int>(coeffs.size()) != nc_) throw std::invalid_argument("wrong number of coefficient fields");
    int64_t nd = 0;
    check(tetmf_fn_num_ref_dofs(src_, level_, &nd));
    if (static_cast<int64_t>(v.data.size()) != nd) throw std::invalid_argument("field shape mismatch");
    for (int i = 0; i < nc_; ++i) {
      if (!coeffs[i]) throw std::invalid_argument("missing coefficient field");
      int64_t nc = 0;
      check(tetmf_fn_num_ref_dofs(c_[i], level_, &nc));
      if (static_cast<int64_t>(coeffs[i]->data.size()) != nc)
        throw std::invalid_argument("coefficient field has wrong space or level");
      check(tetmf_fn_import_ref(c_[i], level_, coeffs[i]->data.data()));
    }
    FieldVector w{v.space, v.level, std::vector<double>(v.data.size())};
    check(tetmf_apply_ref_host(op_, src_, dst_, level_, v.data.data(), w.data.data()));
    return w;
  }

private:
  static void check(int rc) {
    if (rc == TETMF_EINVAL) throw std::invalid_argument(tetmf_last_error());
    if (rc != TETMF_OK) throw std::logic_error(tetmf_last_error());
  }
  Form form_;
  int level_;
  tetmf_ctx* ctx_ = nullptr;
  tetmf_fn* src_ = nullptr;
  tetmf_fn* dst_ = nullptr;
  tetmf_fn* c_[2] = {nullptr, nullptr};
  int nc_ = 0;
  tetmf_op* op_ = nullptr;
};

}  // namespace tetmf

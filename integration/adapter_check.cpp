// integration/adapter_check.cpp -- compiles the reference-side adapter
// (integration/gpu_form_system.hpp) against the reference's own headers and
// sources and checks GpuFormSystem::apply against the reference's
// FormSystem::reference_apply on the same in-memory MacroMesh, seeded input
// and interpolated coefficients. TEST INFRASTRUCTURE: built by
// oracle/Makefile (target `adapter`, with the one-line fill_map fix, DESIGN.md
// "Reference defect") into oracle/_ref/adapter_check; run by
// tests/test_gpu_integration.py on the GPU box. Exit 0 iff every case agrees
// to 1e-12 relative (max norm).
#include "forms.cpp"  // FormSystem's implicit destructor needs StarTables (forms.hpp:75,86)

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <sstream>

#include "gpu_form_system.hpp"

namespace {

double alpha_fn(const tetmf::Vec3& p) { return 1.0 + p[0] * p[0] + p[1] * p[1]; }
double beta_fn(const tetmf::Vec3& p) { return 2.0 + std::sin(M_PI * p[2]); }
double k_fn(const tetmf::Vec3& p) {
  return 1.0 + 0.5 * std::sin(2.0 * M_PI * p[0]) * std::cos(2.0 * M_PI * p[1]) * (1.0 + p[2]);
}

// 2 x 2 x 2 unit cubes, each split like cube6 (mesh.cpp:122-141), in the
// reference's text format -> MacroMesh::load
tetmf::MacroMesh kuhn2() {
  std::ostringstream os;
  auto vid = [](int x, int y, int z) { return x + 3 * (y + 3 * z); };
  for (int z = 0; z <= 2; ++z)
    for (int y = 0; y <= 2; ++y)
      for (int x = 0; x <= 2; ++x) os << "v " << x << " " << y << " " << z << "\n";
  const int perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  for (int cz = 0; cz < 2; ++cz)
    for (int cy = 0; cy < 2; ++cy)
      for (int cx = 0; cx < 2; ++cx)
        for (const auto& p : perm) {
          int a[3] = {0, 0, 0}, b[3];
          a[p[0]] = 1;
          for (int i = 0; i < 3; ++i) b[i] = a[i];
          b[p[1]] = 1;
          int t[4] = {vid(cx, cy, cz), vid(cx + a[0], cy + a[1], cz + a[2]), vid(cx + b[0], cy + b[1], cz + b[2]),
                      vid(cx + 1, cy + 1, cz + 1)};
          // positive orientation: swap the last two if the volume is negative
          const double e1[3] = {double(a[0]), double(a[1]), double(a[2])};
          const double e2[3] = {double(b[0]), double(b[1]), double(b[2])};
          const double e3[3] = {1, 1, 1};
          const double det = e1[0] * (e2[1] * e3[2] - e2[2] * e3[1]) - e1[1] * (e2[0] * e3[2] - e2[2] * e3[0]) +
                             e1[2] * (e2[0] * e3[1] - e2[1] * e3[0]);
          if (det < 0) std::swap(t[2], t[3]);
          os << "t " << t[0] << " " << t[1] << " " << t[2] << " " << t[3] << "\n";
        }
  std::istringstream is(os.str());
  return tetmf::MacroMesh::load(is);
}

double uniform(std::uint64_t i) {
  std::uint64_t z = i * 0x9E3779B97F4A7C15ull + 0x1234567ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return 2.0 * (static_cast<double>(z >> 11) * (1.0 / 9007199254740992.0)) - 1.0;
}

int run(const char* name, const tetmf::MacroMesh& mesh, tetmf::Form form, int level) {
  tetmf::FormSystem ref(form, mesh, level);
  tetmf::FieldVector v{ref.form().trial, level, std::vector<double>(static_cast<std::size_t>(ref.num_dofs()))};
  for (std::size_t i = 0; i < v.data.size(); ++i) v.data[i] = uniform(i);
  std::vector<tetmf::FieldVector> cf;
  if (form == tetmf::Form::N1CurlCurlMass) {
    cf.push_back(tetmf::interpolate(ref.coeff_indexer(0), tetmf::ScalarFn(alpha_fn)));
    cf.push_back(tetmf::interpolate(ref.coeff_indexer(1), tetmf::ScalarFn(beta_fn)));
  } else if (form == tetmf::Form::P2VDiffusion) {
    cf.push_back(tetmf::interpolate(ref.coeff_indexer(0), tetmf::ScalarFn(k_fn)));
  }
  std::vector<const tetmf::FieldVector*> coeffs;
  for (auto& f : cf) coeffs.push_back(&f);
  const tetmf::FieldVector want = ref.reference_apply(v, coeffs);
  tetmf::GpuFormSystem gpu(form, mesh, level);
  const tetmf::FieldVector got = gpu.apply(v, coeffs);
  double num = 0.0, den = 0.0;
  for (std::size_t i = 0; i < want.data.size(); ++i) {
    num = std::max(num, std::fabs(got.data[i] - want.data[i]));
    den = std::max(den, std::fabs(want.data[i]));
  }
  const double err = num / den;
  std::printf("%-10s %-4s L%d  %9zu DoFs  rel err %.3e  %s\n", name, ref.form().name.c_str(), level, want.data.size(),
              err, err <= 1e-12 ? "OK" : "FAIL");
  return err <= 1e-12 ? 0 : 1;
}

}  // namespace

int main() {
  int bad = 0;
  try {
    const auto st = tetmf::MacroMesh::single_tet(), c6 = tetmf::MacroMesh::cube6(), k2 = kuhn2();
    bad += run("single-tet", st, tetmf::Form::P1Diffusion, 4);
    bad += run("cube6", c6, tetmf::Form::P1Diffusion, 4);
    bad += run("cubes2", k2, tetmf::Form::P1Diffusion, 3);
    bad += run("single-tet", st, tetmf::Form::N1CurlCurlMass, 4);
    bad += run("cube6", c6, tetmf::Form::N1CurlCurlMass, 3);
    bad += run("cubes2", k2, tetmf::Form::N1CurlCurlMass, 3);
    bad += run("cube6", c6, tetmf::Form::P2VDiffusion, 2);
    bad += run("single-tet", st, tetmf::Form::P2VDiffusion, 3);
    // error contract: a wrong coefficient count is std::invalid_argument, as in the reference
    tetmf::GpuFormSystem gpu(tetmf::Form::N1CurlCurlMass, c6, 2);
    tetmf::FieldVector v{tetmf::Space::ND1, 2, std::vector<double>(10)};
    try {
      gpu.apply(v, {});
      std::printf("missing invalid_argument\n");
      ++bad;
    } catch (const std::invalid_argument& e) {
      std::printf("invalid_argument as expected: %s\n", e.what());
    }
  } catch (const std::exception& e) {
    std::printf("error: %s\n", e.what());
    return 2;
  }
  return bad ? 1 : 0;
}

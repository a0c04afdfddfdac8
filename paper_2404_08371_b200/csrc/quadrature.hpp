// quadrature.hpp -- the reference's quadrature rules on the unit tetrahedron
// (quadrature.cpp:19-147): the rule an apply integrates with when the caller
// passes one (FormSystem::apply(v, coeffs, rule), forms.hpp:65-66).
//
//   degree 1: centroid;  2: four-point rule (a = 0.5854..., b = 0.1381...,
//   w = 1/24);  4: Keast's 11-point rule (negative centroid weight);
//   3 / 5 / 6: conical products of Gauss-Jacobi rules with 2 / 3 / 4 points
//   per direction (weights (1-x)^2, (1-x)^1, 1; Golub-Welsch)
// Points in reference coordinates (x, y, z), weights sum to 1/6.
#pragma once

#include <vector>

namespace tetmf {

struct QuadRule {
  std::vector<double> x, y, z, w;
  int size() const { return static_cast<int>(w.size()); }
};

// throws (fail_arg) for degrees outside 1..6
QuadRule quadrature_rule(int degree);

} // namespace tetmf

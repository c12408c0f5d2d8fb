// compute_errors / make_reference on the B200 path (errors.cu).
#pragma once

#include <vector>

#include "ctx.cuh"

namespace mlg {

// Closed-form Dirichlet eigenfunction of a rectangle (ExactFunction of
// make_reference, harness.cpp:126-169): amp * sin(mx pi (x-x0)/lx) *
// sin(my pi (y-y0)/ly); mx == 0 means "no closed form" (multiple eigenvalue).
struct ExactMode {
  int mx = 0, my = 0;
  double x0 = -1.0, lx = 2.0, y0 = -1.0, ly = 2.0, amp = 1.0;
};

struct ErrorReport {  // fespace.hpp:108-112
  double eig_err = 0.0, l2_err = 0.0, h1_err = 0.0;
};

struct ReferenceSet {  // corrector.hpp ReferenceSet
  std::vector<double> lambdas;
  std::vector<ExactMode> modes;
};

// compute_errors (fespace.cpp:434-488) on coefficients resident in device
// memory: full-lattice vector, entry of dof d at d_coeffs[d*stride + lane].
ErrorReport compute_errors(Ctx& c, const Level& L, const double* d_coeffs, int stride, int lane,
                           double lambda_h, double lambda_ref, const ExactMode* mode);

// make_reference (harness.cpp:126-169); domain = {x_min, x_max, y_min, y_max}
// or nullptr for the reference's (-1,1)^2 table.
ReferenceSet make_reference(int example, int nev, const double* domain);

// The reference set a configuration's experiment reports against (adds the
// L-shaped domain's table).
ReferenceSet make_reference_for(const Config& cfg, int nev);

}  // namespace mlg

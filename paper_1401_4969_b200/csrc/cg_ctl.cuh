// The scalar state machine of the reference's cg_solve (sparse.cpp:199-258)
// in the one-reduction arrangement used by every batched CG kernel of this
// library (k_cg_iter, k_cg_persist in cg.cu; k_cg_resident in
// cg_resident.cu).  One call per system after each reduction of the five
// dot products a = {r.r, r.z, p.q, q.z, q.D^-1 q}.
#pragma once

#include "cg.cuh"

namespace mlg {

enum Phase { kPhaseInit = 0, kPhaseIter = 1 };

// Scalar recurrences of cg_solve for one system after a launch's reduction.
template <int PH>
__device__ __forceinline__ void update_ctl(CgCtl& c, const double (&a)[kCgDots], double tol,
                                           int maxit, int xdefer = 0) {
  if (PH == kPhaseInit) {
    c.bnorm = sqrt(a[0]);
    c.iters = 0;
    c.alpha = c.beta = c.rho = 0.0;
    c.alpha_prev = 0.0;
    c.xphase = 0;
    c.restart = 1;
    if (c.bnorm == 0.0) {  // sparse.cpp:208-212
      c.status = kConverged;
      c.final_res = 0.0;
      c.mode = kModeSkip;
    } else {
      c.status = kRunning;
      c.mode = kModeNormal;
    }
    return;
  }
  if (c.mode == kModeFlush) {  // the deferred x update is applied: x is current
    c.xphase = 0;
    c.mode = kModeCheck;
    return;
  }
  if (c.mode == kModeNormal) {
    const bool updated = !c.restart;
    if (updated) c.iters += 1;
    if (updated && xdefer) {  // this launch deferred (phase 0) or caught up (phase 1)
      if (c.xphase == 0) {
        c.alpha_prev = c.alpha;
        c.xphase = 1;
      } else {
        c.xphase = 0;
      }
    }
    // The convergence test and the scalar recurrences are independent chains of
    // long-latency FP64 operations (sqrt; two divisions): both are evaluated
    // before the branches so that they overlap (one thread runs this between
    // two barriers of every CG iteration).  Same arithmetic as the branchy
    // form; the speculative quotients are simply unused when a branch returns.
    const double pq = a[2];
    const double rho = a[1];
    const double rnorm = sqrt(a[0]);
    const double alpha = rho / pq;
    const double rho_next = rho - 2.0 * alpha * a[3] + alpha * alpha * a[4];
    const double beta = rho_next / rho;
    if (updated && (rnorm <= tol * c.bnorm || c.iters >= maxit)) {
      // confirm with the true residual (sparse.cpp:232-246), once x is current
      c.mode = c.xphase ? kModeFlush : kModeCheck;
      return;
    }
    if (pq <= 0.0) {  // sparse.cpp:225-226
      c.status = kIndefinite;
      c.mode = kModeSkip;
      return;
    }
    c.alpha = alpha;
    c.beta = beta;
    c.rho = rho;
    c.restart = 0;
  } else if (c.mode == kModeCheck) {
    const double true_rel = sqrt(a[0]) / c.bnorm;
    if (true_rel <= tol) {
      c.status = kConverged;
      c.final_res = true_rel;
      c.mode = kModeSkip;
    } else if (c.iters >= maxit) {
      c.status = kNotConverged;  // sparse.cpp:255-257
      c.final_res = true_rel;
      c.mode = kModeSkip;
    } else {  // restart from the true residual: p = z, no pending update
      c.restart = 1;
      c.alpha = c.beta = 0.0;
      c.xphase = 0;
      c.mode = kModeNormal;
    }
  }
}

}  // namespace mlg

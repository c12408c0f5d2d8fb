// Correction-step orchestration entry points (corrector.cu), used by the C-ABI.
#pragma once

#include <vector>

#include "cg.cuh"

namespace mlg {

struct StepResult {
  std::vector<double> lambdas;
  bool matched = true;
  StepTimes times;
};

struct Workspace;
Workspace& W(Ctx& c);

int nr_for(int nev);
void validate_config(const Config& cfg);

// solve_interior_eigenproblem at `level`; u_out = interleaved full-lattice coeffs.
std::vector<double> coarse_eigensolve(Ctx& c, int level, int nev, DevBuf<double>& u_out);

// one_correction_step: u_in interleaved (nr_for(nev) lanes) at level `from`.
StepResult correction_step(Ctx& c, int from, int to, int nev, const double* lam_in,
                           const double* u_in, DevBuf<double>& u_out);

// augmented_eigensolve on interleaved candidates (k_in lanes used).
std::vector<double> augmented(Ctx& c, int level, int nr, int k_in, const double* glued, int nev,
                              DevBuf<double>& u_out);

// Batched local solves; reports[j * nev + i] for subdomain j, eigenvector i.
int local_solves(Ctx& c, const Level& F, int nr, int nev, const double* res, double tol,
                 int maxit, std::vector<SolveReport>* reports, int only_j = -1);
// The batched local CG of the last local_solves call (X holds e_j per window).
const CgBatch& local_batch(Ctx& c);
// The last local_solves batch, whatever the degree: systems, pooled x, device systems.
struct LocalView {
  std::vector<CgSys> systems;
  const double* x;
  const CgSys* sys_dev;
};
LocalView local_view(Ctx& c);
int strip_solve(Ctx& c, Level& F, int nr, int nev, const double* u, const struct Lam& lam,
                double* glued, double tol, int maxit, std::vector<SolveReport>* reports,
                bool* empty);
void ensure_strip_mask(Ctx& c, Level& F);
void prolong_chain(Ctx& c, int nr, const double* src, int from, int to, double* dst);
const double* restrict_chain(Ctx& c, int nr, const double* src, int from, int slot);
std::vector<double> mdot(Ctx& c, int nr, const Level& L, const double* U, const double* V);
void fix_sign_lanes(Ctx& c, int nr, const Level& L, double* v);

void interleave(Ctx& c, const Level& L, int nr, int k_in, const double* src, int interior_src,
                double* dst);
void deinterleave(Ctx& c, const Level& L, int nr, int k_out, const int* perm, const double* src,
                  int interior_dst, double* dst);
void spmv_full(Ctx& c, const Level& L, int form, const double* x, double* y);
void spmv_interior(Ctx& c, const Level& L, const double* x, double* y);
void restrict_levels(Ctx& c, int nr, const double* src, int from, int to, double* dst);
void glue_full(Ctx& c, int level, const double* corr, const double* u, double* glued);
void residual(Ctx& c, const Level& F, int nr, const double* u, const double* lam, double* out);

}  // namespace mlg

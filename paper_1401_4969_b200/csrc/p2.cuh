// P2 (degree 2) level build and operators (p2.cu).
#pragma once

#include "ctx.cuh"

namespace mlg {

void assemble_p2(Ctx& c, Level& L);
void export_csr_p2(Ctx& c, const Level& L, int form, int* row_ptr, int* cols, double* vals);
// y = A x (form 0) or M x (form 1) on the dof grid, nr interleaved lanes; with
// interior_only the rows of non-interior dofs are 0 (k_dual semantics).
void apply_p2(Ctx& c, const Level& L, int form, int nr, const double* x, double* y,
              bool interior_only);
void interior_dense_p2(Ctx& c, const Level& L, int form, double* d_dense);
void export_space_p2(Ctx& c, const Level& L, int* dof_lattice, int* conn6);
// One refinement C -> C+1 of the P2 prolongation (and its transpose), nr
// interleaved lanes.
void prolong_p2(Ctx& c, const Level& C, int nr, const double* xc, double* xf);
void restrict_p2(Ctx& c, const Level& C, int nr, const double* xf, double* xc);
struct Lam;
// lam * M u - A w at interior dofs (k_residual semantics).
void residual_p2(Ctx& c, const Level& L, int nr, const double* u, const double* w,
                 const Lam& lam, double* out, const unsigned char* only_mask);

}  // namespace mlg

/*
 * mlg_b200.h -- C ABI of the B200 correction-step library (libmlg_b200.so).
 *
 * Drop-in boundary for the hot path of the reference (arXiv 1401.4969,
 * /root/reference/proj): one multilevel correction step -- subdomain residual
 * solves, strip solve, coarse-space-augmented eigensolve -- plus the level
 * build it triggers.  The reference has no FFI of its own; its boundary is the
 * C++ API of include/mleig/corrector.hpp, and every entry point below names
 * the reference function it replaces (file:line under /root/reference/proj).
 *
 * Conventions (mirroring the reference's data layout):
 *   - all arrays are host memory, caller-allocated, 0-based, int32 indices,
 *     float64 values (except the *_device entry points);
 *   - "full" vectors have one entry per dof of the level (boundary included,
 *     dof = iy*(nx+1)+ix, fespace.cpp:230-290); "interior" vectors follow
 *     FeSpace::interior_dofs order (ascending dof id); several vectors are
 *     stored one after another (vector-major);
 *   - a context owns all device state (mesh hierarchy, operators, workspaces)
 *     like Hierarchy owns its LevelSystems (corrector.hpp:63-95); one context
 *     per host thread, calls are synchronous;
 *   - return value 0 on success, otherwise the reference's exception class as
 *     its CLI exit code (tools/mleig_main.cpp:57-66) -- 2 ConfigError,
 *     3 SolverError, 4 IoError, 1 other -- or 5 for a CUDA error; the message
 *     (same text as the reference's exception where one exists) is returned
 *     by mlg_last_error() on the calling thread.
 */
#ifndef MLG_B200_H
#define MLG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MLG_OK 0
#define MLG_ERR_OTHER 1
#define MLG_ERR_CONFIG 2 /* mleig::ConfigError, errors.hpp:10-12 */
#define MLG_ERR_SOLVER 3 /* mleig::SolverError, errors.hpp:15-17 */
#define MLG_ERR_IO 4     /* mleig::IoError,     errors.hpp:20-22 */
#define MLG_ERR_CUDA 5

/* RunConfig (corrector.hpp:21-33). example: 0 = "laplace", 1 = "variable"
 * (CoefficientField, fespace.cpp:105-123), 2 = "reaction": the B200 extension
 * for BASELINE config 4 (no reference code path), -div(a grad u) + c u = lambda u
 * with a = 1 + 0.5 sin(2 pi k1 x) sin(2 pi k2 y), c = 1 + x^2 + y^2 evaluated
 * at triangle centroids, (k1, k2) in {1..4}^2 drawn from `seed` by splitmix64. */
typedef struct mlg_config {
  double x_min, x_max, y_min, y_max; /* DomainRect (mesh.hpp:22-27) */
  double H;                          /* coarse mesh size */
  double delta;                      /* requested overlap (rounded up to the lattice) */
  int m;                             /* subdomain count (perfect square) */
  int n_levels;
  int degree; /* 1 (P1) or 2 (P2, fespace.cpp:230-312) */
  int nev;
  int example;
  int workers; /* accepted for parity; the GPU path has no worker threads */
  double cg_tol;
  int deterministic;
  int device; /* CUDA device ordinal of the context (B200-specific) */
  uint64_t seed; /* example 2 only: coefficient seed */
  /* Corner hole [hole_x_min, hole_x_max] x [hole_y_min, hole_y_max] removed
   * from the rectangle -> an L-shaped domain (BASELINE config 3; B200
   * extension, the reference meshes rectangles only).  All zero = none.  Must
   * lie on the coarse lattice and touch exactly one corner.  Full vectors stay
   * on the bounding lattice: points strictly inside the hole are inactive
   * (zero, empty rows), points on its edges are Dirichlet boundary. */
  double hole_x_min, hole_x_max, hole_y_min, hole_y_max;
} mlg_config;

typedef struct mlg_ctx mlg_ctx;

typedef struct mlg_level_info {
  int64_t num_vertices, num_triangles, num_boundary_edges;
  int64_t ndofs, n_interior, nnz; /* nnz of A (== nnz of M) */
  int nx, ny, level;
  double h_max;
} mlg_level_info;

/* SolveReport (sparse.hpp:103-107) */
typedef struct mlg_solve_report {
  int iterations;
  double final_residual;
  int converged;
} mlg_solve_report;

/* StepTimings (corrector.hpp:97-101) plus device-side evidence. */
typedef struct mlg_step_timings {
  double local_seconds, iface_seconds, aug_seconds; /* CUDA events, as StepTimings */
  double build_seconds;                             /* extend_to + region data of the step */
  int local_iterations_max, strip_iterations_max;
  double spmv_kernel_ms;   /* summed device time of the sampled local-solve CG iteration
                              launches (k_cg_iter, profiling on) */
  int64_t spmv_launches;   /* number of such launches */
  double spmv_rows;        /* window rows those launches swept in CG-update mode (counted
                              on the device) */
  int64_t kernel_launches; /* CG kernel launches of the step */
  double step_seconds;     /* CUDA events on the context stream around the whole call,
                              host<->device copies included for the host-array variant */
  int spmv_uniform_stencil; /* 1: stencil/D^-1 taken from kernel parameters (no
                               coefficient stream: 48 B/row instead of 88); 2: the
                               same with x updates deferred in pairs (44 B/row
                               averaged over a launch pair); 0: general stencil */
  double spmv_check_rows;  /* rows the same launches swept in true-residual mode */
  int64_t spmv_launches_all; /* all launches of that kernel in the step (sampled or not):
                                the kernel's share of the step is
                                spmv_kernel_ms / spmv_launches * spmv_launches_all */
  double strip_kernel_ms;  /* summed device time of EVERY strip-solve CG launch (profiling on) */
  int64_t strip_launches;  /* number of those launches */
  double strip_row_iters;  /* sum over strip systems of unknowns x CG updates (host count) */
  int strip_kernel;        /* CG kernel of the strip batch: 0 k_cg_iter (one launch per
                              iteration), 1 k_cg_persist (one cooperative launch per
                              solve), 2 k_cg_resident (iterates resident on chip) */
  int strip_bytes_per_row; /* algorithmic bytes per unknown and CG update of that kernel */
  int local_kernel;        /* the CG kernel of the local-solve batch (same codes) */
} mlg_step_timings;

const char* mlg_last_error(void);

/* Hierarchy::Hierarchy (corrector.cpp:111-129): validate_config, coarse mesh,
 * partition (decomp.cpp:24-86, delta rounded up corrector.cpp:117-121), level-0
 * space and operators. */
int mlg_create(const mlg_config* cfg, mlg_ctx** out);
void mlg_destroy(mlg_ctx* ctx);

/* Hierarchy::extend_to (corrector.cpp:131-146): refine_regular, register_level,
 * build_space, assemble_form x2, prolongation_matrix -- on device. */
int mlg_extend_to(mlg_ctx* ctx, int level);
int mlg_max_level(mlg_ctx* ctx, int* level);
int mlg_get_level_info(mlg_ctx* ctx, int level, mlg_level_info* out);

/* Mesh arrays (mesh.hpp:32-50): vertices[nv][2], vertex_lattice[nv][2],
 * triangles[nt][3], parent[nt] (level >= 1), boundary_edges[nb][2].  Any
 * pointer may be NULL. */
int mlg_export_mesh(mlg_ctx* ctx, int level, double* vertices, int* vertex_lattice,
                    int* triangles, int* parent, int* boundary_edges);

/* FeSpace (fespace.hpp:52-65): dof_lattice[ndofs][2] (half units),
 * interior_dofs[n_interior], interior_index[ndofs], connectivity[nt][3]
 * (P1) or [nt][6] (P2: v0, v1, v2, m01, m12, m20). */
int mlg_export_space(mlg_ctx* ctx, int level, int* dof_lattice, int* interior_dofs,
                     int* interior_index, int* connectivity3);

/* SparseSymMatrix CSR of the full-space form (sparse.hpp:30-55); form 0 =
 * stiffness (assemble_stiffness), 1 = mass (assemble_mass). */
int mlg_export_csr(mlg_ctx* ctx, int level, int form, int* row_ptr, int* cols, double* values);

/* Partition (decomp.hpp:59-93): rects[m][3][4] = block, overlap, inner as
 * x0,y0,x1,y1 in coarse cells; info[5] = m, side, delta_cells, nx0, ny0. */
int mlg_partition(mlg_ctx* ctx, int* rects, int* info);

/* restrict_space (decomp.cpp:167-217); kind 0 domain, 1 block, 2 overlap,
 * 3 inner, 4 strip.  out may be NULL to query the count. */
int mlg_region_dofs(mlg_ctx* ctx, int level, int kind, int j, int zero_trace, int* out,
                    int64_t* count);
/* Partition::region_elements (decomp.cpp:148-165). */
int mlg_region_elements(mlg_ctx* ctx, int level, int kind, int j, int* out, int64_t* count);

/* SparseSymMatrix::multiply (sparse.cpp:69-76) on full vectors. */
int mlg_spmv(mlg_ctx* ctx, int level, int form, const double* x_full, double* y_full);
/* Hierarchy::prolong / restrict_transpose (corrector.cpp:158-170), full vectors. */
int mlg_prolong(mlg_ctx* ctx, int from_level, int to_level, const double* x, double* y);
int mlg_restrict_transpose(mlg_ctx* ctx, int from_level, int to_level, const double* x,
                           double* y);

/* coarse_eigensolve / solve_interior_eigenproblem (fespace.hpp:128-132,
 * sparse.cpp:326-355): lambdas[nev], coeffs[nev][n_interior]. */
int mlg_coarse_eigensolve(mlg_ctx* ctx, int level, int nev, double* lambdas, double* coeffs);

/* local_bvp_solve (corrector.hpp:112-113, corrector.cpp:198-214). */
int mlg_local_bvp_solve(mlg_ctx* ctx, int level, int j, double lambda, const double* u_full,
                        double cg_tol, double* e_full, mlg_solve_report* report);

/* interface_solve (corrector.hpp:118-120, corrector.cpp:216-254);
 * corrections[m][ndofs]. */
/* The CG of local_bvp_solve with cg_solve's own contract (sparse.hpp:109-116,
 * sparse.cpp:199-258): maxit > 0 replaces the default 10 n, non-convergence is
 * REPORTED (report->converged = 0, final_residual = true relative residual),
 * not thrown; a zero right-hand side returns after 0 iterations.  e_full as in
 * mlg_local_bvp_solve. */
int mlg_local_cg_solve(mlg_ctx* ctx, int level, int j, double lambda, const double* u_full,
                       double cg_tol, int maxit, double* e_full, mlg_solve_report* report);

int mlg_interface_solve(mlg_ctx* ctx, int level, double lambda, const double* u_full,
                        const double* corrections, double cg_tol, double* glued_full,
                        mlg_solve_report* report);

/* augmented_eigensolve (corrector.hpp:127-128, corrector.cpp:256-334);
 * glued[k_in][ndofs] (k_in <= 8); lambdas[nev], coeffs[nev][n_interior]. */
int mlg_augmented_eigensolve(mlg_ctx* ctx, int level, int k_in, const double* glued_full,
                             int nev, double* lambdas, double* coeffs);

/* one_correction_step (corrector.hpp:135-136, corrector.cpp:336-412).
 * coeffs_in[nev][n_interior(from)], coeffs_out[nev][n_interior(to)];
 * matched = CorrectionState::matched_previous.  nev <= 8. */
int mlg_correction_step(mlg_ctx* ctx, int from_level, int to_level, int nev,
                        const double* lambdas_in, const double* coeffs_in, double* lambdas_out,
                        double* coeffs_out, int* matched, mlg_step_timings* timings);

/* Same, with coefficient arrays resident in device memory (same layout).
 * Ordering: before touching d_coeffs_in / d_coeffs_out the call makes the
 * context's stream wait for all work already queued on the input stream
 * (mlg_set_input_stream; default the legacy default stream 0), so a caller that
 * filled the input with asynchronous kernels or copies on that stream need not
 * synchronize first.  The call returns after the outputs are written. */
int mlg_correction_step_device(mlg_ctx* ctx, int from_level, int to_level, int nev,
                               const double* lambdas_in, const double* d_coeffs_in,
                               double* lambdas_out, double* d_coeffs_out, int* matched,
                               mlg_step_timings* timings);

/* multilevel_correction (corrector.cpp:414-462) up to last_level (<= 0: the
 * config's n_levels): lambdas[last_level][nev] (row k-1 = level k), matched
 * and timings per level (may be NULL); final coefficients to host and/or
 * device arrays [nev][n_interior(last)] (either may be NULL). */
int mlg_multilevel_correction(mlg_ctx* ctx, int last_level, double* lambdas,
                              double* final_coeffs, double* d_final_coeffs, int* matched,
                              mlg_step_timings* timings);

/* The CUDA stream (cudaStream_t, as void*) whose queued work the *_device entry
 * points wait for before reading or writing caller device buffers; NULL (the
 * default) = the legacy default stream. */
int mlg_set_input_stream(mlg_ctx* ctx, void* stream);

/* Record CUDA events around every local-solve SpMV launch (roofline evidence). */
int mlg_set_profiling(mlg_ctx* ctx, int on);

/* Assembly kernel evidence of the most recent level built with profiling on:
 * summed CUDA-event time of its operator assembly launch(es) and the dofs they
 * assembled (fespace.cpp:314-341 replaced by k_assemble). */
int mlg_build_profile(mlg_ctx* ctx, double* assemble_ms, double* assemble_dofs);
/* Which assembly kernel that launch was: 0 k_assemble (generic row gather),
 * 1 k_assemble_table (translation-invariant lattice: element matrices from a
 * six-variant table, bitwise the generic result), 2 k_assemble_var. */
int mlg_build_profile_kernel(mlg_ctx* ctx, int* kernel);

/* Interior-stiffness SpMV microbenchmark (extract_submatrix(A, interior) x):
 * average device ms per launch over `reps` launches, and its algorithmic bytes. */
int mlg_bench_spmv(mlg_ctx* ctx, int level, int reps, double* ms_per_launch,
                   double* bytes_per_launch);

/* ---- error reporting and the experiment harness ------------------------
 * (fespace.cpp:434-488 compute_errors, harness.cpp of the reference).  The
 * closed-form reference eigenfunctions of make_reference are separable sine
 * modes, so they cross the ABI as parameters instead of std::function. */

/* amp * sin(mx pi (x-x0)/lx) * sin(my pi (y-y0)/ly); mx == 0: no closed form
 * (the eigenvalue is multiple, harness.cpp:146-152). */
typedef struct mlg_exact_mode {
  int mx, my;
  double x0, lx, y0, ly, amp;
} mlg_exact_mode;

/* ErrorReport (fespace.hpp:108-112); l2/h1 are NaN without a closed form. */
typedef struct mlg_error_report {
  double eig_err, l2_err, h1_err;
} mlg_error_report;

/* make_reference (harness.cpp:126-169): example 0 laplace, 1 variable.
 * domain = {x_min, x_max, y_min, y_max} generalises the reference's (-1,1)^2
 * Laplace table to the configured rectangle (bitwise the reference's table on
 * (-1,1)^2); NULL = the reference's table.  lambdas[nev], modes[nev] (either
 * may be NULL). */
int mlg_make_reference(int example, int nev, const double* domain, double* lambdas,
                       mlg_exact_mode* modes);

/* The reference set run_experiment uses for a configuration: make_reference
 * on the configured rectangle, or the L-shaped domain's table when cfg has
 * the unit corner hole of (-1,1)^2 (config 3). */
int mlg_make_reference_for(const mlg_config* cfg, int nev, double* lambdas,
                           mlg_exact_mode* modes);

/* compute_errors (fespace.cpp:434-488) of a full coefficient vector at
 * `level` against lambda_ref and (if non-NULL with mx > 0) the closed form:
 * 49-point Gauss-Duffy sweep over every element, on device. */
int mlg_compute_errors(mlg_ctx* ctx, int level, const double* coeffs_full, double lambda_h,
                       double lambda_ref, const mlg_exact_mode* reference,
                       mlg_error_report* out);

/* multilevel_correction with a ReferenceSet (corrector.cpp:414-462): as
 * mlg_multilevel_correction plus per-level errors of the first n_refs pairs
 * (LevelTrace::eig_errors / h1_errors, computed on the resident vectors);
 * eig_err / l2_err / h1_err are [last_level][nev] (NaN where undefined), any
 * may be NULL. */
int mlg_multilevel_correction_refs(mlg_ctx* ctx, int last_level, int n_refs,
                                   const double* ref_lambdas, const mlg_exact_mode* ref_modes,
                                   double* lambdas, double* eig_err, double* l2_err,
                                   double* h1_err, double* final_coeffs, int* matched,
                                   mlg_step_timings* timings);

/* parse_config_json / parse_config_file (harness.cpp:58-111): strict JSON
 * (every field required, unknown keys rejected, ints must be integers), then
 * validate_config.  device is set to 0. */
int mlg_parse_config_json(const char* json_text, mlg_config* out);
int mlg_parse_config_file(const char* path, mlg_config* out);

/* estimate_orders (harness.cpp:113-122): orders[n-1]. */
int mlg_estimate_orders(const double* errors, int n, double beta, double* orders);

/* ReportRow (harness.hpp:23-35); optional columns carry a has_* flag. */
typedef struct mlg_report_row {
  int level;
  double h;
  int dofs, eig_index;
  double lambda, eig_err;
  int has_h1;
  double h1_err;
  int has_order;
  double order;
  double local_s, iface_s, aug_s;
} mlg_report_row;

/* run_experiment (harness.cpp:171-206): multilevel correction with the
 * reference set of the example, rows written to csv_path (write_csv,
 * harness.cpp:208-222, %.17g, byte-identical across runs when deterministic).
 * rows may be NULL; n_rows receives n_levels*nev. */
int mlg_run_experiment(const mlg_config* cfg, const char* csv_path, mlg_report_row* rows,
                       int rows_cap, int* n_rows);
int mlg_write_csv(const mlg_report_row* rows, int n, const char* path);

/* print_table (harness.cpp:240-290) into buf (NUL-terminated, truncated to
 * cap); *len = full length. */
int mlg_print_table(const char* csv_path, char* buf, size_t cap, size_t* len);

/* export_vtk (harness.cpp:292-351): final-level eigenfunctions as VTK legacy
 * ASCII point data in out_dir/eigenfunctions.vtk. */
int mlg_export_vtk(const mlg_config* cfg, const char* out_dir);

#ifdef __cplusplus
}
#endif

#endif /* MLG_B200_H */

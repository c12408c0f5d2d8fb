// TEST INFRASTRUCTURE ONLY (oracle).  A thin C-ABI over the UNMODIFIED
// reference library (compiled from /root/reference/proj/src by Makefile), so
// the Python tests and bench.py's CPU baseline leg can drive the reference's
// own entry points through ctypes:
//   Hierarchy ctor / extend_to            corrector.hpp:63-95, corrector.cpp:111-146
//   Mesh / FeSpace / CSR exports           mesh.hpp:32-50, fespace.hpp:52-65, sparse.hpp:30-55
//   restrict_space / region_elements       decomp.hpp:88-104, decomp.cpp:148-217
//   coarse_eigensolve                      fespace.hpp:128-132
//   local_bvp_solve / interface_solve /
//   augmented_eigensolve / one_correction_step   corrector.hpp:112-136
//   cg_solve / dense_gen_eigensolve        sparse.hpp:118-131
//   compute_errors                         fespace.hpp:118-120
//   parse_config_json / run_experiment /
//   print_table / export_vtk / make_reference   harness.hpp:16-67
// Status codes follow the reference's exit-code taxonomy (mleig_main.cpp:57-66):
// 0 ok, 2 ConfigError, 3 SolverError, 4 IoError, 1 anything else.
#include <chrono>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include <sstream>

#include "mleig/corrector.hpp"
#include "mleig/harness.hpp"
#include "mleig/decomp.hpp"
#include "mleig/fespace.hpp"
#include "mleig/mesh.hpp"
#include "mleig/sparse.hpp"

using namespace mleig;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const SolverError& e) {
    g_err = e.what();
    return 3;
  } catch (const IoError& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

Hierarchy& H(void* h) { return *static_cast<Hierarchy*>(h); }

Region region_of(int kind, int j) {
  switch (kind) {
    case 0: return Region::domain();
    case 1: return Region::block(j);
    case 2: return Region::overlap(j);
    case 3: return Region::inner(j);
    case 4: return Region::strip();
  }
  throw ConfigError("unknown region kind");
}

Vector to_vec(const double* p, long n) {
  Vector v(n);
  for (long i = 0; i < n; ++i) v[i] = p[i];
  return v;
}
void from_vec(const Vector& v, double* p) {
  for (long i = 0; i < v.size(); ++i) p[i] = v[i];
}

}  // namespace

extern "C" {

struct RefConfig {
  double x_min, x_max, y_min, y_max;
  double H;
  double delta;
  int m;
  int n_levels;
  int degree;
  int nev;
  int example;  // 0 laplace, 1 variable
  int workers;
  double cg_tol;
  int deterministic;
};

const char* ref_last_error() { return g_err.c_str(); }

int ref_create(const RefConfig* c, void** out) {
  return guarded([&] {
    RunConfig cfg;
    cfg.domain = {c->x_min, c->x_max, c->y_min, c->y_max};
    cfg.H = c->H;
    cfg.delta = c->delta;
    cfg.m = c->m;
    cfg.n_levels = c->n_levels;
    cfg.degree = c->degree;
    cfg.nev = c->nev;
    cfg.example = c->example == 1 ? "variable" : "laplace";
    cfg.workers = c->workers;
    cfg.cg_tol = c->cg_tol;
    cfg.deterministic = c->deterministic != 0;
    *out = new Hierarchy(cfg);
  });
}

void ref_destroy(void* h) { delete static_cast<Hierarchy*>(h); }

int ref_set_workers(void* h, int workers) {
  // RunConfig is const inside Hierarchy; rebuild is the only public way, so
  // this hook is limited to reading.  Kept for ABI symmetry.
  (void)h;
  (void)workers;
  g_err = "workers are fixed at construction";
  return 2;
}

int ref_extend_to(void* h, int level, double* seconds) {
  return guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    H(h).extend_to(level);
    if (seconds)
      *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

int ref_build_region_systems(void* h, int level, double* seconds) {
  return guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    H(h).level(level).build_region_systems(H(h).partition());
    if (seconds)
      *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

// out[0..9] = nv, nt, nb, ndofs, n_int, nnz_a, nnz_m, nx, ny, level
int ref_level_sizes(void* h, int level, long long* out, double* h_max) {
  return guarded([&] {
    const LevelSystem& L = H(h).level(level);
    const Mesh& m = *L.mesh;
    out[0] = static_cast<long long>(m.vertices.size());
    out[1] = static_cast<long long>(m.triangles.size());
    out[2] = static_cast<long long>(m.boundary_edges.size());
    out[3] = L.space.ndofs;
    out[4] = static_cast<long long>(L.space.interior_dofs.size());
    out[5] = L.stiffness.nonzeros();
    out[6] = L.mass.nonzeros();
    out[7] = m.nx;
    out[8] = m.ny;
    out[9] = m.level;
    if (h_max) *h_max = m.h_max;
  });
}

int ref_export_mesh(void* h, int level, double* verts, int* lattice, int* tris, int* parent,
                    int* bedges) {
  return guarded([&] {
    const Mesh& m = *H(h).level(level).mesh;
    for (std::size_t i = 0; i < m.vertices.size(); ++i) {
      if (verts) {
        verts[2 * i] = m.vertices[i].x;
        verts[2 * i + 1] = m.vertices[i].y;
      }
      if (lattice) {
        lattice[2 * i] = m.vertex_lattice[i][0];
        lattice[2 * i + 1] = m.vertex_lattice[i][1];
      }
    }
    if (tris)
      for (std::size_t t = 0; t < m.triangles.size(); ++t)
        for (int k = 0; k < 3; ++k) tris[3 * t + k] = m.triangles[t][k];
    if (parent)
      for (std::size_t t = 0; t < m.parent.size(); ++t) parent[t] = m.parent[t];
    if (bedges)
      for (std::size_t b = 0; b < m.boundary_edges.size(); ++b) {
        bedges[2 * b] = m.boundary_edges[b][0];
        bedges[2 * b + 1] = m.boundary_edges[b][1];
      }
  });
}

int ref_export_space(void* h, int level, int* dof_lattice, int* interior_dofs,
                     int* interior_index, int* conn3) {
  return guarded([&] {
    const FeSpace& s = H(h).level(level).space;
    if (dof_lattice)
      for (int d = 0; d < s.ndofs; ++d) {
        dof_lattice[2 * d] = s.dof_lattice[d][0];
        dof_lattice[2 * d + 1] = s.dof_lattice[d][1];
      }
    if (interior_dofs)
      for (std::size_t i = 0; i < s.interior_dofs.size(); ++i) interior_dofs[i] = s.interior_dofs[i];
    if (interior_index)
      for (int d = 0; d < s.ndofs; ++d) interior_index[d] = s.interior_index[d];
    if (conn3) {  // dofs_per_elem columns (3 for P1, 6 for P2)
      const int nd = s.dofs_per_elem();
      for (std::size_t e = 0; e < s.connectivity.size(); ++e)
        for (int k = 0; k < nd; ++k) conn3[nd * e + k] = s.connectivity[e][k];
    }
  });
}

// form: 0 stiffness, 1 mass.  row_ptr is recovered from the row spans.
int ref_export_csr(void* h, int level, int form, int* row_ptr, int* cols, double* vals) {
  return guarded([&] {
    const LevelSystem& L = H(h).level(level);
    const SparseSymMatrix& a = form == 0 ? L.stiffness : L.mass;
    long long k = 0;
    for (int r = 0; r < a.rows(); ++r) {
      if (row_ptr) row_ptr[r] = static_cast<int>(k);
      auto c = a.row_cols(r);
      auto v = a.row_values(r);
      for (std::size_t i = 0; i < c.size(); ++i, ++k) {
        if (cols) cols[k] = c[i];
        if (vals) vals[k] = v[i];
      }
    }
    if (row_ptr) row_ptr[a.rows()] = static_cast<int>(k);
  });
}

int ref_spmv(void* h, int level, int form, const double* x, double* y) {
  return guarded([&] {
    const LevelSystem& L = H(h).level(level);
    const SparseSymMatrix& a = form == 0 ? L.stiffness : L.mass;
    from_vec(a.apply(to_vec(x, a.rows())), y);
  });
}

int ref_prolong(void* h, int from, int to, const double* x, double* y) {
  return guarded([&] {
    const int n = H(h).level(from).space.ndofs;
    from_vec(H(h).prolong(to_vec(x, n), from, to), y);
  });
}

int ref_restrict_transpose(void* h, int from, int to, const double* x, double* y) {
  return guarded([&] {
    const int n = H(h).level(from).space.ndofs;
    from_vec(H(h).restrict_transpose(to_vec(x, n), from, to), y);
  });
}

// kind: 0 domain, 1 block, 2 overlap, 3 inner, 4 strip.  out may be null.
int ref_region_dofs(void* h, int level, int kind, int j, int zero_trace, int* out,
                    long long* count) {
  return guarded([&] {
    const SubSpace s = restrict_space(H(h).level(level).space, H(h).partition(),
                                      region_of(kind, j), zero_trace != 0);
    *count = static_cast<long long>(s.dofs.size());
    if (out)
      for (std::size_t i = 0; i < s.dofs.size(); ++i) out[i] = s.dofs[i];
  });
}

int ref_region_elements(void* h, int level, int kind, int j, int* out, long long* count) {
  return guarded([&] {
    const auto& e = H(h).partition().region_elements(level, region_of(kind, j));
    *count = static_cast<long long>(e.size());
    if (out)
      for (std::size_t i = 0; i < e.size(); ++i) out[i] = e[i];
  });
}

// rects: m x 3 x 4 ints (block, overlap, inner) as x0,y0,x1,y1;
// info: m, side, delta_cells, coarse_nx, coarse_ny
int ref_partition(void* h, int* rects, int* info) {
  return guarded([&] {
    const Partition& p = H(h).partition();
    info[0] = p.num_subdomains();
    info[1] = p.grid_side();
    info[2] = p.overlap_cells();
    info[3] = p.coarse_nx();
    info[4] = p.coarse_ny();
    if (rects)
      for (int j = 0; j < p.num_subdomains(); ++j) {
        const IRect rs[3] = {p.block_rect(j), p.overlap_rect(j), p.inner_rect(j)};
        for (int k = 0; k < 3; ++k) {
          int* o = rects + 12 * j + 4 * k;
          o[0] = rs[k].x0;
          o[1] = rs[k].y0;
          o[2] = rs[k].x1;
          o[3] = rs[k].y1;
        }
      }
  });
}

int ref_coarse_eigensolve(void* h, int level, int nev, double* lambdas, double* coeffs) {
  return guarded([&] {
    H(h).extend_to(level);
    const LevelSystem& L = H(h).level(level);
    const auto pairs = coarse_eigensolve(L.space, L.stiffness, L.mass, nev);
    const long n = static_cast<long>(L.space.interior_dofs.size());
    for (int i = 0; i < nev; ++i) {
      lambdas[i] = pairs[i].lambda;
      from_vec(pairs[i].coeffs, coeffs + i * n);
    }
  });
}

int ref_local_bvp_solve(void* h, int level, int j, double lambda, const double* u_full,
                        double tol, double* e_full, int* iters, double* final_res) {
  return guarded([&] {
    LevelSystem& L = H(h).level(level);
    L.build_region_systems(H(h).partition());
    SolveReport rep;
    const Vector e = local_bvp_solve(L, j, lambda, to_vec(u_full, L.space.ndofs), tol, &rep);
    from_vec(e, e_full);
    if (iters) *iters = rep.iterations;
    if (final_res) *final_res = rep.final_residual;
  });
}

// Timing samples for bench.py's reference arm (bounded samples of a correction
// step whose full run takes tens of minutes at 4096^2):
//  * ref_local_bvp_time: one local_bvp_solve task exactly as one_correction_step
//    runs it (corrector.cpp:364-370 -> :198-214), timed around the call only;
//    concurrent calls from several host threads are what parallel_tasks does
//    (region systems are built first, then only read).
//  * ref_strip_cg_sample: the reference's cg_solve (sparse.cpp:199-258) on the
//    level's strip system with interface_solve's load form (corrector.cpp:238-242,
//    glued = u), capped at maxit iterations, timed around cg_solve only.
int ref_local_bvp_time(void* h, int level, int j, double lambda, const double* u_full,
                       double tol, double* seconds, int* iters) {
  return guarded([&] {
    LevelSystem& L = H(h).level(level);
    L.build_region_systems(H(h).partition());
    const Vector u = to_vec(u_full, L.space.ndofs);
    SolveReport rep;
    const auto t0 = std::chrono::steady_clock::now();
    const Vector e = local_bvp_solve(L, j, lambda, u, tol, &rep);
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (iters) *iters = rep.iterations;
  });
}

int ref_strip_cg_sample(void* h, int level, double lambda, const double* u_full, double tol,
                        int maxit, double* seconds, int* iters) {
  return guarded([&] {
    LevelSystem& L = H(h).level(level);
    L.build_region_systems(H(h).partition());
    const Vector u = to_vec(u_full, L.space.ndofs);
    const Vector load = lambda * L.mass.apply(u) - L.stiffness.apply(u);
    const RegionSystem& strip = L.strip_system;
    Vector rhs(static_cast<int>(strip.dofs.size()));
    for (std::size_t i = 0; i < strip.dofs.size(); ++i)
      rhs[static_cast<int>(i)] = load[strip.dofs[i]];
    const auto t0 = std::chrono::steady_clock::now();
    auto [x, rep] = cg_solve(strip.a_sub, rhs, tol, maxit);
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (iters) *iters = rep.iterations;
  });
}

int ref_interface_solve(void* h, int level, double lambda, const double* u_full,
                        const double* corrections, double tol, double* glued, int* iters,
                        double* final_res) {
  return guarded([&] {
    LevelSystem& L = H(h).level(level);
    L.build_region_systems(H(h).partition());
    const int m = H(h).partition().num_subdomains();
    const long n = L.space.ndofs;
    std::vector<Vector> corr;
    for (int j = 0; j < m; ++j) corr.push_back(to_vec(corrections + j * n, n));
    SolveReport rep;
    const Vector g =
        interface_solve(L, H(h).partition(), lambda, to_vec(u_full, n), corr, tol, &rep);
    from_vec(g, glued);
    if (iters) *iters = rep.iterations;
    if (final_res) *final_res = rep.final_residual;
  });
}

int ref_augmented_eigensolve(void* h, int level, int k_in, const double* glued, int nev,
                             double* lambdas, double* coeffs) {
  return guarded([&] {
    const long n = H(h).level(level).space.ndofs;
    std::vector<Vector> g;
    for (int l = 0; l < k_in; ++l) g.push_back(to_vec(glued + l * n, n));
    const auto pairs = augmented_eigensolve(H(h), level, g, nev);
    const long ni = static_cast<long>(H(h).level(level).space.interior_dofs.size());
    for (std::size_t i = 0; i < pairs.size(); ++i) {
      lambdas[i] = pairs[i].lambda;
      from_vec(pairs[i].coeffs, coeffs + static_cast<long>(i) * ni);
    }
  });
}

int ref_correction_step(void* h, int from, int to, int nev, const double* lam_in,
                        const double* coeffs_in, double* lam_out, double* coeffs_out,
                        int* matched, double* timings3) {
  return guarded([&] {
    H(h).extend_to(std::max(from, to));
    CorrectionState st;
    st.level = from;
    const long nin = static_cast<long>(H(h).level(from).space.interior_dofs.size());
    for (int i = 0; i < nev; ++i) {
      EigenPair p;
      p.lambda = lam_in[i];
      p.coeffs = to_vec(coeffs_in + i * nin, nin);
      p.level = from;
      st.pairs.push_back(std::move(p));
    }
    StepTimings t;
    const CorrectionState out = one_correction_step(H(h), st, to, &t);
    const long nout = static_cast<long>(H(h).level(to).space.interior_dofs.size());
    for (int i = 0; i < nev; ++i) {
      lam_out[i] = out.pairs[i].lambda;
      if (coeffs_out) from_vec(out.pairs[i].coeffs, coeffs_out + i * nout);
    }
    if (matched) *matched = out.matched_previous ? 1 : 0;
    if (timings3) {
      timings3[0] = t.local_seconds;
      timings3[1] = t.iface_seconds;
      timings3[2] = t.aug_seconds;
    }
  });
}

// Full multilevel run (corrector.cpp:414-462); lambdas is n_levels x nev,
// final_coeffs (may be null) is nev x n_int(final level).
int ref_multilevel(void* h, double* lambdas, double* final_coeffs, int* matched,
                   double* timings) {
  return guarded([&] {
    const MultilevelResult r = multilevel_correction(H(h));
    for (std::size_t k = 0; k < r.levels.size(); ++k) {
      const LevelTrace& t = r.levels[k];
      for (std::size_t i = 0; i < t.lambdas.size(); ++i)
        lambdas[k * t.lambdas.size() + i] = t.lambdas[i];
      if (matched) matched[k] = t.matched_previous ? 1 : 0;
      if (timings) {
        timings[3 * k] = t.timings.local_seconds;
        timings[3 * k + 1] = t.timings.iface_seconds;
        timings[3 * k + 2] = t.timings.aug_seconds;
      }
    }
    if (final_coeffs) {
      const LevelTrace& last = r.levels.back();
      const long n = static_cast<long>(last.pairs.at(0).coeffs.size());
      for (std::size_t i = 0; i < last.pairs.size(); ++i)
        from_vec(last.pairs[i].coeffs, final_coeffs + static_cast<long>(i) * n);
    }
  });
}

// cg_solve on the symmetric CSR (full storage) given by the arrays.
int ref_cg_solve_csr(int n, const int* row_ptr, const int* cols, const double* vals,
                     const double* rhs, double tol, int maxit, double* x, int* iters,
                     double* final_res, int* converged) {
  return guarded([&] {
    std::vector<Triplet> upper;
    for (int r = 0; r < n; ++r)
      for (int k = row_ptr[r]; k < row_ptr[r + 1]; ++k)
        if (cols[k] >= r) upper.push_back({r, cols[k], vals[k]});
    const auto a = SparseSymMatrix::from_upper_triplets(n, std::move(upper));
    auto [sol, rep] = cg_solve(a, to_vec(rhs, n), tol, maxit);
    from_vec(sol, x);
    *iters = rep.iterations;
    *final_res = rep.final_residual;
    *converged = rep.converged ? 1 : 0;
  });
}

// FNV-1a-64 over raw bytes, chained from h (SURVEY.md Appendix B digests).
unsigned long long ref_fnv1a64(const unsigned char* p, unsigned long long n,
                               unsigned long long h) {
  for (unsigned long long i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 1099511628211ULL;
  }
  return h;
}

// a, b column-major n x n; vecs n x nev column-major.
int ref_dense_gen_eigensolve(int n, const double* a, const double* b, int nev, double* lambdas,
                             double* vecs) {
  return guarded([&] {
    Eigen::MatrixXd A(n, n), B(n, n);
    for (long i = 0; i < static_cast<long>(n) * n; ++i) {
      A.data()[i] = a[i];
      B.data()[i] = b[i];
    }
    const auto pairs = dense_gen_eigensolve(A, B, nev);
    for (int i = 0; i < nev; ++i) {
      lambdas[i] = pairs[i].lambda;
      from_vec(pairs[i].vec, vecs + static_cast<long>(i) * n);
    }
  });
}

// ---- harness and error reporting (harness.hpp, fespace.hpp:103-120) ----
static void to_ref(const RunConfig& cfg, RefConfig* c) {
  c->x_min = cfg.domain.x_min;
  c->x_max = cfg.domain.x_max;
  c->y_min = cfg.domain.y_min;
  c->y_max = cfg.domain.y_max;
  c->H = cfg.H;
  c->delta = cfg.delta;
  c->m = cfg.m;
  c->n_levels = cfg.n_levels;
  c->degree = cfg.degree;
  c->nev = cfg.nev;
  c->example = cfg.example == "variable" ? 1 : (cfg.example == "laplace" ? 0 : -1);
  c->workers = cfg.workers;
  c->cg_tol = cfg.cg_tol;
  c->deterministic = cfg.deterministic ? 1 : 0;
}

static RunConfig from_ref(const RefConfig* c) {
  RunConfig cfg;
  cfg.domain = {c->x_min, c->x_max, c->y_min, c->y_max};
  cfg.H = c->H;
  cfg.delta = c->delta;
  cfg.m = c->m;
  cfg.n_levels = c->n_levels;
  cfg.degree = c->degree;
  cfg.nev = c->nev;
  cfg.example = c->example == 1 ? "variable" : "laplace";
  cfg.workers = c->workers;
  cfg.cg_tol = c->cg_tol;
  cfg.deterministic = c->deterministic != 0;
  return cfg;
}

int ref_parse_config_json(const char* text, RefConfig* out) {
  return guarded([&] { to_ref(parse_config_json(text), out); });
}

int ref_parse_config_file(const char* path, RefConfig* out) {
  return guarded([&] { to_ref(parse_config_file(path), out); });
}

int ref_estimate_orders(const double* e, int n, double beta, double* out) {
  return guarded([&] {
    const auto o = estimate_orders(std::vector<double>(e, e + n), beta);
    for (std::size_t k = 0; k < o.size(); ++k) out[k] = o[k];
  });
}

// lambdas[nev]; has_fn[nev]; fn values at the probe points (x,y)[np] -> vals[nev][np][3]
// (value, du/dx, du/dy) for the indices with a closed form.
int ref_make_reference(const char* example, int nev, double* lambdas, int* has_fn, int np,
                       const double* pts, double* vals) {
  return guarded([&] {
    const ReferenceSet r = make_reference(example, nev);
    for (int i = 0; i < nev; ++i) {
      lambdas[i] = r.lambdas[i];
      auto it = r.eigenfunctions.find(i);
      has_fn[i] = it != r.eigenfunctions.end();
      if (has_fn[i] && vals)
        for (int k = 0; k < np; ++k) {
          const double x = pts[2 * k], y = pts[2 * k + 1];
          const auto g = it->second.gradient(x, y);
          double* o = vals + (static_cast<long>(i) * np + k) * 3;
          o[0] = it->second.value(x, y);
          o[1] = g[0];
          o[2] = g[1];
        }
    }
  });
}

// compute_errors with the make_reference("laplace") eigenfunction of index
// ref_index (< 0: none), on a full coefficient vector of `level`.
int ref_compute_errors(void* h, int level, const double* coeffs_full, double lambda_h,
                       double lambda_ref, int ref_index, double* out3) {
  return guarded([&] {
    const LevelSystem& L = H(h).level(level);
    const ReferenceSet r = make_reference("laplace", std::max(ref_index + 1, 1));
    const ExactFunction* fn = nullptr;
    if (ref_index >= 0) fn = &r.eigenfunctions.at(ref_index);
    const ErrorReport e = compute_errors(L.space, H(h).field(), to_vec(coeffs_full, L.space.ndofs),
                                         lambda_h, lambda_ref, fn);
    out3[0] = e.eig_err;
    out3[1] = e.l2_err;
    out3[2] = e.h1_err;
  });
}

int ref_run_experiment(const RefConfig* c, const char* csv_path) {
  return guarded([&] { run_experiment(from_ref(c), csv_path); });
}

int ref_print_table(const char* csv_path, char* buf, unsigned long cap, unsigned long* len) {
  return guarded([&] {
    std::ostringstream os;
    print_table(csv_path, os);
    const std::string s = os.str();
    *len = s.size();
    if (buf && cap > 0) {
      const std::size_t n = std::min<std::size_t>(cap - 1, s.size());
      std::memcpy(buf, s.data(), n);
      buf[n] = '\0';
    }
  });
}

int ref_export_vtk(const RefConfig* c, const char* out_dir) {
  return guarded([&] { export_vtk(from_ref(c), out_dir); });
}

}  // extern "C"

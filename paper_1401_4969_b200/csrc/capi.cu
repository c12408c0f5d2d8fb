// extern "C" boundary (include/mlg_b200.h): marshals host arrays, maps the
// exception taxonomy to status codes, and calls the device implementation.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/mlg_b200.h"
#include "corrector.cuh"
#include "errors.cuh"
#include "vec_kernels.cuh"

struct mlg_ctx {
  std::unique_ptr<mlg::Ctx> c;
};

namespace mlg {
std::string& last_error_slot() {
  static thread_local std::string s;
  return s;
}
}  // namespace mlg

namespace {

// The message slot is thread-local: look it up on the calling thread every
// time (a namespace-scope reference would bind the loader thread's slot).
template <class F>
int guarded(F&& f) {
  std::string& g_err = mlg::last_error_slot();
  try {
    f();
    g_err.clear();
    return MLG_OK;
  } catch (const mlg::ConfigError& e) {
    g_err = e.what();
    return MLG_ERR_CONFIG;
  } catch (const mlg::SolverError& e) {
    g_err = e.what();
    return MLG_ERR_SOLVER;
  } catch (const mlg::IoError& e) {
    g_err = e.what();
    return MLG_ERR_IO;
  } catch (const mlg::CudaError& e) {
    g_err = e.what();
    return MLG_ERR_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MLG_ERR_OTHER;
  }
}

mlg::Ctx& C(mlg_ctx* x) {
  if (!x || !x->c) throw mlg::ConfigError("null context");
  MLG_CUDA(cudaSetDevice(x->c->cfg.device));  // one context per device, any host thread
  return *x->c;
}

void fill_timings(mlg_step_timings* t, const mlg::StepTimes& s, const mlg::Ctx& c) {
  if (!t) return;
  t->local_seconds = s.local_s;
  t->iface_seconds = s.iface_s;
  t->aug_seconds = s.aug_s;
  t->build_seconds = s.build_s;
  t->local_iterations_max = s.local_iters_max;
  t->strip_iterations_max = s.strip_iters_max;
  t->spmv_kernel_ms = c.times.ka_ms_sum;
  t->spmv_launches = c.times.ka_launches;
  t->spmv_rows = c.times.ka_rows;
  t->spmv_check_rows = c.times.ka_check_rows;
  t->kernel_launches = mlg::launch_counter().load() - c.times.launch_base;
  t->spmv_uniform_stencil = c.times.ka_uniform;
  t->spmv_launches_all = c.times.ka_launches_all;
  t->strip_kernel_ms = c.times.ks_ms;
  t->strip_launches = c.times.ks_launches;
  t->strip_row_iters = c.times.ks_row_iters;
  t->strip_kernel = c.times.ks_kernel;
  t->local_kernel = c.times.ka_kernel;
  t->strip_bytes_per_row = c.times.ks_bytes_per_row;
}

void reset_kernel_stats(mlg::Ctx& c) {
  c.times.ka_ms_sum = 0;
  c.times.ka_launches = 0;
  c.times.ka_launches_all = 0;
  c.times.ka_rows = 0;
  c.times.ka_check_rows = 0;
  c.times.kernel_launches = 0;
  c.times.ks_ms = 0;
  c.times.ks_launches = 0;
  c.times.ks_row_iters = 0;
  c.times.ks_kernel = 0;
  c.times.ks_bytes_per_row = 0;
  c.times.launch_base = mlg::launch_counter().load();
}

struct Region {
  int kind, j;
};

// restrict_space membership in vertex-lattice units (decomp.cpp:167-217).
bool keep_dof(const mlg::Partition& p, int kind, int j, bool zero_trace, int S, int ix, int iy) {
  auto in_rect = [&](const mlg::IRect& r, bool strict) {
    if (strict) return ix > r.x0 * S && ix < r.x1 * S && iy > r.y0 * S && iy < r.y1 * S;
    return ix >= r.x0 * S && ix <= r.x1 * S && iy >= r.y0 * S && iy <= r.y1 * S;
  };
  switch (kind) {
    case 0: return true;
    case 1: return in_rect(p.blocks.at(j), zero_trace);
    case 2: return in_rect(p.overlaps.at(j), zero_trace);
    case 3: return in_rect(p.inners.at(j), zero_trace);
    case 4:
      for (int q = 0; q < p.m; ++q)
        if (in_rect(p.inners[q], !zero_trace)) return false;
      return true;
  }
  throw mlg::ConfigError("unknown region id");
}

mlg::ExactMode from_c(const mlg_exact_mode& m) {
  mlg::ExactMode r;
  r.mx = m.mx;
  r.my = m.my;
  r.x0 = m.x0;
  r.lx = m.lx;
  r.y0 = m.y0;
  r.ly = m.ly;
  r.amp = m.amp;
  return r;
}

mlg_exact_mode to_c(const mlg::ExactMode& m) {
  return mlg_exact_mode{m.mx, m.my, m.x0, m.lx, m.y0, m.ly, m.amp};
}

// multilevel_correction (corrector.cpp:414-462) with the optional ReferenceSet
// of its `record` lambda: errors of the resident (interleaved) coefficients at
// every level, outside the step timers like the reference.
void multilevel_impl(mlg_ctx* ctx, int last_level, int n_refs, const double* ref_lambdas,
                     const mlg_exact_mode* ref_modes, double* lambdas, double* eig_err,
                     double* l2_err, double* h1_err, double* final_coeffs,
                     double* d_final_coeffs, int* matched, mlg_step_timings* timings) {
  mlg::Ctx& c = C(ctx);
  const int nlev = last_level > 0 ? last_level : c.cfg.n_levels;
  const int nev = c.cfg.nev;
  const int nr = mlg::nr_for(nev);
  mlg::DevBuf<double> u, u2;
  auto record = [&](int k, const std::vector<double>& lam) {
    std::copy(lam.begin(), lam.end(), lambdas + static_cast<std::size_t>(k - 1) * nev);
    for (int i = 0; i < nev; ++i) {
      const std::size_t o = static_cast<std::size_t>(k - 1) * nev + i;
      double ee = std::nan(""), l2 = std::nan(""), h1 = std::nan("");
      if (ref_lambdas && i < n_refs) {
        mlg::ExactMode md;
        const bool fn = ref_modes && ref_modes[i].mx > 0;
        if (fn) md = from_c(ref_modes[i]);
        const mlg::ErrorReport r = mlg::compute_errors(c, c.level(k), u.get(), nr, i, lam[i],
                                                       ref_lambdas[i], fn ? &md : nullptr);
        ee = r.eig_err;
        if (fn) {
          l2 = r.l2_err;
          h1 = r.h1_err;
        }
      }
      if (eig_err) eig_err[o] = ee;
      if (l2_err) l2_err[o] = l2;
      if (h1_err) h1_err[o] = h1;
    }
  };
  std::vector<double> lam = mlg::coarse_eigensolve(c, 1, nev, u);
  record(1, lam);
  if (matched) matched[0] = 1;
  if (timings) std::memset(&timings[0], 0, sizeof(mlg_step_timings));
  for (int k = 1; k < nlev; ++k) {
    reset_kernel_stats(c);
    const mlg::StepResult r = mlg::correction_step(c, k, k + 1, nev, lam.data(), u.get(), u2);
    std::swap(u, u2);
    lam = r.lambdas;
    if (matched) matched[k] = r.matched ? 1 : 0;
    if (timings) fill_timings(&timings[k], r.times, c);
    record(k + 1, lam);
  }
  const mlg::Level& L = c.level(nlev);
  if (d_final_coeffs) {
    c.order_after_input();  // the caller's buffer may still be in use on its stream
    mlg::deinterleave(c, L, nr, nev, nullptr, u.get(), 1, d_final_coeffs);
  }
  if (final_coeffs) {
    mlg::DevBuf<double> out(L.nint() * nev);
    mlg::deinterleave(c, L, nr, nev, nullptr, u.get(), 1, out.get());
    out.download(final_coeffs, L.nint() * nev, c.stream);
  }
  c.sync();
}

}  // namespace

extern "C" {

const char* mlg_last_error(void) { return mlg::last_error_slot().c_str(); }

int mlg_create(const mlg_config* cfg, mlg_ctx** out) {
  return guarded([&] {
    if (!cfg || !out) throw mlg::ConfigError("null argument");
    mlg::Config c;
    c.x_min = cfg->x_min;
    c.x_max = cfg->x_max;
    c.y_min = cfg->y_min;
    c.y_max = cfg->y_max;
    c.H = cfg->H;
    c.delta = cfg->delta;
    c.m = cfg->m;
    c.n_levels = cfg->n_levels;
    c.degree = cfg->degree;
    c.nev = cfg->nev;
    c.example = cfg->example;
    c.workers = cfg->workers;
    c.cg_tol = cfg->cg_tol;
    c.deterministic = cfg->deterministic;
    c.device = cfg->device;
    c.seed = cfg->seed;
    c.hole_x0 = cfg->hole_x_min;
    c.hole_x1 = cfg->hole_x_max;
    c.hole_y0 = cfg->hole_y_min;
    c.hole_y1 = cfg->hole_y_max;
    auto h = std::make_unique<mlg_ctx>();
    h->c = std::make_unique<mlg::Ctx>(c);
    *out = h.release();
  });
}

void mlg_destroy(mlg_ctx* ctx) { delete ctx; }

int mlg_extend_to(mlg_ctx* ctx, int level) {
  return guarded([&] { C(ctx).extend_to(level); });
}

int mlg_max_level(mlg_ctx* ctx, int* level) {
  return guarded([&] { *level = C(ctx).max_level(); });
}

int mlg_get_level_info(mlg_ctx* ctx, int level, mlg_level_info* out) {
  return guarded([&] {
    const mlg::Level& L = C(ctx).level(level);
    out->num_vertices = L.nv;
    out->num_triangles = L.nt;
    out->num_boundary_edges = L.nb;
    out->ndofs = L.ndofs();
    out->n_interior = L.nint();
    out->nnz = mlg::csr_nnz(L);
    out->nx = L.nx;
    out->ny = L.ny;
    out->level = L.level;
    out->h_max = L.h_max;
  });
}

int mlg_export_mesh(mlg_ctx* ctx, int level, double* vertices, int* vertex_lattice,
                    int* triangles, int* parent, int* boundary_edges) {
  return guarded([&] {
    mlg::Ctx& c = C(ctx);
    mlg::export_mesh(c, c.level(level), vertices, vertex_lattice, triangles, parent,
                     boundary_edges);
  });
}

int mlg_export_space(mlg_ctx* ctx, int level, int* dof_lattice, int* interior_dofs,
                     int* interior_index, int* connectivity3) {
  return guarded([&] {
    mlg::Ctx& c = C(ctx);
    mlg::export_space(c, c.level(level), dof_lattice, interior_dofs, interior_index,
                      connectivity3);
  });
}

int mlg_export_csr(mlg_ctx* ctx, int level, int form, int* row_ptr, int* cols, double* values) {
  return guarded([&] {
    mlg::Ctx& c = C(ctx);
    if (form != 0 && form != 1) throw mlg::ConfigError("form must be 0 (stiffness) or 1 (mass)");
    mlg::export_csr(c, c.level(level), form, row_ptr, cols, values);
  });
}

int mlg_partition(mlg_ctx* ctx, int* rects, int* info) {
  return guarded([&] {
    const mlg::Partition& p = C(ctx).part;
    info[0] = p.m;
    info[1] = p.side;
    info[2] = p.delta_cells;
    info[3] = p.nx0;
    info[4] = p.ny0;
    if (rects)
      for (int j = 0; j < p.m; ++j) {
        const mlg::IRect rs[3] = {p.blocks[j], p.overlaps[j], p.inners[j]};
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

int mlg_region_dofs(mlg_ctx* ctx, int level, int kind, int j, int zero_trace, int* out,
                    int64_t* count) {
  return guarded([&] {
    mlg::Ctx& c = C(ctx);
    const mlg::Level& L = c.level(level);
    if (kind < 0 || kind > 4) throw mlg::ConfigError("unknown region id");
    if ((kind >= 1 && kind <= 3) && (j < 0 || j >= c.part.m))
      throw mlg::ConfigError("subdomain index out of range");
    const int S = 1 << level;
    const mlg::IMap im = L.imap();
    int64_t n = 0;
    for (int iy = 1; iy < L.ny; ++iy)
      for (int ix = 1; ix < L.nx; ++ix)
        if (im.interior(ix, iy) && keep_dof(c.part, kind, j, zero_trace != 0, S, ix, iy)) {
          if (out) out[n] = iy * (L.nx + 1) + ix;
          ++n;
        }
    *count = n;
  });
}

int mlg_region_elements(mlg_ctx* ctx, int level, int kind, int j, int* out, int64_t* count) {
  return guarded([&] {
    mlg::Ctx& c = C(ctx);
    const mlg::Level& L = c.level(level);
    const mlg::Partition& p = c.part;
    const std::vector<int>* base = nullptr;
    std::vector<int> all;
    switch (kind) {
      case 0:
        all.resize(static_cast<std::size_t>(p.nt0));
        for (std::size_t e = 0; e < all.size(); ++e) all[e] = static_cast<int>(e);
        base = &all;
        break;
      case 1: base = &p.block_elems.at(j); break;
      case 2: base = &p.overlap_elems.at(j); break;
      case 3: base = &p.inner_elems.at(j); break;
      case 4: base = &p.strip_elems; break;
      default: throw mlg::ConfigError("unknown region id");
    }
    const int64_t span = int64_t(1) << (2 * L.level);  // descendants of a level-0 element
    *count = static_cast<int64_t>(base->size()) * span;
    if (out) {
      int64_t k = 0;
      for (int t0 : *base)
        for (int64_t d = 0; d < span; ++d) out[k++] = static_cast<int>(t0 * span + d);
    }
  });
}

int mlg_spmv(mlg_ctx* ctx, int level, int form, const double* x_full, double* y_full) {
  return guarded([&] {
    mlg::Ctx& c = C(ctx);
    const mlg::Level& L = c.level(level);
    mlg::DevBuf<double> x(L.ndofs()), y(L.ndofs());
    x.upload(x_full, L.ndofs(), c.stream);
    mlg::spmv_full(c, L, form, x.get(), y.get());
    y.download(y_full, L.ndofs(), c.stream);
    c.sync();
  });
}

int mlg_prolong(mlg_ctx* ctx, int from_level, int to_level, const double* x, double* y) {
  return guarded([&] {
    mlg::Ctx& c = C(ctx);
    if (from_level > to_level) throw mlg::ConfigError("prolong goes from coarse to fine");
    c.extend_to(to_level);
    const mlg::Level& A = c.level(from_level);
    const mlg::Level& B = c.level(to_level);
    mlg::DevBuf<double> dx(A.ndofs()), dy(B.ndofs());
    dx.upload(x, A.ndofs(), c.stream);
    mlg::prolong_chain(c, 1, dx.get(), from_level, to_level, dy.get());
    dy.download(y, B.ndofs(), c.stream);
    c.sync();
  });
}

int mlg_restrict_transpose(mlg_ctx* ctx, int from_level, int to_level, const double* x,
                           double* y) {
  return guarded([&] {
    mlg::Ctx& c = C(ctx);
    if (from_level < to_level)
      throw mlg::ConfigError("restrict_transpose goes from fine to coarse");
    const mlg::Level& A = c.level(from_level);
    const mlg::Level& B = c.level(to_level);
    mlg::DevBuf<double> dx(A.ndofs()), dy(B.ndofs());
    dx.upload(x, A.ndofs(), c.stream);
    mlg::restrict_levels(c, 1, dx.get(), from_level, to_level, dy.get());
    dy.download(y, B.ndofs(), c.stream);
    c.sync();
  });
}

int mlg_coarse_eigensolve(mlg_ctx* ctx, int level, int nev, double* lambdas, double* coeffs) {
  return guarded([&] {
    mlg::Ctx& c = C(ctx);
    mlg::DevBuf<double> u;
    const auto lam = mlg::coarse_eigensolve(c, level, nev, u);
    const mlg::Level& L = c.level(level);
    std::copy(lam.begin(), lam.end(), lambdas);
    if (coeffs) {
      mlg::DevBuf<double> out(L.nint() * nev);
      mlg::deinterleave(c, L, mlg::nr_for(nev), nev, nullptr, u.get(), 1, out.get());
      out.download(coeffs, L.nint() * nev, c.stream);
      c.sync();
    }
  });
}

namespace {
// local_bvp_solve (corrector.cpp:198-214) on one subdomain; maxit > 0 overrides
// cg_solve's default 10 n (sparse.cpp:204).
void local_solve_impl(mlg_ctx* ctx, int level, int j, double lambda, const double* u_full,
                      double cg_tol, int maxit, double* e_full, mlg_solve_report* report,
                      bool throw_unconverged) {
    mlg::Ctx& c = C(ctx);
    mlg::Level& F = c.level(level);
    if (j < 0 || j >= c.part.m) throw mlg::ConfigError("subdomain index out of range");
    if (!(cg_tol > 0.0)) throw mlg::ConfigError("cg_solve: tolerance must be positive");
    const int64_t nd = F.ndofs();
    mlg::DevBuf<double> u(nd), res(nd);
    u.upload(u_full, nd, c.stream);
    // boundary entries do not enter (the reference's u_full is zero there)
    mlg::DevBuf<double> ui(nd);
    mlg::interleave(c, F, 1, 1, u.get(), 0, ui.get());
    mlg::residual(c, F, 1, ui.get(), &lambda, res.get());
    std::vector<mlg::SolveReport> rep;
    mlg::local_solves(c, F, 1, 1, res.get(), cg_tol, maxit, &rep, j);
    const mlg::LocalView b = mlg::local_view(c);
    const mlg::CgSys s = b.systems[0];
    std::vector<double> x(static_cast<std::size_t>(s.h) * s.pitch);  // window rows, pitched
    MLG_CUDA(cudaMemcpyAsync(x.data(), b.x + s.voff, sizeof(double) * x.size(),
                             cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    std::fill(e_full, e_full + nd, 0.0);
    for (int ly = 0; ly < s.h; ++ly)
      for (int lx = 0; lx < s.w; ++lx)
        e_full[static_cast<int64_t>(s.y0 + ly) * (F.gx() + 1) + (s.x0 + lx)] =
            x[static_cast<std::size_t>(ly) * s.pitch + lx];
    if (report) {
      report->iterations = rep[0].iterations;
      report->final_residual = rep[0].final_residual;
      report->converged = rep[0].converged;
    }
    if (throw_unconverged && !rep[0].converged)
      throw mlg::SolverError("subdomain " + std::to_string(j + 1) +
                             " solve did not converge (" + std::to_string(rep[0].iterations) +
                             " iterations, residual " + std::to_string(rep[0].final_residual) +
                             ")");
}
}  // namespace

int mlg_local_bvp_solve(mlg_ctx* ctx, int level, int j, double lambda, const double* u_full,
                        double cg_tol, double* e_full, mlg_solve_report* report) {
  return guarded([&] {
    local_solve_impl(ctx, level, j, lambda, u_full, cg_tol, 0, e_full, report, true);
  });
}

int mlg_local_cg_solve(mlg_ctx* ctx, int level, int j, double lambda, const double* u_full,
                       double cg_tol, int maxit, double* e_full, mlg_solve_report* report) {
  return guarded([&] {
    if (maxit < 0) throw mlg::ConfigError("maxit must be nonnegative");
    local_solve_impl(ctx, level, j, lambda, u_full, cg_tol, maxit, e_full, report, false);
  });
}

int mlg_interface_solve(mlg_ctx* ctx, int level, double lambda, const double* u_full,
                        const double* corrections, double cg_tol, double* glued_full,
                        mlg_solve_report* report) {
  return guarded([&] {
    mlg::Ctx& c = C(ctx);
    mlg::Level& F = c.level(level);
    if (!(cg_tol > 0.0)) throw mlg::ConfigError("cg_solve: tolerance must be positive");
    const int64_t nd = F.ndofs();
    const int m = c.part.m;
    mlg::DevBuf<double> u(nd), ui(nd), corr(static_cast<std::size_t>(nd) * m), glued(nd);
    u.upload(u_full, nd, c.stream);
    mlg::interleave(c, F, 1, 1, u.get(), 0, ui.get());
    corr.upload(corrections, static_cast<std::size_t>(nd) * m, c.stream);
    mlg::glue_full(c, level, corr.get(), ui.get(), glued.get());
    std::vector<mlg::SolveReport> rep;
    bool empty = false;
    mlg::Lam lam{};
    lam.v[0] = lambda;
    mlg::strip_solve(c, F, 1, 1, ui.get(), lam, glued.get(), cg_tol, 0, &rep, &empty);
    glued.download(glued_full, nd, c.stream);
    c.sync();
    if (report) {
      report->iterations = empty ? 0 : rep[0].iterations;
      report->final_residual = empty ? 0.0 : rep[0].final_residual;
      report->converged = empty ? 1 : rep[0].converged;
    }
    if (!empty && !rep[0].converged)
      throw mlg::SolverError("strip solve did not converge (" +
                             std::to_string(rep[0].iterations) + " iterations, residual " +
                             std::to_string(rep[0].final_residual) + ")");
  });
}

int mlg_augmented_eigensolve(mlg_ctx* ctx, int level, int k_in, const double* glued_full,
                             int nev, double* lambdas, double* coeffs) {
  return guarded([&] {
    mlg::Ctx& c = C(ctx);
    mlg::Level& F = c.level(level);
    if (k_in < 0 || k_in > 8) throw mlg::ConfigError("at most 8 candidates on the B200 path");
    const int nr = mlg::nr_for(std::max(std::max(k_in, nev), 1));
    const int64_t nd = F.ndofs();
    mlg::DevBuf<double> g(static_cast<std::size_t>(nd) * std::max(k_in, 1)), gi(nd * nr), u;
    if (k_in > 0) g.upload(glued_full, static_cast<std::size_t>(nd) * k_in, c.stream);
    mlg::interleave(c, F, nr, k_in, g.get(), 0, gi.get());
    const auto lam = mlg::augmented(c, level, nr, k_in, gi.get(), nev, u);
    std::copy(lam.begin(), lam.end(), lambdas);
    if (coeffs) {
      mlg::DevBuf<double> out(F.nint() * nev);
      mlg::deinterleave(c, F, nr, nev, nullptr, u.get(), 1, out.get());
      out.download(coeffs, F.nint() * nev, c.stream);
      c.sync();
    }
  });
}

namespace {
// Timing events of one C-ABI call, destroyed on every exit path.
struct EventPair {
  cudaEvent_t a = nullptr, b = nullptr;
  EventPair() {
    MLG_CUDA(cudaEventCreate(&a));
    MLG_CUDA(cudaEventCreate(&b));
  }
  ~EventPair() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
  EventPair(const EventPair&) = delete;
  EventPair& operator=(const EventPair&) = delete;
};
}  // namespace

static int step_impl(mlg_ctx* ctx, int from_level, int to_level, int nev,
                     const double* lambdas_in, const double* coeffs_in, bool device_in,
                     double* lambdas_out, double* coeffs_out, bool device_out, int* matched,
                     mlg_step_timings* timings) {
  return guarded([&] {
    mlg::Ctx& c = C(ctx);
    if (nev < 1) throw mlg::ConfigError("correction step needs at least one eigenpair");
    const int nr = mlg::nr_for(nev);
    const mlg::Level& A = c.level(from_level);
    reset_kernel_stats(c);
    if (device_in || device_out) c.order_after_input();  // caller's writes to its buffers
    EventPair ev;
    MLG_CUDA(cudaEventRecord(ev.a, c.stream));
    // grow-only context buffers: no allocation inside a steady-state step
    mlg::DevBuf<double>& in_ri = c.io_in;
    mlg::DevBuf<double>& u_in = c.io_u_in;
    mlg::DevBuf<double>& u_out = c.io_u_out;
    u_in.ensure(A.ndofs() * nr);
    const double* src = coeffs_in;
    if (!device_in) {
      in_ri.ensure(A.nint() * nev);
      in_ri.upload(coeffs_in, A.nint() * nev, c.stream);
      src = in_ri.get();
    }
    mlg::interleave(c, A, nr, nev, src, 1, u_in.get());
    const mlg::StepResult r =
        mlg::correction_step(c, from_level, to_level, nev, lambdas_in, u_in.get(), u_out);
    const mlg::Level& B = c.level(to_level);
    std::copy(r.lambdas.begin(), r.lambdas.end(), lambdas_out);
    if (coeffs_out) {
      if (device_out) {
        mlg::deinterleave(c, B, nr, nev, nullptr, u_out.get(), 1, coeffs_out);
      } else {
        mlg::DevBuf<double>& out = c.io_out;
        out.ensure(B.nint() * nev);
        mlg::deinterleave(c, B, nr, nev, nullptr, u_out.get(), 1, out.get());
        out.download(coeffs_out, B.nint() * nev, c.stream);
      }
    }
    MLG_CUDA(cudaEventRecord(ev.b, c.stream));
    c.sync();
    float ms = 0.f;
    MLG_CUDA(cudaEventElapsedTime(&ms, ev.a, ev.b));
    if (matched) *matched = r.matched ? 1 : 0;
    fill_timings(timings, r.times, c);
    if (timings) timings->step_seconds = ms * 1e-3;
  });
}

int mlg_correction_step(mlg_ctx* ctx, int from_level, int to_level, int nev,
                        const double* lambdas_in, const double* coeffs_in, double* lambdas_out,
                        double* coeffs_out, int* matched, mlg_step_timings* timings) {
  return step_impl(ctx, from_level, to_level, nev, lambdas_in, coeffs_in, false, lambdas_out,
                   coeffs_out, false, matched, timings);
}

int mlg_correction_step_device(mlg_ctx* ctx, int from_level, int to_level, int nev,
                               const double* lambdas_in, const double* d_coeffs_in,
                               double* lambdas_out, double* d_coeffs_out, int* matched,
                               mlg_step_timings* timings) {
  return step_impl(ctx, from_level, to_level, nev, lambdas_in, d_coeffs_in, true, lambdas_out,
                   d_coeffs_out, true, matched, timings);
}

int mlg_multilevel_correction(mlg_ctx* ctx, int last_level, double* lambdas,
                              double* final_coeffs, double* d_final_coeffs, int* matched,
                              mlg_step_timings* timings) {
  return guarded([&] {
    multilevel_impl(ctx, last_level, 0, nullptr, nullptr, lambdas, nullptr, nullptr, nullptr,
                    final_coeffs, d_final_coeffs, matched, timings);
  });
}

int mlg_multilevel_correction_refs(mlg_ctx* ctx, int last_level, int n_refs,
                                   const double* ref_lambdas, const mlg_exact_mode* ref_modes,
                                   double* lambdas, double* eig_err, double* l2_err,
                                   double* h1_err, double* final_coeffs, int* matched,
                                   mlg_step_timings* timings) {
  return guarded([&] {
    multilevel_impl(ctx, last_level, n_refs, ref_lambdas, ref_modes, lambdas, eig_err, l2_err,
                    h1_err, final_coeffs, nullptr, matched, timings);
  });
}

int mlg_make_reference(int example, int nev, const double* domain, double* lambdas,
                       mlg_exact_mode* modes) {
  return guarded([&] {
    const mlg::ReferenceSet r = mlg::make_reference(example, nev, domain);
    for (int i = 0; i < nev; ++i) {
      if (lambdas) lambdas[i] = r.lambdas[static_cast<std::size_t>(i)];
      if (modes) modes[i] = to_c(r.modes[static_cast<std::size_t>(i)]);
    }
  });
}

int mlg_make_reference_for(const mlg_config* cfg, int nev, double* lambdas,
                           mlg_exact_mode* modes) {
  return guarded([&] {
    if (!cfg) throw mlg::ConfigError("null argument");
    mlg::Config c;
    c.x_min = cfg->x_min;
    c.x_max = cfg->x_max;
    c.y_min = cfg->y_min;
    c.y_max = cfg->y_max;
    c.example = cfg->example;
    c.hole_x0 = cfg->hole_x_min;
    c.hole_x1 = cfg->hole_x_max;
    c.hole_y0 = cfg->hole_y_min;
    c.hole_y1 = cfg->hole_y_max;
    const mlg::ReferenceSet r = mlg::make_reference_for(c, nev);
    for (int i = 0; i < nev; ++i) {
      if (lambdas) lambdas[i] = r.lambdas[static_cast<std::size_t>(i)];
      if (modes) modes[i] = to_c(r.modes[static_cast<std::size_t>(i)]);
    }
  });
}

int mlg_compute_errors(mlg_ctx* ctx, int level, const double* coeffs_full, double lambda_h,
                       double lambda_ref, const mlg_exact_mode* reference,
                       mlg_error_report* out) {
  return guarded([&] {
    mlg::Ctx& c = C(ctx);
    const mlg::Level& L = c.level(level);
    if (!coeffs_full || !out) throw mlg::ConfigError("compute_errors: null argument");
    mlg::DevBuf<double> d(static_cast<std::size_t>(L.ndofs()));
    d.upload(coeffs_full, static_cast<std::size_t>(L.ndofs()), c.stream);
    mlg::ExactMode md;
    if (reference) md = from_c(*reference);
    const mlg::ErrorReport r = mlg::compute_errors(c, L, d.get(), 1, 0, lambda_h, lambda_ref,
                                                   reference ? &md : nullptr);
    *out = {r.eig_err, r.l2_err, r.h1_err};
  });
}

int mlg_set_input_stream(mlg_ctx* ctx, void* stream) {
  return guarded([&] { C(ctx).input_stream = static_cast<cudaStream_t>(stream); });
}

int mlg_build_profile(mlg_ctx* ctx, double* assemble_ms, double* assemble_dofs) {
  return guarded([&] {
    const mlg::Ctx& c = C(ctx);
    if (assemble_ms) *assemble_ms = c.asm_ms;
    if (assemble_dofs) *assemble_dofs = c.asm_dofs;
  });
}

int mlg_build_profile_kernel(mlg_ctx* ctx, int* kernel) {
  return guarded([&] {
    if (kernel) *kernel = C(ctx).asm_kernel;
  });
}

int mlg_set_profiling(mlg_ctx* ctx, int on) {
  return guarded([&] { C(ctx).profile = on != 0; });
}

int mlg_bench_spmv(mlg_ctx* ctx, int level, int reps, double* ms_per_launch,
                   double* bytes_per_launch) {
  return guarded([&] {
    mlg::Ctx& c = C(ctx);
    const mlg::Level& L = c.level(level);
    const int64_t n = L.nint();
    mlg::DevBuf<double> x(n), y(n);
    std::vector<double> h(static_cast<std::size_t>(n));
    unsigned long long s = 20261019ULL;
    for (auto& v : h) {  // splitmix64 -> uniform(-1,1)
      s += 0x9E3779B97F4A7C15ULL;
      unsigned long long z = s;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
      z ^= z >> 31;
      v = 2.0 * (static_cast<double>(z >> 11) * 0x1.0p-53) - 1.0;
    }
    x.upload(h.data(), h.size(), c.stream);
    for (int k = 0; k < 3; ++k) mlg::spmv_interior(c, L, x.get(), y.get());
    cudaEvent_t e0, e1;
    MLG_CUDA(cudaEventCreate(&e0));
    MLG_CUDA(cudaEventCreate(&e1));
    MLG_CUDA(cudaEventRecord(e0, c.stream));
    for (int k = 0; k < reps; ++k) mlg::spmv_interior(c, L, x.get(), y.get());
    MLG_CUDA(cudaEventRecord(e1, c.stream));
    MLG_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    MLG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms_per_launch = ms / std::max(reps, 1);
    // stencil row (4 x f64) + x + y per interior row
    *bytes_per_launch = static_cast<double>(n) * (32.0 + 8.0 + 8.0);
  });
}

}  // extern "C"

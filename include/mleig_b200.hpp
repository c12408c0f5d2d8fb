// mleig_b200.hpp -- header-only C++17 host mirror of the reference's corrector
// API (/root/reference/proj/include/mleig/corrector.hpp), implemented over the
// C ABI of libmlg_b200.so (mlg_b200.h).  A reference caller switches by
// replacing `#include "mleig/corrector.hpp"` with this header, the namespace
// mleig with mleig_b200, and linking -lmlg_b200.
//
// Same entry points, argument meaning and exception classes as the reference:
//   Hierarchy (corrector.hpp:63-95), coarse_eigensolve (fespace.hpp:128-132),
//   local_bvp_solve / interface_solve / augmented_eigensolve (corrector.hpp:112-128),
//   one_correction_step (corrector.hpp:135-136), multilevel_correction
//   (corrector.hpp:164-165).  Vectors are std::vector<double> in the
//   reference's layouts (full = all dofs, coeffs = interior dofs).
#pragma once

#include <algorithm>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "mlg_b200.h"

namespace mleig_b200 {

struct ConfigError : std::runtime_error {  // errors.hpp:10-12
  using std::runtime_error::runtime_error;
};
struct SolverError : std::runtime_error {  // errors.hpp:15-17
  using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {  // errors.hpp:20-22
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int status) {
  if (status == MLG_OK) return;
  const std::string msg = mlg_last_error();
  switch (status) {
    case MLG_ERR_CONFIG: throw ConfigError(msg);
    case MLG_ERR_SOLVER: throw SolverError(msg);
    case MLG_ERR_IO: throw IoError(msg);
    case MLG_ERR_CUDA: throw CudaError(msg);
    default: throw std::runtime_error(msg);
  }
}

struct DomainRect {  // mesh.hpp:22-27
  double x_min = -1.0, x_max = 1.0, y_min = -1.0, y_max = 1.0;
};

struct RunConfig {  // corrector.hpp:21-33
  DomainRect domain{};
  double H = 0.25;
  double delta = 0.1;
  int m = 4;
  int n_levels = 5;
  int degree = 1;
  int nev = 5;
  std::string example = "laplace";
  double cg_tol = 1e-10;
  int workers = 1;
  bool deterministic = true;
  int device = 0;
};

struct SolveReport {  // sparse.hpp:103-107
  int iterations = 0;
  double final_residual = 0.0;
  bool converged = false;
};

struct StepTimings {  // corrector.hpp:97-101
  double local_seconds = 0.0;
  double iface_seconds = 0.0;
  double aug_seconds = 0.0;
};

struct EigenPair {  // sparse.hpp:133-137
  double lambda = 0.0;
  std::vector<double> coeffs;
  int level = 0;
};

struct CorrectionState {  // corrector.hpp:103-107
  int level = 0;
  std::vector<EigenPair> pairs;
  bool matched_previous = true;
};

struct LevelTrace {  // corrector.hpp:151-159 (errors are the caller's business)
  int level = 0;
  double h = 0.0;
  int interior_dofs = 0;
  std::vector<double> lambdas;
  StepTimings timings;
  bool matched_previous = true;
  std::vector<EigenPair> pairs;
};

struct MultilevelResult {
  std::vector<LevelTrace> levels;
};

class Hierarchy {
 public:
  explicit Hierarchy(const RunConfig& config) : config_(config) {
    mlg_config c{};
    c.x_min = config.domain.x_min;
    c.x_max = config.domain.x_max;
    c.y_min = config.domain.y_min;
    c.y_max = config.domain.y_max;
    c.H = config.H;
    c.delta = config.delta;
    c.m = config.m;
    c.n_levels = config.n_levels;
    c.degree = config.degree;
    c.nev = config.nev;
    c.example = config.example == "laplace" ? 0 : (config.example == "variable" ? 1 : -1);
    if (c.example < 0)
      throw ConfigError("unknown example id \"" + config.example +
                        "\" (expected laplace or variable)");
    c.workers = config.workers;
    c.cg_tol = config.cg_tol;
    c.deterministic = config.deterministic ? 1 : 0;
    c.device = config.device;
    check(mlg_create(&c, &ctx_));
  }
  ~Hierarchy() { mlg_destroy(ctx_); }
  Hierarchy(const Hierarchy&) = delete;
  Hierarchy& operator=(const Hierarchy&) = delete;

  const RunConfig& config() const { return config_; }
  void extend_to(int level) { check(mlg_extend_to(ctx_, level)); }
  int max_level() const {
    int k = 0;
    check(mlg_max_level(ctx_, &k));
    return k;
  }
  mlg_level_info info(int level) const {
    mlg_level_info i{};
    check(mlg_get_level_info(ctx_, level, &i));
    return i;
  }
  std::vector<double> prolong(const std::vector<double>& full, int from_level, int to_level) {
    extend_to(to_level);
    std::vector<double> y(static_cast<std::size_t>(info(to_level).ndofs));
    check(mlg_prolong(ctx_, from_level, to_level, full.data(), y.data()));
    return y;
  }
  std::vector<double> restrict_transpose(const std::vector<double>& full, int from_level,
                                         int to_level) const {
    std::vector<double> y(static_cast<std::size_t>(info(to_level).ndofs));
    check(mlg_restrict_transpose(ctx_, from_level, to_level, full.data(), y.data()));
    return y;
  }
  std::vector<double> expand_interior(int level, const std::vector<double>& coeffs) const {
    const mlg_level_info i = info(level);
    std::vector<double> full(static_cast<std::size_t>(i.ndofs), 0.0);
    std::size_t k = 0;
    for (int iy = 1; iy < i.ny; ++iy)
      for (int ix = 1; ix < i.nx; ++ix) full[static_cast<std::size_t>(iy) * (i.nx + 1) + ix] = coeffs[k++];
    return full;
  }
  mlg_ctx* handle() const { return ctx_; }

 private:
  RunConfig config_;
  mlg_ctx* ctx_ = nullptr;
};

inline std::vector<EigenPair> coarse_eigensolve(Hierarchy& hy, int level, int nev) {
  hy.extend_to(level);
  const std::size_t n = static_cast<std::size_t>(hy.info(level).n_interior);
  std::vector<double> lam(static_cast<std::size_t>(nev)), co(n * nev);
  check(mlg_coarse_eigensolve(hy.handle(), level, nev, lam.data(), co.data()));
  std::vector<EigenPair> out(static_cast<std::size_t>(nev));
  for (int i = 0; i < nev; ++i)
    out[i] = {lam[i], std::vector<double>(co.begin() + i * n, co.begin() + (i + 1) * n), level};
  return out;
}

inline std::vector<double> local_bvp_solve(Hierarchy& hy, int level, int j, double lambda,
                                           const std::vector<double>& u_full, double cg_tol,
                                           SolveReport* report = nullptr) {
  std::vector<double> e(u_full.size());
  mlg_solve_report r{};
  check(mlg_local_bvp_solve(hy.handle(), level, j, lambda, u_full.data(), cg_tol, e.data(), &r));
  if (report) *report = {r.iterations, r.final_residual, r.converged != 0};
  return e;
}

inline std::vector<double> interface_solve(Hierarchy& hy, int level, double lambda,
                                           const std::vector<double>& u_full,
                                           const std::vector<std::vector<double>>& corrections,
                                           double cg_tol, SolveReport* report = nullptr) {
  std::vector<double> flat;
  for (const auto& c : corrections) flat.insert(flat.end(), c.begin(), c.end());
  std::vector<double> g(u_full.size());
  mlg_solve_report r{};
  check(mlg_interface_solve(hy.handle(), level, lambda, u_full.data(), flat.data(), cg_tol,
                            g.data(), &r));
  if (report) *report = {r.iterations, r.final_residual, r.converged != 0};
  return g;
}

inline std::vector<EigenPair> augmented_eigensolve(Hierarchy& hy, int fine_level,
                                                   const std::vector<std::vector<double>>& glued,
                                                   int nev) {
  std::vector<double> flat;
  for (const auto& g : glued) flat.insert(flat.end(), g.begin(), g.end());
  const std::size_t n = static_cast<std::size_t>(hy.info(fine_level).n_interior);
  std::vector<double> lam(static_cast<std::size_t>(nev)), co(n * nev);
  check(mlg_augmented_eigensolve(hy.handle(), fine_level, static_cast<int>(glued.size()),
                                 flat.data(), nev, lam.data(), co.data()));
  std::vector<EigenPair> out(static_cast<std::size_t>(nev));
  for (int i = 0; i < nev; ++i)
    out[i] = {lam[i], std::vector<double>(co.begin() + i * n, co.begin() + (i + 1) * n),
              fine_level};
  return out;
}

inline CorrectionState one_correction_step(Hierarchy& hy, const CorrectionState& state,
                                           int to_level, StepTimings* timings = nullptr) {
  const int nev = static_cast<int>(state.pairs.size());
  if (nev == 0) throw ConfigError("correction step needs at least one eigenpair");
  std::vector<double> lam_in(static_cast<std::size_t>(nev)), cin;
  for (int i = 0; i < nev; ++i) {
    lam_in[i] = state.pairs[i].lambda;
    cin.insert(cin.end(), state.pairs[i].coeffs.begin(), state.pairs[i].coeffs.end());
  }
  hy.extend_to(std::max(to_level, state.level));
  const std::size_t n = static_cast<std::size_t>(hy.info(to_level).n_interior);
  std::vector<double> lam_out(static_cast<std::size_t>(nev)), cout(n * nev);
  int matched = 0;
  mlg_step_timings t{};
  check(mlg_correction_step(hy.handle(), state.level, to_level, nev, lam_in.data(), cin.data(),
                            lam_out.data(), cout.data(), &matched, &t));
  if (timings) *timings = {t.local_seconds, t.iface_seconds, t.aug_seconds};
  CorrectionState out;
  out.level = to_level;
  out.matched_previous = matched != 0;
  for (int i = 0; i < nev; ++i)
    out.pairs.push_back(
        {lam_out[i], std::vector<double>(cout.begin() + i * n, cout.begin() + (i + 1) * n),
         to_level});
  return out;
}

// multilevel_correction (corrector.cpp:414-462): level-1 direct solve, then
// one correction step per level; the whole loop stays on the device.
inline MultilevelResult multilevel_correction(Hierarchy& hy) {
  const int nlev = hy.config().n_levels, nev = hy.config().nev;
  hy.extend_to(nlev);
  std::vector<double> lam(static_cast<std::size_t>(nlev) * nev);
  std::vector<int> matched(static_cast<std::size_t>(nlev));
  std::vector<mlg_step_timings> t(static_cast<std::size_t>(nlev));
  const std::size_t n = static_cast<std::size_t>(hy.info(nlev).n_interior);
  std::vector<double> co(n * nev);
  check(mlg_multilevel_correction(hy.handle(), nlev, lam.data(), co.data(), nullptr,
                                  matched.data(), t.data()));
  MultilevelResult r;
  for (int k = 1; k <= nlev; ++k) {
    LevelTrace tr;
    const mlg_level_info i = hy.info(k);
    tr.level = k;
    tr.h = i.h_max;
    tr.interior_dofs = static_cast<int>(i.n_interior);
    tr.lambdas.assign(lam.begin() + (k - 1) * nev, lam.begin() + k * nev);
    tr.timings = {t[k - 1].local_seconds, t[k - 1].iface_seconds, t[k - 1].aug_seconds};
    tr.matched_previous = matched[k - 1] != 0;
    if (k == nlev)
      for (int e = 0; e < nev; ++e)
        tr.pairs.push_back(
            {tr.lambdas[e], std::vector<double>(co.begin() + e * n, co.begin() + (e + 1) * n), k});
    r.levels.push_back(std::move(tr));
  }
  return r;
}

}  // namespace mleig_b200

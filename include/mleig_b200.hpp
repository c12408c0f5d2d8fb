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
#include <array>
#include <cmath>
#include <map>
#include <optional>
#include <ostream>
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
  unsigned long long seed = 0;  // example "reaction" (BASELINE config 4)
  DomainRect hole{0.0, 0.0, 0.0, 0.0};  // corner hole: L-shaped domain (config 3)
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

struct LevelTrace {  // corrector.hpp:151-159
  int level = 0;
  double h = 0.0;
  int interior_dofs = 0;
  std::vector<double> lambdas;
  std::vector<double> eig_errors;  // NaN without a ReferenceSet
  std::vector<double> h1_errors;   // NaN without a closed-form eigenfunction
  StepTimings timings;
  bool matched_previous = true;
  std::vector<EigenPair> pairs;
};

struct MultilevelResult {
  std::vector<LevelTrace> levels;
};

inline mlg_config to_c(const RunConfig& config) {
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
  c.example = config.example == "laplace"    ? 0
              : config.example == "variable" ? 1
              : config.example == "reaction" ? 2
                                             : -1;
  c.seed = config.seed;
  c.hole_x_min = config.hole.x_min;
  c.hole_x_max = config.hole.x_max;
  c.hole_y_min = config.hole.y_min;
  c.hole_y_max = config.hole.y_max;
  if (c.example < 0)
    throw ConfigError("unknown example id \"" + config.example +
                      "\" (expected laplace or variable)");
  c.workers = config.workers;
  c.cg_tol = config.cg_tol;
  c.deterministic = config.deterministic ? 1 : 0;
  c.device = config.device;
  return c;
}

inline RunConfig from_c(const mlg_config& c) {
  RunConfig r;
  r.domain = {c.x_min, c.x_max, c.y_min, c.y_max};
  r.H = c.H;
  r.delta = c.delta;
  r.m = c.m;
  r.n_levels = c.n_levels;
  r.degree = c.degree;
  r.nev = c.nev;
  r.example = c.example == 2 ? "reaction" : (c.example == 1 ? "variable" : "laplace");
  r.seed = c.seed;
  r.hole = {c.hole_x_min, c.hole_x_max, c.hole_y_min, c.hole_y_max};
  r.cg_tol = c.cg_tol;
  r.workers = c.workers;
  r.deterministic = c.deterministic != 0;
  r.device = c.device;
  return r;
}

class Hierarchy {
 public:
  explicit Hierarchy(const RunConfig& config) : config_(config) {
    const mlg_config c = to_c(config);
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
    std::vector<int> d(static_cast<std::size_t>(i.n_interior));
    check(mlg_export_space(ctx_, level, nullptr, d.data(), nullptr, nullptr));
    for (std::size_t k = 0; k < d.size(); ++k) full[static_cast<std::size_t>(d[k])] = coeffs[k];
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

// ---- reference sets and error reporting (fespace.hpp:103-120, harness.cpp:126-169) ----
struct ExactFunction {  // a separable sine mode (make_reference's closed forms)
  mlg_exact_mode mode{};
  double value(double x, double y) const {
    constexpr double kPi = 3.14159265358979323846;
    return mode.amp * (std::sin(mode.mx * kPi * (x - mode.x0) / mode.lx) *
                       std::sin(mode.my * kPi * (y - mode.y0) / mode.ly));
  }
  std::array<double, 2> gradient(double x, double y) const {
    constexpr double kPi = 3.14159265358979323846;
    const double ax = mode.mx * kPi / mode.lx, ay = mode.my * kPi / mode.ly;
    return {mode.amp * (ax * std::cos(ax * (x - mode.x0)) * std::sin(ay * (y - mode.y0))),
            mode.amp * (ay * std::sin(ax * (x - mode.x0)) * std::cos(ay * (y - mode.y0)))};
  }
};

struct ReferenceSet {  // corrector.hpp
  std::vector<double> lambdas;
  std::map<int, ExactFunction> eigenfunctions;
};

inline int example_id(const std::string& example) {
  if (example == "laplace") return 0;
  if (example == "variable") return 1;
  if (example == "reaction") return 2;
  throw ConfigError("no reference data for example \"" + example + "\"");
}

// make_reference(example, nev): the reference's table ((-1,1)^2 for laplace).
inline ReferenceSet make_reference(const std::string& example, int nev,
                                   const DomainRect* domain = nullptr) {
  const int ex = example_id(example);
  std::vector<double> lam(static_cast<std::size_t>(std::max(nev, 0)));
  std::vector<mlg_exact_mode> modes(lam.size());
  const double dom[4] = {domain ? domain->x_min : -1.0, domain ? domain->x_max : 1.0,
                         domain ? domain->y_min : -1.0, domain ? domain->y_max : 1.0};
  check(mlg_make_reference(ex, nev, domain ? dom : nullptr, lam.data(), modes.data()));
  ReferenceSet r;
  r.lambdas = lam;
  for (int i = 0; i < nev; ++i)
    if (modes[i].mx > 0) r.eigenfunctions[i] = ExactFunction{modes[i]};
  return r;
}

struct ErrorReport {  // fespace.hpp:108-112
  double eig_err = 0.0, l2_err = 0.0, h1_err = 0.0;
};

// compute_errors (fespace.cpp:434-488); the sweep runs on the device.
inline ErrorReport compute_errors(Hierarchy& hy, int level, const std::vector<double>& coeffs_full,
                                  double lambda_h, double lambda_ref,
                                  const ExactFunction* reference) {
  mlg_error_report r{};
  check(mlg_compute_errors(hy.handle(), level, coeffs_full.data(), lambda_h, lambda_ref,
                           reference ? &reference->mode : nullptr, &r));
  return {r.eig_err, r.l2_err, r.h1_err};
}

// multilevel_correction (corrector.cpp:414-462): level-1 direct solve, then
// one correction step per level; the whole loop stays on the device, and with
// a ReferenceSet the per-level errors are computed there too.
inline MultilevelResult multilevel_correction(Hierarchy& hy, const ReferenceSet* refs = nullptr) {
  const int nlev = hy.config().n_levels, nev = hy.config().nev;
  hy.extend_to(nlev);
  const std::size_t nn = static_cast<std::size_t>(nlev) * nev;
  std::vector<double> lam(nn), ee(nn, std::nan("")), h1(nn, std::nan(""));
  std::vector<int> matched(static_cast<std::size_t>(nlev));
  std::vector<mlg_step_timings> t(static_cast<std::size_t>(nlev));
  const std::size_t n = static_cast<std::size_t>(hy.info(nlev).n_interior);
  std::vector<double> co(n * nev);
  if (refs) {
    const int nref = std::min(static_cast<int>(refs->lambdas.size()), nev);
    std::vector<mlg_exact_mode> modes(static_cast<std::size_t>(std::max(nref, 1)));
    for (int i = 0; i < nref; ++i) {
      auto it = refs->eigenfunctions.find(i);
      if (it != refs->eigenfunctions.end()) modes[i] = it->second.mode;
    }
    check(mlg_multilevel_correction_refs(hy.handle(), nlev, nref, refs->lambdas.data(),
                                         modes.data(), lam.data(), ee.data(), nullptr, h1.data(),
                                         co.data(), matched.data(), t.data()));
  } else {
    check(mlg_multilevel_correction(hy.handle(), nlev, lam.data(), co.data(), nullptr,
                                    matched.data(), t.data()));
  }
  MultilevelResult r;
  for (int k = 1; k <= nlev; ++k) {
    LevelTrace tr;
    const mlg_level_info i = hy.info(k);
    tr.level = k;
    tr.h = i.h_max;
    tr.interior_dofs = static_cast<int>(i.n_interior);
    tr.lambdas.assign(lam.begin() + (k - 1) * nev, lam.begin() + k * nev);
    tr.eig_errors.assign(ee.begin() + (k - 1) * nev, ee.begin() + k * nev);
    tr.h1_errors.assign(h1.begin() + (k - 1) * nev, h1.begin() + k * nev);
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

// ---- experiment harness (harness.hpp; native code in libmlg_b200.so) ----
inline RunConfig parse_config_json(const std::string& json_text) {
  mlg_config c{};
  check(mlg_parse_config_json(json_text.c_str(), &c));
  return from_c(c);
}

inline RunConfig parse_config_file(const std::string& path) {
  mlg_config c{};
  check(mlg_parse_config_file(path.c_str(), &c));
  return from_c(c);
}

inline std::vector<double> estimate_orders(const std::vector<double>& errors, double beta) {
  std::vector<double> out(errors.empty() ? 0 : errors.size() - 1);
  std::vector<double> tmp(std::max<std::size_t>(out.size(), 1));
  check(mlg_estimate_orders(errors.data(), static_cast<int>(errors.size()), beta, tmp.data()));
  std::copy(tmp.begin(), tmp.begin() + out.size(), out.begin());
  return out;
}

struct ReportRow {  // harness.hpp:23-35
  int level = 0;
  double h = 0.0;
  int dofs = 0;
  int eig_index = 0;
  double lambda = 0.0;
  double eig_err = 0.0;
  std::optional<double> h1_err;
  std::optional<double> order;
  double local_s = 0.0, iface_s = 0.0, aug_s = 0.0;
};

struct ExperimentReport {  // harness.hpp:37-41
  RunConfig config;
  std::vector<ReportRow> rows;
};

inline ExperimentReport run_experiment(const RunConfig& config, const std::string& csv_path) {
  const mlg_config c = to_c(config);
  std::vector<mlg_report_row> rows(static_cast<std::size_t>(std::max(config.n_levels * config.nev, 1)));
  int n = 0;
  check(mlg_run_experiment(&c, csv_path.c_str(), rows.data(), static_cast<int>(rows.size()), &n));
  ExperimentReport rep;
  rep.config = config;
  for (int k = 0; k < n; ++k) {
    const mlg_report_row& r = rows[k];
    ReportRow o;
    o.level = r.level;
    o.h = r.h;
    o.dofs = r.dofs;
    o.eig_index = r.eig_index;
    o.lambda = r.lambda;
    o.eig_err = r.eig_err;
    if (r.has_h1) o.h1_err = r.h1_err;
    if (r.has_order) o.order = r.order;
    o.local_s = r.local_s;
    o.iface_s = r.iface_s;
    o.aug_s = r.aug_s;
    rep.rows.push_back(o);
  }
  return rep;
}

inline void write_csv(const ExperimentReport& report, const std::string& path) {
  std::vector<mlg_report_row> rows;
  for (const ReportRow& r : report.rows)
    rows.push_back({r.level, r.h, r.dofs, r.eig_index, r.lambda, r.eig_err, r.h1_err ? 1 : 0,
                    r.h1_err.value_or(0.0), r.order ? 1 : 0, r.order.value_or(0.0), r.local_s,
                    r.iface_s, r.aug_s});
  check(mlg_write_csv(rows.data(), static_cast<int>(rows.size()), path.c_str()));
}

inline void print_table(const std::string& csv_path, std::ostream& os) {
  size_t len = 0;
  check(mlg_print_table(csv_path.c_str(), nullptr, 0, &len));
  std::string buf(len + 1, '\0');
  check(mlg_print_table(csv_path.c_str(), buf.data(), buf.size(), &len));
  os << buf.c_str();
}

inline void export_vtk(const RunConfig& config, const std::string& out_dir) {
  const mlg_config c = to_c(config);
  check(mlg_export_vtk(&c, out_dir.c_str()));
}

}  // namespace mleig_b200

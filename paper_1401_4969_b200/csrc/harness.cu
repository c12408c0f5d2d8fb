// Experiment harness around the B200 path (the reference's harness.cpp):
// strict JSON config parsing, convergence orders, the CSV report, the table
// pretty-printer and the VTK export.  Host C++ over the library's own C ABI;
// the compute (multilevel correction, error sweeps) runs on the device.
//
//   parse_config_json / parse_config_file   harness.cpp:58-111
//   estimate_orders                         harness.cpp:113-122
//   run_experiment / write_csv              harness.cpp:171-222 (%.17g columns)
//   print_table                             harness.cpp:240-290
//   export_vtk                              harness.cpp:292-351
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <sys/stat.h>
#include <vector>

#include "../../include/mlg_b200.h"
#include "common.cuh"

namespace {

template <class F>
int hguard(F&& f) {  // same taxonomy as capi.cu's guard, same message slot
  std::string& h_err = mlg::last_error_slot();
  try {
    f();
    h_err.clear();
    return MLG_OK;
  } catch (const mlg::ConfigError& e) {
    h_err = e.what();
    return MLG_ERR_CONFIG;
  } catch (const mlg::SolverError& e) {
    h_err = e.what();
    return MLG_ERR_SOLVER;
  } catch (const mlg::IoError& e) {
    h_err = e.what();
    return MLG_ERR_IO;
  } catch (const mlg::CudaError& e) {
    h_err = e.what();
    return MLG_ERR_CUDA;
  } catch (const std::exception& e) {
    h_err = e.what();
    return MLG_ERR_OTHER;
  }
}

// Re-raise a status of a nested C-ABI call as the matching exception.
void ok(int st) {
  if (st == MLG_OK) return;
  const std::string msg = mlg_last_error();
  switch (st) {
    case MLG_ERR_CONFIG: throw mlg::ConfigError(msg);
    case MLG_ERR_SOLVER: throw mlg::SolverError(msg);
    case MLG_ERR_IO: throw mlg::IoError(msg);
    case MLG_ERR_CUDA: throw mlg::CudaError(msg);
    default: throw std::runtime_error(msg);
  }
}

// ---- minimal strict JSON (RFC 8259 values) --------------------------------
struct JVal {
  enum Kind { Null, Bool, Int, Float, Str, Arr, Obj } kind = Null;
  bool b = false;
  double num = 0.0;
  long long i = 0;
  std::string s;
  std::vector<JVal> arr;
  std::map<std::string, JVal> obj;  // sorted keys, last duplicate wins
};

struct JParser {
  const std::string& t;
  std::size_t p = 0;
  [[noreturn]] void fail(const std::string& what) {
    throw mlg::ConfigError("config is not valid JSON: " + what + " at byte " +
                           std::to_string(p));
  }
  void ws() {
    while (p < t.size() && (t[p] == ' ' || t[p] == '\t' || t[p] == '\n' || t[p] == '\r')) ++p;
  }
  bool lit(const char* w) {
    const std::size_t n = std::strlen(w);
    if (t.compare(p, n, w) == 0) {
      p += n;
      return true;
    }
    return false;
  }
  std::string str() {
    if (t[p] != '"') fail("expected string");
    ++p;
    std::string out;
    while (true) {
      if (p >= t.size()) fail("unterminated string");
      const char c = t[p++];
      if (c == '"') break;
      if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
      if (c != '\\') {
        out.push_back(c);
        continue;
      }
      if (p >= t.size()) fail("bad escape");
      const char e = t[p++];
      switch (e) {
        case '"': out.push_back('"'); break;
        case '\\': out.push_back('\\'); break;
        case '/': out.push_back('/'); break;
        case 'b': out.push_back('\b'); break;
        case 'f': out.push_back('\f'); break;
        case 'n': out.push_back('\n'); break;
        case 'r': out.push_back('\r'); break;
        case 't': out.push_back('\t'); break;
        case 'u': {
          if (p + 4 > t.size()) fail("bad \\u escape");
          const unsigned cp = static_cast<unsigned>(std::stoul(t.substr(p, 4), nullptr, 16));
          p += 4;
          if (cp < 0x80) {
            out.push_back(static_cast<char>(cp));
          } else if (cp < 0x800) {
            out.push_back(static_cast<char>(0xC0 | (cp >> 6)));
            out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
          } else {
            out.push_back(static_cast<char>(0xE0 | (cp >> 12)));
            out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
            out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
          }
          break;
        }
        default: fail("bad escape");
      }
    }
    return out;
  }
  JVal number() {
    const std::size_t s0 = p;
    bool integer = true;
    if (t[p] == '-') ++p;
    if (p >= t.size() || !std::isdigit(static_cast<unsigned char>(t[p]))) fail("bad number");
    if (t[p] == '0') {
      ++p;
    } else {
      while (p < t.size() && std::isdigit(static_cast<unsigned char>(t[p]))) ++p;
    }
    if (p < t.size() && t[p] == '.') {
      integer = false;
      ++p;
      if (p >= t.size() || !std::isdigit(static_cast<unsigned char>(t[p]))) fail("bad number");
      while (p < t.size() && std::isdigit(static_cast<unsigned char>(t[p]))) ++p;
    }
    if (p < t.size() && (t[p] == 'e' || t[p] == 'E')) {
      integer = false;
      ++p;
      if (p < t.size() && (t[p] == '+' || t[p] == '-')) ++p;
      if (p >= t.size() || !std::isdigit(static_cast<unsigned char>(t[p]))) fail("bad number");
      while (p < t.size() && std::isdigit(static_cast<unsigned char>(t[p]))) ++p;
    }
    JVal v;
    const std::string tok = t.substr(s0, p - s0);
    v.num = std::strtod(tok.c_str(), nullptr);
    if (integer) {
      errno = 0;
      v.i = std::strtoll(tok.c_str(), nullptr, 10);
      v.kind = errno == ERANGE ? JVal::Float : JVal::Int;
    } else {
      v.kind = JVal::Float;
    }
    return v;
  }
  JVal value(int depth = 0) {
    if (depth > 64) fail("nesting too deep");
    ws();
    if (p >= t.size()) fail("unexpected end of input");
    JVal v;
    const char c = t[p];
    if (c == '{') {
      ++p;
      v.kind = JVal::Obj;
      ws();
      if (p < t.size() && t[p] == '}') {
        ++p;
        return v;
      }
      while (true) {
        ws();
        if (p >= t.size()) fail("unexpected end of input");
        std::string k = str();
        ws();
        if (p >= t.size() || t[p] != ':') fail("expected ':'");
        ++p;
        v.obj[k] = value(depth + 1);
        ws();
        if (p < t.size() && t[p] == ',') {
          ++p;
          continue;
        }
        if (p < t.size() && t[p] == '}') {
          ++p;
          return v;
        }
        fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      ++p;
      v.kind = JVal::Arr;
      ws();
      if (p < t.size() && t[p] == ']') {
        ++p;
        return v;
      }
      while (true) {
        v.arr.push_back(value(depth + 1));
        ws();
        if (p < t.size() && t[p] == ',') {
          ++p;
          continue;
        }
        if (p < t.size() && t[p] == ']') {
          ++p;
          return v;
        }
        fail("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.kind = JVal::Str;
      v.s = str();
      return v;
    }
    if (lit("true")) {
      v.kind = JVal::Bool;
      v.b = true;
      return v;
    }
    if (lit("false")) {
      v.kind = JVal::Bool;
      return v;
    }
    if (lit("null")) return v;
    if (c == '-' || std::isdigit(static_cast<unsigned char>(c))) return number();
    fail("unexpected character");
  }
  JVal document() {
    JVal v = value();
    ws();
    if (p != t.size()) fail("trailing characters");
    return v;
  }
};

const JVal* field(const JVal& j, const std::string& key) {
  auto it = j.obj.find(key);
  return it == j.obj.end() ? nullptr : &it->second;
}

double require_number(const JVal& j, const std::string& key) {
  const JVal* v = field(j, key);
  if (!v || (v->kind != JVal::Int && v->kind != JVal::Float))
    throw mlg::ConfigError("config field \"" + key + "\" must be a number");
  return v->kind == JVal::Int ? static_cast<double>(v->i) : v->num;
}

int require_int(const JVal& j, const std::string& key) {
  const JVal* v = field(j, key);
  if (!v || v->kind != JVal::Int)
    throw mlg::ConfigError("config field \"" + key + "\" must be an integer");
  return static_cast<int>(v->i);
}

bool require_bool(const JVal& j, const std::string& key) {
  const JVal* v = field(j, key);
  if (!v || v->kind != JVal::Bool)
    throw mlg::ConfigError("config field \"" + key + "\" must be a boolean");
  return v->b;
}

std::string require_string(const JVal& j, const std::string& key) {
  const JVal* v = field(j, key);
  if (!v || v->kind != JVal::Str)
    throw mlg::ConfigError("config field \"" + key + "\" must be a string");
  return v->s;
}

std::string format_double(double v) {  // harness.cpp:51-55
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

// validate_config (corrector.cpp:76-88) without touching the device.
void validate(const mlg_config& c) {
  if (!(c.x_min < c.x_max) || !(c.y_min < c.y_max))
    throw mlg::ConfigError("domain rectangle must have positive side lengths");
  if (!(c.H > 0.0)) throw mlg::ConfigError("H must be positive");
  if (!(c.delta > 0.0)) throw mlg::ConfigError("delta must be positive");
  if (c.n_levels < 1) throw mlg::ConfigError("n_levels must be at least 1");
  if (c.degree != 1 && c.degree != 2) throw mlg::ConfigError("degree must be 1 or 2");
  if (c.nev < 1) throw mlg::ConfigError("nev must be at least 1");
  if (!(c.cg_tol > 0.0)) throw mlg::ConfigError("cg_tol must be positive");
  if (c.workers < 1) throw mlg::ConfigError("workers must be at least 1");
  if (c.example < 0 || c.example > 2)
    throw mlg::ConfigError("unknown example id (expected laplace, variable or reaction)");
}

mlg_config parse_json(const std::string& text) {
  JParser P{text};
  const JVal j = P.document();
  if (j.kind != JVal::Obj) throw mlg::ConfigError("config must be a JSON object");
  static const std::vector<std::string> keys = {"domain",  "H",       "delta",  "m",
                                                "n_levels", "degree", "nev",    "example",
                                                "cg_tol",   "workers", "deterministic"};
  // "seed" is the one key beyond the reference's schema, accepted only with the
  // B200 extension example "reaction" (BASELINE config 4).
  const JVal* exv = field(j, "example");
  const bool reaction = exv && exv->kind == JVal::Str && exv->s == "reaction";
  for (const auto& kv : j.obj)
    if (std::find(keys.begin(), keys.end(), kv.first) == keys.end() &&
        !(reaction && kv.first == "seed"))
      throw mlg::ConfigError("unknown config field \"" + kv.first + "\"");
  for (const auto& k : keys)
    if (!field(j, k)) throw mlg::ConfigError("missing config field \"" + k + "\"");
  const JVal& d = *field(j, "domain");
  if (d.kind != JVal::Obj) throw mlg::ConfigError("config field \"domain\" must be an object");
  static const std::vector<std::string> dkeys = {"x_min", "x_max", "y_min", "y_max"};
  for (const auto& kv : d.obj)
    if (std::find(dkeys.begin(), dkeys.end(), kv.first) == dkeys.end())
      throw mlg::ConfigError("unknown domain field \"" + kv.first + "\"");
  mlg_config c{};
  c.x_min = require_number(d, "x_min");
  c.x_max = require_number(d, "x_max");
  c.y_min = require_number(d, "y_min");
  c.y_max = require_number(d, "y_max");
  c.H = require_number(j, "H");
  c.delta = require_number(j, "delta");
  c.m = require_int(j, "m");
  c.n_levels = require_int(j, "n_levels");
  c.degree = require_int(j, "degree");
  c.nev = require_int(j, "nev");
  const std::string ex = require_string(j, "example");
  c.cg_tol = require_number(j, "cg_tol");
  c.workers = require_int(j, "workers");
  c.deterministic = require_bool(j, "deterministic") ? 1 : 0;
  c.device = 0;
  if (ex == "laplace") {
    c.example = 0;
  } else if (ex == "variable") {
    c.example = 1;
  } else if (ex == "reaction") {
    c.example = 2;
    if (field(j, "seed")) {
      const JVal* sv = field(j, "seed");
      if (sv->kind != JVal::Int || sv->i < 0)
        throw mlg::ConfigError("config field \"seed\" must be a nonnegative integer");
      c.seed = static_cast<uint64_t>(sv->i);
    }
  } else {
    validate(c);  // the reference reports field errors first, then the example
    throw mlg::ConfigError("unknown example id \"" + ex + "\" (expected laplace or variable)");
  }
  validate(c);
  return c;
}

std::string slurp(const std::string& path, bool config) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw mlg::IoError(std::string(config ? "cannot open config file " : "cannot open CSV file ") + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

struct Ctx {  // RAII over mlg_create / mlg_destroy
  mlg_ctx* h = nullptr;
  explicit Ctx(const mlg_config& c) { ok(mlg_create(&c, &h)); }
  ~Ctx() { mlg_destroy(h); }
};

std::vector<mlg_report_row> experiment_rows(const mlg_config& cfg) {
  validate(cfg);
  const int nev = cfg.nev, nl = cfg.n_levels;
  std::vector<double> ref_l(static_cast<std::size_t>(nev));
  std::vector<mlg_exact_mode> ref_m(static_cast<std::size_t>(nev));
  ok(mlg_make_reference_for(&cfg, nev, ref_l.data(), ref_m.data()));
  Ctx ctx(cfg);
  ok(mlg_extend_to(ctx.h, nl));
  const std::size_t nn = static_cast<std::size_t>(nl) * nev;
  std::vector<double> lam(nn), ee(nn), l2(nn), h1(nn);
  std::vector<int> matched(static_cast<std::size_t>(nl));
  std::vector<mlg_step_timings> t(static_cast<std::size_t>(nl));
  ok(mlg_multilevel_correction_refs(ctx.h, nl, nev, ref_l.data(), ref_m.data(), lam.data(),
                                    ee.data(), l2.data(), h1.data(), nullptr, matched.data(),
                                    t.data()));
  std::vector<mlg_report_row> rows;
  for (int k = 1; k <= nl; ++k) {
    mlg_level_info li{};
    ok(mlg_get_level_info(ctx.h, k, &li));
    for (int i = 0; i < nev; ++i) {
      const std::size_t o = static_cast<std::size_t>(k - 1) * nev + i;
      mlg_report_row r{};
      r.level = k;
      r.h = li.h_max;
      r.dofs = static_cast<int>(li.n_interior);
      r.eig_index = i + 1;
      r.lambda = lam[o];
      r.eig_err = ee[o];
      r.has_h1 = std::isnan(h1[o]) ? 0 : 1;
      r.h1_err = r.has_h1 ? h1[o] : 0.0;
      if (k > 1) {
        const double prev = ee[o - nev], cur = ee[o];
        if (prev > 0.0 && cur > 0.0) {
          r.has_order = 1;
          r.order = std::log(prev / cur) / std::log(2.0);
        }
      }
      if (!cfg.deterministic) {
        r.local_s = t[static_cast<std::size_t>(k - 1)].local_seconds;
        r.iface_s = t[static_cast<std::size_t>(k - 1)].iface_seconds;
        r.aug_s = t[static_cast<std::size_t>(k - 1)].aug_seconds;
      }
      rows.push_back(r);
    }
  }
  return rows;
}

void write_csv(const mlg_report_row* rows, int n, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw mlg::IoError("cannot open output file " + path);
  out << "level,h,dofs,eig_index,lambda,eig_err,h1_err,order,local_s,iface_s,aug_s\n";
  for (int k = 0; k < n; ++k) {
    const mlg_report_row& r = rows[k];
    out << r.level << ',' << format_double(r.h) << ',' << r.dofs << ',' << r.eig_index << ','
        << format_double(r.lambda) << ',' << format_double(r.eig_err) << ',';
    if (r.has_h1) out << format_double(r.h1_err);
    out << ',';
    if (r.has_order) out << format_double(r.order);
    out << ',' << format_double(r.local_s) << ',' << format_double(r.iface_s) << ','
        << format_double(r.aug_s) << '\n';
  }
  if (!out) throw mlg::IoError("failed while writing " + path);
}

std::vector<std::string> split_csv(const std::string& line) {
  std::vector<std::string> out(1);
  for (const char c : line) {
    if (c == ',')
      out.emplace_back();
    else
      out.back().push_back(c);
  }
  return out;
}

std::string table(const std::string& csv_path) {
  std::ifstream in(csv_path);
  if (!in) throw mlg::IoError("cannot open CSV file " + csv_path);
  std::string line;
  if (!std::getline(in, line)) throw mlg::IoError("empty CSV file " + csv_path);
  if (split_csv(line).size() != 11)
    throw mlg::ConfigError("unexpected CSV header in " + csv_path);
  struct Row {
    int level, dofs, eig_index;
    double h, lambda, eig_err;
    std::string h1_err, order;
  };
  std::vector<Row> rows;
  int max_index = 0;
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    const auto f = split_csv(line);
    if (f.size() != 11) throw mlg::ConfigError("malformed CSV row in " + csv_path);
    Row r{std::stoi(f[0]), std::stoi(f[2]), std::stoi(f[3]), std::stod(f[1]),
          std::stod(f[4]), std::stod(f[5]), f[6], f[7]};
    rows.push_back(r);
    max_index = std::max(max_index, r.eig_index);
  }
  std::ostringstream os;
  for (int i = 1; i <= max_index; ++i) {
    os << "eigenvalue " << i << ":\n";
    os << "  level        h     dofs        lambda       eig_err     order    h1_err\n";
    for (const Row& r : rows) {
      if (r.eig_index != i) continue;
      os << "  " << std::setw(5) << r.level << ' ' << std::setw(8) << std::setprecision(6) << r.h
         << ' ' << std::setw(8) << r.dofs << ' ' << std::setw(13) << std::setprecision(10)
         << r.lambda << ' ' << std::setw(13) << std::setprecision(6) << r.eig_err << ' '
         << std::setw(9) << (r.order.empty() ? "-" : r.order.substr(0, 7)) << ' '
         << std::setw(9) << (r.h1_err.empty() ? "-" : r.h1_err.substr(0, 9)) << '\n';
    }
  }
  return os.str();
}

void make_dirs(const std::string& dir) {
  std::string cur;
  for (std::size_t i = 0; i <= dir.size(); ++i) {
    if (i == dir.size() || dir[i] == '/') {
      if (!cur.empty() && ::mkdir(cur.c_str(), 0777) != 0 && errno != EEXIST)
        throw mlg::IoError("cannot create output directory " + dir);
    }
    if (i < dir.size()) cur.push_back(dir[i]);
  }
}

void vtk(const mlg_config& cfg, const std::string& out_dir) {
  validate(cfg);
  Ctx ctx(cfg);
  const int nl = cfg.n_levels, nev = cfg.nev;
  ok(mlg_extend_to(ctx.h, nl));
  mlg_level_info li{};
  ok(mlg_get_level_info(ctx.h, nl, &li));
  std::vector<double> lam(static_cast<std::size_t>(nl) * nev);
  std::vector<double> co(static_cast<std::size_t>(li.n_interior) * nev);
  ok(mlg_multilevel_correction(ctx.h, nl, lam.data(), co.data(), nullptr, nullptr, nullptr));
  std::vector<double> xy(static_cast<std::size_t>(li.num_vertices) * 2);
  std::vector<int> lat(static_cast<std::size_t>(li.num_vertices) * 2);
  std::vector<int> tri(static_cast<std::size_t>(li.num_triangles) * 3);
  ok(mlg_export_mesh(ctx.h, nl, xy.data(), lat.data(), tri.data(), nullptr, nullptr));
  make_dirs(out_dir);
  const std::string path = out_dir + "/eigenfunctions.vtk";
  std::ofstream out(path, std::ios::binary);
  if (!out) throw mlg::IoError("cannot open output file " + path);
  out << "# vtk DataFile Version 3.0\n";
  out << "eigenfunctions level " << nl << "\n";
  out << "ASCII\nDATASET UNSTRUCTURED_GRID\n";
  out << "POINTS " << li.num_vertices << " double\n";
  for (int64_t v = 0; v < li.num_vertices; ++v)
    out << format_double(xy[2 * v]) << ' ' << format_double(xy[2 * v + 1]) << " 0\n";
  out << "CELLS " << li.num_triangles << ' ' << 4 * li.num_triangles << '\n';
  for (int64_t t = 0; t < li.num_triangles; ++t)
    out << "3 " << tri[3 * t] << ' ' << tri[3 * t + 1] << ' ' << tri[3 * t + 2] << '\n';
  out << "CELL_TYPES " << li.num_triangles << '\n';
  for (int64_t t = 0; t < li.num_triangles; ++t) out << "5\n";
  out << "POINT_DATA " << li.num_vertices << '\n';
  const int w = li.nx - 1;
  for (int i = 0; i < nev; ++i) {
    out << "SCALARS eig_" << (i + 1) << " double 1\nLOOKUP_TABLE default\n";
    const double* c = co.data() + static_cast<std::size_t>(i) * li.n_interior;
    for (int64_t v = 0; v < li.num_vertices; ++v) {
      // P1: the dof at vertex lattice (lx,ly); interior ones follow the
      // row-major interior order, boundary values are 0 (expand_interior).
      const int lx = lat[2 * v], ly = lat[2 * v + 1];
      const bool interior = lx > 0 && ly > 0 && lx < li.nx && ly < li.ny;
      const double val = interior ? c[static_cast<std::size_t>(ly - 1) * w + (lx - 1)] : 0.0;
      out << format_double(val) << '\n';
    }
  }
  if (!out) throw mlg::IoError("failed while writing " + path);
}

}  // namespace

extern "C" {

int mlg_parse_config_json(const char* json_text, mlg_config* out) {
  const int st = hguard([&] {
    if (!json_text || !out) throw mlg::ConfigError("null argument");
    *out = parse_json(json_text);
  });
  return st;
}

int mlg_parse_config_file(const char* path, mlg_config* out) {
  return hguard([&] {
    if (!path || !out) throw mlg::ConfigError("null argument");
    *out = parse_json(slurp(path, true));
  });
}

int mlg_estimate_orders(const double* errors, int n, double beta, double* orders) {
  return hguard([&] {
    if (!(beta > 1.0)) throw mlg::ConfigError("estimate_orders: beta must exceed 1");
    for (int k = 0; k < n; ++k)
      if (!(errors[k] > 0.0)) throw mlg::ConfigError("estimate_orders: errors must be positive");
    for (int k = 1; k < n; ++k) orders[k - 1] = std::log(errors[k - 1] / errors[k]) / std::log(beta);
  });
}

int mlg_run_experiment(const mlg_config* cfg, const char* csv_path, mlg_report_row* rows,
                       int rows_cap, int* n_rows) {
  return hguard([&] {
    if (!cfg || !csv_path) throw mlg::ConfigError("null argument");
    const std::vector<mlg_report_row> r = experiment_rows(*cfg);
    write_csv(r.data(), static_cast<int>(r.size()), csv_path);
    if (n_rows) *n_rows = static_cast<int>(r.size());
    if (rows)
      for (int k = 0; k < std::min(rows_cap, static_cast<int>(r.size())); ++k) rows[k] = r[k];
  });
}

int mlg_write_csv(const mlg_report_row* rows, int n, const char* path) {
  return hguard([&] {
    if (!path || (n > 0 && !rows)) throw mlg::ConfigError("null argument");
    write_csv(rows, n, path);
  });
}

int mlg_print_table(const char* csv_path, char* buf, size_t cap, size_t* len) {
  return hguard([&] {
    if (!csv_path) throw mlg::ConfigError("null argument");
    const std::string s = table(csv_path);
    if (len) *len = s.size();
    if (buf && cap > 0) {
      const std::size_t n = std::min(cap - 1, s.size());
      std::memcpy(buf, s.data(), n);
      buf[n] = '\0';
    }
  });
}

int mlg_export_vtk(const mlg_config* cfg, const char* out_dir) {
  return hguard([&] {
    if (!cfg || !out_dir) throw mlg::ConfigError("null argument");
    vtk(*cfg, out_dir);
  });
}

}  // extern "C"

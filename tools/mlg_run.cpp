// mlg_run: C++ host driver over the drop-in API (include/mleig_b200.hpp), the
// B200 counterpart of the reference's CLI (tools/mleig_main.cpp:13-71):
//
//   mlg_run run <config.json> -o <out.csv> [--threads N]   run_experiment + CSV
//   mlg_run table <report.csv>                              print_table
//   mlg_run export-vtk <config.json> -o <dir> [--threads N] export_vtk
//
// plus a positional shortcut that prints the CSV columns of a multilevel run
// without the error columns:
//
//   mlg_run x_min x_max y_min y_max H delta m n_levels nev [cg_tol] [device]
//
// Exit codes as mleig_main.cpp:57-66: 0 ok, 2 config, 3 solver, 4 i/o, 1 other.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <iostream>
#include <string>

#include "mleig_b200.hpp"

namespace {

int usage(const char* argv0) {
  std::fprintf(stderr,
               "usage: %s run <config.json> -o <out.csv> [--threads N]\n"
               "       %s table <report.csv>\n"
               "       %s export-vtk <config.json> -o <dir> [--threads N]\n"
               "       %s x_min x_max y_min y_max H delta m n_levels nev [cg_tol] [device]\n",
               argv0, argv0, argv0, argv0);
  return 2;
}

int positional(int argc, char** argv) {
  if (argc < 10) return usage(argv[0]);
  mleig_b200::RunConfig cfg;
  cfg.domain = {std::atof(argv[1]), std::atof(argv[2]), std::atof(argv[3]), std::atof(argv[4])};
  cfg.H = std::atof(argv[5]);
  cfg.delta = std::atof(argv[6]);
  cfg.m = std::atoi(argv[7]);
  cfg.n_levels = std::atoi(argv[8]);
  cfg.nev = std::atoi(argv[9]);
  if (argc > 10) cfg.cg_tol = std::atof(argv[10]);
  if (argc > 11) cfg.device = std::atoi(argv[11]);
  mleig_b200::Hierarchy hy(cfg);
  const mleig_b200::MultilevelResult r = mleig_b200::multilevel_correction(hy);
  std::printf("level,h,dofs,eig_index,lambda,eig_err,h1_err,order,local_s,iface_s,aug_s\n");
  for (const auto& t : r.levels)
    for (std::size_t i = 0; i < t.lambdas.size(); ++i)
      std::printf("%d,%.17g,%d,%zu,%.17g,,,,%.17g,%.17g,%.17g\n", t.level, t.h, t.interior_dofs,
                  i + 1, t.lambdas[i], t.timings.local_seconds, t.timings.iface_seconds,
                  t.timings.aug_seconds);
  return 0;
}

int subcommand(int argc, char** argv) {
  const std::string cmd = argv[1];
  std::string input, out;
  int threads = 0;
  for (int k = 2; k < argc; ++k) {
    const std::string a = argv[k];
    if ((a == "-o" || a == "--output") && k + 1 < argc) {
      out = argv[++k];
    } else if (a == "--threads" && k + 1 < argc) {
      threads = std::atoi(argv[++k]);
    } else if (input.empty() && !a.empty() && a[0] != '-') {
      input = a;
    } else {
      return usage(argv[0]);
    }
  }
  if (cmd == "table") {
    if (input.empty()) return usage(argv[0]);
    mleig_b200::print_table(input, std::cout);
    return 0;
  }
  if ((cmd != "run" && cmd != "export-vtk") || input.empty() || out.empty())
    return usage(argv[0]);
  mleig_b200::RunConfig config = mleig_b200::parse_config_file(input);
  if (threads > 0) config.workers = threads;
  if (cmd == "run") {
    mleig_b200::run_experiment(config, out);
    std::cout << "wrote " << out << "\n";
  } else {
    mleig_b200::export_vtk(config, out);
    std::cout << "wrote " << out << "/eigenfunctions.vtk\n";
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return usage(argv[0]);
  try {
    const char c = argv[1][0];
    const bool numeric = (c >= '0' && c <= '9') || c == '-' || c == '.' || c == '+';
    return numeric ? positional(argc, argv) : subcommand(argc, argv);
  } catch (const mleig_b200::ConfigError& e) {
    std::cerr << "config error: " << e.what() << "\n";
    return 2;
  } catch (const mleig_b200::SolverError& e) {
    std::cerr << "solver error: " << e.what() << "\n";
    return 3;
  } catch (const mleig_b200::IoError& e) {
    std::cerr << "i/o error: " << e.what() << "\n";
    return 4;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}

// mlg_run: C++ host driver over the drop-in API (include/mleig_b200.hpp), the
// B200 counterpart of `mleig run` (tools/mleig_main.cpp:13-71 of the reference):
// runs multilevel_correction for a configuration given on the command line and
// prints the reference's CSV columns (harness.cpp:223-237; error columns are
// left empty -- reporting is outside the hot path).
//
//   mlg_run x_min x_max y_min y_max H delta m n_levels nev [cg_tol] [device]
#include <cstdio>
#include <cstdlib>
#include <exception>

#include "mleig_b200.hpp"

int main(int argc, char** argv) {
  if (argc < 10) {
    std::fprintf(stderr,
                 "usage: %s x_min x_max y_min y_max H delta m n_levels nev [cg_tol] [device]\n",
                 argv[0]);
    return 2;
  }
  mleig_b200::RunConfig cfg;
  cfg.domain = {std::atof(argv[1]), std::atof(argv[2]), std::atof(argv[3]), std::atof(argv[4])};
  cfg.H = std::atof(argv[5]);
  cfg.delta = std::atof(argv[6]);
  cfg.m = std::atoi(argv[7]);
  cfg.n_levels = std::atoi(argv[8]);
  cfg.nev = std::atoi(argv[9]);
  if (argc > 10) cfg.cg_tol = std::atof(argv[10]);
  if (argc > 11) cfg.device = std::atoi(argv[11]);
  try {
    mleig_b200::Hierarchy hy(cfg);
    const mleig_b200::MultilevelResult r = mleig_b200::multilevel_correction(hy);
    std::printf("level,h,dofs,eig_index,lambda,eig_err,h1_err,order,local_s,iface_s,aug_s\n");
    for (const auto& t : r.levels)
      for (std::size_t i = 0; i < t.lambdas.size(); ++i)
        std::printf("%d,%.17g,%d,%zu,%.17g,,,,%.17g,%.17g,%.17g\n", t.level, t.h,
                    t.interior_dofs, i + 1, t.lambdas[i], t.timings.local_seconds,
                    t.timings.iface_seconds, t.timings.aug_seconds);
    return 0;
  } catch (const mleig_b200::ConfigError& e) {  // exit codes of mleig_main.cpp:57-66
    std::fprintf(stderr, "config error: %s\n", e.what());
    return 2;
  } catch (const mleig_b200::SolverError& e) {
    std::fprintf(stderr, "solver error: %s\n", e.what());
    return 3;
  } catch (const mleig_b200::IoError& e) {
    std::fprintf(stderr, "io error: %s\n", e.what());
    return 4;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}

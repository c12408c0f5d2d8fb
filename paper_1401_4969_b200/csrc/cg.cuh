// Batched Jacobi-PCG over many lattice-window systems at once (the local
// Dirichlet solves of all subdomains x eigenvectors, or the strip solves).
// Semantics are the reference's cg_solve (sparse.cpp:199-258), per system:
// x0 = 0; zero rhs returns after 0 iterations; stop when ||r|| <= tol ||b||
// *confirmed by the true residual* (else restart from it); maxit = 10 n;
// p'Ap <= 0 is an error; non-convergence is reported.
#pragma once

#include <vector>

#include "ctx.cuh"

namespace mlg {

// A system is a rectangular window [x0, x0+w) x [y0, y0+h) of the fine full
// lattice (interior dofs only), optionally restricted by a byte mask, for ONE
// right-hand side (lane `rhs` of the rhs-interleaved source vector); its
// matrix is the window (mask) restriction of the level's stiffness, exactly
// extract_submatrix (sparse.cpp:156-174).  Vectors are window-compact,
// row-major.
//
// Work decomposition: a warp task is one column strip (32 lanes covering
// kCgCols output columns plus a 2-column halo each side) of `krows` window
// rows, swept bottom to top; a CTA ("tile") runs kCgWarps consecutive tasks of
// one system and owns one partial-sum slot.
struct CgSys {
  int x0, y0, w, h;
  int pitch;       // row pitch in the pooled vectors (w + 1: one shared zero column)
  int rhs;         // lane of the rhs-interleaved source (b) vector
  long long voff;  // first row in the pooled vectors
  int toff;        // first tile id (partials index)
  int ntiles;
  int nrows;       // unknowns: window points minus closed G_j (strip) / hole points
  int maxit;
  int nstrips, nrb, ntasks, krows;
  int tmap_off;  // >= 0: tasks are task_map[tmap_off + i] (strip tasks with strip rows)
};

// Pooled-vector index of window point (lx, ly).  Every window is stored with a
// zero frame -- one zero column shared between consecutive rows (pitch w + 1)
// and a zero row above and below -- so stencil reads that leave the window
// read zeros.
__host__ __device__ __forceinline__ long long cg_index(const CgSys& s, int ly, int lx) {
  return s.voff + static_cast<long long>(ly) * s.pitch + lx;
}

struct CgTile {
  int sys;
  int t;
};

struct CgCtl {
  double alpha, beta, rho, bnorm, final_res;
  int mode, restart, iters, status;
  // Deferred x updates (HBM-streaming batches): xphase 1 = the last launch
  // left x += alpha_prev * p_prev pending (p_prev is in the "new" p buffer of
  // the following launch); the next launch applies both updates at once.
  double alpha_prev;
  int xphase;
};

enum : int { kModeSkip = 0, kModeNormal = 1, kModeCheck = 2, kModeFlush = 3 };
enum : int { kRunning = 0, kConverged = 1, kNotConverged = 2, kIndefinite = 3 };

#ifndef MLG_CG_WARPS
#define MLG_CG_WARPS 4
#endif
constexpr int kCgWarps = MLG_CG_WARPS;  // warps (tasks) per CTA
constexpr int kCgCols = 28;     // output columns per warp task (2 halo lanes each side)
constexpr int kCgRows = 64;     // max window rows per warp task (register pipeline)
constexpr int kCgRowsAsync = 64;  // ... (shared-memory pipeline: prologue amortised)
constexpr int kCgPadRows = 6;  // padding rows after the pooled vectors (prefetch overrun)
constexpr int kCgDots = 5;      // partial sums per tile

struct CgResult {
  std::vector<SolveReport> reports;  // [sys]
  int iters_max = 0;
};

class CgBatch {
 public:
  static constexpr int kBlock = 32 * kCgWarps;

  // Lays out systems (computing voff/toff/ntiles) and sizes the pools.
  // bsrc: rhs-interleaved full-lattice source, bstride = its lane count.
  void setup(Ctx& c, const Level& L, std::vector<CgSys> systems, const unsigned char* mask,
             const double* bsrc, int bstride);
  // Runs to completion; throws SolverError for p'Ap <= 0.
  CgResult solve(Ctx& c, double tol, int maxit_override = 0);

  const double* x() const { return X.get(); }
  const std::vector<CgSys>& systems() const { return sys_h; }
  const CgSys* sys_dev() const { return sys_d.get(); }

 private:
  double tile_cost(const CgTile& t, const std::vector<int>& tmap) const;
  // SM-resident path (cg_resident.cu): every system of the batch runs with its
  // iterates held on chip; false when the batch does not fit (caller falls back).
  bool solve_resident(Ctx& c, double tol, CgResult& res);
  std::vector<CgTile> balance_tiles(const std::vector<CgTile>& tiles, int grid) const;
  const Level* L = nullptr;
  const unsigned char* mask = nullptr;
  const double* bsrc = nullptr;
  int bstride = 1;
  bool use_async = false;  // HBM-streaming batches: shared-memory row pipeline
  bool use_persist = false;  // L2-resident batches: one cooperative launch per solve
  std::vector<CgSys> sys_h;
  std::vector<int> tmap_h;  // host copy of task_map
  long long total_rows = 0;
  int total_tiles = 0;
  DevBuf<CgSys> sys_d;
  DevBuf<CgTile> tiles_d;
  DevBuf<int> task_map;
  DevBuf<CgCtl> ctl_d;
  DevBuf<unsigned> counters;  // per-system tile arrival counters (last-tile reduction)
  DevBuf<unsigned long long> prof_rows;
  DevBuf<unsigned> gsync;  // grid barrier (count, generation) of the persistent kernel
  DevBuf<int> active_d;    // systems still running  // rows swept by the sampled (profiled) launches
  DevBuf<double> X, R0, R1, P0, P1, part;
  // resident path: lane system lists, per-lane barrier counters, partial sums
  // and boundary-row exchange buffers
  DevBuf<int> res_lanes;
  DevBuf<unsigned> res_bar;
  DevBuf<double> res_part, res_halo, res_bslab;
};

}  // namespace mlg

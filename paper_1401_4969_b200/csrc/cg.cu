// Batched Jacobi-PCG (sparse.cpp:199-258) for lattice-window systems.
//
// One CG iteration = 4 launches on the context stream:
//   k_cg_a   (streaming)  p = z + beta p  (z = D^-1 r, recomputed for the 6
//                         neighbours from r and p_old, so p is never re-read
//                         after its update), q = A p with the window-masked
//                         7-point stencil in the reference's column order,
//                         partial p.q per tile;  or, for a right-hand side
//                         whose recurrence residual met the tolerance, the
//                         true residual b - A x (the reference's
//                         confirmation step, sparse.cpp:232-246).
//   k_cg_reduce<A>        one warp per (system, rhs): alpha = rho / p.q
//   k_cg_b   (streaming)  x += alpha p, r -= alpha q, partial r.r and r.z
//   k_cg_reduce<B>        beta, convergence test, mode of the next k_cg_a
// Partial sums are reduced in a fixed tree (no floating-point atomics), so the
// result is run-to-run bitwise deterministic (SURVEY finding 10).  Every
// (system, rhs) keeps its own scalars and stops independently; tiles of
// finished systems are dropped from the launch list between chunks.
#include <algorithm>
#include <cmath>
#include <string>

#include "cg.cuh"
#include "stencil.cuh"

namespace mlg {
namespace {

constexpr int kBlock = CgBatch::kBlock;
constexpr int kRPT = CgBatch::kRowsPerThread;
constexpr int kTile = CgBatch::kTile;

template <int NR>
__global__ void __launch_bounds__(kBlock) k_cg_init(const CgSys* sys, const CgTile* tiles,
                                                    const double* dinv, int nxp1,
                                                    const unsigned char* mask,
                                                    const double* bsrc, double* X, double* R,
                                                    double* part) {
  const CgTile tl = tiles[blockIdx.x];
  const CgSys S = sys[tl.sys];
  double acc[2 * NR];
#pragma unroll
  for (int k = 0; k < 2 * NR; ++k) acc[k] = 0.0;
  const int row0 = tl.t * kTile;
  for (int k = 0; k < kRPT; ++k) {
    const int i = row0 + k * kBlock + threadIdx.x;
    if (i >= S.nrows) break;
    const long long v = (S.voff + i) * NR;
    double b[NR], z0[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) z0[r] = 0.0;
    Nbhd h;
    if (!decode(S, i, nxp1, mask, &h)) {
      stv<NR>(X + v, z0);
      stv<NR>(R + v, z0);
      continue;
    }
    ldv<NR>(bsrc + h.g * NR, b);
    const double dv = dinv[h.g];
    stv<NR>(X + v, z0);
    stv<NR>(R + v, b);
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      acc[2 * r] += b[r] * b[r];
      acc[2 * r + 1] += b[r] * xmul(dv, b[r]);
    }
  }
  block_reduce_store<2 * NR>(acc, part + static_cast<long long>(S.toff + tl.t) * 2 * NR);
}

template <int NR>
__global__ void __launch_bounds__(kBlock)
    k_cg_a(const CgSys* sys, const CgTile* tiles, const CgCtl* ctl, const Stencil* st,
           const double* dinv, int nxp1, const unsigned char* mask, const double* bsrc,
           const double* X, double* R, const double* Pin, double* Pout, double* Q,
           double* part) {
  const CgTile tl = tiles[blockIdx.x];
  const CgSys S = sys[tl.sys];
  __shared__ double s_beta[NR];
  __shared__ int s_mode[NR], s_restart[NR];
  if (threadIdx.x < NR) {
    const CgCtl c = ctl[tl.sys * NR + threadIdx.x];
    s_beta[threadIdx.x] = c.beta;
    s_mode[threadIdx.x] = c.mode_a;
    s_restart[threadIdx.x] = c.restart;
  }
  __syncthreads();
  bool any_normal = false, any_check = false;
  double beta[NR];
  bool rst[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    any_normal |= s_mode[r] == kModeNormal;
    any_check |= s_mode[r] == kModeCheck;
    beta[r] = s_beta[r];
    rst[r] = s_restart[r] != 0;
  }
  if (!any_normal && !any_check) return;
  double acc[2 * NR];
#pragma unroll
  for (int k = 0; k < 2 * NR; ++k) acc[k] = 0.0;
  const int row0 = tl.t * kTile;
  const double* Rb = R + S.voff * NR;
  const double* Pb = Pin + S.voff * NR;
  if (any_normal) {
    auto pnew = [&](int j, long long gj, double (&o)[NR]) {
      double rv[NR], pv[NR];
      ldv<NR>(Rb + static_cast<long long>(j) * NR, rv);
      ldv<NR>(Pb + static_cast<long long>(j) * NR, pv);
      const double dv = dinv[gj];
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const double z = xmul(dv, rv[r]);
        o[r] = rst[r] ? z : xadd(z, xmul(beta[r], pv[r]));
      }
    };
    for (int k = 0; k < kRPT; ++k) {
      const int i = row0 + k * kBlock + threadIdx.x;
      if (i >= S.nrows) break;
      Nbhd h;
      if (!decode(S, i, nxp1, mask, &h)) continue;
      double pc[NR], q[NR];
      stencil_apply<NR>(h, i, S.w, nxp1, st, pnew, pc, q);
      const long long v = (S.voff + i) * NR;
      stv<NR>(Pout + v, pc);
      stv<NR>(Q + v, q);
#pragma unroll
      for (int r = 0; r < NR; ++r) acc[2 * r] += pc[r] * q[r];
    }
  }
  if (any_check) {
    // True residual r = b - A x for the right-hand sides under confirmation.
#pragma unroll
    for (int r = 0; r < NR; ++r)
      if (s_mode[r] == kModeCheck) acc[2 * r] = acc[2 * r + 1] = 0.0;
    const double* Xb = X + S.voff * NR;
    auto xval = [&](int j, long long, double (&o)[NR]) {
      ldv<NR>(Xb + static_cast<long long>(j) * NR, o);
    };
    for (int k = 0; k < kRPT; ++k) {
      const int i = row0 + k * kBlock + threadIdx.x;
      if (i >= S.nrows) break;
      Nbhd h;
      if (!decode(S, i, nxp1, mask, &h)) continue;
      double xs[NR], ax[NR], b[NR], rv[NR];
      stencil_apply<NR>(h, i, S.w, nxp1, st, xval, xs, ax);
      ldv<NR>(bsrc + h.g * NR, b);
      const long long v = (S.voff + i) * NR;
      ldv<NR>(R + v, rv);
      const double dv = dinv[h.g];
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        if (s_mode[r] != kModeCheck) continue;
        const double rt = xsub(b[r], ax[r]);
        rv[r] = rt;
        acc[2 * r] += rt * rt;
        acc[2 * r + 1] += rt * xmul(dv, rt);
      }
      stv<NR>(R + v, rv);
    }
  }
  block_reduce_store<2 * NR>(acc, part + static_cast<long long>(S.toff + tl.t) * 2 * NR);
}

template <int NR>
__global__ void __launch_bounds__(kBlock)
    k_cg_b(const CgSys* sys, const CgTile* tiles, const CgCtl* ctl, const double* dinv, int nxp1,
           const unsigned char* mask, double* X, double* R, const double* P, const double* Q,
           double* part) {
  const CgTile tl = tiles[blockIdx.x];
  const CgSys S = sys[tl.sys];
  __shared__ double s_alpha[NR];
  __shared__ int s_mode[NR];
  if (threadIdx.x < NR) {
    const CgCtl c = ctl[tl.sys * NR + threadIdx.x];
    s_alpha[threadIdx.x] = c.alpha;
    s_mode[threadIdx.x] = c.mode_b;
  }
  __syncthreads();
  bool any = false, upd[NR];
  double alpha[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    upd[r] = s_mode[r] == kModeNormal;
    any |= upd[r];
    alpha[r] = s_alpha[r];
  }
  if (!any) return;
  double acc[2 * NR];
#pragma unroll
  for (int k = 0; k < 2 * NR; ++k) acc[k] = 0.0;
  const int row0 = tl.t * kTile;
  for (int k = 0; k < kRPT; ++k) {
    const int i = row0 + k * kBlock + threadIdx.x;
    if (i >= S.nrows) break;
    long long g = 0;
    if (mask) {
      const int lx = i % S.w, ly = i / S.w;
      g = static_cast<long long>(S.y0 + ly) * nxp1 + (S.x0 + lx);
      if (!mask[g]) continue;
    } else {
      g = static_cast<long long>(S.y0 + i / S.w) * nxp1 + (S.x0 + i % S.w);
    }
    const long long v = (S.voff + i) * NR;
    double x[NR], r[NR], p[NR], q[NR];
    ldv<NR>(X + v, x);
    ldv<NR>(R + v, r);
    ldv<NR>(P + v, p);
    ldv<NR>(Q + v, q);
    const double dv = dinv[g];
#pragma unroll
    for (int k2 = 0; k2 < NR; ++k2) {
      if (!upd[k2]) continue;
      x[k2] = xadd(x[k2], xmul(alpha[k2], p[k2]));
      r[k2] = xsub(r[k2], xmul(alpha[k2], q[k2]));
      acc[2 * k2] += r[k2] * r[k2];
      acc[2 * k2 + 1] += r[k2] * xmul(dv, r[k2]);
    }
    stv<NR>(X + v, x);
    stv<NR>(R + v, r);
  }
  block_reduce_store<2 * NR>(acc, part + static_cast<long long>(S.toff + tl.t) * 2 * NR);
}

enum Phase { kPhaseInit = 0, kPhaseA = 1, kPhaseB = 2 };

template <int PH>
__global__ void k_cg_reduce(const CgSys* sys, int nsys, int nr, CgCtl* ctl, const double* part,
                            double tol) {
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= nsys * nr) return;
  const int s = wid / nr, r = wid % nr;
  CgCtl c = ctl[wid];
  if (PH == kPhaseA && c.mode_a == kModeSkip) return;
  if (PH == kPhaseB && c.mode_b == kModeSkip) return;
  const CgSys S = sys[s];
  double a0 = 0.0, a1 = 0.0;
  for (int t = lane; t < S.ntiles; t += 32) {
    const double* p = part + (static_cast<long long>(S.toff + t) * nr + r) * 2;
    a0 += p[0];
    a1 += p[1];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a0 += __shfl_xor_sync(0xffffffffu, a0, o);
    a1 += __shfl_xor_sync(0xffffffffu, a1, o);
  }
  if (lane != 0) return;
  if (PH == kPhaseInit) {
    c.bnorm = sqrt(a0);
    c.iters = 0;
    c.alpha = c.beta = 0.0;
    c.mode_b = kModeSkip;
    if (c.bnorm == 0.0) {  // sparse.cpp:208-212
      c.status = kConverged;
      c.final_res = 0.0;
      c.mode_a = kModeSkip;
    } else {
      c.status = kRunning;
      c.rho = a1;
      c.restart = 1;
      c.mode_a = kModeNormal;
    }
  } else if (PH == kPhaseA) {
    if (c.mode_a == kModeNormal) {
      const double pq = a0;
      if (pq <= 0.0) {  // sparse.cpp:225-226
        c.status = kIndefinite;
        c.mode_a = c.mode_b = kModeSkip;
      } else {
        c.alpha = c.rho / pq;
        c.mode_b = kModeNormal;
        c.mode_a = kModeSkip;
      }
    } else {  // confirmation with the true residual (sparse.cpp:232-246)
      const double true_rel = sqrt(a0) / c.bnorm;
      if (true_rel <= tol) {
        c.status = kConverged;
        c.final_res = true_rel;
        c.mode_a = c.mode_b = kModeSkip;
      } else if (c.iters >= S.maxit) {
        c.status = kNotConverged;  // sparse.cpp:255-257
        c.final_res = true_rel;
        c.mode_a = c.mode_b = kModeSkip;
      } else {
        c.rho = a1;
        c.restart = 1;
        c.mode_a = kModeNormal;
        c.mode_b = kModeSkip;
      }
    }
  } else {  // kPhaseB
    c.iters += 1;
    c.mode_b = kModeSkip;
    if (sqrt(a0) <= tol * c.bnorm || c.iters >= S.maxit) {
      c.mode_a = kModeCheck;
    } else {
      c.beta = a1 / c.rho;
      c.rho = a1;
      c.restart = 0;
      c.mode_a = kModeNormal;
    }
  }
  ctl[wid] = c;
}

template <int NR>
void launch_init(unsigned ntiles, cudaStream_t st, const CgSys* sys, const CgTile* tiles,
                 const Level& L, const unsigned char* mask, const double* bsrc, double* X,
                 double* R, double* part) {
  k_cg_init<NR><<<ntiles, kBlock, 0, st>>>(sys, tiles, L.dinv.get(), L.nx + 1, mask, bsrc, X, R,
                                           part);
}
template <int NR>
void launch_a(unsigned ntiles, cudaStream_t st, const CgSys* sys, const CgTile* tiles,
              const CgCtl* ctl, const Level& L, const unsigned char* mask, const double* bsrc,
              const double* X, double* R, const double* Pin, double* Pout, double* Q,
              double* part) {
  k_cg_a<NR><<<ntiles, kBlock, 0, st>>>(sys, tiles, ctl, L.stA.get(), L.dinv.get(), L.nx + 1,
                                        mask, bsrc, X, R, Pin, Pout, Q, part);
}
template <int NR>
void launch_b(unsigned ntiles, cudaStream_t st, const CgSys* sys, const CgTile* tiles,
              const CgCtl* ctl, const Level& L, const unsigned char* mask, double* X, double* R,
              const double* P, const double* Q, double* part) {
  k_cg_b<NR><<<ntiles, kBlock, 0, st>>>(sys, tiles, ctl, L.dinv.get(), L.nx + 1, mask, X, R, P,
                                        Q, part);
}

#define MLG_NR_DISPATCH(nr, fn, ...)                                      \
  do {                                                                    \
    switch (nr) {                                                         \
      case 1: fn<1>(__VA_ARGS__); break;                                  \
      case 2: fn<2>(__VA_ARGS__); break;                                  \
      case 4: fn<4>(__VA_ARGS__); break;                                  \
      case 8: fn<8>(__VA_ARGS__); break;                                  \
      default: throw ConfigError("unsupported right-hand-side batch width"); \
    }                                                                     \
  } while (0)

}  // namespace

void CgBatch::setup(Ctx& c, const Level& lev, std::vector<CgSys> systems, int nr_,
                    const unsigned char* mask_, const double* bsrc_) {
  L = &lev;
  nr = nr_;
  mask = mask_;
  bsrc = bsrc_;
  total_rows = 0;
  total_tiles = 0;
  for (CgSys& s : systems) {
    s.nrows = s.w * s.h;
    s.voff = total_rows;
    s.ntiles = std::max(1, (s.nrows + kTile - 1) / kTile);
    s.toff = total_tiles;
    s.maxit = 10 * std::max(s.nrows, 1);
    total_rows += s.nrows;
    total_tiles += s.ntiles;
  }
  sys_h = std::move(systems);
  const std::size_t nv = static_cast<std::size_t>(total_rows) * nr;
  X.ensure(nv);
  R.ensure(nv);
  P0.ensure(nv);
  P1.ensure(nv);
  Q.ensure(nv);
  partA.ensure(static_cast<std::size_t>(total_tiles) * 2 * nr);
  partB.ensure(static_cast<std::size_t>(total_tiles) * 2 * nr);
  sys_d.ensure(sys_h.size());
  sys_d.upload(sys_h.data(), sys_h.size(), c.stream);
  ctl_d.ensure(sys_h.size() * nr);
  tiles_d.ensure(total_tiles);
}

CgResult CgBatch::solve(Ctx& c, double tol, int maxit_override) {
  const int nsys = static_cast<int>(sys_h.size());
  if (maxit_override > 0) {
    for (CgSys& s : sys_h) s.maxit = maxit_override;
    sys_d.upload(sys_h.data(), sys_h.size(), c.stream);
  }
  std::vector<CgTile> tiles;
  long long active_rows = 0;
  auto rebuild = [&](const std::vector<char>& active) {
    tiles.clear();
    active_rows = 0;
    for (int s = 0; s < nsys; ++s)
      if (active[s]) {
        active_rows += sys_h[s].nrows;
        for (int t = 0; t < sys_h[s].ntiles; ++t) tiles.push_back({s, t});
      }
    tiles_d.upload(tiles.data(), tiles.size(), c.stream);
  };
  std::vector<char> active(nsys, 1);
  rebuild(active);
  const unsigned red_blocks = grid_for(static_cast<std::int64_t>(nsys) * nr * 32, 128);
  cudaStream_t st = c.stream;

  MLG_NR_DISPATCH(nr, launch_init, static_cast<unsigned>(tiles.size()), st, sys_d.get(),
                  tiles_d.get(), *L, mask, bsrc, X.get(), R.get(), partA.get());
  MLG_LAUNCH_CHECK();
  k_cg_reduce<kPhaseInit><<<red_blocks, 128, 0, st>>>(sys_d.get(), nsys, nr, ctl_d.get(),
                                                      partA.get(), tol);
  MLG_LAUNCH_CHECK();

  std::vector<CgCtl> ctl(static_cast<std::size_t>(nsys) * nr);
  double* pin = P0.get();
  double* pout = P1.get();
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> evs;
  int chunk = 16;
  int iters_done = 0;
  while (true) {
    for (int it = 0; it < chunk && !tiles.empty(); ++it) {
      const unsigned nt = static_cast<unsigned>(tiles.size());
      const bool prof = c.profile && mask == nullptr;
      if (prof) {
        c.times.ka_rows += static_cast<double>(active_rows);
        MLG_CUDA(cudaEventCreate(&ev0));
        MLG_CUDA(cudaEventCreate(&ev1));
        MLG_CUDA(cudaEventRecord(ev0, st));
      }
      MLG_NR_DISPATCH(nr, launch_a, nt, st, sys_d.get(), tiles_d.get(), ctl_d.get(), *L, mask,
                      bsrc, X.get(), R.get(), pin, pout, Q.get(), partA.get());
      MLG_LAUNCH_CHECK();
      if (prof) {
        MLG_CUDA(cudaEventRecord(ev1, st));
        evs.emplace_back(ev0, ev1);
      }
      k_cg_reduce<kPhaseA><<<red_blocks, 128, 0, st>>>(sys_d.get(), nsys, nr, ctl_d.get(),
                                                       partA.get(), tol);
      MLG_LAUNCH_CHECK();
      MLG_NR_DISPATCH(nr, launch_b, nt, st, sys_d.get(), tiles_d.get(), ctl_d.get(), *L, mask,
                      X.get(), R.get(), pout, Q.get(), partB.get());
      MLG_LAUNCH_CHECK();
      k_cg_reduce<kPhaseB><<<red_blocks, 128, 0, st>>>(sys_d.get(), nsys, nr, ctl_d.get(),
                                                       partB.get(), tol);
      MLG_LAUNCH_CHECK();
      std::swap(pin, pout);
      c.times.kernel_launches += 4;
    }
    iters_done += chunk;
    ctl_d.download(ctl.data(), ctl.size(), st);
    c.sync();
    bool running = false;
    bool changed = false;
    for (int s = 0; s < nsys; ++s) {
      bool sys_running = false;
      for (int r = 0; r < nr; ++r) {
        const CgCtl& k = ctl[static_cast<std::size_t>(s) * nr + r];
        if (k.status == kIndefinite)
          throw SolverError("cg_solve: matrix is not positive definite (p'Mp <= 0)");
        if (k.status == kRunning) sys_running = true;
      }
      if (active[s] && !sys_running) {
        active[s] = 0;
        changed = true;
      }
      running |= sys_running;
    }
    if (!running) break;
    if (changed) rebuild(active);
    chunk = std::min(64, chunk * 2);
  }
  if (!evs.empty()) {
    for (auto& e : evs) {
      float ms = 0.f;
      MLG_CUDA(cudaEventElapsedTime(&ms, e.first, e.second));
      c.times.ka_ms_sum += ms;
      c.times.ka_launches += 1;
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
  }
  CgResult res;
  res.reports.resize(ctl.size());
  for (std::size_t k = 0; k < ctl.size(); ++k) {
    res.reports[k].iterations = ctl[k].iters;
    res.reports[k].final_residual = ctl[k].final_res;
    res.reports[k].converged = ctl[k].status == kConverged ? 1 : 0;
    res.iters_max = std::max(res.iters_max, ctl[k].iters);
  }
  return res;
}

}  // namespace mlg

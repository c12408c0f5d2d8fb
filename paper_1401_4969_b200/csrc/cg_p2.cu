// Batched Jacobi-PCG for P2 systems (windows of the half-lattice dof grid,
// 25-slot operators): the local Dirichlet solves and the strip solve of a
// degree-2 correction step.  Same semantics as the reference's cg_solve
// (sparse.cpp:199-258): x0 = 0; zero rhs -> 0 iterations; alpha = rho/p'q
// (p'q <= 0 is an error); stop on ||r|| <= tol ||b|| confirmed by the true
// residual b - A x, else restart from it; maxit = 10 n; the final residual is
// reported when maxit runs out.
//
// Each iteration is three sweeps over the batch (q = A p | x, r update | p
// update), every per-system scalar decided on the device between them by one
// block per system summing its tiles' partials in a fixed order -- bitwise
// reproducible, no host round trip inside an iteration.  Vectors live in the
// P1 path's pooled layout (CgSys.voff / pitch, cg.cuh) with a two-deep zero
// frame (pitch w + 2, two zero rows above and below), so the 5x5 stencil
// needs no bounds tests and the glue / strip-scatter kernels read them as
// they read the P1 batch.  This path favours simplicity over bandwidth: the
// degree-2 step is an extension, the P1 kernels in cg.cu are the hot path.
#include <algorithm>

#include "cg_p2.cuh"
#include "stencil.cuh"

namespace mlg {
namespace {

constexpr int kT = 256;  // threads (= window points) per tile

enum : int { kNormal = 0, kCheck = 1, kRestart = 2, kPupd = 3, kFinal = 4, kDone = 5 };

struct P2Ctl {
  double rho, alpha, beta, bnorm, final_res;
  int state, iters, converged, indefinite;
};

struct P2Args {
  const double* st;  // level operator, 25 slots per dof
  const unsigned* pat;
  int gxp1;          // dof-grid row length
  const unsigned char* mask;  // strip systems: dof in the system
  const double* bsrc;
  int bstride;
};

__device__ __forceinline__ bool point_of(const CgSys& S, long long k, int* lx, int* ly) {
  *ly = static_cast<int>(k / S.w);
  *lx = static_cast<int>(k % S.w);
  return k < S.nrows;
}

__device__ __forceinline__ long long gdof(const CgSys& S, const P2Args& A, int lx, int ly) {
  return static_cast<long long>(S.y0 + ly) * A.gxp1 + (S.x0 + lx);
}

__device__ __forceinline__ bool in_sys(const CgSys& S, const P2Args& A, int lx, int ly) {
  return A.mask == nullptr || A.mask[gdof(S, A, lx, ly)];
}

// (A v) at window point (lx, ly): the 25 slots in ascending column order; the
// zero frame and the never-written non-system points supply the zeros.
__device__ __forceinline__ double apply_row(const CgSys& S, const P2Args& A, const double* v,
                                            int lx, int ly) {
  const long long d = gdof(S, A, lx, ly);
  const long long c = cg_index(S, ly, lx);
  const unsigned m = A.pat[d];
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 25; ++q)
    if (m >> q & 1u) s = fma(A.st[d * 25 + q], v[c + (q / 5 - 2) * S.pitch + (q % 5 - 2)], s);
  return s;
}

template <int K>
__device__ __forceinline__ void tile_store(double (&acc)[K], double* out) {
  block_reduce_store<K, kT>(acc, out);
}

// Sum of a system's tile partials (2 per tile) by one block of kF threads:
// thread t takes tiles t, t + kF, ...; then a fixed tree -- the same order on
// every run.  The result is valid in thread 0.
constexpr int kF = 256;
__device__ __forceinline__ void sys_sum(const CgSys& S, const double* part, double* a0,
                                        double* a1) {
  double acc[2] = {0.0, 0.0};
  for (int t = threadIdx.x; t < S.ntiles; t += kF) {
    acc[0] += part[2LL * (S.toff + t)];
    acc[1] += part[2LL * (S.toff + t) + 1];
  }
  __shared__ double red[2];
  block_reduce_store<2, kF>(acc, red);
  __syncthreads();
  *a0 = red[0];
  *a1 = red[1];
}

__global__ void __launch_bounds__(kT) k_p2cg_init(const CgSys* sys, const int* tile_sys,
                                                  const int* tile_t, P2Args A, double* X,
                                                  double* R, double* P, double* part) {
  const CgSys S = sys[tile_sys[blockIdx.x]];
  const long long k = static_cast<long long>(tile_t[blockIdx.x]) * kT + threadIdx.x;
  double acc[2] = {0.0, 0.0};
  int lx, ly;
  if (point_of(S, k, &lx, &ly) && in_sys(S, A, lx, ly)) {
    const long long d = gdof(S, A, lx, ly);
    const long long v = cg_index(S, ly, lx);
    const double b = A.bsrc[d * A.bstride + S.rhs];
    const double z = (1.0 / A.st[d * 25 + 12]) * b;  // JacobiPreconditioner::apply
    X[v] = 0.0;
    R[v] = b;
    P[v] = z;
    acc[0] = b * b;
    acc[1] = b * z;
  }
  tile_store<2>(acc, part + 2LL * blockIdx.x);
}

__global__ void __launch_bounds__(kF) k_p2cg_init_final(int nsys, const CgSys* sys,
                                                         const double* part, double tol,
                                                         P2Ctl* ctl) {
  const int s = blockIdx.x;
  const CgSys S = sys[s];
  double bb, rz;
  sys_sum(S, part, &bb, &rz);
  if (threadIdx.x) return;
  P2Ctl c{};
  c.bnorm = sqrt(bb);
  c.rho = rz;
  c.state = c.bnorm == 0.0 ? kDone : kNormal;
  c.converged = c.bnorm == 0.0 ? 1 : 0;
  ctl[s] = c;
}

// Sweep A: NORMAL q = A p (p'q); CHECK / FINAL r = b - A x (r'r, r'z).
__global__ void __launch_bounds__(kT) k_p2cg_a(const CgSys* sys, const int* tile_sys,
                                               const int* tile_t, P2Args A, const P2Ctl* ctl,
                                               const double* X, double* R, const double* P,
                                               double* Q, double* part) {
  const int s = tile_sys[blockIdx.x];
  const CgSys S = sys[s];
  const int st = ctl[s].state;
  const long long k = static_cast<long long>(tile_t[blockIdx.x]) * kT + threadIdx.x;
  double acc[2] = {0.0, 0.0};
  int lx, ly;
  if ((st == kNormal || st == kCheck || st == kFinal) && point_of(S, k, &lx, &ly) &&
      in_sys(S, A, lx, ly)) {
    const long long v = cg_index(S, ly, lx);
    if (st == kNormal) {
      const double q = apply_row(S, A, P, lx, ly);
      Q[v] = q;
      acc[0] = P[v] * q;
    } else {
      const long long d = gdof(S, A, lx, ly);
      const double rt = A.bsrc[d * A.bstride + S.rhs] - apply_row(S, A, X, lx, ly);
      R[v] = rt;
      acc[0] = rt * rt;
      acc[1] = rt * ((1.0 / A.st[d * 25 + 12]) * rt);
    }
  }
  tile_store<2>(acc, part + 2LL * blockIdx.x);
}

__global__ void __launch_bounds__(kF) k_p2cg_a_final(int nsys, const CgSys* sys,
                                                      const double* part, double tol,
                                                      P2Ctl* ctl) {
  const int s = blockIdx.x;
  const CgSys S = sys[s];
  P2Ctl c = ctl[s];
  if (c.state != kNormal && c.state != kCheck && c.state != kFinal) return;  // block-uniform
  double a0, a1;
  sys_sum(S, part, &a0, &a1);
  if (threadIdx.x) return;
  if (c.state == kNormal) {
    if (a0 <= 0.0) {
      c.indefinite = 1;
      c.state = kDone;
    } else {
      c.alpha = c.rho / a0;
    }
  } else {
    const double rel = sqrt(a0) / c.bnorm;
    if (c.state == kFinal) {
      c.final_res = rel;
      c.converged = rel <= tol;
      c.state = kDone;
    } else if (rel <= tol) {
      c.final_res = rel;
      c.converged = 1;
      c.state = kDone;
    } else if (c.iters >= S.maxit) {  // the loop ends on this restart
      c.final_res = rel;
      c.state = kDone;
    } else {
      c.rho = a1;
      c.state = kRestart;
    }
  }
  ctl[s] = c;
}

// Sweep B: NORMAL x += alpha p, r -= alpha q (r'r, r'z); RESTART p = z.
__global__ void __launch_bounds__(kT) k_p2cg_b(const CgSys* sys, const int* tile_sys,
                                               const int* tile_t, P2Args A, const P2Ctl* ctl,
                                               double* X, double* R, double* P, const double* Q,
                                               double* part) {
  const int s = tile_sys[blockIdx.x];
  const CgSys S = sys[s];
  const P2Ctl c = ctl[s];
  const long long k = static_cast<long long>(tile_t[blockIdx.x]) * kT + threadIdx.x;
  double acc[2] = {0.0, 0.0};
  int lx, ly;
  if ((c.state == kNormal || c.state == kRestart) && point_of(S, k, &lx, &ly) &&
      in_sys(S, A, lx, ly)) {
    const long long v = cg_index(S, ly, lx);
    const double dv = 1.0 / A.st[gdof(S, A, lx, ly) * 25 + 12];
    if (c.state == kNormal) {
      X[v] = X[v] + c.alpha * P[v];
      const double r = R[v] - c.alpha * Q[v];
      R[v] = r;
      acc[0] = r * r;
      acc[1] = r * (dv * r);
    } else {
      P[v] = dv * R[v];
    }
  }
  tile_store<2>(acc, part + 2LL * blockIdx.x);
}

__global__ void __launch_bounds__(kF) k_p2cg_b_final(int nsys, const CgSys* sys,
                                                      const double* part, double tol,
                                                      P2Ctl* ctl) {
  const int s = blockIdx.x;
  const CgSys S = sys[s];
  P2Ctl c = ctl[s];
  if (c.state == kRestart) {
    if (threadIdx.x == 0) {
      c.state = kNormal;
      ctl[s] = c;
    }
    return;
  }
  if (c.state == kNormal) {  // block-uniform
    double rr, rz;
    sys_sum(S, part, &rr, &rz);
    if (threadIdx.x) return;
    c.iters += 1;
    if (sqrt(rr) <= tol * c.bnorm) {
      c.state = kCheck;
    } else if (c.iters >= S.maxit) {
      c.state = kFinal;
    } else {
      c.beta = rz / c.rho;
      c.rho = rz;
      c.state = kPupd;
    }
    ctl[s] = c;
  }
}

// Sweep C: p = z + beta p.
__global__ void __launch_bounds__(kT) k_p2cg_c(const CgSys* sys, const int* tile_sys,
                                               const int* tile_t, P2Args A, P2Ctl* ctl,
                                               const double* R, double* P) {
  const int s = tile_sys[blockIdx.x];
  const CgSys S = sys[s];
  const P2Ctl c = ctl[s];
  if (c.state != kPupd) return;
  const long long k = static_cast<long long>(tile_t[blockIdx.x]) * kT + threadIdx.x;
  int lx, ly;
  if (point_of(S, k, &lx, &ly) && in_sys(S, A, lx, ly)) {
    const long long v = cg_index(S, ly, lx);
    const double dv = 1.0 / A.st[gdof(S, A, lx, ly) * 25 + 12];
    P[v] = dv * R[v] + c.beta * P[v];
  }
}

__global__ void k_p2cg_c_final(int nsys, P2Ctl* ctl, int* running) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nsys) return;
  if (ctl[s].state == kPupd) ctl[s].state = kNormal;
  if (ctl[s].state != kDone) atomicAdd(running, 1);
}

}  // namespace

void CgBatchP2::setup(Ctx& c, const Level& L, std::vector<CgSys> systems,
                      const unsigned char* mask, const double* bsrc, int bstride) {
  L_ = &L;
  mask_ = mask;
  bsrc_ = bsrc;
  bstride_ = bstride;
  int max_pitch = 1;
  for (const CgSys& s : systems) max_pitch = std::max(max_pitch, s.w + 2);
  long long cursor = 2LL * max_pitch + 4;
  std::vector<int> ts, tt;
  for (CgSys& s : systems) {
    s.nrows = s.w * s.h;
    s.pitch = s.w + 2;
    s.voff = cursor + 2LL * s.pitch + 2;
    s.ntiles = std::max(1, (s.nrows + kT - 1) / kT);
    s.toff = static_cast<int>(ts.size());
    s.maxit = 10 * std::max(s.nrows, 1);
    for (int t = 0; t < s.ntiles; ++t) {
      ts.push_back(static_cast<int>(&s - systems.data()));
      tt.push_back(t);
    }
    cursor += static_cast<long long>(s.h + 4) * s.pitch;
  }
  rows_ = cursor + 4LL * max_pitch + 64;
  sys_h_ = std::move(systems);
  ntiles_ = static_cast<int>(ts.size());
  sys_d_.ensure(sys_h_.size());
  sys_d_.upload(sys_h_.data(), sys_h_.size(), c.stream);
  tsys_.ensure(ts.size());
  tsys_.upload(ts.data(), ts.size(), c.stream);
  tt_.ensure(tt.size());
  tt_.upload(tt.data(), tt.size(), c.stream);
  for (DevBuf<double>* v : {&X_, &R_, &P_, &Q_}) {
    v->ensure(static_cast<std::size_t>(rows_));
    MLG_CUDA(cudaMemsetAsync(v->get(), 0, sizeof(double) * rows_, c.stream));
  }
  part_.ensure(2ULL * ntiles_);
  ctl_.ensure(sys_h_.size() * sizeof(P2Ctl));
  running_.ensure(1);
  c.sync();  // host vectors above are temporaries
}

CgResult CgBatchP2::solve(Ctx& c, double tol) {
  const int nsys = static_cast<int>(sys_h_.size());
  CgResult out;
  out.reports.resize(sys_h_.size());
  if (nsys == 0) return out;
  P2Args A{L_->p2A.get(), L_->p2pat.get(), L_->gx() + 1, mask_, bsrc_, bstride_};
  auto* ctl = reinterpret_cast<P2Ctl*>(ctl_.get());
  const CgSys* sd = sys_d_.get();
  const int* ts = tsys_.get();
  const int* tt = tt_.get();
  const unsigned sb = static_cast<unsigned>((nsys + 127) / 128);
  const unsigned nb = static_cast<unsigned>(nsys);  // one block per system (sys_sum)
  k_p2cg_init<<<ntiles_, kT, 0, c.stream>>>(sd, ts, tt, A, X_.get(), R_.get(), P_.get(),
                                           part_.get());
  MLG_LAUNCH_CHECK();
  k_p2cg_init_final<<<nb, kF, 0, c.stream>>>(nsys, sd, part_.get(), tol, ctl);
  MLG_LAUNCH_CHECK();
  long long max_maxit = 0;
  for (const CgSys& s : sys_h_) max_maxit = std::max<long long>(max_maxit, s.maxit);
  constexpr int kChunk = 64;
  for (long long it = 0; it <= max_maxit + 2; it += kChunk) {
    for (int k = 0; k < kChunk; ++k) {
      k_p2cg_a<<<ntiles_, kT, 0, c.stream>>>(sd, ts, tt, A, ctl, X_.get(), R_.get(), P_.get(),
                                            Q_.get(), part_.get());
      k_p2cg_a_final<<<nb, kF, 0, c.stream>>>(nsys, sd, part_.get(), tol, ctl);
      k_p2cg_b<<<ntiles_, kT, 0, c.stream>>>(sd, ts, tt, A, ctl, X_.get(), R_.get(), P_.get(),
                                            Q_.get(), part_.get());
      k_p2cg_b_final<<<nb, kF, 0, c.stream>>>(nsys, sd, part_.get(), tol, ctl);
      k_p2cg_c<<<ntiles_, kT, 0, c.stream>>>(sd, ts, tt, A, ctl, R_.get(), P_.get());
      running_.zero(c.stream);
      k_p2cg_c_final<<<sb, 128, 0, c.stream>>>(nsys, ctl, running_.get());
      MLG_LAUNCH_CHECK();
    }
    int running = 0;
    running_.download(&running, 1, c.stream);
    c.sync();
    if (running == 0) break;
  }
  std::vector<P2Ctl> h(static_cast<std::size_t>(nsys));
  MLG_CUDA(cudaMemcpyAsync(h.data(), ctl, sizeof(P2Ctl) * nsys, cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  for (int s = 0; s < nsys; ++s) {
    if (h[s].indefinite) throw SolverError("cg_solve: matrix is not positive definite (p'Mp <= 0)");
    if (h[s].state != kDone) throw SolverError("cg_solve: P2 CG did not terminate");
    SolveReport r;
    r.iterations = h[s].iters;
    r.final_residual = h[s].final_res;
    r.converged = h[s].converged;
    out.reports[static_cast<std::size_t>(s)] = r;
    out.iters_max = std::max(out.iters_max, r.iterations);
  }
  return out;
}

}  // namespace mlg

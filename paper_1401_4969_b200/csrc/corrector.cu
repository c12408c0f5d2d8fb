// The correction step (Algorithm 4.1 of the paper, corrector.cpp:198-412) on
// one B200: hierarchy/partition bookkeeping on the host, everything of size N
// in HBM.
//
//   Hierarchy ctor / extend_to   corrector.cpp:111-146
//   build_partition              decomp.cpp:24-86 (+ delta rounding corrector.cpp:117-121)
//   local_bvp_solve              corrector.cpp:198-214  -> residual once per eigenvector,
//                                 all (eigenvector x subdomain) systems in ONE batched CG
//   interface_solve              corrector.cpp:216-254  -> glue gather + strip CG
//   augmented_eigensolve         corrector.cpp:256-334  -> Gram blocks on device, restriction
//                                 chain, dense gen-eig with cuSOLVER sygvd, expansion
//   one_correction_step          corrector.cpp:336-412
//   solve_interior_eigenproblem  sparse.cpp:326-355 (level-1 direct solve)
#include <algorithm>
#include <cfloat>
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>

#include "cg_p2.cuh"
#include "corrector.cuh"
#include "p2.cuh"
#include "vec_kernels.cuh"

namespace mlg {
namespace {

constexpr int kB = 256;

// ---- prolongation / restriction (fespace.cpp:355-400, sparse.cpp:129-154) ----

// y = P x for one refinement: fine dof at a coarse vertex -> 1.0 x_c, at an
// axis or SW-NE diagonal edge midpoint -> 0.5 x_a + 0.5 x_b (a < b), summed
// from 0.0 in ascending coarse column order.
// With a hole (fine scale hf) the fine points strictly inside it carry no row
// of P (they lie in no coarse element): 0.
__device__ __forceinline__ bool point_live(const Hole& h, int nx, int ny, int ix, int iy) {
  return !h.any() || cell_active(h, nx, ny, ix, iy) || cell_active(h, nx, ny, ix - 1, iy) ||
         cell_active(h, nx, ny, ix, iy - 1) || cell_active(h, nx, ny, ix - 1, iy - 1);
}

template <int NR>
__global__ void k_prolong(int nxc, int nxf, int nyf, Hole hf, const double* xc, double* xf) {
  const long long d = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (d >= static_cast<long long>(nxf + 1) * (nyf + 1)) return;
  const int fx = static_cast<int>(d % (nxf + 1)), fy = static_cast<int>(d / (nxf + 1));
  const long long sc = nxc + 1;
  double y[NR], a[NR], b[NR];
  if (!point_live(hf, nxf, nyf, fx, fy)) {
#pragma unroll
    for (int r = 0; r < NR; ++r) y[r] = 0.0;
  } else if (!(fx & 1) && !(fy & 1)) {
    ldv<NR>(xc + (static_cast<long long>(fy / 2) * sc + fx / 2) * NR, a);
#pragma unroll
    for (int r = 0; r < NR; ++r) y[r] = xadd(0.0, xmul(1.0, a[r]));
  } else {
    const int ax = fx >> 1, ay = fy >> 1;             // lower/left endpoint
    const int bx = (fx + 1) >> 1, by = (fy + 1) >> 1;  // upper/right endpoint
    ldv<NR>(xc + (static_cast<long long>(ay) * sc + ax) * NR, a);
    ldv<NR>(xc + (static_cast<long long>(by) * sc + bx) * NR, b);
#pragma unroll
    for (int r = 0; r < NR; ++r) y[r] = xadd(xadd(0.0, xmul(0.5, a[r])), xmul(0.5, b[r]));
  }
  stv<NR>(xf + d * NR, y);
}

// y = P^T x: coarse c gathers its <=7 fine rows in ascending fine-row order
// (multiply_transpose scatters row by row), weights 0.5 / 1.0.
template <int NR>
__global__ void k_restrict(int nxf, int nyf, int nxc, int nyc, Hole hf, const double* xf,
                           double* xc) {
  const long long d = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (d >= static_cast<long long>(nxc + 1) * (nyc + 1)) return;
  const int cx = static_cast<int>(d % (nxc + 1)), cy = static_cast<int>(d / (nxc + 1));
  const int X = 2 * cx, Y = 2 * cy;
  const long long sf = nxf + 1;
  double y[NR], t[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) y[r] = 0.0;
  auto acc = [&](int fx, int fy, double w) {
    if (fx < 0 || fy < 0 || fx > nxf || fy > nyf) return;
    if (!point_live(hf, nxf, nyf, fx, fy)) return;  // no row of P
    ldv<NR>(xf + (static_cast<long long>(fy) * sf + fx) * NR, t);
#pragma unroll
    for (int r = 0; r < NR; ++r) y[r] = xadd(y[r], xmul(w, t[r]));
  };
  acc(X - 1, Y - 1, 0.5);
  acc(X, Y - 1, 0.5);
  acc(X - 1, Y, 0.5);
  acc(X, Y, 1.0);
  acc(X + 1, Y, 0.5);
  acc(X, Y + 1, 0.5);
  acc(X + 1, Y + 1, 0.5);
  stv<NR>(xc + d * NR, y);
}

// ---- residual / dual products ----

// res = lam * (M u) - (A u) at interior dofs (corrector.cpp:201,237); 0 on the boundary.
template <int NR>
__global__ void k_residual(IMap im, const Stencil* stA, const Stencil* stM,
                           const double* u, const double* w, Lam lam, double* out,
                           const unsigned char* only_mask) {
  const int nx = im.nx, ny = im.ny;
  const long long d = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (d >= static_cast<long long>(nx + 1) * (ny + 1)) return;
  const int ix = static_cast<int>(d % (nx + 1)), iy = static_cast<int>(d / (nx + 1));
  double y[NR];
  // Non-interior points get 0 (the CG windows of a domain with a hole cover
  // hole points, which must see a zero rhs); masked-out interior points are
  // never read.
  if (!im.interior(ix, iy)) {
#pragma unroll
    for (int r = 0; r < NR; ++r) y[r] = 0.0;
    stv<NR>(out + d * NR, y);
    return;
  }
  if (only_mask && !only_mask[d]) return;
  double mu[NR], aw[NR];
  full_row<NR>(stM, u, ix, iy, nx, ny, mu);
  full_row<NR>(stA, w, ix, iy, nx, ny, aw);
#pragma unroll
  for (int r = 0; r < NR; ++r) y[r] = xsub(xmul(lam.v[r], mu[r]), aw[r]);
  stv<NR>(out + d * NR, y);
}

// ya = A x, ym = M x at interior rows (boundary rows 0; they never reach the
// interior of a coarser level nor a dot product with an interior vector).
template <int NR>
__global__ void k_dual(IMap im, const Stencil* stA, const Stencil* stM, const double* x,
                       double* ya, double* ym) {
  const int nx = im.nx, ny = im.ny;
  const long long d = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (d >= static_cast<long long>(nx + 1) * (ny + 1)) return;
  const int ix = static_cast<int>(d % (nx + 1)), iy = static_cast<int>(d / (nx + 1));
  double y[NR];
  const bool inner = im.interior(ix, iy);
  if (ya) {
    if (inner) full_row<NR>(stA, x, ix, iy, nx, ny, y);
    else
      for (int r = 0; r < NR; ++r) y[r] = 0.0;
    stv<NR>(ya + d * NR, y);
  }
  if (ym) {
    if (inner) full_row<NR>(stM, x, ix, iy, nx, ny, y);
    else
      for (int r = 0; r < NR; ++r) y[r] = 0.0;
    stv<NR>(ym + d * NR, y);
  }
}

// Full-space single-vector SpMV over ALL rows (boundary rows included), the
// exact SparseSymMatrix::multiply; test/parity hook and SpMV microbenchmark.
__global__ void k_full_spmv(int nx, int ny, const Stencil* st, const double* x, double* y) {
  const long long d = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (d >= static_cast<long long>(nx + 1) * (ny + 1)) return;
  const int ix = static_cast<int>(d % (nx + 1)), iy = static_cast<int>(d / (nx + 1));
  double o[1];
  full_row<1>(st, x, ix, iy, nx, ny, o);
  y[d] = o[0];
}

// Interior-restricted SpMV (the matrix extract_submatrix(A, interior_dofs)),
// x and y in interior order; the local-solve operator on the whole interior.
__global__ void k_interior_spmv(int nx, int ny, const Stencil* st, const double* x, double* y) {
  const long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const int w = nx - 1, h = ny - 1;
  if (k >= static_cast<long long>(w) * h) return;
  const int i = static_cast<int>(k % w), j = static_cast<int>(k / w);
  const long long s = nx + 1;
  const long long g = static_cast<long long>(j + 1) * s + (i + 1);
  double a = 0.0;
  if (j > 0 && i > 0) a = xadd(a, xmul(st[g - s - 1].ne, x[k - w - 1]));
  if (j > 0) a = xadd(a, xmul(st[g - s].n, x[k - w]));
  if (i > 0) a = xadd(a, xmul(st[g - 1].e, x[k - 1]));
  const Stencil c = st[g];
  a = xadd(a, xmul(c.c, x[k]));
  if (i < w - 1) a = xadd(a, xmul(c.e, x[k + 1]));
  if (j < h - 1) a = xadd(a, xmul(c.n, x[k + w]));
  if (j < h - 1 && i < w - 1) a = xadd(a, xmul(c.ne, x[k + w + 1]));
  y[k] = a;
}

// ---- deterministic multi-dot: D[r][s] = sum_d U[d][r] * V[d][s] ----
template <int NR>
__global__ void __launch_bounds__(kB) k_mdot(long long n, const double* U, const double* V,
                                             double* part) {
  double acc[NR * NR];
#pragma unroll
  for (int k = 0; k < NR * NR; ++k) acc[k] = 0.0;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long d = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; d < n;
       d += stride) {
    double u[NR], v[NR];
    ldv<NR>(U + d * NR, u);
    ldv<NR>(V + d * NR, v);
#pragma unroll
    for (int r = 0; r < NR; ++r)
#pragma unroll
      for (int s = 0; s < NR; ++s) acc[r * NR + s] += u[r] * v[s];
  }
  block_reduce_store<NR * NR>(acc, part + static_cast<long long>(blockIdx.x) * NR * NR);
}

__global__ void k_mdot_final(int nblocks, int kk, const double* part, double* out) {
  const int k = threadIdx.x;
  if (k >= kk) return;
  double s = 0.0;
  for (int b = 0; b < nblocks; ++b) s += part[static_cast<long long>(b) * kk + k];
  out[k] = s;
}

// ---- glue / strip (corrector.cpp:216-254) ----

struct PartDev {
  int side, bw, bh;  // blocks in coarse cells
  int scale;         // 2^level
  int m;
  IRect inner[256];
  IRect overlap[256];
  short blk2j[256];  // block (bottom-up row-major) -> subdomain, -1: removed (hole)
};

// Subdomain whose closed inner region G_j contains the fine lattice point,
// or -1 (then the point belongs to the strip).  G_j lies inside the closed
// block D_j and never touches an interior block side, so the block found by
// integer division is the only candidate.
__device__ __forceinline__ int inner_owner(const PartDev& P, int ix, int iy) {
  const int c = min(ix / (P.bw * P.scale), P.side - 1);
  const int rb = min(iy / (P.bh * P.scale), P.side - 1);
  const int j = P.blk2j[rb * P.side + c];
  if (j < 0) return -1;
  const IRect& g = P.inner[j];
  if (ix >= g.x0 * P.scale && ix <= g.x1 * P.scale && iy >= g.y0 * P.scale &&
      iy <= g.y1 * P.scale)
    return j;
  return -1;
}

__global__ void k_strip_mask(IMap im, PartDev P, unsigned char* mask) {
  const int nx = im.nx, ny = im.ny;
  const long long d = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (d >= static_cast<long long>(nx + 1) * (ny + 1)) return;
  const int ix = static_cast<int>(d % (nx + 1)), iy = static_cast<int>(d / (nx + 1));
  const bool interior = im.interior(ix, iy);
  mask[d] = (interior && inner_owner(P, ix, iy) < 0) ? 1 : 0;
}

// glued = u + e_j on the closed G_j (bitwise, corrector.cpp:223-231); 0 elsewhere.
// e_j of eigenvector r comes from the batched local CG: system j*nev + r
// (window-compact X) ...
template <int NR>
__global__ void k_glue_cg(IMap im, PartDev P, int nev, const CgSys* sys, const double* X,
                          const double* u, double* glued) {
  const int nx = im.nx, ny = im.ny;
  const long long d = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (d >= static_cast<long long>(nx + 1) * (ny + 1)) return;
  const int ix = static_cast<int>(d % (nx + 1)), iy = static_cast<int>(d / (nx + 1));
  double y[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) y[r] = 0.0;
  if (im.interior(ix, iy)) {
    const int j = inner_owner(P, ix, iy);
    if (j >= 0) {
      double uu[NR];
      ldv<NR>(u + d * NR, uu);
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        if (r >= nev) break;
        const CgSys S = sys[j * nev + r];
        y[r] = xadd(uu[r], X[cg_index(S, iy - S.y0, ix - S.x0)]);
      }
    }
  }
  stv<NR>(glued + d * NR, y);
}

// ... or from caller-provided full-space corrections (NR = 1 test entry point).
__global__ void k_glue_full(IMap im, PartDev P, long long ndofs, const double* corr,
                            const double* u, double* glued) {
  const int nx = im.nx;
  const long long d = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (d >= ndofs) return;
  const int ix = static_cast<int>(d % (nx + 1)), iy = static_cast<int>(d / (nx + 1));
  double y = 0.0;
  if (im.interior(ix, iy)) {
    const int j = inner_owner(P, ix, iy);
    if (j >= 0) y = xadd(u[d], corr[static_cast<long long>(j) * ndofs + d]);
  }
  glued[d] = y;
}

// glued[strip dofs, lane r] = x of strip system r (same window for all r).
template <int NR>
__global__ void k_strip_scatter(int nx, int nev, const CgSys* sys, const unsigned char* mask,
                                const double* X, double* glued) {
  const CgSys S0 = sys[0];
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<long long>(S0.w) * S0.h) return;  // every window point (nrows = strip unknowns)
  const int ly = static_cast<int>(i / S0.w), lx = static_cast<int>(i % S0.w);
  const long long d = static_cast<long long>(S0.y0 + ly) * (nx + 1) + (S0.x0 + lx);
  if (!mask[d]) return;
  double x[NR];
  ldv<NR>(glued + d * NR, x);
#pragma unroll
  for (int r = 0; r < NR; ++r)
    if (r < nev) x[r] = X[cg_index(sys[r], ly, lx)];
  stv<NR>(glued + d * NR, x);
}

// ---- layout conversions ----

// rhs-major [k][n_src] (full or interior order) -> interleaved full lattice.
template <int NR>
__global__ void k_interleave(IMap im, int k_in, const double* src, int interior_src,
                             double* dst) {
  const int nx = im.nx, ny = im.ny;
  const long long d = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long nd = static_cast<long long>(nx + 1) * (ny + 1);
  if (d >= nd) return;
  const int ix = static_cast<int>(d % (nx + 1)), iy = static_cast<int>(d / (nx + 1));
  const long long ki = im.index(ix, iy);
  const long long ni = im.count();
  double y[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    double v = 0.0;
    if (r < k_in) {
      if (interior_src) {
        if (ki >= 0) v = src[r * ni + ki];
      } else {
        v = src[r * nd + d];
      }
    }
    y[r] = v;
  }
  stv<NR>(dst + d * NR, y);
}

// interleaved full lattice -> rhs-major (interior or full order), lanes perm[r].
template <int NR>
__global__ void k_deinterleave(IMap im, int k_out, const int* perm, const double* src,
                               int interior_dst, double* dst) {
  const int nx = im.nx, ny = im.ny;
  const long long d = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long nd = static_cast<long long>(nx + 1) * (ny + 1);
  if (d >= nd) return;
  const int ix = static_cast<int>(d % (nx + 1)), iy = static_cast<int>(d / (nx + 1));
  const long long ki = im.index(ix, iy);
  if (interior_dst && ki < 0) return;
  const long long ni = im.count();
  double v[NR];
  ldv<NR>(src + d * NR, v);
  const long long o = interior_dst ? ki : d;
  const long long n = interior_dst ? ni : nd;
  for (int r = 0; r < k_out; ++r) dst[r * n + o] = v[perm ? perm[r] : r];
}

// Interior coarse dofs of a full-lattice vector -> column-major mc x NR.
template <int NR>
__global__ void k_gather_coarse(IMap im, const double* src, double* dst) {
  const long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long mc = im.count();
  if (k >= mc) return;
  int ix, iy;
  im.point(k, &ix, &iy);
  const long long d = static_cast<long long>(iy) * (im.nx + 1) + ix;
  double v[NR];
  ldv<NR>(src + d * NR, v);
#pragma unroll
  for (int r = 0; r < NR; ++r) dst[r * mc + k] = v[r];
}

// full[:, i] += c[i][l] * glued[:, keep[l]] for l = 0..k-1 (corrector.cpp:318-320).
template <int NR>
__global__ void k_candidates(long long nd, int k, const int* keep, const double* coef,
                             const double* glued, double* full) {
  const long long d = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (d >= nd) return;
  double f[NR], g[NR];
  ldv<NR>(full + d * NR, f);
  ldv<NR>(glued + d * NR, g);
  for (int l = 0; l < k; ++l) {
    const double gl = g[keep[l]];
#pragma unroll
    for (int r = 0; r < NR; ++r) f[r] = xadd(f[r], xmul(coef[r * 8 + l], gl));
  }
  stv<NR>(full + d * NR, f);
}

// v[:, r] /= s[r] (restrict_interior(full) / sqrt(q), corrector.cpp:327)
template <int NR>
__global__ void k_div_lanes(long long nd, Lam s, double* v) {
  const long long d = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (d >= nd) return;
  double x[NR];
  ldv<NR>(v + d * NR, x);
#pragma unroll
  for (int r = 0; r < NR; ++r) x[r] = xdiv(x[r], s.v[r]);
  stv<NR>(v + d * NR, x);
}

// fix_sign (sparse.cpp:260-271): first index of max |v|, per lane.
struct AbsMax {
  double a;
  long long i;
};
__device__ __forceinline__ AbsMax better(AbsMax x, AbsMax y) {
  if (y.a > x.a || (y.a == x.a && y.i < x.i)) return y;
  return x;
}
template <int NR>
__global__ void __launch_bounds__(kB) k_absmax(int nx, int ny, const double* v, AbsMax* part) {
  const long long nd = static_cast<long long>(nx + 1) * (ny + 1);
  AbsMax best[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) best[r] = {-1.0, LLONG_MAX};
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long d = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; d < nd;
       d += stride) {
    const int ix = static_cast<int>(d % (nx + 1)), iy = static_cast<int>(d / (nx + 1));
    if (ix == 0 || iy == 0 || ix == nx || iy == ny) continue;
    double x[NR];
    ldv<NR>(v + d * NR, x);
#pragma unroll
    for (int r = 0; r < NR; ++r) best[r] = better(best[r], AbsMax{fabs(x[r]), d});
  }
  __shared__ AbsMax sh[kB];
  for (int r = 0; r < NR; ++r) {
    sh[threadIdx.x] = best[r];
    __syncthreads();
    for (int o = kB / 2; o > 0; o >>= 1) {
      if (threadIdx.x < o) sh[threadIdx.x] = better(sh[threadIdx.x], sh[threadIdx.x + o]);
      __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x * NR + r] = sh[0];
    __syncthreads();
  }
}

template <int NR>
__global__ void k_absmax_final(int nblocks, const AbsMax* part, const double* v, double* sign) {
  const int r = threadIdx.x;
  if (r >= NR) return;
  AbsMax b{-1.0, LLONG_MAX};
  for (int k = 0; k < nblocks; ++k) b = better(b, part[k * NR + r]);
  sign[r] = (b.i != LLONG_MAX && v[b.i * NR + r] < 0.0) ? -1.0 : 1.0;
}

template <int NR>
__global__ void k_apply_sign(long long nd, const double* sign, double* v) {
  const long long d = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (d >= nd) return;
  double x[NR];
  ldv<NR>(v + d * NR, x);
#pragma unroll
  for (int r = 0; r < NR; ++r)
    if (sign[r] < 0.0) x[r] = -x[r];
  stv<NR>(v + d * NR, x);
}

template <int NR>
__global__ void k_permute_lanes(long long nd, Lam permf, const double* src, double* dst) {
  const long long d = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (d >= nd) return;
  double x[NR], y[NR];
  ldv<NR>(src + d * NR, x);
#pragma unroll
  for (int r = 0; r < NR; ++r) y[r] = x[static_cast<int>(permf.v[r])];
  stv<NR>(dst + d * NR, y);
}

// Dense augmented pair (corrector.cpp:299-311), column-major dim x dim.
__global__ void k_build_aug(int mc, int k, const int* keep, const double* cc, const double* cu,
                            const double* uu, int nr, double* out) {
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const int dim = mc + k;
  if (idx >= static_cast<long long>(dim) * dim) return;
  const int i = static_cast<int>(idx % dim), j = static_cast<int>(idx / dim);
  double v;
  if (i < mc && j < mc) v = cc[static_cast<long long>(j) * mc + i];
  else if (i < mc) v = cu[static_cast<long long>(keep[j - mc]) * mc + i];
  else if (j < mc) v = cu[static_cast<long long>(keep[i - mc]) * mc + j];
  else v = uu[keep[i - mc] * nr + keep[j - mc]];
  out[idx] = v;
}

// ---- augmented eigenproblem with ONE candidate: arrowhead form ----------
// corrector.cpp:256-334 solves the (mc+1) pencil [[A_cc, a],[a', a_uu]] vs
// [[B_cc, b],[b', b_uu]] densely.  With the cached coarse spectrum
// A_cc V = B_cc V Lam (V'B_cc V = I) and c = V'b, d = V'a, the B-orthogonal
// change of basis x = [V (w_c - c x_u); x_u], x_u = w_u / sqrt(s_b) with the
// Schur complement s_b = b_uu - c'c turns it into the standard symmetric
// arrowhead problem [[Lam, e],[e', f]] w = mu w, e = (d - Lam c)/sqrt(s_b),
// f = (a_uu - 2 c'd + c'Lam c)/s_b, whose eigenvalues below lam_0 are the roots
// of the secular function g(mu) = f - mu - sum e_i^2 / (lam_i - mu) -- no dense
// factorisation per step.  s_b is exactly the reference's dependence test
// (b_uu - b'B_cc^{-1} b, corrector.cpp:285-292): below 1e-10^2 the candidate is
// dropped and the coarse pair (lam_0, V_0) is the answer.  One CTA; root by
// safeguarded Newton on g inside its bracket, block reductions in fixed order.
constexpr int kArrowThreads = 1024;

__device__ __forceinline__ void block_sum2(double& a, double& b, double* red) {
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) {
    red[warp] = a;
    red[32 + warp] = b;
  }
  __syncthreads();
  a = 0.0;
  b = 0.0;
  for (int k = 0; k < static_cast<int>(blockDim.x >> 5); ++k) {
    a += red[k];
    b += red[32 + k];
  }
}

__global__ void __launch_bounds__(kArrowThreads) k_aug_arrow(
    int mc, const double* lamc, const double* V, const double* a_cu, const double* b_cu,
    const double* auu, const double* buu, double* work, double* out_lam, double* out_cp,
    double* out_coef, int* out_flag) {
  __shared__ double red[64];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  double* c = work;
  double* d = work + mc;
  double* e = work + 2 * mc;
  for (int i = warp; i < mc; i += nw) {  // c = V'b, d = V'a (column i of V is contiguous)
    double sc = 0.0, sd = 0.0;
    const double* vi = V + static_cast<long long>(i) * mc;
    for (int j = lane; j < mc; j += 32) {
      const double v = vi[j];
      sc += v * b_cu[j];
      sd += v * a_cu[j];
    }
    for (int o = 16; o > 0; o >>= 1) {
      sc += __shfl_xor_sync(0xffffffffu, sc, o);
      sd += __shfl_xor_sync(0xffffffffu, sd, o);
    }
    if (lane == 0) {
      c[i] = sc;
      d[i] = sd;
    }
  }
  __syncthreads();
  double cc = 0.0, cd = 0.0, clc = 0.0, dummy = 0.0;
  for (int i = tid; i < mc; i += blockDim.x) {
    cc += c[i] * c[i];
    cd += c[i] * d[i];
    clc += lamc[i] * c[i] * c[i];
  }
  block_sum2(cc, cd, red);
  block_sum2(clc, dummy, red);
  const double s_b = buu[0] - cc;
  if (!(sqrt(fmax(s_b, 0.0)) >= 1e-10)) {  // dropped: the coarse pair
    for (int r = tid; r < mc; r += blockDim.x) out_cp[r] = V[r];
    if (tid == 0) {
      out_lam[0] = lamc[0];
      out_coef[0] = 0.0;
      *out_flag = 2;
    }
    return;
  }
  const double sq = sqrt(s_b);
  const double f = (auu[0] - 2.0 * cd + clc) / s_b;
  double ee = 0.0;
  for (int i = tid; i < mc; i += blockDim.x) {
    const double v = (d[i] - lamc[i] * c[i]) / sq;
    e[i] = v;
    ee += v * v;
  }
  block_sum2(ee, dummy, red);
  __syncthreads();
  // smallest root of g in (lo, lam_0); start from the 2x2 problem [[lam_0, e_0],[e_0, f]]
  const double l0 = lamc[0], e0 = e[0];
  double lo = fmin(l0, f) - sqrt(ee) - 1.0, hi = l0;
  const double h = 0.5 * (l0 - f);
  double mu = 0.5 * (l0 + f) - sqrt(h * h + e0 * e0);
  if (!(mu > lo && mu < hi)) mu = 0.5 * (lo + hi);
  for (int it = 0; it < 200; ++it) {
    double s1 = 0.0, s2 = 0.0;
    for (int i = tid; i < mc; i += blockDim.x) {
      const double t = e[i] / (lamc[i] - mu);
      s1 += e[i] * t;
      s2 += t * t;
    }
    block_sum2(s1, s2, red);
    const double g = f - mu - s1, gp = -1.0 - s2;
    if (g > 0.0)
      lo = mu;
    else if (g < 0.0)
      hi = mu;
    else
      break;
    double nx = mu - g / gp;
    if (!(nx > lo && nx < hi)) nx = 0.5 * (lo + hi);
    const bool done = fabs(nx - mu) <= 2.0 * DBL_EPSILON * fabs(mu) || !(hi - lo > 2.0 * DBL_EPSILON * fabs(hi));
    mu = nx;
    if (done) break;
  }
  // mu on (or within rounding of) the pole lam_0: deflated case, left to the dense path
  if (!(l0 - mu > 8.0 * DBL_EPSILON * fabs(l0))) {
    if (tid == 0) *out_flag = 1;
    return;
  }
  // eigenvector w = [e_i / (mu - lam_i); 1] / ||.||, then back to the pencil's basis
  double nn = 0.0;
  for (int i = tid; i < mc; i += blockDim.x) {
    const double t = e[i] / (mu - lamc[i]);
    nn += t * t;
  }
  block_sum2(nn, dummy, red);
  const double scale = 1.0 / sqrt(1.0 + nn);
  const double xu = scale / sq;
  for (int i = tid; i < mc; i += blockDim.x) d[i] = e[i] / (mu - lamc[i]) * scale - c[i] * xu;
  __syncthreads();
  for (int r = tid; r < mc; r += blockDim.x) {  // x_c = V t, V column-major
    double acc = 0.0;
    for (int i = 0; i < mc; ++i) acc += V[static_cast<long long>(i) * mc + r] * d[i];
    out_cp[r] = acc;
  }
  if (tid == 0) {
    out_lam[0] = mu;
    out_coef[0] = xu;
    *out_flag = 0;
  }
}

#define NR_DISPATCH(nr, kernel, grid, ...)                                      \
  do {                                                                          \
    switch (nr) {                                                               \
      case 1: kernel<1><<<grid, kB, 0, c.stream>>>(__VA_ARGS__); break;         \
      case 2: kernel<2><<<grid, kB, 0, c.stream>>>(__VA_ARGS__); break;         \
      case 4: kernel<4><<<grid, kB, 0, c.stream>>>(__VA_ARGS__); break;         \
      case 8: kernel<8><<<grid, kB, 0, c.stream>>>(__VA_ARGS__); break;         \
      default: throw ConfigError("unsupported right-hand-side batch width");    \
    }                                                                           \
    MLG_LAUNCH_CHECK();                                                         \
  } while (0)

PartDev part_dev(const Ctx& c, int level) {
  PartDev P{};
  const Partition& p = c.part;
  P.side = p.side;
  P.bw = p.nx0 / p.side;
  P.bh = p.ny0 / p.side;
  P.scale = (c.cfg.degree == 2 ? 2 : 1) << level;  // dof-grid points per coarse cell
  P.m = p.m;
  if (p.m > 256) throw ConfigError("more than 256 subdomains are not supported on this path");
  for (int j = 0; j < p.m; ++j) {
    P.inner[j] = p.inners[j];
    P.overlap[j] = p.overlaps[j];
  }
  for (int b = 0; b < p.side * p.side; ++b) P.blk2j[b] = static_cast<short>(p.blk2j[b]);
  return P;
}

struct Timer {
  cudaEvent_t e;
  explicit Timer(cudaStream_t s) {
    MLG_CUDA(cudaEventCreate(&e));
    MLG_CUDA(cudaEventRecord(e, s));
  }
  ~Timer() { cudaEventDestroy(e); }
  double since(const Timer& a) const {
    float ms = 0.f;
    MLG_CUDA(cudaEventSynchronize(e));
    MLG_CUDA(cudaEventElapsedTime(&ms, a.e, e));
    return ms * 1e-3;
  }
};

}  // namespace

int nr_for(int nev) {
  if (nev <= 1) return 1;
  if (nev <= 2) return 2;
  if (nev <= 4) return 4;
  if (nev <= 8) return 8;
  throw ConfigError("nev > 8 is not supported on the B200 path");
}

// ---------------------------------------------------------------------------
// Ctx
// ---------------------------------------------------------------------------

void validate_config(const Config& cfg) {  // corrector.cpp:76-88
  if (!(cfg.x_min < cfg.x_max) || !(cfg.y_min < cfg.y_max))
    throw ConfigError("domain rectangle must have positive side lengths");
  if (!(cfg.H > 0.0)) throw ConfigError("H must be positive");
  if (!(cfg.delta > 0.0)) throw ConfigError("delta must be positive");
  if (cfg.n_levels < 1) throw ConfigError("n_levels must be at least 1");
  if (cfg.degree != 1 && cfg.degree != 2) throw ConfigError("degree must be 1 or 2");
  if (cfg.nev < 1) throw ConfigError("nev must be at least 1");
  if (!(cfg.cg_tol > 0.0)) throw ConfigError("cg_tol must be positive");
  if (cfg.workers < 1) throw ConfigError("workers must be at least 1");
  if (cfg.example < 0 || cfg.example > 2)
    throw ConfigError("unknown example id (expected laplace, variable or reaction)");

}

static void build_partition(Ctx& c) {  // decomp.cpp:24-121 + corrector.cpp:117-121
  const Level& L0 = *c.levels[0];
  const double cell = L0.dx;
  const int delta_cells = std::max(1, static_cast<int>(std::ceil(c.cfg.delta / cell - 1e-9)));
  const double delta = delta_cells * cell;
  int m = c.cfg.m;  // the block grid; a hole drops the blocks it contains
  const int side = static_cast<int>(std::lround(std::sqrt(static_cast<double>(m))));
  if (m < 1 || side * side != m) throw ConfigError("subdomain count m must be a perfect square");
  const double hx = L0.dx, hy = L0.dy;
  if (std::abs(hx - hy) > 1e-12 * std::max(hx, hy))
    throw ConfigError("partition requires square coarse cells");
  if (L0.nx % side != 0 || L0.ny % side != 0)
    throw ConfigError("block grid does not align with the coarse mesh");
  if (!(delta > 0.0)) throw ConfigError("overlap width delta must be positive");
  const double ratio = delta / hx;
  const int dc = static_cast<int>(std::lround(ratio));
  if (dc < 1 || std::abs(ratio - dc) > 1e-9)
    throw ConfigError("overlap width delta must be a positive multiple of the coarse cell size");
  const int bw = L0.nx / side, bh = L0.ny / side;
  if (2 * dc >= bw || 2 * dc >= bh)
    throw ConfigError("overlap width leaves a degenerate inner region (2*delta >= block side)");
  Partition& p = c.part;
  p.side = side;
  p.delta_cells = dc;
  p.nx0 = L0.nx;
  p.ny0 = L0.ny;
  p.cell_h = hx;
  p.nt0 = static_cast<int>(L0.nt);
  p.blk2j.assign(static_cast<std::size_t>(side) * side, -1);
  // Domains with a corner hole (config 3, B200 extension): blocks inside the
  // hole are dropped ("subdomains on the grid clipped to the domain").
  const Hole& H0 = L0.hole;
  auto block_in_hole = [&](int col, int rb) {
    return H0.any() && col * bw >= H0.x0 && (col + 1) * bw <= H0.x1 && rb * bh >= H0.y0 &&
           (rb + 1) * bh <= H0.y1;
  };
  if (H0.any() && (H0.x0 % bw || H0.x1 % bw || H0.y0 % bh || H0.y1 % bh))
    throw ConfigError("hole does not align with the subdomain block grid");
  m = 0;
  for (int r = 0; r < side; ++r)
    for (int col = 0; col < side; ++col) {
      const int rb = side - 1 - r;
      if (block_in_hole(col, rb)) continue;
      p.blk2j[static_cast<std::size_t>(rb) * side + col] = m++;
      IRect d;
      d.x0 = col * bw;
      d.x1 = (col + 1) * bw;
      d.y1 = L0.ny - r * bh;
      d.y0 = d.y1 - bh;
      p.blocks.push_back(d);
      IRect om;
      om.x0 = std::max(0, d.x0 - dc);
      om.x1 = std::min(L0.nx, d.x1 + dc);
      om.y0 = std::max(0, d.y0 - dc);
      om.y1 = std::min(L0.ny, d.y1 + dc);
      p.overlaps.push_back(om);
      IRect g;  // decomp.cpp:73-80; with a hole its edges are shrunk from like
                // interior block sides (the strip then runs along them too),
                // which keeps G_j the closed form the strip CG kernels use
      g.x0 = (d.x0 == 0) ? 0 : d.x0 + dc;
      g.x1 = (d.x1 == L0.nx) ? L0.nx : d.x1 - dc;
      g.y0 = (d.y0 == 0) ? 0 : d.y0 + dc;
      g.y1 = (d.y1 == L0.ny) ? L0.ny : d.y1 - dc;
      p.inners.push_back(g);
    }
  p.m = m;
  // Level-0 element sets by integer centroid-in-open-rect (decomp.cpp:13-18,101-121);
  // element 2*cell is the lower triangle (centroid*3 = (3ix+2, 3iy+1)), 2*cell+1
  // the upper one ((3ix+1, 3iy+2)).
  p.block_elems.assign(m, {});
  p.overlap_elems.assign(m, {});
  p.inner_elems.assign(m, {});
  p.strip_elems.clear();
  auto open_in = [](const IRect& r, int cx3, int cy3) {
    return cx3 > 3 * r.x0 && cx3 < 3 * r.x1 && cy3 > 3 * r.y0 && cy3 < 3 * r.y1;
  };
  std::vector<int> cell_of;  // element pair -> lattice cell (holes skip removed cells)
  for (int cy = 0; cy < L0.ny; ++cy)
    for (int cx = 0; cx < L0.nx; ++cx)
      if (!H0.cell_in(cx, cy)) cell_of.push_back(cy * L0.nx + cx);
  for (int e = 0; e < 2 * static_cast<int>(cell_of.size()); ++e) {
    const int cell_id = cell_of[e / 2], ix = cell_id % L0.nx, iy = cell_id / L0.nx;
    const int cx3 = (e & 1) ? 3 * ix + 1 : 3 * ix + 2;
    const int cy3 = (e & 1) ? 3 * iy + 2 : 3 * iy + 1;
    bool in_inner = false;
    for (int j = 0; j < m; ++j) {
      if (open_in(p.blocks[j], cx3, cy3)) p.block_elems[j].push_back(e);
      if (open_in(p.overlaps[j], cx3, cy3)) p.overlap_elems[j].push_back(e);
      if (open_in(p.inners[j], cx3, cy3)) {
        p.inner_elems[j].push_back(e);
        in_inner = true;
      }
    }
    if (!in_inner) p.strip_elems.push_back(e);
  }
}

struct Workspace {
  CgBatch local, strip;
  CgBatchP2 local2, strip2;  // degree-2 batches (cg_p2.cu)
  DevBuf<double> corr;
  DevBuf<double> aug_ctmp, aug_uu_a, aug_uu_b, aug_cp, aug_c0;
  DevBuf<double> u, res, glued, au, bu, full, mfull, load, tmp_c0, tmp_c1, a_cu, b_cu;
  DevBuf<double> part, dots, dense_a, dense_b, eigw, work, sign;
  DevBuf<AbsMax> amax;
  DevBuf<int> info, keep;
  DevBuf<double> coef;
  std::vector<DevBuf<double>> chain;  // restriction chain buffers per level
};

Ctx::Ctx(const Config& config) : cfg(config) {
  validate_config(cfg);
  MLG_CUDA(cudaSetDevice(cfg.device));
  MLG_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  if (cusolverDnCreate(&solver) != CUSOLVER_STATUS_SUCCESS)
    throw CudaError("cusolverDnCreate failed");
  cusolverDnSetStream(solver, stream);
  ws = std::make_shared<Workspace>();
  build_level0(*this);
  build_partition(*this);
  assemble_level(*this, *levels[0]);
  sync();
}

Ctx::~Ctx() {
  ws.reset();
  levels.clear();
  for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
  if (input_ready) cudaEventDestroy(input_ready);
  if (solver) cusolverDnDestroy(solver);
  if (stream) cudaStreamDestroy(stream);
}

void Ctx::extend_to(int level) {
  if (level < 0) throw ConfigError("level must be nonnegative");
  while (max_level() < level) {
    auto next = std::make_unique<Level>();
    refine_level(*this, *levels.back(), *next);
    assemble_level(*this, *next);
    levels.push_back(std::move(next));
  }
  sync();
}

Workspace& W(Ctx& c) { return *static_cast<Workspace*>(c.ws.get()); }

void Ctx::ensure_coarse_dense() {
  if (coarse_ready) return;
  const Level& L0 = *levels[0];
  mc = static_cast<int>(L0.nint());
  coarse_a.alloc(static_cast<std::size_t>(mc) * mc);
  coarse_b.alloc(static_cast<std::size_t>(mc) * mc);
  coarse_bchol.alloc(static_cast<std::size_t>(mc) * mc);
  interior_dense(*this, L0, 0, coarse_a.get());
  interior_dense(*this, L0, 1, coarse_b.get());
  MLG_CUDA(cudaMemcpyAsync(coarse_bchol.get(), coarse_b.get(), sizeof(double) * mc * mc,
                           cudaMemcpyDeviceToDevice, stream));
  int lwork = 0;
  cusolverDnDpotrf_bufferSize(solver, CUBLAS_FILL_MODE_LOWER, mc, coarse_bchol.get(), mc, &lwork);
  Workspace& w = W(*this);
  w.work.ensure(std::max(lwork, 1));
  w.info.ensure(1);
  cusolverDnDpotrf(solver, CUBLAS_FILL_MODE_LOWER, mc, coarse_bchol.get(), mc, w.work.get(),
                   lwork, w.info.get());
  int info = 0;
  w.info.download(&info, 1, stream);
  sync();
  if (info != 0) throw SolverError("coarse mass block is not SPD");
  coarse_ready = true;
}

void Ctx::ensure_coarse_spectrum() {
  if (spectrum_ready) return;
  ensure_coarse_dense();
  Workspace& w = W(*this);
  coarse_lam.alloc(static_cast<std::size_t>(mc));
  coarse_vec.alloc(static_cast<std::size_t>(mc) * mc);
  DevBuf<double> b(static_cast<std::size_t>(mc) * mc);
  MLG_CUDA(cudaMemcpyAsync(coarse_vec.get(), coarse_a.get(), sizeof(double) * mc * mc,
                           cudaMemcpyDeviceToDevice, stream));
  MLG_CUDA(cudaMemcpyAsync(b.get(), coarse_b.get(), sizeof(double) * mc * mc,
                           cudaMemcpyDeviceToDevice, stream));
  int lwork = 0;
  cusolverDnDsygvd_bufferSize(solver, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR,
                              CUBLAS_FILL_MODE_LOWER, mc, coarse_vec.get(), mc, b.get(), mc,
                              coarse_lam.get(), &lwork);
  w.work.ensure(std::max(lwork, 1));
  w.info.ensure(1);
  if (cusolverDnDsygvd(solver, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR,
                       CUBLAS_FILL_MODE_LOWER, mc, coarse_vec.get(), mc, b.get(), mc,
                       coarse_lam.get(), w.work.get(), lwork,
                       w.info.get()) != CUSOLVER_STATUS_SUCCESS)
    throw CudaError("cusolverDnDsygvd failed to launch");
  int info = 0;
  w.info.download(&info, 1, stream);
  sync();
  if (info != 0) throw SolverError("coarse pencil eigensolve failed");
  spectrum_ready = true;
}

// ---------------------------------------------------------------------------
// building blocks
// ---------------------------------------------------------------------------

void prolong_chain(Ctx& c, int nr, const double* src, int from, int to, double* dst) {
  // dst must hold ndofs(to) * nr; intermediate levels use workspace.
  Workspace& w = W(c);
  if (from == to) {
    MLG_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * c.level(to).ndofs() * nr,
                             cudaMemcpyDeviceToDevice, c.stream));
    return;
  }
  const double* cur = src;
  DevBuf<double>* bufs[2] = {&w.tmp_c0, &w.tmp_c1};
  for (int k = from + 1; k <= to; ++k) {
    const Level& F = c.level(k);
    const Level& C = c.level(k - 1);
    double* out;
    if (k == to) {
      out = dst;
    } else {
      bufs[k & 1]->ensure(F.ndofs() * nr);
      out = bufs[k & 1]->get();
    }
    if (F.deg == 2) {
      prolong_p2(c, C, nr, cur, out);
    } else {
      NR_DISPATCH(nr, k_prolong, grid_for(F.ndofs(), kB), C.nx, F.nx, F.ny, F.hole, cur, out);
    }
    cur = out;
  }
}

// Restriction (P^T chain, corrector.cpp:165-170) from level `from` down to 0;
// returns a pointer to the level-0 full-lattice result (workspace owned).
const double* restrict_chain(Ctx& c, int nr, const double* src, int from, int slot) {
  Workspace& w = W(c);
  if (w.chain.size() < 2 * static_cast<std::size_t>(from + 1)) w.chain.resize(2 * (from + 1));
  const double* cur = src;
  for (int k = from; k > 0; --k) {
    const Level& F = c.level(k);
    const Level& C = c.level(k - 1);
    DevBuf<double>& out = w.chain[2 * (k - 1) + slot];
    out.ensure(C.ndofs() * nr);
    if (F.deg == 2)
      restrict_p2(c, C, nr, cur, out.get());
    else
      NR_DISPATCH(nr, k_restrict, grid_for(C.ndofs(), kB), F.nx, F.ny, C.nx, C.ny, F.hole, cur,
                  out.get());
    cur = out.get();
  }
  return cur;
}

// D = U^T V over a level's full lattice (nr x nr, row-major), to host.
std::vector<double> mdot(Ctx& c, int nr, const Level& L, const double* U, const double* V) {
  Workspace& w = W(c);
  const int nb = 296;
  w.part.ensure(static_cast<std::size_t>(nb) * nr * nr);
  w.dots.ensure(nr * nr);
  NR_DISPATCH(nr, k_mdot, nb, L.ndofs(), U, V, w.part.get());
  k_mdot_final<<<1, 64, 0, c.stream>>>(nb, nr * nr, w.part.get(), w.dots.get());
  MLG_LAUNCH_CHECK();
  std::vector<double> out(nr * nr);
  w.dots.download(out.data(), out.size(), c.stream);
  c.sync();
  return out;
}

// mdot into device memory (no host round trip): d_out[r*nr+s].
void mdot_dev(Ctx& c, int nr, const Level& L, const double* U, const double* V, double* d_out) {
  Workspace& w = W(c);
  const int nb = 296;
  w.part.ensure(static_cast<std::size_t>(nb) * nr * nr);
  NR_DISPATCH(nr, k_mdot, nb, L.ndofs(), U, V, w.part.get());
  k_mdot_final<<<1, 64, 0, c.stream>>>(nb, nr * nr, w.part.get(), d_out);
  MLG_LAUNCH_CHECK();
}

void fix_sign_lanes(Ctx& c, int nr, const Level& L, double* v) {
  Workspace& w = W(c);
  const int nb = 296;
  w.amax.ensure(static_cast<std::size_t>(nb) * nr);
  w.sign.ensure(nr);
  NR_DISPATCH(nr, k_absmax, nb, L.gx(), L.gy(), v, w.amax.get());
  switch (nr) {
    case 1: k_absmax_final<1><<<1, 32, 0, c.stream>>>(nb, w.amax.get(), v, w.sign.get()); break;
    case 2: k_absmax_final<2><<<1, 32, 0, c.stream>>>(nb, w.amax.get(), v, w.sign.get()); break;
    case 4: k_absmax_final<4><<<1, 32, 0, c.stream>>>(nb, w.amax.get(), v, w.sign.get()); break;
    case 8: k_absmax_final<8><<<1, 32, 0, c.stream>>>(nb, w.amax.get(), v, w.sign.get()); break;
  }
  MLG_LAUNCH_CHECK();
  NR_DISPATCH(nr, k_apply_sign, grid_for(L.ndofs(), kB), L.ndofs(), w.sign.get(), v);
}

// Reference fix_sign on a host dense vector (sparse.cpp:260-271).
static void fix_sign_host(std::vector<double>& v) {
  std::size_t idx = 0;
  double best = -1.0;
  for (std::size_t i = 0; i < v.size(); ++i) {
    const double a = std::abs(v[i]);
    if (a > best) {
      best = a;
      idx = i;
    }
  }
  if (!v.empty() && v[idx] < 0.0)
    for (double& x : v) x = -x;
}

struct DensePair {
  double lambda;
  std::vector<double> vec;
};

// order_ties (sparse.cpp:277-293)
static void order_ties(std::vector<DensePair>& pairs) {
  auto lex_less = [](const std::vector<double>& a, const std::vector<double>& b) {
    for (std::size_t i = 0; i < a.size(); ++i)
      if (a[i] != b[i]) return a[i] < b[i];
    return false;
  };
  std::size_t i = 0;
  while (i < pairs.size()) {
    std::size_t j = i + 1;
    const double tol = 1e-12 * std::max(1.0, std::abs(pairs[i].lambda));
    while (j < pairs.size() && std::abs(pairs[j].lambda - pairs[i].lambda) <= tol) ++j;
    std::sort(pairs.begin() + i, pairs.begin() + j, [&](const DensePair& a, const DensePair& b) {
      return lex_less(a.vec, b.vec);
    });
    i = j;
  }
}

// dense_gen_eigensolve (sparse.cpp:297-324) with cuSOLVER sygvd on device;
// a and b (device, column-major n x n) are overwritten.
std::vector<DensePair> dense_gen_eigensolve_dev(Ctx& c, int n, double* a, double* b, int nev) {
  if (nev < 1 || nev > n) throw ConfigError("dense_gen_eigensolve: invalid nev");
  Workspace& w = W(c);
  w.eigw.ensure(n);
  w.info.ensure(1);
  int lwork = 0;
  static const int variant = [] {  // A/B hook: 0 sygvd, 1 sygvdx (lowest nev), 2 sygvj
    const char* e = std::getenv("MLG_AUG");
    return e ? std::atoi(e) : 0;
  }();
  cusolverStatus_t st;
  if (variant == 1) {
    int h_meig = 0;
    cusolverDnDsygvdx_bufferSize(c.solver, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR,
                                 CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, n, a, n, b, n, 0.0,
                                 0.0, 1, nev, &h_meig, w.eigw.get(), &lwork);
    w.work.ensure(std::max(lwork, 1));
    st = cusolverDnDsygvdx(c.solver, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR,
                           CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, n, a, n, b, n, 0.0, 0.0,
                           1, nev, &h_meig, w.eigw.get(), w.work.get(), lwork, w.info.get());
  } else if (variant == 2) {
    syevjInfo_t params = nullptr;
    cusolverDnCreateSyevjInfo(&params);
    cusolverDnDsygvj_bufferSize(c.solver, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR,
                                CUBLAS_FILL_MODE_LOWER, n, a, n, b, n, w.eigw.get(), &lwork,
                                params);
    w.work.ensure(std::max(lwork, 1));
    st = cusolverDnDsygvj(c.solver, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR,
                          CUBLAS_FILL_MODE_LOWER, n, a, n, b, n, w.eigw.get(), w.work.get(),
                          lwork, w.info.get(), params);
    c.sync();
    cusolverDnDestroySyevjInfo(params);
  } else {
    cusolverDnDsygvd_bufferSize(c.solver, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR,
                                CUBLAS_FILL_MODE_LOWER, n, a, n, b, n, w.eigw.get(), &lwork);
    w.work.ensure(std::max(lwork, 1));
    st = cusolverDnDsygvd(c.solver, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR,
                          CUBLAS_FILL_MODE_LOWER, n, a, n, b, n, w.eigw.get(), w.work.get(),
                          lwork, w.info.get());
  }
  if (st != CUSOLVER_STATUS_SUCCESS) throw CudaError("cusolverDnDsygvd failed to launch");
  int info = 0;
  std::vector<double> lam(nev);
  std::vector<double> vecs(static_cast<std::size_t>(n) * nev);
  w.info.download(&info, 1, c.stream);
  w.eigw.download(lam.data(), nev, c.stream);
  MLG_CUDA(cudaMemcpyAsync(vecs.data(), a, sizeof(double) * n * nev, cudaMemcpyDeviceToHost,
                           c.stream));
  c.sync();
  if (info > n) throw SolverError("dense_gen_eigensolve: mass block is not SPD");
  if (info != 0) throw SolverError("dense_gen_eigensolve: eigensolver did not converge");
  std::vector<DensePair> pairs(nev);
  for (int i = 0; i < nev; ++i) {
    pairs[i].lambda = lam[i];
    pairs[i].vec.assign(vecs.begin() + static_cast<std::ptrdiff_t>(i) * n,
                        vecs.begin() + static_cast<std::ptrdiff_t>(i + 1) * n);
    fix_sign_host(pairs[i].vec);
  }
  order_ties(pairs);
  return pairs;
}

// ---------------------------------------------------------------------------
// Level-1 direct solve: solve_interior_eigenproblem (sparse.cpp:326-355)
// ---------------------------------------------------------------------------
// Degree dispatch of the operator kernels the step uses.
static void residual_any(Ctx& c, const Level& F, int nr, const double* u, const double* w,
                         const Lam& lam, double* out, const unsigned char* mask) {
  if (F.deg == 2) {
    residual_p2(c, F, nr, u, w, lam, out, mask);
    return;
  }
  NR_DISPATCH(nr, k_residual, grid_for(F.ndofs(), kB), F.imap(), F.stA.get(), F.stM.get(), u, w,
              lam, out, mask);
}

static void dual_any(Ctx& c, const Level& F, int nr, const double* x, double* ya, double* ym) {
  if (F.deg == 2) {
    if (ya) apply_p2(c, F, 0, nr, x, ya, true);
    if (ym) apply_p2(c, F, 1, nr, x, ym, true);
    return;
  }
  NR_DISPATCH(nr, k_dual, grid_for(F.ndofs(), kB), F.imap(), F.stA.get(), F.stM.get(), x, ya,
              ym);
}

std::vector<double> coarse_eigensolve(Ctx& c, int level, int nev, DevBuf<double>& u_out) {
  c.extend_to(level);
  Level& L = c.level(level);
  const long long dim = L.nint();
  if (dim > 5000)
    throw ConfigError("interior dimension " + std::to_string(dim) +
                      " exceeds the dense eigensolver threshold 5000");
  if (nev < 1 || nev > dim) throw ConfigError("nev out of range for the interior dimension");
  const int nr = nr_for(nev);
  Workspace& w = W(c);
  w.dense_a.ensure(dim * dim);
  w.dense_b.ensure(dim * dim);
  interior_dense(c, L, 0, w.dense_a.get());
  interior_dense(c, L, 1, w.dense_b.get());
  const auto pairs = dense_gen_eigensolve_dev(c, static_cast<int>(dim), w.dense_a.get(),
                                              w.dense_b.get(), nev);
  // coeffs -> device (interior order), expand, normalise by sqrt(v' B v), fix_sign.
  std::vector<double> host(static_cast<std::size_t>(dim) * nev);
  for (int i = 0; i < nev; ++i)
    std::copy(pairs[i].vec.begin(), pairs[i].vec.end(), host.begin() + static_cast<long>(i) * dim);
  DevBuf<double> tmp(host.size());
  tmp.upload(host.data(), host.size(), c.stream);
  u_out.ensure(L.ndofs() * nr);
  NR_DISPATCH(nr, k_interleave, grid_for(L.ndofs(), kB), L.imap(), nev, tmp.get(), 1,
              u_out.get());
  w.mfull.ensure(L.ndofs() * nr);
  dual_any(c, L, nr, u_out.get(), nullptr, w.mfull.get());
  const auto q = mdot(c, nr, L, u_out.get(), w.mfull.get());
  Lam s{};
  for (int r = 0; r < 8; ++r) s.v[r] = 1.0;
  for (int i = 0; i < nev; ++i) {
    const double qi = q[i * nr + i];
    if (qi <= 0.0) throw SolverError("eigenvector with nonpositive mass norm");
    s.v[i] = std::sqrt(qi);
  }
  NR_DISPATCH(nr, k_div_lanes, grid_for(L.ndofs(), kB), L.ndofs(), s, u_out.get());
  fix_sign_lanes(c, nr, L, u_out.get());
  std::vector<double> lam(nev);
  for (int i = 0; i < nev; ++i) lam[i] = pairs[i].lambda;
  c.sync();
  return lam;
}

// ---------------------------------------------------------------------------
// Step 1: batched local residual solves (corrector.cpp:198-214, 361-369)
// ---------------------------------------------------------------------------
static std::vector<CgSys> local_systems(const Ctx& c, int level) {
  const int S = (c.cfg.degree == 2 ? 2 : 1) << level;  // dof-grid points per coarse cell
  std::vector<CgSys> sys;
  for (int j = 0; j < c.part.m; ++j) {
    const IRect& o = c.part.overlaps[j];
    CgSys s{};
    s.x0 = o.x0 * S + 1;
    s.y0 = o.y0 * S + 1;
    s.w = (o.x1 - o.x0) * S - 1;
    s.h = (o.y1 - o.y0) * S - 1;
    sys.push_back(s);
  }
  return sys;
}

static std::string fmt_report(const SolveReport& r) {
  return "(" + std::to_string(r.iterations) + " iterations, residual " +
         std::to_string(r.final_residual) + ")";
}

// All local corrections e_{i,j} in one batched CG: system j*nev + i solves
// subdomain j for eigenvector i (lane i of the interleaved residual); e_{i,j}
// lives in its window-compact X (never expanded to N-length vectors).
int local_solves(Ctx& c, const Level& F, int nr, int nev, const double* res, double tol,
                 int maxit, std::vector<SolveReport>* reports, int only_j) {
  Workspace& w = W(c);
  const std::vector<CgSys> win = local_systems(c, F.level);
  std::vector<CgSys> sys;
  for (int j = 0; j < c.part.m; ++j) {
    if (only_j >= 0 && j != only_j) continue;
    for (int i = 0; i < nev; ++i) {
      CgSys s = win[j];
      s.rhs = i;
      sys.push_back(s);
    }
  }
  if (F.deg == 2) {
    w.local2.setup(c, F, std::move(sys), nullptr, res, nr);
    const CgResult r = w.local2.solve(c, tol);
    if (reports) *reports = r.reports;
    return r.iters_max;
  }
  w.local.setup(c, F, std::move(sys), nullptr, res, nr);
  const CgResult r = w.local.solve(c, tol, maxit);
  if (reports) *reports = r.reports;
  return r.iters_max;
}

void ensure_strip_mask(Ctx& c, Level& F) {
  if (!F.strip_mask.empty()) return;
  StripGeom& g = F.strip_geom;
  g.side = c.part.side;
  g.bw = c.part.nx0 / c.part.side;
  g.bh = c.part.ny0 / c.part.side;
  g.dc = c.part.delta_cells;
  g.nx0 = c.part.nx0;
  g.ny0 = c.part.ny0;
  g.scale = 1 << F.level;
  F.strip_mask.alloc(F.ndofs());
  k_strip_mask<<<grid_for(F.ndofs(), kB), kB, 0, c.stream>>>(F.imap(), part_dev(c, F.level),
                                                             F.strip_mask.get());
  MLG_LAUNCH_CHECK();
}

// Step 2 after gluing: strip solve on the interior window masked to the strip.
int strip_solve(Ctx& c, Level& F, int nr, int nev, const double* u, const Lam& lam,
                double* glued, double tol, int maxit, std::vector<SolveReport>* reports,
                bool* empty) {
  Workspace& w = W(c);
  ensure_strip_mask(c, F);
  bool any_strip = false;
  for (int j = 0; j < c.part.m && !any_strip; ++j) {
    const IRect& g = c.part.inners[j];
    any_strip = !(g.x0 == 0 && g.y0 == 0 && g.x1 == c.part.nx0 && g.y1 == c.part.ny0);
  }
  *empty = !any_strip;
  if (!any_strip) return 0;  // m = 1: G_1 is the whole domain, the strip is empty
  w.load.ensure(F.ndofs() * nr);
  residual_any(c, F, nr, u, glued, lam, w.load.get(), F.strip_mask.get());
  std::vector<CgSys> sys;
  for (int i = 0; i < nev; ++i) {
    CgSys s{};
    s.x0 = 1;
    s.y0 = 1;
    s.w = F.gx() - 1;
    s.h = F.gy() - 1;
    s.rhs = i;
    sys.push_back(s);
  }
  const long long rows = static_cast<long long>(F.gx() - 1) * (F.gy() - 1);
  if (F.deg == 2) {
    w.strip2.setup(c, F, std::move(sys), F.strip_mask.get(), w.load.get(), nr);
    const CgResult r = w.strip2.solve(c, tol);
    if (reports) *reports = r.reports;
    NR_DISPATCH(nr, k_strip_scatter, grid_for(rows, kB), F.gx(), nev, w.strip2.sys_dev(),
                F.strip_mask.get(), w.strip2.x(), glued);
    return r.iters_max;
  }
  w.strip.setup(c, F, std::move(sys), F.strip_mask.get(), w.load.get(), nr);
  const CgResult r = w.strip.solve(c, tol, maxit);
  if (reports) *reports = r.reports;
  NR_DISPATCH(nr, k_strip_scatter, grid_for(rows, kB), F.nx, nev, w.strip.sys_dev(),
              F.strip_mask.get(), w.strip.x(), glued);
  return r.iters_max;
}

// ---------------------------------------------------------------------------
// Step 3: augmented eigensolve (corrector.cpp:256-334)
// glued: full-lattice interleaved (nr lanes, first k_in used).  Output: sorted
// lambdas; u_out = normalised, sign-fixed coefficients (interleaved, nr lanes).
// ---------------------------------------------------------------------------
// Expansion of the augmented eigenvectors (corrector.cpp:318-332): prolong the
// coarse parts (device, [nev][mc]) through all levels, add coef x candidates,
// M-normalise, fix_sign, stable sort by lambda.
static std::vector<double> expand_augmented(Ctx& c, Level& F, int level, int nr, int nev, int k,
                                            const double* d_cp, const std::vector<double>& lam_in,
                                            const double* glued, DevBuf<double>& u_out) {
  const Level& L0 = c.level(0);
  Workspace& w = W(c);
  const long long nd = F.ndofs();
  DevBuf<double>& c0 = w.aug_c0;
  c0.ensure(L0.ndofs() * nr);
  NR_DISPATCH(nr, k_interleave, grid_for(L0.ndofs(), kB), L0.imap(), nev, d_cp, 1, c0.get());
  w.full.ensure(nd * nr);
  prolong_chain(c, nr, c0.get(), 0, level, w.full.get());
  NR_DISPATCH(nr, k_candidates, grid_for(nd, kB), nd, k, w.keep.get(), w.coef.get(), glued,
              w.full.get());
  w.mfull.ensure(nd * nr);
  dual_any(c, F, nr, w.full.get(), nullptr, w.mfull.get());
  const auto q = mdot(c, nr, F, w.full.get(), w.mfull.get());
  Lam s{};
  for (int r = 0; r < 8; ++r) s.v[r] = 1.0;
  for (int i = 0; i < nev; ++i) {
    const double qi = q[i * nr + i];
    if (qi <= 0.0) throw SolverError("augmented eigenvector with nonpositive mass norm");
    s.v[i] = std::sqrt(qi);
  }
  NR_DISPATCH(nr, k_div_lanes, grid_for(nd, kB), nd, s, w.full.get());
  fix_sign_lanes(c, nr, F, w.full.get());
  // stable sort by lambda (corrector.cpp:331-332)
  std::vector<int> order(nev);
  for (int i = 0; i < nev; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return lam_in[a] < lam_in[b]; });
  Lam perm{};
  for (int r = 0; r < 8; ++r) perm.v[r] = r < nev ? order[r] : r;
  u_out.ensure(nd * nr);
  NR_DISPATCH(nr, k_permute_lanes, grid_for(nd, kB), nd, perm, w.full.get(), u_out.get());
  std::vector<double> lam(nev);
  for (int i = 0; i < nev; ++i) lam[i] = lam_in[order[i]];
  c.sync();
  return lam;
}

static bool arrow_enabled() {  // A/B hook: MLG_AUG=0/1/2 forces the dense cuSOLVER path
  static const bool on = [] {
    const char* e = std::getenv("MLG_AUG");
    return e == nullptr || e[0] == '\0' || std::strcmp(e, "arrow") == 0;
  }();
  return on;
}

std::vector<double> augmented(Ctx& c, int level, int nr, int k_in, const double* glued, int nev,
                              DevBuf<double>& u_out) {
  Level& F = c.level(level);
  const Level& L0 = c.level(0);
  c.ensure_coarse_dense();
  const int mc = c.mc;
  Workspace& w = W(c);
  const long long nd = F.ndofs();
  w.au.ensure(nd * nr);
  w.bu.ensure(nd * nr);
  dual_any(c, F, nr, glued, w.au.get(), w.bu.get());
  const double* a0 = restrict_chain(c, nr, w.au.get(), level, 0);
  const double* b0 = restrict_chain(c, nr, w.bu.get(), level, 1);
  w.a_cu.ensure(static_cast<std::size_t>(mc) * nr);
  w.b_cu.ensure(static_cast<std::size_t>(mc) * nr);
  NR_DISPATCH(nr, k_gather_coarse, grid_for(mc, kB), L0.imap(), a0, w.a_cu.get());
  NR_DISPATCH(nr, k_gather_coarse, grid_for(mc, kB), L0.imap(), b0, w.b_cu.get());
  w.coef.ensure(64);
  w.keep.ensure(8);

  if (nev == 1 && k_in == 1 && nr == 1 && arrow_enabled()) {
    c.ensure_coarse_spectrum();
    w.dots.ensure(4);
    mdot_dev(c, 1, F, glued, w.au.get(), w.dots.get());
    mdot_dev(c, 1, F, glued, w.bu.get(), w.dots.get() + 1);
    w.aug_ctmp.ensure(static_cast<std::size_t>(3) * mc);
    w.aug_cp.ensure(static_cast<std::size_t>(mc));
    w.aug_uu_a.ensure(2);
    w.info.ensure(1);
    MLG_CUDA(cudaMemsetAsync(w.coef.get(), 0, 64 * sizeof(double), c.stream));
    const int zero = 0;
    w.keep.upload(&zero, 1, c.stream);
    k_aug_arrow<<<1, kArrowThreads, 0, c.stream>>>(
        mc, c.coarse_lam.get(), c.coarse_vec.get(), w.a_cu.get(), w.b_cu.get(), w.dots.get(),
        w.dots.get() + 1, w.aug_ctmp.get(), w.aug_uu_a.get(), w.aug_cp.get(), w.coef.get(),
        w.info.get());
    MLG_LAUNCH_CHECK();
    double mu = 0.0;
    int flag = 0;
    w.aug_uu_a.download(&mu, 1, c.stream);
    w.info.download(&flag, 1, c.stream);
    c.sync();
    if (flag != 1)  // 0: candidate kept, 2: dropped (coef 0); 1: deflated -> dense path
      return expand_augmented(c, F, level, nr, 1, 1, w.aug_cp.get(), {mu}, glued, u_out);
  }

  const auto a_uu = mdot(c, nr, F, glued, w.au.get());
  const auto b_uu = mdot(c, nr, F, glued, w.bu.get());
  // Dependence drop through the cached coarse Cholesky (corrector.cpp:285-292).
  std::vector<double> bcu(static_cast<std::size_t>(mc) * nr), csol(bcu.size());
  DevBuf<double>& ctmp = w.aug_ctmp;
  ctmp.ensure(bcu.size());
  MLG_CUDA(cudaMemcpyAsync(ctmp.get(), w.b_cu.get(), sizeof(double) * bcu.size(),
                           cudaMemcpyDeviceToDevice, c.stream));
  cusolverDnDpotrs(c.solver, CUBLAS_FILL_MODE_LOWER, mc, k_in, c.coarse_bchol.get(), mc,
                   ctmp.get(), mc, w.info.get());
  w.b_cu.download(bcu.data(), bcu.size(), c.stream);
  ctmp.download(csol.data(), csol.size(), c.stream);
  c.sync();
  std::vector<int> keep;
  for (int l = 0; l < k_in; ++l) {
    double dotv = 0.0;
    for (int i = 0; i < mc; ++i) dotv += bcu[l * mc + i] * csol[l * mc + i];
    const double res2 = b_uu[l * nr + l] - dotv;
    if (std::sqrt(std::max(res2, 0.0)) >= 1e-10) keep.push_back(l);
  }
  const int k = static_cast<int>(keep.size());
  const int dim = mc + k;
  if (nev < 1 || nev > dim)
    throw ConfigError("augmented eigenproblem smaller than the requested nev");

  w.keep.upload(keep.data(), keep.size(), c.stream);
  DevBuf<double>& uu_a = w.aug_uu_a;
  DevBuf<double>& uu_b = w.aug_uu_b;
  uu_a.ensure(nr * nr);
  uu_b.ensure(nr * nr);
  uu_a.upload(a_uu.data(), a_uu.size(), c.stream);
  uu_b.upload(b_uu.data(), b_uu.size(), c.stream);
  w.dense_a.ensure(static_cast<std::size_t>(dim) * dim);
  w.dense_b.ensure(static_cast<std::size_t>(dim) * dim);
  const long long nn = static_cast<long long>(dim) * dim;
  k_build_aug<<<grid_for(nn, kB), kB, 0, c.stream>>>(mc, k, w.keep.get(), c.coarse_a.get(),
                                                     w.a_cu.get(), uu_a.get(), nr,
                                                     w.dense_a.get());
  k_build_aug<<<grid_for(nn, kB), kB, 0, c.stream>>>(mc, k, w.keep.get(), c.coarse_b.get(),
                                                     w.b_cu.get(), uu_b.get(), nr,
                                                     w.dense_b.get());
  MLG_LAUNCH_CHECK();
  // The reference's explicit LLT check on b_aug happens inside sygvd (info > n).
  const auto pairs = dense_gen_eigensolve_dev(c, dim, w.dense_a.get(), w.dense_b.get(), nev);

  std::vector<double> coarse_part(static_cast<std::size_t>(mc) * nev);
  std::vector<double> coef(8 * 8, 0.0);
  std::vector<double> lam(nev);
  for (int i = 0; i < nev; ++i) {
    std::copy(pairs[i].vec.begin(), pairs[i].vec.begin() + mc,
              coarse_part.begin() + static_cast<long>(i) * mc);
    for (int l = 0; l < k; ++l) coef[i * 8 + l] = pairs[i].vec[mc + l];
    lam[i] = pairs[i].lambda;
  }
  DevBuf<double>& cp = w.aug_cp;
  cp.ensure(coarse_part.size());
  cp.upload(coarse_part.data(), coarse_part.size(), c.stream);
  w.coef.upload(coef.data(), 64, c.stream);
  return expand_augmented(c, F, level, nr, nev, k, cp.get(), lam, glued, u_out);
}

// ---------------------------------------------------------------------------
// one_correction_step (corrector.cpp:336-412)
// ---------------------------------------------------------------------------
StepResult correction_step(Ctx& c, int from, int to, int nev, const double* lam_in,
                           const double* u_in, DevBuf<double>& u_out) {
  if (nev < 1) throw ConfigError("correction step needs at least one eigenpair");
  if (to != from + 1 && to != from)
    throw ConfigError("correction step targets the next level (or the same level)");
  const auto t_build0 = std::chrono::steady_clock::now();
  c.extend_to(to);
  Level& F = c.level(to);
  ensure_strip_mask(c, F);
  c.sync();
  StepResult out;
  out.times.build_s =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t_build0).count();
  const int nr = nr_for(nev);
  Workspace& w = W(c);
  const long long nd = F.ndofs();
  w.u.ensure(nd * nr);
  prolong_chain(c, nr, u_in, from, to, w.u.get());
  Lam lam{};
  for (int i = 0; i < nev; ++i) lam.v[i] = lam_in[i];

  Timer t0(c.stream);
  w.res.ensure(nd * nr);
  residual_any(c, F, nr, w.u.get(), w.u.get(), lam, w.res.get(), nullptr);
  std::vector<SolveReport> lrep;
  out.times.local_iters_max =
      local_solves(c, F, nr, nev, w.res.get(), c.cfg.cg_tol, 0, &lrep);
  for (int i = 0; i < nev; ++i)  // task order i*m + j (parallel_tasks with one worker)
    for (int j = 0; j < c.part.m; ++j) {
      const SolveReport& r = lrep[static_cast<std::size_t>(j) * nev + i];
      if (!r.converged)
        throw SolverError("subdomain " + std::to_string(j + 1) + " solve did not converge " +
                          fmt_report(r));
    }
  Timer t1(c.stream);

  w.glued.ensure(nd * nr);
  NR_DISPATCH(nr, k_glue_cg, grid_for(nd, kB), F.imap(), part_dev(c, to), nev,
              F.deg == 2 ? w.local2.sys_dev() : w.local.sys_dev(),
              F.deg == 2 ? w.local2.x() : w.local.x(), w.u.get(), w.glued.get());
  std::vector<SolveReport> srep;
  bool empty = false;
  out.times.strip_iters_max =
      strip_solve(c, F, nr, nev, w.u.get(), lam, w.glued.get(), c.cfg.cg_tol, 0, &srep,
                  &empty);
  for (int i = 0; i < nev && !empty; ++i)
    if (!srep[i].converged)
      throw SolverError("strip solve did not converge " + fmt_report(srep[i]));
  Timer t2(c.stream);

  out.lambdas = augmented(c, to, nr, nev, w.glued.get(), nev, u_out);
  Timer t3(c.stream);

  // matching diagnostic (corrector.cpp:383-399)
  w.mfull.ensure(nd * nr);
  dual_any(c, F, nr, u_out.get(), nullptr, w.mfull.get());
  const auto m = mdot(c, nr, F, w.u.get(), w.mfull.get());
  out.matched = true;
  for (int i2 = 0; i2 < nev; ++i2) {
    int best = 0;
    double best_val = -1.0;
    for (int i = 0; i < nev; ++i) {
      const double v = std::abs(m[i * nr + i2]);
      if (v > best_val) {
        best_val = v;
        best = i;
      }
    }
    if (best != i2) out.matched = false;
  }
  out.times.local_s = t1.since(t0);
  out.times.iface_s = t2.since(t1);
  out.times.aug_s = t3.since(t2);
  return out;
}

// ---------------------------------------------------------------------------
// Hooks for the C-ABI's sub-step and kernel-level entry points.
// ---------------------------------------------------------------------------
const CgBatch& local_batch(Ctx& c) { return W(c).local; }

void interleave(Ctx& c, const Level& L, int nr, int k_in, const double* src, int interior_src,
                double* dst) {
  NR_DISPATCH(nr, k_interleave, grid_for(L.ndofs(), kB), L.imap(), k_in, src, interior_src,
              dst);
}

void deinterleave(Ctx& c, const Level& L, int nr, int k_out, const int* perm, const double* src,
                  int interior_dst, double* dst) {
  NR_DISPATCH(nr, k_deinterleave, grid_for(L.ndofs(), kB), L.imap(), k_out, perm, src,
              interior_dst, dst);
}

void spmv_full(Ctx& c, const Level& L, int form, const double* x, double* y) {
  if (L.deg == 2) {
    apply_p2(c, L, form, 1, x, y, false);
    return;
  }
  k_full_spmv<<<grid_for(L.ndofs(), kB), kB, 0, c.stream>>>(
      L.nx, L.ny, form == 0 ? L.stA.get() : L.stM.get(), x, y);
  MLG_LAUNCH_CHECK();
}

void spmv_interior(Ctx& c, const Level& L, const double* x, double* y) {
  k_interior_spmv<<<grid_for(L.nint(), kB), kB, 0, c.stream>>>(L.nx, L.ny, L.stA.get(), x, y);
  MLG_LAUNCH_CHECK();
}

void restrict_levels(Ctx& c, int nr, const double* src, int from, int to, double* dst) {
  Workspace& w = W(c);
  const double* cur = src;
  DevBuf<double>* bufs[2] = {&w.tmp_c0, &w.tmp_c1};
  if (from == to) {
    MLG_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * c.level(to).ndofs() * nr,
                             cudaMemcpyDeviceToDevice, c.stream));
    return;
  }
  for (int k = from; k > to; --k) {
    const Level& F = c.level(k);
    const Level& C = c.level(k - 1);
    double* out;
    if (k - 1 == to) {
      out = dst;
    } else {
      bufs[k & 1]->ensure(C.ndofs() * nr);
      out = bufs[k & 1]->get();
    }
    if (F.deg == 2) {
      restrict_p2(c, C, nr, cur, out);
    } else {
      NR_DISPATCH(nr, k_restrict, grid_for(C.ndofs(), kB), F.nx, F.ny, C.nx, C.ny, F.hole, cur,
                  out);
    }
    cur = out;
  }
}

void glue_full(Ctx& c, int level, const double* corr, const double* u, double* glued) {
  const Level& F = c.level(level);
  k_glue_full<<<grid_for(F.ndofs(), kB), kB, 0, c.stream>>>(F.imap(), part_dev(c, level),
                                                           F.ndofs(), corr, u, glued);
  MLG_LAUNCH_CHECK();
}

void residual(Ctx& c, const Level& F, int nr, const double* u, const double* lam, double* out) {
  Lam l{};
  for (int r = 0; r < nr; ++r) l.v[r] = lam[r];
  residual_any(c, F, nr, u, u, l, out, nullptr);
}

LocalView local_view(Ctx& c) {
  Workspace& w = W(c);
  if (c.cfg.degree == 2) return {w.local2.systems(), w.local2.x(), w.local2.sys_dev()};
  return {w.local.systems(), w.local.x(), w.local.sys_dev()};
}

}  // namespace mlg

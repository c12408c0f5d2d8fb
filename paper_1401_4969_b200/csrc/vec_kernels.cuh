// Level-wide vector kernels of the correction step (full lattice, NR
// right-hand sides interleaved).  Each one restates a reference expression
// with the same per-element operation order so values match bitwise where the
// reference's own result is order-defined.
#pragma once

#include "stencil.cuh"

namespace mlg {

struct Lam {
  double v[8];
};

// Full-space row product (SparseSymMatrix::multiply, sparse.cpp:69-76): all
// 7-point neighbours inside [0,nx]x[0,ny] take part, boundary entries of the
// vector are whatever it holds (zero for our interior vectors).
template <int NR>
__device__ __forceinline__ void full_row(const Stencil* st, const double* x, int ix, int iy,
                                         int nx, int ny, double (&y)[NR]) {
  const long long s = nx + 1;
  const long long g = static_cast<long long>(iy) * s + ix;
  double t[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) y[r] = 0.0;
  auto acc = [&](long long gj, double a) {
    ldv<NR>(x + gj * NR, t);
#pragma unroll
    for (int r = 0; r < NR; ++r) y[r] = xadd(y[r], xmul(a, t[r]));
  };
  if (iy > 0 && ix > 0) acc(g - s - 1, st[g - s - 1].ne);
  if (iy > 0) acc(g - s, st[g - s].n);
  if (ix > 0) acc(g - 1, st[g - 1].e);
  const Stencil c = st[g];
  acc(g, c.c);
  if (ix < nx) acc(g + 1, c.e);
  if (iy < ny) acc(g + s, c.n);
  if (iy < ny && ix < nx) acc(g + s + 1, c.ne);
}

}  // namespace mlg

// Device helpers shared by the stencil kernels: rhs-interleaved vector
// loads/stores, deterministic block reductions, and the window/mask-restricted
// 7-point row product in the reference's CSR column order (SW,S,W,C,E,N,NE),
// each term rounded separately like SparseSymMatrix::multiply (sparse.cpp:69-76).
#pragma once

#include "cg.cuh"

namespace mlg {

template <int NR>
__device__ __forceinline__ void ldv(const double* p, double (&o)[NR]) {
  if constexpr (NR == 1) {
    o[0] = *p;
  } else {
    const double2* q = reinterpret_cast<const double2*>(p);
#pragma unroll
    for (int k = 0; k < NR / 2; ++k) {
      const double2 t = q[k];
      o[2 * k] = t.x;
      o[2 * k + 1] = t.y;
    }
  }
}

template <int NR>
__device__ __forceinline__ void stv(double* p, const double (&o)[NR]) {
  if constexpr (NR == 1) {
    *p = o[0];
  } else {
    double2* q = reinterpret_cast<double2*>(p);
#pragma unroll
    for (int k = 0; k < NR / 2; ++k) q[k] = make_double2(o[2 * k], o[2 * k + 1]);
  }
}

template <int K, int kBlock = 256>
__device__ __forceinline__ void block_reduce_store(double (&acc)[K], double* out) {
  __shared__ double red[kBlock / 32][K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double v = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    acc[k] = v;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) red[warp][k] = acc[k];
  __syncthreads();
  if (threadIdx.x < K) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kBlock / 32; ++w) s += red[w][threadIdx.x];
    out[threadIdx.x] = s;
  }
}

// Neighbourhood of window row i: presence flags (window + mask) and the
// global dof ids.  Order of the 7 slots = ascending column order of the
// reference's CSR row: SW, S, W, C, E, N, NE.
struct Nbhd {
  long long g;
  int lx, ly;
  bool sw, s, w, e, n, ne;
};

__device__ __forceinline__ bool decode(const CgSys& S, int i, int nxp1,
                                       const unsigned char* mask, Nbhd* h) {
  h->lx = i % S.w;
  h->ly = i / S.w;
  h->g = static_cast<long long>(S.y0 + h->ly) * nxp1 + (S.x0 + h->lx);
  if (mask && !mask[h->g]) return false;
  const bool W = h->lx > 0, E = h->lx < S.w - 1, So = h->ly > 0, N = h->ly < S.h - 1;
  h->w = W;
  h->e = E;
  h->s = So;
  h->n = N;
  h->sw = W && So;
  h->ne = E && N;
  if (mask) {
    const long long g = h->g;
    h->w = h->w && mask[g - 1];
    h->e = h->e && mask[g + 1];
    h->s = h->s && mask[g - nxp1];
    h->n = h->n && mask[g + nxp1];
    h->sw = h->sw && mask[g - nxp1 - 1];
    h->ne = h->ne && mask[g + nxp1 + 1];
  }
  return true;
}

// y = A_window v  with v produced per neighbour by `val(local_row, dof, out)`.
template <int NR, class F>
__device__ __forceinline__ void stencil_apply(const Nbhd& h, int i, int w, int nxp1,
                                              const Stencil* st, F&& val, double (&self)[NR],
                                              double (&y)[NR]) {
  double t[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) y[r] = 0.0;
  const long long g = h.g;
  if (h.sw) {
    val(i - w - 1, g - nxp1 - 1, t);
    const double a = st[g - nxp1 - 1].ne;
#pragma unroll
    for (int r = 0; r < NR; ++r) y[r] = xadd(y[r], xmul(a, t[r]));
  }
  if (h.s) {
    val(i - w, g - nxp1, t);
    const double a = st[g - nxp1].n;
#pragma unroll
    for (int r = 0; r < NR; ++r) y[r] = xadd(y[r], xmul(a, t[r]));
  }
  if (h.w) {
    val(i - 1, g - 1, t);
    const double a = st[g - 1].e;
#pragma unroll
    for (int r = 0; r < NR; ++r) y[r] = xadd(y[r], xmul(a, t[r]));
  }
  const Stencil sc = st[g];
  val(i, g, self);
#pragma unroll
  for (int r = 0; r < NR; ++r) y[r] = xadd(y[r], xmul(sc.c, self[r]));
  if (h.e) {
    val(i + 1, g + 1, t);
#pragma unroll
    for (int r = 0; r < NR; ++r) y[r] = xadd(y[r], xmul(sc.e, t[r]));
  }
  if (h.n) {
    val(i + w, g + nxp1, t);
#pragma unroll
    for (int r = 0; r < NR; ++r) y[r] = xadd(y[r], xmul(sc.n, t[r]));
  }
  if (h.ne) {
    val(i + w + 1, g + nxp1 + 1, t);
#pragma unroll
    for (int r = 0; r < NR; ++r) y[r] = xadd(y[r], xmul(sc.ne, t[r]));
  }
}


}  // namespace mlg

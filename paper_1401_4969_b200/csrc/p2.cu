// P2 (degree 2) spaces on the device: level build and operators, bit-exact
// with the reference.
//
//   build_space(mesh, 2)        fespace.cpp:230-312  dofs = vertices + edge
//                               midpoints, numbered by sorted half-lattice key
//   local_matrix / default_rule fespace.cpp:185-222  degree-6 rule (12 points)
//                               for every P2 form, P2 shape values/gradients
//                               fespace.cpp:128-161
//   assemble_form               fespace.cpp:314-341 + from_upper_triplets
//                               sparse.cpp:24-61 (sums in ascending element id)
//   prolongation_matrix         fespace.cpp:355-400 (nodal interpolation)
//
// B200 design.  On the structured lattice every half-lattice point is a P2
// dof (vertices at even/even, axis-edge midpoints at odd/even and even/odd,
// diagonal midpoints at odd/odd), so the reference's sorted-key numbering is
// dof = Y * (2nx+1) + X in closed form.  A dof couples with the dofs of the
// <= 6 triangles around it, all inside the 5x5 half-lattice block centred on
// it: each level stores, per dof, the 25 slot values of A and M (row-major
// offsets dy, dx = -2..2, i.e. ascending column order) and a 25-bit mask of
// the structurally present couplings.  One thread per dof recomputes the
// element matrices of its triangles with the reference's unfused operation
// sequence and sums each slot in ascending element id, so every value --
// including the mirrored lower triangle -- is bitwise the reference's.
#include <cub/device/device_scan.cuh>

#include <algorithm>

#include "p2.cuh"
#include "stencil.cuh"
#include "vec_kernels.cuh"

namespace mlg {
namespace {

constexpr int kBlock = 256;

__constant__ double kQ6p2[12][4];  // make_degree6 (fespace.cpp:49-75)

struct P2Geom {
  int nx, ny;  // cells
  double x0, y0, dx, dy;
  const unsigned* geo;
  int example;
};

__device__ __forceinline__ int upk6(int i, int j) {  // packed upper 6x6, i <= j
  return i * 6 - (i * (i - 1)) / 2 + (j - i);
}

// Element matrices of one triangle (vertices in element order), degree 2,
// upper packed (21 entries): local_matrix (fespace.cpp:185-217) for the
// Laplace (A = I, phi = 1) or the variable field.
__device__ void elem_p2(const double vx[3], const double vy[3], int example, double a[21],
                        double m[21]) {
  const double area2 = xsub(xmul(xsub(vx[1], vx[0]), xsub(vy[2], vy[0])),
                            xmul(xsub(vx[2], vx[0]), xsub(vy[1], vy[0])));
  const double area = xmul(0.5, area2);
  double gl[3][2];
  gl[0][0] = xdiv(xsub(vy[1], vy[2]), area2);
  gl[0][1] = xdiv(xsub(vx[2], vx[1]), area2);
  gl[1][0] = xdiv(xsub(vy[2], vy[0]), area2);
  gl[1][1] = xdiv(xsub(vx[0], vx[2]), area2);
  gl[2][0] = xdiv(xsub(vy[0], vy[1]), area2);
  gl[2][1] = xdiv(xsub(vx[1], vx[0]), area2);
  for (int k = 0; k < 21; ++k) a[k] = m[k] = 0.0;
  for (int q = 0; q < 12; ++q) {
    const double l[3] = {kQ6p2[q][0], kQ6p2[q][1], kQ6p2[q][2]};
    const double w = xmul(kQ6p2[q][3], area);
    const double x = xadd(xadd(xmul(l[0], vx[0]), xmul(l[1], vx[1])), xmul(l[2], vx[2]));
    const double y = xadd(xadd(xmul(l[0], vy[0]), xmul(l[1], vy[1])), xmul(l[2], vy[2]));
    double d0 = 1.0, d1 = 0.0, d2 = 1.0, phi = 1.0;  // CoefficientField::laplace
    if (example == 1) {  // CoefficientField::variable (fespace.cpp:114-123)
      d0 = exp(xadd(1.0, xmul(x, x)));
      d1 = exp(xmul(x, y));
      d2 = exp(xadd(1.0, xmul(y, y)));
      phi = xmul(xadd(1.0, xmul(x, x)), xadd(1.0, xmul(y, y)));
    }
    // shape_gradients / shape_values, degree 2 (fespace.cpp:128-161)
    double g[6][2], v[6];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double f = xsub(xmul(4.0, l[i]), 1.0);
      g[i][0] = xmul(f, gl[i][0]);
      g[i][1] = xmul(f, gl[i][1]);
      v[i] = xmul(l[i], xsub(xmul(2.0, l[i]), 1.0));
    }
    const int ea[3] = {0, 1, 2}, eb[3] = {1, 2, 0};
#pragma unroll
    for (int e = 0; e < 3; ++e) {
      g[3 + e][0] = xmul(4.0, xadd(xmul(l[ea[e]], gl[eb[e]][0]), xmul(l[eb[e]], gl[ea[e]][0])));
      g[3 + e][1] = xmul(4.0, xadd(xmul(l[ea[e]], gl[eb[e]][1]), xmul(l[eb[e]], gl[ea[e]][1])));
      v[3 + e] = xmul(xmul(4.0, l[ea[e]]), l[eb[e]]);
    }
    const double wphi = xmul(w, phi);
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      const double agx = xadd(xmul(d0, g[i][0]), xmul(d1, g[i][1]));
      const double agy = xadd(xmul(d1, g[i][0]), xmul(d2, g[i][1]));
#pragma unroll
      for (int j = i; j < 6; ++j) {
        const int k = upk6(i, j);
        a[k] = xadd(a[k], xmul(w, xadd(xmul(agx, g[j][0]), xmul(agy, g[j][1]))));
        m[k] = xadd(m[k], xmul(xmul(wphi, v[i]), v[j]));
      }
    }
  }
}

// Half-lattice offsets (in cell units x2) of canonical vertex k of the L/U
// triangle: L (0,0),(2,0),(2,2)  U (0,0),(2,2),(0,2).
__device__ __forceinline__ void canon_half(int upper, int k, int* x, int* y) {
  if (k == 0) {
    *x = 0;
    *y = 0;
  } else if (k == 1) {
    *x = 2;
    *y = upper ? 2 : 0;
  } else {
    *x = upper ? 0 : 2;
    *y = 2;
  }
}

// The 6 dofs (half-lattice points relative to the cell origin) of triangle
// (upper, rot) in element order: v0, v1, v2, m01, m12, m20.
__device__ __forceinline__ void tri_dofs(int upper, int rot, int px[6], int py[6]) {
#pragma unroll
  for (int j = 0; j < 3; ++j) canon_half(upper, (rot + j) % 3, &px[j], &py[j]);
  px[3] = (px[0] + px[1]) / 2;
  py[3] = (py[0] + py[1]) / 2;
  px[4] = (px[1] + px[2]) / 2;
  py[4] = (py[1] + py[2]) / 2;
  px[5] = (px[2] + px[0]) / 2;
  py[5] = (py[2] + py[0]) / 2;
}

struct P2Contrib {
  unsigned e;
  double a, m;
};

// One thread per dof (X, Y) of the half lattice: all slots of its row.
__global__ void __launch_bounds__(kBlock) k_p2_assemble(P2Geom G, double* A, double* M,
                                                        unsigned* pat) {
  const int gx = 2 * G.nx, gy = 2 * G.ny;
  const long long d = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (d >= static_cast<long long>(gx + 1) * (gy + 1)) return;
  const int X = static_cast<int>(d % (gx + 1)), Y = static_cast<int>(d / (gx + 1));
  // contributions per slot: at most 6 triangles touch a row, each adds one
  // value per slot it covers
  P2Contrib cs[25][6];
  unsigned char n[25];
#pragma unroll
  for (int s = 0; s < 25; ++s) n[s] = 0;
  const int cxa = (X - 1) >> 1, cxb = X >> 1, cya = (Y - 1) >> 1, cyb = Y >> 1;
  for (int cy = cya; cy <= cyb; ++cy)
    for (int cx = cxa; cx <= cxb; ++cx) {
      if (cx < 0 || cy < 0 || cx >= G.nx || cy >= G.ny) continue;
      for (int upper = 0; upper < 2; ++upper) {
        const unsigned code = G.geo[2 * (static_cast<long long>(cy) * G.nx + cx) + upper];
        if (code == 0xFFFFFFFFu) continue;
        const int rot = static_cast<int>(code & 3u);
        int px[6], py[6];
        tri_dofs(upper, rot, px, py);
        int me = -1;
        for (int i = 0; i < 6; ++i)
          if (2 * cx + px[i] == X && 2 * cy + py[i] == Y) me = i;
        if (me < 0) continue;
        double vx[3], vy[3];
        for (int j = 0; j < 3; ++j) {
          vx[j] = lattice_coord(G.x0, cx + px[j] / 2, G.dx);
          vy[j] = lattice_coord(G.y0, cy + py[j] / 2, G.dy);
        }
        double a[21], m[21];
        elem_p2(vx, vy, G.example, a, m);
        for (int j = 0; j < 6; ++j) {
          const int s = (2 * cy + py[j] - Y + 2) * 5 + (2 * cx + px[j] - X + 2);
          const int k = upk6(min(me, j), max(me, j));
          cs[s][n[s]] = P2Contrib{code >> 2, a[k], m[k]};
          ++n[s];
        }
      }
    }
  unsigned mask = 0;
  for (int s = 0; s < 25; ++s) {
    // ascending element id, summed from 0.0 (sparse.cpp:36-46)
    for (int i = 1; i < n[s]; ++i) {
      const P2Contrib t = cs[s][i];
      int k = i;
      while (k > 0 && cs[s][k - 1].e > t.e) {
        cs[s][k] = cs[s][k - 1];
        --k;
      }
      cs[s][k] = t;
    }
    double sa = 0.0, sm = 0.0;
    for (int i = 0; i < n[s]; ++i) {
      sa = xadd(sa, cs[s][i].a);
      sm = xadd(sm, cs[s][i].m);
    }
    A[d * 25 + s] = sa;
    M[d * 25 + s] = sm;
    if (n[s]) mask |= 1u << s;
  }
  pat[d] = mask;
}

__device__ __forceinline__ long long slot_col(long long d, int s, int gx) {
  return d + static_cast<long long>(s / 5 - 2) * (gx + 1) + (s % 5 - 2);
}

__global__ void k_p2_count(long long nd, const unsigned* pat, int* cnt) {
  const long long d = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (d > nd) return;
  cnt[d] = d == nd ? 0 : __popc(pat[d]);
}

__global__ void k_p2_export(long long nd, int gx, const double* st, const unsigned* pat,
                            const int* rp, int* cols, double* vals) {
  const long long d = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (d >= nd) return;
  long long k = rp[d];
  const unsigned m = pat[d];
  for (int s = 0; s < 25; ++s)
    if (m >> s & 1u) {
      if (cols) cols[k] = static_cast<int>(slot_col(d, s, gx));
      if (vals) vals[k] = st[d * 25 + s];
      ++k;
    }
}

// SparseSymMatrix::multiply (sparse.cpp:69-76): s = 0; s += v * x in column
// order; rows of non-interior dofs give 0 when interior_only (k_dual semantics).
template <int NR>
__global__ void k_p2_apply(IMap im, const double* st, const unsigned* pat, const double* x,
                           double* y, int interior_only) {
  const int gx = im.nx;
  const long long nd = static_cast<long long>(gx + 1) * (im.ny + 1);
  const long long d = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (d >= nd) return;
  const int X = static_cast<int>(d % (gx + 1)), Y = static_cast<int>(d / (gx + 1));
  double acc[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) acc[r] = 0.0;
  if (!interior_only || im.interior(X, Y)) {
    const unsigned m = pat[d];
    for (int s = 0; s < 25; ++s)
      if (m >> s & 1u) {
        const double v = st[d * 25 + s];
        double xv[NR];
        ldv<NR>(x + slot_col(d, s, gx) * NR, xv);
#pragma unroll
        for (int r = 0; r < NR; ++r) acc[r] = xadd(acc[r], xmul(v, xv[r]));
      }
  }
  stv<NR>(y + d * NR, acc);
}

__global__ void k_p2_dense(IMap im, const double* st, const unsigned* pat, double* dense) {
  const long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long n = im.count();
  if (k >= n) return;
  int X, Y;
  im.point(k, &X, &Y);
  const long long d = static_cast<long long>(Y) * (im.nx + 1) + X;
  const unsigned m = pat[d];
  for (int s = 0; s < 25; ++s) {
    if (!(m >> s & 1u)) continue;
    const long long col = im.index(X + s % 5 - 2, Y + s / 5 - 2);
    if (col >= 0) dense[col * n + k] = st[d * 25 + s];
  }
}

__global__ void k_p2_space(int nx, int ny, int* dof_lattice) {
  const int gx = 2 * nx;
  const long long d = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (d >= static_cast<long long>(gx + 1) * (2 * ny + 1)) return;
  dof_lattice[2 * d] = static_cast<int>(d % (gx + 1));
  dof_lattice[2 * d + 1] = static_cast<int>(d / (gx + 1));
}

__global__ void k_p2_connectivity(long long nt, const int* tri, const int* lat, int nx,
                                  int* conn6) {
  const long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (t >= nt) return;
  const long long st = 2LL * nx + 1;
  int px[3], py[3];
  for (int k = 0; k < 3; ++k) {
    const int v = tri[3 * t + k];
    px[k] = 2 * lat[2 * v];
    py[k] = 2 * lat[2 * v + 1];
    conn6[6 * t + k] = static_cast<int>(py[k] * st + px[k]);
  }
  const int ea[3] = {0, 1, 2}, eb[3] = {1, 2, 0};
  for (int e = 0; e < 3; ++e)
    conn6[6 * t + 3 + e] = static_cast<int>(((py[ea[e]] + py[eb[e]]) / 2) * st +
                                            (px[ea[e]] + px[eb[e]]) / 2);
}

// prolongation_matrix (fespace.cpp:355-400) row of fine dof (FX, FY): the P2
// interpolant of the coarse triangle containing the point, entries in
// ascending coarse dof order (nonzeros only).  Coarse half-lattice = FX/2.
struct PRow {
  int n;
  long long col[6];
  double val[6];
};

__device__ PRow p2_row(int nxc, int nyc, int FX, int FY) {
  // coarse cell and triangle containing the point (fine half units: 4 per cell)
  const int cx = min(FX >> 2, nxc - 1), cy = min(FY >> 2, nyc - 1);
  const int u = FX - 4 * cx, v = FY - 4 * cy;  // 0..4
  const int upper = v > u ? 1 : 0;           // above the SW-NE diagonal
  // canonical (rotation-0) vertex order; the P2 interpolant does not depend on
  // the vertex order, the nonzero columns are re-sorted below
  long long x[3], y[3];
  for (int k = 0; k < 3; ++k) {
    int hx, hy;
    canon_half(upper, k, &hx, &hy);
    x[k] = 4LL * cx + 2 * hx;
    y[k] = 4LL * cy + 2 * hy;
  }
  const double denom = static_cast<double>((x[1] - x[0]) * (y[2] - y[0]) - (x[2] - x[0]) * (y[1] - y[0]));
  const double l1 = static_cast<double>((FX - x[0]) * (y[2] - y[0]) - (x[2] - x[0]) * (FY - y[0])) / denom;
  const double l2 = static_cast<double>((x[1] - x[0]) * (FY - y[0]) - (FX - x[0]) * (y[1] - y[0])) / denom;
  const double l[3] = {1.0 - l1 - l2, l1, l2};
  double val[6];
  for (int i = 0; i < 3; ++i) val[i] = l[i] * (2.0 * l[i] - 1.0);
  val[3] = 4.0 * l[0] * l[1];
  val[4] = 4.0 * l[1] * l[2];
  val[5] = 4.0 * l[2] * l[0];
  const long long sc = 2LL * nxc + 1;
  long long hx[6], hy[6];
  for (int k = 0; k < 3; ++k) {
    hx[k] = x[k] / 2;
    hy[k] = y[k] / 2;
  }
  hx[3] = (hx[0] + hx[1]) / 2;
  hy[3] = (hy[0] + hy[1]) / 2;
  hx[4] = (hx[1] + hx[2]) / 2;
  hy[4] = (hy[1] + hy[2]) / 2;
  hx[5] = (hx[2] + hx[0]) / 2;
  hy[5] = (hy[2] + hy[0]) / 2;
  PRow r;
  r.n = 0;
  for (int c = 0; c < 6; ++c) {
    if (val[c] == 0.0) continue;
    const long long col = hy[c] * sc + hx[c];
    int k = r.n++;
    while (k > 0 && r.col[k - 1] > col) {
      r.col[k] = r.col[k - 1];
      r.val[k] = r.val[k - 1];
      --k;
    }
    r.col[k] = col;
    r.val[k] = val[c];
  }
  return r;
}

// y = P x (SparseMatrix::multiply, sparse.cpp:129-136: from 0.0, column order)
template <int NR>
__global__ void k_p2_prolong(int nxc, int nyc, const double* xc, double* xf) {
  const int gx = 4 * nxc, gy = 4 * nyc;
  const long long d = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (d >= static_cast<long long>(gx + 1) * (gy + 1)) return;
  const PRow r = p2_row(nxc, nyc, static_cast<int>(d % (gx + 1)), static_cast<int>(d / (gx + 1)));
  double s[NR], t[NR];
#pragma unroll
  for (int q = 0; q < NR; ++q) s[q] = 0.0;
  for (int k = 0; k < r.n; ++k) {
    ldv<NR>(xc + r.col[k] * NR, t);
#pragma unroll
    for (int q = 0; q < NR; ++q) s[q] = xadd(s[q], xmul(r.val[k], t[q]));
  }
  stv<NR>(xf + d * NR, s);
}

// y = P^T x (multiply_transpose, sparse.cpp:144-148: rows in ascending order):
// coarse dof c gathers the fine rows around it (a 9x9 fine half-lattice block).
template <int NR>
__global__ void k_p2_restrict(int nxc, int nyc, const double* xf, double* xc) {
  const int gxc = 2 * nxc, gyc = 2 * nyc, gxf = 4 * nxc, gyf = 4 * nyc;
  const long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (c >= static_cast<long long>(gxc + 1) * (gyc + 1)) return;
  const int CX = static_cast<int>(c % (gxc + 1)), CY = static_cast<int>(c / (gxc + 1));
  double s[NR], t[NR];
#pragma unroll
  for (int q = 0; q < NR; ++q) s[q] = 0.0;
  for (int FY = max(2 * CY - 4, 0); FY <= min(2 * CY + 4, gyf); ++FY)
    for (int FX = max(2 * CX - 4, 0); FX <= min(2 * CX + 4, gxf); ++FX) {
      const PRow r = p2_row(nxc, nyc, FX, FY);
      for (int k = 0; k < r.n; ++k)
        if (r.col[k] == c) {
          ldv<NR>(xf + (static_cast<long long>(FY) * (gxf + 1) + FX) * NR, t);
#pragma unroll
          for (int q = 0; q < NR; ++q) s[q] = xadd(s[q], xmul(r.val[k], t[q]));
        }
    }
  stv<NR>(xc + c * NR, s);
}

// res = lam * (M u) - (A w) at interior dofs (corrector.cpp:201,237), 0 at
// non-interior ones; with only_mask, masked-out interior dofs are not written.
template <int NR>
__global__ void k_p2_residual(IMap im, const double* stA, const double* stM, const unsigned* pat,
                              const double* u, const double* w, Lam lam, double* out,
                              const unsigned char* only_mask) {
  const int gx = im.nx;
  const long long nd = static_cast<long long>(gx + 1) * (im.ny + 1);
  const long long d = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (d >= nd) return;
  const int X = static_cast<int>(d % (gx + 1)), Y = static_cast<int>(d / (gx + 1));
  double y[NR];
  if (!im.interior(X, Y)) {
#pragma unroll
    for (int r = 0; r < NR; ++r) y[r] = 0.0;
    stv<NR>(out + d * NR, y);
    return;
  }
  if (only_mask && !only_mask[d]) return;
  double mu[NR], aw[NR], t[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) mu[r] = aw[r] = 0.0;
  const unsigned m = pat[d];
  for (int s = 0; s < 25; ++s)
    if (m >> s & 1u) {
      const long long col = slot_col(d, s, gx);
      ldv<NR>(u + col * NR, t);
#pragma unroll
      for (int r = 0; r < NR; ++r) mu[r] = xadd(mu[r], xmul(stM[d * 25 + s], t[r]));
      ldv<NR>(w + col * NR, t);
#pragma unroll
      for (int r = 0; r < NR; ++r) aw[r] = xadd(aw[r], xmul(stA[d * 25 + s], t[r]));
    }
#pragma unroll
  for (int r = 0; r < NR; ++r) y[r] = xsub(xmul(lam.v[r], mu[r]), aw[r]);
  stv<NR>(out + d * NR, y);
}

void upload_q6(Ctx& c) {
  const double a1 = 0.501426509658179, b1 = 0.249286745170910, w1 = 0.116786275726379;
  const double a2 = 0.873821971016996, b2 = 0.063089014491502, w2 = 0.050844906370207;
  const double a3 = 0.053145049844816, b3 = 0.310352451033785, c3 = 0.636502499121399,
               w3 = 0.082851075618374;
  const double q[12][4] = {{a1, b1, b1, w1}, {b1, a1, b1, w1}, {b1, b1, a1, w1},
                           {a2, b2, b2, w2}, {b2, a2, b2, w2}, {b2, b2, a2, w2},
                           {a3, b3, c3, w3}, {a3, c3, b3, w3}, {b3, a3, c3, w3},
                           {b3, c3, a3, w3}, {c3, a3, b3, w3}, {c3, b3, a3, w3}};
  MLG_CUDA(cudaMemcpyToSymbolAsync(kQ6p2, q, sizeof(q), 0, cudaMemcpyHostToDevice, c.stream));
  c.sync();
}

}  // namespace

void assemble_p2(Ctx& c, Level& L) {
  if (L.hole.any()) throw ConfigError("P2 elements on a domain with a hole are not supported");
  if (c.cfg.example == 2) throw ConfigError("P2 elements with the reaction example are not supported");
  upload_q6(c);
  const long long nd = L.ndofs();
  L.p2A.alloc(static_cast<std::size_t>(nd) * 25);
  L.p2M.alloc(static_cast<std::size_t>(nd) * 25);
  L.p2pat.alloc(static_cast<std::size_t>(nd));
  P2Geom G{L.nx, L.ny, c.cfg.x_min, c.cfg.y_min, L.dx, L.dy, L.geo.get(), c.cfg.example};
  k_p2_assemble<<<grid_for(nd, kBlock), kBlock, 0, c.stream>>>(G, L.p2A.get(), L.p2M.get(),
                                                               L.p2pat.get());
  MLG_LAUNCH_CHECK();
  // nnz = sum of row masks
  DevBuf<int> cnt(nd + 1), rp(nd + 1);
  k_p2_count<<<grid_for(nd + 1, kBlock), kBlock, 0, c.stream>>>(nd, L.p2pat.get(), cnt.get());
  MLG_LAUNCH_CHECK();
  std::size_t tb = 0;
  MLG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.get(), rp.get(), static_cast<int>(nd + 1),
                                         c.stream));
  void* tmp = c.scratch_bytes(tb);
  MLG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt.get(), rp.get(), static_cast<int>(nd + 1),
                                         c.stream));
  int nnz = 0;
  MLG_CUDA(cudaMemcpyAsync(&nnz, rp.get() + nd, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  L.p2nnz = nnz;
}

void export_csr_p2(Ctx& c, const Level& L, int form, int* row_ptr, int* cols, double* vals) {
  const long long nd = L.ndofs();
  DevBuf<int> cnt(nd + 1), rp(nd + 1);
  k_p2_count<<<grid_for(nd + 1, kBlock), kBlock, 0, c.stream>>>(nd, L.p2pat.get(), cnt.get());
  MLG_LAUNCH_CHECK();
  std::size_t tb = 0;
  MLG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.get(), rp.get(), static_cast<int>(nd + 1),
                                         c.stream));
  void* tmp = c.scratch_bytes(tb);
  MLG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt.get(), rp.get(), static_cast<int>(nd + 1),
                                         c.stream));
  DevBuf<int> cl(cols ? L.p2nnz : 0);
  DevBuf<double> vl(vals ? L.p2nnz : 0);
  k_p2_export<<<grid_for(nd, kBlock), kBlock, 0, c.stream>>>(
      nd, 2 * L.nx, form == 0 ? L.p2A.get() : L.p2M.get(), L.p2pat.get(), rp.get(),
      cols ? cl.get() : nullptr, vals ? vl.get() : nullptr);
  MLG_LAUNCH_CHECK();
  if (row_ptr) rp.download(row_ptr, nd + 1, c.stream);
  if (cols) cl.download(cols, L.p2nnz, c.stream);
  if (vals) vl.download(vals, L.p2nnz, c.stream);
  c.sync();
}

void apply_p2(Ctx& c, const Level& L, int form, int nr, const double* x, double* y,
              bool interior_only) {
  const long long nd = L.ndofs();
  const double* st = form == 0 ? L.p2A.get() : L.p2M.get();
  switch (nr) {
    case 1: k_p2_apply<1><<<grid_for(nd, kBlock), kBlock, 0, c.stream>>>(L.imap(), st, L.p2pat.get(), x, y, interior_only); break;
    case 2: k_p2_apply<2><<<grid_for(nd, kBlock), kBlock, 0, c.stream>>>(L.imap(), st, L.p2pat.get(), x, y, interior_only); break;
    case 4: k_p2_apply<4><<<grid_for(nd, kBlock), kBlock, 0, c.stream>>>(L.imap(), st, L.p2pat.get(), x, y, interior_only); break;
    case 8: k_p2_apply<8><<<grid_for(nd, kBlock), kBlock, 0, c.stream>>>(L.imap(), st, L.p2pat.get(), x, y, interior_only); break;
    default: throw ConfigError("unsupported right-hand-side batch width");
  }
  MLG_LAUNCH_CHECK();
}

void interior_dense_p2(Ctx& c, const Level& L, int form, double* d_dense) {
  const long long n = L.nint();
  MLG_CUDA(cudaMemsetAsync(d_dense, 0, sizeof(double) * n * n, c.stream));
  k_p2_dense<<<grid_for(n, kBlock), kBlock, 0, c.stream>>>(
      L.imap(), form == 0 ? L.p2A.get() : L.p2M.get(), L.p2pat.get(), d_dense);
  MLG_LAUNCH_CHECK();
}

void export_space_p2(Ctx& c, const Level& L, int* dof_lattice, int* conn6) {
  const long long nd = L.ndofs();
  if (dof_lattice) {
    DevBuf<int> d(2 * nd);
    k_p2_space<<<grid_for(nd, kBlock), kBlock, 0, c.stream>>>(L.nx, L.ny, d.get());
    MLG_LAUNCH_CHECK();
    d.download(dof_lattice, 2 * nd, c.stream);
  }
  if (conn6) {
    DevBuf<int> cn(6 * L.nt);
    k_p2_connectivity<<<grid_for(L.nt, kBlock), kBlock, 0, c.stream>>>(L.nt, L.tri.get(),
                                                                       L.lat.get(), L.nx, cn.get());
    MLG_LAUNCH_CHECK();
    cn.download(conn6, 6 * L.nt, c.stream);
  }
  c.sync();
}

#define P2_NR(nr, kernel, grid, ...)                                              \
  do {                                                                            \
    switch (nr) {                                                                 \
      case 1: kernel<1><<<grid, kBlock, 0, c.stream>>>(__VA_ARGS__); break;       \
      case 2: kernel<2><<<grid, kBlock, 0, c.stream>>>(__VA_ARGS__); break;       \
      case 4: kernel<4><<<grid, kBlock, 0, c.stream>>>(__VA_ARGS__); break;       \
      case 8: kernel<8><<<grid, kBlock, 0, c.stream>>>(__VA_ARGS__); break;       \
      default: throw ConfigError("unsupported right-hand-side batch width");      \
    }                                                                             \
    MLG_LAUNCH_CHECK();                                                           \
  } while (0)

void prolong_p2(Ctx& c, const Level& C, int nr, const double* xc, double* xf) {
  const long long nf = static_cast<long long>(4 * C.nx + 1) * (4 * C.ny + 1);
  P2_NR(nr, k_p2_prolong, grid_for(nf, kBlock), C.nx, C.ny, xc, xf);
}

void restrict_p2(Ctx& c, const Level& C, int nr, const double* xf, double* xc) {
  P2_NR(nr, k_p2_restrict, grid_for(C.ndofs(), kBlock), C.nx, C.ny, xf, xc);
}

void residual_p2(Ctx& c, const Level& L, int nr, const double* u, const double* w,
                 const Lam& lam, double* out, const unsigned char* only_mask) {
  P2_NR(nr, k_p2_residual, grid_for(L.ndofs(), kBlock), L.imap(), L.p2A.get(), L.p2M.get(),
        L.p2pat.get(), u, w, lam, out, only_mask);
}

}  // namespace mlg

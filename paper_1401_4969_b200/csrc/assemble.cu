// Level build, floating-point part: P1 stiffness and mass assembly, bit-exact
// with the reference's element-order triplet accumulation.
//
//   local_matrix / element_geometry  fespace.cpp:169-217 (3-point edge-midpoint
//                                    rule, quad_degree2 fespace.cpp:41-47, for the
//                                    Laplace field; 12-point quad_degree6
//                                    fespace.cpp:49-75 for the variable field)
//   assemble_form                    fespace.cpp:314-341
//   SparseSymMatrix::from_upper_triplets  sparse.cpp:24-61 (stable (row,col)
//                                    sort => duplicates summed from 0.0 in
//                                    ascending element id; mirrored bitwise)
//
// B200 design (row gather, no sort): entry (r,c) of the global matrix is the
// sum, over the <=6 triangles that contain both dofs, of local[i][j] in
// ascending element id.  Every triangle of the structured lattice is found
// through the per-level slot table `geo` (cell, L/U) -> (elem<<2 | rotation)
// that refinement writes, so one thread per dof gathers its <=6 triangles,
// recomputes their element matrices with the reference's exact operation
// sequence (unfused __d*_rn), sorts the contributions by element id and sums
// them.  Output is the 4-entry upper stencil {C,E,N,NE} of A and M per dof
// (64 B/dof written, coalesced); CSR export is a second closed-form pass.
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>

#include "ctx.cuh"
#include "p2.cuh"

namespace mlg {
namespace {

constexpr int kBlock = 256;

struct Contrib {
  unsigned e;
  double a, m;
};

// Element-local entries (i<=j) of the P1 Laplace stiffness and unit mass for
// a triangle with vertices v0,v1,v2 in element order (fespace.cpp:169-217).
__device__ __forceinline__ void local_entry(double v0x, double v0y, double v1x, double v1y,
                                            double v2x, double v2y, int i, int j, double* a_out,
                                            double* m_out) {
  const double area2 = xsub(xmul(xsub(v1x, v0x), xsub(v2y, v0y)),
                            xmul(xsub(v2x, v0x), xsub(v1y, v0y)));
  const double area = xmul(0.5, area2);
  double g[3][2];
  g[0][0] = xdiv(xsub(v1y, v2y), area2);
  g[0][1] = xdiv(xsub(v2x, v1x), area2);
  g[1][0] = xdiv(xsub(v2y, v0y), area2);
  g[1][1] = xdiv(xsub(v0x, v2x), area2);
  g[2][0] = xdiv(xsub(v0y, v1y), area2);
  g[2][1] = xdiv(xsub(v1x, v0x), area2);
  const double w = xmul(1.0 / 3.0, area);  // rule.weights[q] * g.area, same for all q
  // stiffness with A = I (CoefficientField::laplace, fespace.cpp:105-112)
  const double agx = xadd(xmul(1.0, g[i][0]), xmul(0.0, g[i][1]));
  const double agy = xadd(xmul(0.0, g[i][0]), xmul(1.0, g[i][1]));
  const double s = xmul(w, xadd(xmul(agx, g[j][0]), xmul(agy, g[j][1])));
  double a = 0.0;
  a = xadd(a, s);
  a = xadd(a, s);
  a = xadd(a, s);
  // mass with phi = 1: points {.5,.5,0},{0,.5,.5},{.5,0,.5}
  const double P[3][3] = {{0.5, 0.5, 0.0}, {0.0, 0.5, 0.5}, {0.5, 0.0, 0.5}};
  double m = 0.0;
#pragma unroll
  for (int q = 0; q < 3; ++q) m = xadd(m, xmul(xmul(xmul(w, 1.0), P[q][i]), P[q][j]));
  *a_out = a;
  *m_out = m;
}

struct LevelGeom {
  int nx, ny;
  double x0, y0, dx, dy;
  const unsigned* geo;
  int k1 = 0, k2 = 0;  // example 2 (reaction) modes
};

// Example 2 (BASELINE config 4, no reference code path): piecewise-constant
// coefficients at the centroid, a = 1 + 0.5 sin(2 pi k1 x) sin(2 pi k2 y),
// c = 1 + x^2 + y^2; element stiffness a*K + c*M (K, M the P1 Laplace
// stiffness and mass of local_entry), element mass M.  The tests' numpy restatement
// restates the same operation sequence.
__device__ __forceinline__ void reaction_entry(double v0x, double v0y, double v1x, double v1y,
                                               double v2x, double v2y, int k1, int k2,
                                               double* a_io, double m) {
  const double kTwoPi = 6.283185307179586476925286766559;
  const double xc = xdiv(xadd(xadd(v0x, v1x), v2x), 3.0);
  const double yc = xdiv(xadd(xadd(v0y, v1y), v2y), 3.0);
  const double ac = xadd(1.0, xmul(xmul(0.5, sin(xmul(xmul(kTwoPi, k1), xc))),
                                   sin(xmul(xmul(kTwoPi, k2), yc))));
  const double cc = xadd(xadd(1.0, xmul(xc, xc)), xmul(yc, yc));
  *a_io = xadd(xmul(ac, *a_io), xmul(cc, m));
}

// Canonical vertex k of the L/U triangle of cell (cx,cy):
//   L: (cx,cy), (cx+1,cy), (cx+1,cy+1)     U: (cx,cy), (cx+1,cy+1), (cx,cy+1)
__device__ __forceinline__ void canon_vertex(int cx, int cy, int upper, int k, int* x, int* y) {
  if (k == 0) {
    *x = cx;
    *y = cy;
  } else if (k == 1) {
    *x = cx + 1;
    *y = cy + (upper ? 1 : 0);
  } else {
    *x = cx + (upper ? 0 : 1);
    *y = cy + 1;
  }
}

// Contribution of triangle (cell, upper) to the pair of canonical vertices
// (kd, kn) (kd == kn for a diagonal entry).
template <int EX>
__device__ __forceinline__ bool contribution(const LevelGeom& G, int cx, int cy, int upper,
                                             int kd, int kn, Contrib* out) {
  if (cx < 0 || cy < 0 || cx >= G.nx || cy >= G.ny) return false;
  const unsigned code = G.geo[2 * (static_cast<std::int64_t>(cy) * G.nx + cx) + upper];
  if (code == 0xFFFFFFFFu) return false;  // removed cell (domain with a hole)
  const int rot = static_cast<int>(code & 3u);
  double vx[3], vy[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    int lx, ly;
    canon_vertex(cx, cy, upper, (rot + j) % 3, &lx, &ly);
    vx[j] = lattice_coord(G.x0, lx, G.dx);
    vy[j] = lattice_coord(G.y0, ly, G.dy);
  }
  const int ld = (kd - rot + 3) % 3, ln = (kn - rot + 3) % 3;
  local_entry(vx[0], vy[0], vx[1], vy[1], vx[2], vy[2], min(ld, ln), max(ld, ln), &out->a,
              &out->m);
  if (EX == 2)
    reaction_entry(vx[0], vy[0], vx[1], vy[1], vx[2], vy[2], G.k1, G.k2, &out->a, out->m);
  out->e = code >> 2;
  return true;
}

// Sum in ascending element id, from 0.0 (sparse.cpp:36-46).
template <int N>
__device__ __forceinline__ void ordered_sum(Contrib* c, int n, double* a, double* m) {
  for (int i = 1; i < n; ++i) {  // insertion sort, n <= 6
    Contrib t = c[i];
    int k = i;
    while (k > 0 && c[k - 1].e > t.e) {
      c[k] = c[k - 1];
      --k;
    }
    c[k] = t;
  }
  double sa = 0.0, sm = 0.0;
  for (int i = 0; i < n; ++i) {
    sa = xadd(sa, c[i].a);
    sm = xadd(sm, c[i].m);
  }
  *a = sa;
  *m = sm;
}

// ---- CoefficientField::variable (fespace.cpp:114-123) with quad_degree6 ----
// Upper entries of the element matrices of one triangle in element-local
// vertex order, packed (0,0),(0,1),(0,2),(1,1),(1,2),(2,2); the reference's
// operation sequence of local_matrix (fespace.cpp:185-217) for degree 1:
// per quadrature point w = weight*area, x = l0*v0x + l1*v1x + l2*v2x,
// stiffness += w*(agx*g_j0 + agy*g_j1) with a = diffusion(x,y), mass +=
// ((w*phi)*l_i)*l_j -- every operation rounded separately (the reference is
// built for baseline x86-64: no FMA contraction).  exp() is CUDA's (<= 1 ulp),
// so entries agree with the reference to a few ulp, not bitwise.
__device__ __forceinline__ int upk(int i, int j) { return i * 3 - (i * (i - 1)) / 2 + (j - i); }

__constant__ double kQ6[12][4];  // l0, l1, l2, weight (make_degree6, fespace.cpp:49-75)

__device__ void elem_variable(double v0x, double v0y, double v1x, double v1y, double v2x,
                              double v2y, double a[6], double m[6]) {
  const double area2 = xsub(xmul(xsub(v1x, v0x), xsub(v2y, v0y)),
                            xmul(xsub(v2x, v0x), xsub(v1y, v0y)));
  const double area = xmul(0.5, area2);
  double g[3][2];
  g[0][0] = xdiv(xsub(v1y, v2y), area2);
  g[0][1] = xdiv(xsub(v2x, v1x), area2);
  g[1][0] = xdiv(xsub(v2y, v0y), area2);
  g[1][1] = xdiv(xsub(v0x, v2x), area2);
  g[2][0] = xdiv(xsub(v0y, v1y), area2);
  g[2][1] = xdiv(xsub(v1x, v0x), area2);
#pragma unroll
  for (int k = 0; k < 6; ++k) a[k] = m[k] = 0.0;
  for (int q = 0; q < 12; ++q) {
    const double l0 = kQ6[q][0], l1 = kQ6[q][1], l2 = kQ6[q][2];
    const double w = xmul(kQ6[q][3], area);
    const double x = xadd(xadd(xmul(l0, v0x), xmul(l1, v1x)), xmul(l2, v2x));
    const double y = xadd(xadd(xmul(l0, v0y), xmul(l1, v1y)), xmul(l2, v2y));
    const double d0 = exp(xadd(1.0, xmul(x, x)));
    const double d1 = exp(xmul(x, y));
    const double d2 = exp(xadd(1.0, xmul(y, y)));
    const double phi = xmul(xadd(1.0, xmul(x, x)), xadd(1.0, xmul(y, y)));
    const double l[3] = {l0, l1, l2};
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double agx = xadd(xmul(d0, g[i][0]), xmul(d1, g[i][1]));
      const double agy = xadd(xmul(d1, g[i][0]), xmul(d2, g[i][1]));
#pragma unroll
      for (int j = i; j < 3; ++j) {
        a[upk(i, j)] = xadd(a[upk(i, j)], xmul(w, xadd(xmul(agx, g[j][0]), xmul(agy, g[j][1]))));
        m[upk(i, j)] = xadd(m[upk(i, j)], xmul(xmul(xmul(w, phi), l[i]), l[j]));
      }
    }
  }
}

// Element matrix of triangle (cell, upper) in its mesh vertex order; returns
// false outside the lattice.
__device__ __forceinline__ bool elem_matrix_var(const LevelGeom& G, int cx, int cy, int upper,
                                                double a[6], double m[6], unsigned* e,
                                                int* rot) {
  if (cx < 0 || cy < 0 || cx >= G.nx || cy >= G.ny) return false;
  const unsigned code = G.geo[2 * (static_cast<std::int64_t>(cy) * G.nx + cx) + upper];
  if (code == 0xFFFFFFFFu) return false;  // removed cell (domain with a hole)
  *rot = static_cast<int>(code & 3u);
  *e = code >> 2;
  double vx[3], vy[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    int lx, ly;
    canon_vertex(cx, cy, upper, (*rot + j) % 3, &lx, &ly);
    vx[j] = lattice_coord(G.x0, lx, G.dx);
    vy[j] = lattice_coord(G.y0, ly, G.dy);
  }
  elem_variable(vx[0], vy[0], vx[1], vy[1], vx[2], vy[2], a, m);
  return true;
}

__device__ __forceinline__ void push_entry(const double a[6], const double m[6], unsigned e,
                                           int rot, int kd, int kn, Contrib* list, int* n) {
  const int ld = (kd - rot + 3) % 3, ln = (kn - rot + 3) % 3;
  const int k = upk(min(ld, ln), max(ld, ln));
  list[*n] = Contrib{e, a[k], m[k]};
  ++*n;
}

// Variable-coefficient assembly: one thread per dof computes each of its <= 6
// triangles' element matrices once (12 quadrature points, 3 exp each) and
// scatters the entries it owns into the C/E/N/NE lists, summed in ascending
// element id as in k_assemble.
__global__ void __launch_bounds__(kBlock) k_assemble_var(LevelGeom G, Stencil* stA,
                                                         Stencil* stM, double* dinv) {
  const std::int64_t d = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  const std::int64_t nd = static_cast<std::int64_t>(G.nx + 1) * (G.ny + 1);
  if (d >= nd) return;
  const int ix = static_cast<int>(d % (G.nx + 1)), iy = static_cast<int>(d / (G.nx + 1));
  Contrib cd[6], ce[2], cn[2], cne[2];
  int nd_ = 0, ne_ = 0, nn_ = 0, nne_ = 0;
  double a[6], m[6];
  unsigned e;
  int rot;
  // T0 = L(ix,iy): diag k0; E (0,1); NE (0,2)
  if (elem_matrix_var(G, ix, iy, 0, a, m, &e, &rot)) {
    push_entry(a, m, e, rot, 0, 0, cd, &nd_);
    push_entry(a, m, e, rot, 0, 1, ce, &ne_);
    push_entry(a, m, e, rot, 0, 2, cne, &nne_);
  }
  // T1 = U(ix,iy): diag k0; N (0,2); NE (0,1)
  if (elem_matrix_var(G, ix, iy, 1, a, m, &e, &rot)) {
    push_entry(a, m, e, rot, 0, 0, cd, &nd_);
    push_entry(a, m, e, rot, 0, 2, cn, &nn_);
    push_entry(a, m, e, rot, 0, 1, cne, &nne_);
  }
  // T2 = L(ix-1,iy): diag k1; N (1,2)
  if (elem_matrix_var(G, ix - 1, iy, 0, a, m, &e, &rot)) {
    push_entry(a, m, e, rot, 1, 1, cd, &nd_);
    push_entry(a, m, e, rot, 1, 2, cn, &nn_);
  }
  // T3 = U(ix,iy-1): diag k2; E (2,1)
  if (elem_matrix_var(G, ix, iy - 1, 1, a, m, &e, &rot)) {
    push_entry(a, m, e, rot, 2, 2, cd, &nd_);
    push_entry(a, m, e, rot, 2, 1, ce, &ne_);
  }
  if (elem_matrix_var(G, ix - 1, iy - 1, 0, a, m, &e, &rot))  // T4 = L(ix-1,iy-1): k2
    push_entry(a, m, e, rot, 2, 2, cd, &nd_);
  if (elem_matrix_var(G, ix - 1, iy - 1, 1, a, m, &e, &rot))  // T5 = U(ix-1,iy-1): k1
    push_entry(a, m, e, rot, 1, 1, cd, &nd_);
  Stencil A{0.0, 0.0, 0.0, 0.0}, M{0.0, 0.0, 0.0, 0.0};
  ordered_sum<6>(cd, nd_, &A.c, &M.c);
  ordered_sum<2>(ce, ne_, &A.e, &M.e);
  ordered_sum<2>(cn, nn_, &A.n, &M.n);
  ordered_sum<2>(cne, nne_, &A.ne, &M.ne);
  stA[d] = A;
  stM[d] = M;
  dinv[d] = A.c != 0.0 ? 1.0 / A.c : 0.0;  // inactive points of a hole: empty rows
}

template <int EX>
__global__ void __launch_bounds__(kBlock) k_assemble(LevelGeom G, Stencil* stA, Stencil* stM,
                                                     double* dinv) {
  const std::int64_t d = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  const std::int64_t nd = static_cast<std::int64_t>(G.nx + 1) * (G.ny + 1);
  if (d >= nd) return;
  const int ix = static_cast<int>(d % (G.nx + 1)), iy = static_cast<int>(d / (G.nx + 1));
  Contrib c[6];
  int n;
  Stencil A{0.0, 0.0, 0.0, 0.0}, M{0.0, 0.0, 0.0, 0.0};
  // diagonal: the six triangles around (ix,iy) with the dof's canonical index
  n = 0;
  n += contribution<EX>(G, ix, iy, 0, 0, 0, c + n);
  n += contribution<EX>(G, ix, iy, 1, 0, 0, c + n);
  n += contribution<EX>(G, ix - 1, iy, 0, 1, 1, c + n);
  n += contribution<EX>(G, ix, iy - 1, 1, 2, 2, c + n);
  n += contribution<EX>(G, ix - 1, iy - 1, 0, 2, 2, c + n);
  n += contribution<EX>(G, ix - 1, iy - 1, 1, 1, 1, c + n);
  ordered_sum<6>(c, n, &A.c, &M.c);
  if (ix < G.nx) {  // E: L(ix,iy) (0,1), U(ix,iy-1) (2,1)
    n = 0;
    n += contribution<EX>(G, ix, iy, 0, 0, 1, c + n);
    n += contribution<EX>(G, ix, iy - 1, 1, 2, 1, c + n);
    ordered_sum<2>(c, n, &A.e, &M.e);
  }
  if (iy < G.ny) {  // N: U(ix,iy) (0,2), L(ix-1,iy) (1,2)
    n = 0;
    n += contribution<EX>(G, ix, iy, 1, 0, 2, c + n);
    n += contribution<EX>(G, ix - 1, iy, 0, 1, 2, c + n);
    ordered_sum<2>(c, n, &A.n, &M.n);
  }
  if (ix < G.nx && iy < G.ny) {  // NE: L(ix,iy) (0,2), U(ix,iy) (0,1)
    n = 0;
    n += contribution<EX>(G, ix, iy, 0, 0, 2, c + n);
    n += contribution<EX>(G, ix, iy, 1, 0, 1, c + n);
    ordered_sum<2>(c, n, &A.ne, &M.ne);
  }
  stA[d] = A;
  stM[d] = M;
  dinv[d] = A.c != 0.0 ? 1.0 / A.c : 0.0;  // JacobiPreconditioner inv_diag (0 for inactive points)
}

// ---- translation-invariant lattices: table-driven assembly (HBM-bound) ----
// local_entry reads the vertex coordinates only through differences between
// two vertices of the same triangle: 0 (same column / row, exact), or
// +-(x(cx+1) - x(cx)), +-(y(cy+1) - y(cy)) (negation is exact).  When every
// column step is bitwise one value EX and every row step one value EY (always
// the case for the BASELINE lattices, whose dx is a power of two), the element
// matrices of a triangle depend only on (lower/upper, rotation): six variants.
// k_lattice_steps proves the premise on the device; k_assemble_table then
// reads the variants, evaluated ONCE per level by k_assemble_table_build with
// local_entry itself (the reference's operation sequence), into shared memory
// and each dof only looks its <= 12 entries up, orders
// them by element id and sums from 0.0 -- bitwise the generic kernel, without
// its 72 FP64 divisions per dof.  Any other lattice keeps k_assemble.
__global__ void k_lattice_steps(LevelGeom G, int* flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < G.nx) {
    const double e0 = xsub(lattice_coord(G.x0, 1, G.dx), lattice_coord(G.x0, 0, G.dx));
    const double e = xsub(lattice_coord(G.x0, i + 1, G.dx), lattice_coord(G.x0, i, G.dx));
    if (__double_as_longlong(e) != __double_as_longlong(e0)) atomicAnd(flag, 0);
  }
  if (i < G.ny) {
    const double e0 = xsub(lattice_coord(G.y0, 1, G.dy), lattice_coord(G.y0, 0, G.dy));
    const double e = xsub(lattice_coord(G.y0, i + 1, G.dy), lattice_coord(G.y0, i, G.dy));
    if (__double_as_longlong(e) != __double_as_longlong(e0)) atomicAnd(flag, 0);
  }
}

constexpr int kTabEntries = 2 * 3 * 3 * 3;  // (upper, rot, kd, kn)
__device__ __forceinline__ int tab_index(int upper, int rot, int kd, int kn) {
  return ((upper * 3 + rot) * 3 + kd) * 3 + kn;
}

// Sort key: element id above the 6-bit table index; all ones = absent.  KEY is
// unsigned when (max element id << 6) fits 32 bits, else unsigned long long.
template <typename KEY>
__device__ __forceinline__ void cswap(KEY& a, KEY& b) {
  const KEY lo = min(a, b), hi = max(a, b);
  a = lo;
  b = hi;
}

__device__ __forceinline__ void st_stencil(Stencil* p, const Stencil& s) {
  // one 32-byte store per thread (sm_100: 256-bit global stores)
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(s.c), "d"(s.e), "d"(s.n),
               "d"(s.ne)
               : "memory");
}

// The table: entry (upper, rot, kd, kn) of A at [i], of M at [kTabEntries + i],
// evaluated once per level with local_entry itself.
__global__ void k_assemble_table_build(LevelGeom G, double* tab) {
  if (threadIdx.x < kTabEntries) {
    const int kn = threadIdx.x % 3, kd = threadIdx.x / 3 % 3, rot = threadIdx.x / 9 % 3,
              upper = threadIdx.x / 27;
    double vx[3], vy[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      int lx, ly;
      canon_vertex(0, 0, upper, (rot + j) % 3, &lx, &ly);
      vx[j] = lattice_coord(G.x0, lx, G.dx);
      vy[j] = lattice_coord(G.y0, ly, G.dy);
    }
    const int ld = (kd - rot + 3) % 3, ln = (kn - rot + 3) % 3;
    double a, m;
    local_entry(vx[0], vy[0], vx[1], vy[1], vx[2], vy[2], min(ld, ln), max(ld, ln), &a, &m);
    tab[threadIdx.x] = a;
    tab[kTabEntries + threadIdx.x] = m;
  }
}

template <typename KEY>
__global__ void __launch_bounds__(kBlock) k_assemble_table(LevelGeom G, const double* tab,
                                                           Stencil* stA, Stencil* stM,
                                                           double* dinv) {
  constexpr KEY kAbsent = ~static_cast<KEY>(0);
  __shared__ double tabA[kTabEntries], tabM[kTabEntries];
  if (threadIdx.x < kTabEntries) {
    tabA[threadIdx.x] = __ldg(tab + threadIdx.x);
    tabM[threadIdx.x] = __ldg(tab + kTabEntries + threadIdx.x);
  }
  __syncthreads();
  const std::int64_t d = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  const std::int64_t nd = static_cast<std::int64_t>(G.nx + 1) * (G.ny + 1);
  if (d >= nd) return;
  const int ix = static_cast<int>(d % (G.nx + 1)), iy = static_cast<int>(d / (G.nx + 1));
  // geo codes of the four cells around the dof: (L, U) pairs, 0xFFFFFFFF = absent
  const uint2 none = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
  const uint2* geo2 = reinterpret_cast<const uint2*>(G.geo);
  const bool xin = ix < G.nx, yin = iy < G.ny, xm = ix > 0, ym = iy > 0;
  const std::int64_t cell = static_cast<std::int64_t>(iy) * G.nx + ix;
  const uint2 g11 = xin && yin ? __ldg(geo2 + cell) : none;              // cell (ix, iy)
  const uint2 g01 = xm && yin ? __ldg(geo2 + cell - 1) : none;           // cell (ix-1, iy)
  const uint2 g10 = xin && ym ? __ldg(geo2 + cell - G.nx) : none;        // cell (ix, iy-1)
  const uint2 g00 = xm && ym ? __ldg(geo2 + cell - G.nx - 1) : none;     // cell (ix-1, iy-1)
  auto key = [](unsigned code, int upper, int kd, int kn) -> KEY {
    if (code == 0xFFFFFFFFu) return kAbsent;
    return (static_cast<KEY>(code >> 2) << 6) |
           static_cast<unsigned>(tab_index(upper, static_cast<int>(code & 3u), kd, kn));
  };
  auto pair_sum = [&](KEY k0, KEY k1, double* a, double* m) {
    cswap(k0, k1);
    double sa = 0.0, sm = 0.0;
    if (k0 != kAbsent) {
      sa = xadd(sa, tabA[k0 & 63u]);
      sm = xadd(sm, tabM[k0 & 63u]);
    }
    if (k1 != kAbsent) {
      sa = xadd(sa, tabA[k1 & 63u]);
      sm = xadd(sm, tabM[k1 & 63u]);
    }
    *a = sa;
    *m = sm;
  };
  Stencil A, M;
  {  // diagonal: the six triangles around the dof (same list as k_assemble)
    KEY k0 = key(g11.x, 0, 0, 0), k1 = key(g11.y, 1, 0, 0), k2 = key(g01.x, 0, 1, 1),
        k3 = key(g10.y, 1, 2, 2), k4 = key(g00.x, 0, 2, 2), k5 = key(g00.y, 1, 1, 1);
    // 12-comparator sorting network for 6 keys
    cswap(k0, k5); cswap(k1, k3); cswap(k2, k4);
    cswap(k1, k2); cswap(k3, k4);
    cswap(k0, k3); cswap(k2, k5);
    cswap(k0, k1); cswap(k2, k3); cswap(k4, k5);
    cswap(k1, k2); cswap(k3, k4);
    double sa = 0.0, sm = 0.0;
    const KEY ks[6] = {k0, k1, k2, k3, k4, k5};
#pragma unroll
    for (int i = 0; i < 6; ++i)
      if (ks[i] != kAbsent) {
        sa = xadd(sa, tabA[ks[i] & 63u]);
        sm = xadd(sm, tabM[ks[i] & 63u]);
      }
    A.c = sa;
    M.c = sm;
  }
  pair_sum(key(g11.x, 0, 0, 1), key(g10.y, 1, 2, 1), &A.e, &M.e);   // E
  pair_sum(key(g11.y, 1, 0, 2), key(g01.x, 0, 1, 2), &A.n, &M.n);   // N
  pair_sum(key(g11.x, 0, 0, 2), key(g11.y, 1, 0, 1), &A.ne, &M.ne); // NE
  st_stencil(stA + d, A);
  st_stencil(stM + d, M);
  dinv[d] = A.c != 0.0 ? 1.0 / A.c : 0.0;
}

// row_ptr of the full 7-point pattern in closed form.
__device__ __forceinline__ long long row_start(int ix, int iy, int nx, int ny) {
  const long long r = static_cast<long long>(iy) * (3LL * nx + 1) +
                      (2LL * nx + 1) * (max(iy - 1, 0) + min(iy, ny));
  const long long w = ix + max(ix - 1, 0) + ix + (iy > 0 ? ix + max(ix - 1, 0) : 0) +
                      (iy < ny ? 2LL * ix : 0);
  return r + w;
}

__global__ void k_export_csr(int nx, int ny, long long nnz, const Stencil* st, int* row_ptr,
                             int* cols, double* vals) {
  const std::int64_t d = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  const std::int64_t nd = static_cast<std::int64_t>(nx + 1) * (ny + 1);
  if (d > nd) return;
  if (d == nd) {
    if (row_ptr) row_ptr[nd] = static_cast<int>(nnz);
    return;
  }
  const int ix = static_cast<int>(d % (nx + 1)), iy = static_cast<int>(d / (nx + 1));
  long long k = row_start(ix, iy, nx, ny);
  if (row_ptr) row_ptr[d] = static_cast<int>(k);
  const std::int64_t s = nx + 1;
  auto put = [&](std::int64_t col, double v) {
    if (cols) cols[k] = static_cast<int>(col);
    if (vals) vals[k] = v;
    ++k;
  };
  if (iy > 0 && ix > 0) put(d - s - 1, st[d - s - 1].ne);
  if (iy > 0) put(d - s, st[d - s].n);
  if (ix > 0) put(d - 1, st[d - 1].e);
  put(d, st[d].c);
  if (ix < nx) put(d + 1, st[d].e);
  if (iy < ny) put(d + s, st[d].n);
  if (iy < ny && ix < nx) put(d + s + 1, st[d].ne);
}

// to_dense(extract_submatrix(a, interior_dofs)) (sparse.cpp:156-184),
// column-major n x n with n = (nx-1)(ny-1); entries mirror bitwise.
__global__ void k_interior_dense(IMap im, const Stencil* st, double* dense) {
  const std::int64_t k = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  const std::int64_t n = im.count();
  if (k >= n) return;
  int ix, iy;
  im.point(k, &ix, &iy);
  const std::int64_t s = im.nx + 1;
  const std::int64_t d = static_cast<std::int64_t>(iy) * s + ix;
  auto put = [&](int jx, int jy, double v) {
    const long long col_k = im.index(jx, jy);
    if (col_k >= 0) dense[col_k * n + k] = v;
  };
  put(ix - 1, iy - 1, st[d - s - 1].ne);
  put(ix, iy - 1, st[d - s].n);
  put(ix - 1, iy, st[d - 1].e);
  put(ix, iy, st[d].c);
  put(ix + 1, iy, st[d].e);
  put(ix, iy + 1, st[d].n);
  put(ix + 1, iy + 1, st[d].ne);
}

// ---- domains with a corner hole (config 3) ----
// Structural existence of the couplings of row (ix,iy) in the order SW, S, W,
// C, E, N, NE (a coupling exists iff an element contains both dofs).
__device__ __forceinline__ void hole_row_pattern(const Hole& h, int nx, int ny, int ix, int iy,
                                                 bool e[7]) {
  const bool c00 = cell_active(h, nx, ny, ix - 1, iy - 1), c10 = cell_active(h, nx, ny, ix, iy - 1);
  const bool c01 = cell_active(h, nx, ny, ix - 1, iy), c11 = cell_active(h, nx, ny, ix, iy);
  e[0] = c00;
  e[1] = c00 || c10;
  e[2] = c00 || c01;
  e[3] = c00 || c10 || c01 || c11;
  e[4] = c10 || c11;
  e[5] = c01 || c11;
  e[6] = c11;
}

__global__ void k_csr_count_hole(int nx, int ny, Hole h, int* cnt) {
  const std::int64_t d = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  const std::int64_t nd = static_cast<std::int64_t>(nx + 1) * (ny + 1);
  if (d > nd) return;
  if (d == nd) {
    cnt[d] = 0;
    return;
  }
  const int ix = static_cast<int>(d % (nx + 1)), iy = static_cast<int>(d / (nx + 1));
  bool e[7];
  hole_row_pattern(h, nx, ny, ix, iy, e);
  int n = 0;
  for (int k = 0; k < 7; ++k) n += e[k];
  cnt[d] = n;
}

__global__ void k_export_csr_hole(int nx, int ny, Hole h, const Stencil* st, const int* rp,
                                  int* cols, double* vals) {
  const std::int64_t d = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  const std::int64_t nd = static_cast<std::int64_t>(nx + 1) * (ny + 1);
  if (d >= nd) return;
  const int ix = static_cast<int>(d % (nx + 1)), iy = static_cast<int>(d / (nx + 1));
  bool e[7];
  hole_row_pattern(h, nx, ny, ix, iy, e);
  const std::int64_t s = nx + 1;
  const std::int64_t col[7] = {d - s - 1, d - s, d - 1, d, d + 1, d + s, d + s + 1};
  long long k = rp[d];
  for (int q = 0; q < 7; ++q) {
    if (!e[q]) continue;
    double v;
    switch (q) {
      case 0: v = st[d - s - 1].ne; break;
      case 1: v = st[d - s].n; break;
      case 2: v = st[d - 1].e; break;
      case 3: v = st[d].c; break;
      case 4: v = st[d].e; break;
      case 5: v = st[d].n; break;
      default: v = st[d].ne; break;
    }
    if (cols) cols[k] = static_cast<int>(col[q]);
    if (vals) vals[k] = v;
    ++k;
  }
}

// CG operator of a domain with a hole: extract_submatrix(A, interior) on the
// bounding lattice -- couplings touching a non-interior point are 0 and
// non-interior rows are identity, so a window that covers part of the hole
// keeps exact zeros there (zero rhs, zero iterates) and every dot product
// equals the restricted system's.
__global__ void k_cg_stencil(IMap im, const Stencil* st, const double* dinv, Stencil* out,
                             double* dinv_out) {
  const std::int64_t d = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  const int nx = im.nx, ny = im.ny;
  if (d >= static_cast<std::int64_t>(nx + 1) * (ny + 1)) return;
  const int ix = static_cast<int>(d % (nx + 1)), iy = static_cast<int>(d / (nx + 1));
  if (!im.interior(ix, iy)) {
    out[d] = Stencil{1.0, 0.0, 0.0, 0.0};
    dinv_out[d] = 1.0;
    return;
  }
  const Stencil a = st[d];
  out[d] = Stencil{a.c, im.interior(ix + 1, iy) ? a.e : 0.0, im.interior(ix, iy + 1) ? a.n : 0.0,
                   im.interior(ix + 1, iy + 1) ? a.ne : 0.0};
  dinv_out[d] = dinv[d];
}

// Clears *flag if any interior row of st / dinv differs bitwise from the first one.
__global__ void k_uniform_check(IMap im, const Stencil* st, const double* dinv, int* flag) {
  const std::int64_t k = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (k >= im.count()) return;
  int ix, iy, ix0, iy0;
  im.point(k, &ix, &iy);
  im.point(0, &ix0, &iy0);
  const std::int64_t d = static_cast<std::int64_t>(iy) * (im.nx + 1) + ix;
  const std::int64_t d0 = static_cast<std::int64_t>(iy0) * (im.nx + 1) + ix0;
  const Stencil a = st[d], b = st[d0];
  const bool same = __double_as_longlong(a.c) == __double_as_longlong(b.c) &&
                    __double_as_longlong(a.e) == __double_as_longlong(b.e) &&
                    __double_as_longlong(a.n) == __double_as_longlong(b.n) &&
                    __double_as_longlong(a.ne) == __double_as_longlong(b.ne) &&
                    __double_as_longlong(dinv[d]) == __double_as_longlong(dinv[d0]);
  if (!same) atomicAnd(flag, 0);
}

}  // namespace

std::int64_t csr_nnz(const Level& L) {
  if (L.deg == 2) return L.p2nnz;
  if (L.hole.any())  // diagonal per vertex + 2 per mesh edge, E = (3T + B) / 2
    return L.nv + 3 * L.nt + L.nb;
  const std::int64_t n = L.nx, m = L.ny;
  // sum over rows: (3nx+1)(ny+1) + (2nx+1)*2ny
  return (3 * n + 1) * (m + 1) + (2 * n + 1) * 2 * m;
}

void assemble_level(Ctx& c, Level& L) {
  if (L.deg == 2) {  // P2 operators on the half lattice (p2.cu)
    assemble_p2(c, L);
    return;
  }
  const std::int64_t nd = L.ndofs();
  L.stA.alloc(nd);
  L.stM.alloc(nd);
  L.dinv.alloc(nd);
  LevelGeom G{L.nx, L.ny, c.cfg.x_min, c.cfg.y_min, L.dx, L.dy, L.geo.get()};
  DevBuf<double> tab;  // element-matrix table of k_assemble_table (outlives the event pair)
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  if (c.profile) {  // roofline evidence: the assembly launch alone
    ev0 = c.event(0);
    ev1 = c.event(1);
    MLG_CUDA(cudaEventRecord(ev0, c.stream));
  }
  if (c.cfg.example == 1) {
    {  // make_degree6 (fespace.cpp:49-75), same point order
      const double a1 = 0.501426509658179, b1 = 0.249286745170910, w1 = 0.116786275726379;
      const double a2 = 0.873821971016996, b2 = 0.063089014491502, w2 = 0.050844906370207;
      const double a3 = 0.053145049844816, b3 = 0.310352451033785, c3 = 0.636502499121399,
                   w3 = 0.082851075618374;
      const double q[12][4] = {{a1, b1, b1, w1}, {b1, a1, b1, w1}, {b1, b1, a1, w1},
                               {a2, b2, b2, w2}, {b2, a2, b2, w2}, {b2, b2, a2, w2},
                               {a3, b3, c3, w3}, {a3, c3, b3, w3}, {b3, a3, c3, w3},
                               {b3, c3, a3, w3}, {c3, a3, b3, w3}, {c3, b3, a3, w3}};
      MLG_CUDA(cudaMemcpyToSymbolAsync(kQ6, q, sizeof(q), 0, cudaMemcpyHostToDevice,
                                       c.stream));
      c.sync();  // q is a host temporary
    }
    k_assemble_var<<<grid_for(nd, kBlock), kBlock, 0, c.stream>>>(G, L.stA.get(), L.stM.get(),
                                                                  L.dinv.get());
  } else if (c.cfg.example == 2) {
    reaction_modes(c.cfg.seed, &G.k1, &G.k2);
    k_assemble<2><<<grid_for(nd, kBlock), kBlock, 0, c.stream>>>(G, L.stA.get(), L.stM.get(),
                                                                 L.dinv.get());
  } else {
    // translation-invariant lattice (all column steps bitwise equal, all row
    // steps bitwise equal): table-driven kernel, else the generic gather
    const char* tenv = std::getenv("MLG_ASSEMBLE_TABLE");  // A/B and test hook: 0 disables
    const bool no_table = tenv && tenv[0] == '0';
    int uniform_steps = 0;
    if (!no_table) {
      DevBuf<int> flag(1);
      const int one = 1;
      flag.upload(&one, 1, c.stream);
      k_lattice_steps<<<grid_for(std::max(L.nx, L.ny), kBlock), kBlock, 0, c.stream>>>(
          G, flag.get());
      MLG_LAUNCH_CHECK();
      flag.download(&uniform_steps, 1, c.stream);
      c.sync();
    }
    L.asm_table = uniform_steps;
    if (uniform_steps) tab.alloc(2 * kTabEntries);
    if (c.profile) MLG_CUDA(cudaEventRecord(ev0, c.stream));  // the assembly launches alone
    if (uniform_steps) {
      k_assemble_table_build<<<1, 64, 0, c.stream>>>(G, tab.get());
      MLG_LAUNCH_CHECK();
    }
    if (uniform_steps && (static_cast<std::uint64_t>(L.nt) << 6) < 0xFFFFFFFFull)
      k_assemble_table<unsigned><<<grid_for(nd, kBlock), kBlock, 0, c.stream>>>(
          G, tab.get(), L.stA.get(), L.stM.get(), L.dinv.get());
    else if (uniform_steps)
      k_assemble_table<unsigned long long><<<grid_for(nd, kBlock), kBlock, 0, c.stream>>>(
          G, tab.get(), L.stA.get(), L.stM.get(), L.dinv.get());
    else
      k_assemble<0><<<grid_for(nd, kBlock), kBlock, 0, c.stream>>>(G, L.stA.get(), L.stM.get(),
                                                                   L.dinv.get());
  }
  MLG_LAUNCH_CHECK();
  if (c.profile) {
    MLG_CUDA(cudaEventRecord(ev1, c.stream));
    MLG_CUDA(cudaEventSynchronize(ev1));
    float ms = 0.f;
    MLG_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
    c.asm_ms = ms;
    c.asm_dofs = static_cast<double>(nd);
    c.asm_kernel = c.cfg.example == 1 ? 2 : L.asm_table;
  }
  // Constant-coefficient detection for the CG fast path (MLG_GENERAL_STENCIL=1
  // forces the general per-row path, used by the tests to cover both).
  L.uniform = 0;
  if (L.hole.any()) {  // CG operator with identity rows on the non-interior points
    L.stCG.alloc(nd);
    L.dinvCG.alloc(nd);
    k_cg_stencil<<<grid_for(nd, kBlock), kBlock, 0, c.stream>>>(L.imap(), L.stA.get(),
                                                                L.dinv.get(), L.stCG.get(),
                                                                L.dinvCG.get());
    MLG_LAUNCH_CHECK();
    // the CG sweeps exclude the closed hole (its points and the re-entrant
    // edges) by geometry, so the fast path applies when the interior rows agree
    L.strip_geom.hx0 = L.hole.x0;
    L.strip_geom.hx1 = L.hole.x1;
    L.strip_geom.hy0 = L.hole.y0;
    L.strip_geom.hy1 = L.hole.y1;
  }
  const char* env = std::getenv("MLG_GENERAL_STENCIL");
  const IMap im = L.imap();
  if (L.nx >= 2 && L.ny >= 2 && im.count() > 0 && !(env && env[0] == '1')) {
    DevBuf<int> flag(1);
    const int one = 1;
    flag.upload(&one, 1, c.stream);
    k_uniform_check<<<grid_for(im.count(), kBlock), kBlock, 0, c.stream>>>(
        im, L.stA.get(), L.dinv.get(), flag.get());
    MLG_LAUNCH_CHECK();
    int f = 0;
    flag.download(&f, 1, c.stream);
    int ix0, iy0;
    im.point(0, &ix0, &iy0);
    const std::int64_t d0 = static_cast<std::int64_t>(iy0) * (L.nx + 1) + ix0;
    MLG_CUDA(cudaMemcpyAsync(&L.ust, L.stA.get() + d0, sizeof(Stencil), cudaMemcpyDeviceToHost,
                             c.stream));
    MLG_CUDA(cudaMemcpyAsync(&L.udinv, L.dinv.get() + d0, sizeof(double),
                             cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    L.uniform = f;
  }
}

void export_csr(Ctx& c, const Level& L, int form, int* row_ptr, int* cols, double* vals) {
  if (L.deg == 2) {
    export_csr_p2(c, L, form, row_ptr, cols, vals);
    return;
  }
  if (L.hole.any()) {
    const std::int64_t nd = L.ndofs();
    DevBuf<int> cnt(nd + 1), rp(nd + 1);
    k_csr_count_hole<<<grid_for(nd + 1, kBlock), kBlock, 0, c.stream>>>(L.nx, L.ny, L.hole,
                                                                       cnt.get());
    MLG_LAUNCH_CHECK();
    std::size_t tb = 0;
    MLG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.get(), rp.get(),
                                           static_cast<int>(nd + 1), c.stream));
    void* tmp = c.scratch_bytes(tb);
    MLG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt.get(), rp.get(), static_cast<int>(nd + 1),
                                           c.stream));
    int nnz = 0;
    MLG_CUDA(cudaMemcpyAsync(&nnz, rp.get() + nd, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    DevBuf<int> cl(cols ? nnz : 0);
    DevBuf<double> vl(vals ? nnz : 0);
    k_export_csr_hole<<<grid_for(nd, kBlock), kBlock, 0, c.stream>>>(
        L.nx, L.ny, L.hole, form == 0 ? L.stA.get() : L.stM.get(), rp.get(),
        cols ? cl.get() : nullptr, vals ? vl.get() : nullptr);
    MLG_LAUNCH_CHECK();
    if (row_ptr) rp.download(row_ptr, nd + 1, c.stream);
    if (cols) cl.download(cols, nnz, c.stream);
    if (vals) vl.download(vals, nnz, c.stream);
    c.sync();
    return;
  }
  const std::int64_t nd = L.ndofs(), nnz = csr_nnz(L);
  DevBuf<int> rp(row_ptr ? nd + 1 : 0), cl(cols ? nnz : 0);
  DevBuf<double> vl(vals ? nnz : 0);
  k_export_csr<<<grid_for(nd + 1, kBlock), kBlock, 0, c.stream>>>(
      L.nx, L.ny, nnz, form == 0 ? L.stA.get() : L.stM.get(), row_ptr ? rp.get() : nullptr,
      cols ? cl.get() : nullptr, vals ? vl.get() : nullptr);
  MLG_LAUNCH_CHECK();
  if (row_ptr) rp.download(row_ptr, nd + 1, c.stream);
  if (cols) cl.download(cols, nnz, c.stream);
  if (vals) vl.download(vals, nnz, c.stream);
  c.sync();
}

void interior_dense(Ctx& c, const Level& L, int form, double* d_dense) {
  if (L.deg == 2) {
    interior_dense_p2(c, L, form, d_dense);
    return;
  }
  const std::int64_t n = L.nint();
  MLG_CUDA(cudaMemsetAsync(d_dense, 0, sizeof(double) * n * n, c.stream));
  k_interior_dense<<<grid_for(n, kBlock), kBlock, 0, c.stream>>>(
      L.imap(), form == 0 ? L.stA.get() : L.stM.get(), d_dense);
  MLG_LAUNCH_CHECK();
}

}  // namespace mlg

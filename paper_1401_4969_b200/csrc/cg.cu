// Batched Jacobi-PCG (sparse.cpp:199-258) for lattice-window systems: ONE
// launch per CG iteration for all systems of a batch.
//
// Iteration scheme (the one-reduction rearrangement of PCG; same iterates in
// exact arithmetic, reductions in a fixed order):  launch k applies the
// pending update of iteration k-1 and prepares iteration k in a single sweep:
//     q_old = A p_old              (recomputed, never stored)
//     r = r - alpha q_old,  x = x + alpha p_old,  z = D^-1 r
//     p = z + beta p_old,   q = A p
//     partials  r.r, r.z, p.q, q.z, q.D^-1 q
// The tile that finishes last reduces the partials of its system and sets
// alpha = rho / p.q with rho = r.z (exact), rho_next = rho - 2 alpha q.z +
// alpha^2 q.D^-1q (so beta = rho_next / rho is known before the next sweep),
// and applies the reference's stopping rule: ||r|| <= tol ||b|| triggers a
// true-residual launch (b - A x; restart from it if it fails, sparse.cpp:232-246).
// Per row and iteration this moves x, r, p in and out (48 B) instead of the
// 80 B of the classic two-kernel form, and needs one launch instead of two.
//
// Memory pattern (B200): each warp sweeps a 32-column strip of its window
// upwards; the two stencil applications use a 4-row register window of the old
// iterate and a 3-row window of the new p, neighbours in x from warp shuffles,
// so every value is read from HBM once per iteration.  Lanes 2..29 produce
// output; lanes 0,1,30,31 are the strip's 2-deep halo.  When the level's
// interior stiffness rows are bitwise identical (UNI: constant-coefficient
// lattice) the stencil and D^-1 come from kernel parameters.
//
// Partial sums are reduced in a fixed order by whichever tile finishes last
// (no floating-point atomics): results are run-to-run bitwise deterministic
// (SURVEY finding 10).  Every system stops independently; tiles of finished
// systems are dropped between chunks.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <queue>
#include <type_traits>

#include "cg.cuh"
#include "cg_ctl.cuh"
#include "stencil.cuh"

namespace mlg {
namespace {

constexpr int kBlock = CgBatch::kBlock;
// Persistent kernel: systems with at most this many tiles are reduced
// redundantly by every CTA holding one of their tiles after the grid barrier;
// larger systems keep the last-tile reduction before it (reading hundreds of
// partials per CTA costs more than the atomic round trip).
#ifndef MLG_CG_REPL
#define MLG_CG_REPL 96
#endif
constexpr int kReplTiles = MLG_CG_REPL;
constexpr unsigned kFull = 0xffffffffu;

#ifdef MLG_CG_TRACE
__device__ unsigned long long g_trace[4096][8];  // per-CTA timestamps of one iteration
__device__ unsigned g_kind[4096];                // per-CTA tile kinds (persistent kernel)
#endif

// Iterate loads.  The persistent kernel (CG) re-reads rows that other CTAs
// rewrote in an earlier iteration of the same launch, so it must bypass the
// (non-coherent) L1: ld.global.cg.
template <bool CG>
__device__ __forceinline__ double ldv(const double* p) {
  if constexpr (CG)
    return __ldcg(p);
  else
    return *p;
}

struct SweepArgs {
  const Stencil* st;
  const double* dinv;
  int nxp1;
  const unsigned char* mask;  // non-null: system restricted to the strip
  StripGeom sg;               // closed form of that restriction (no mask loads)
  Stencil ust;                // interior stencil when the level is uniform
  double udinv;
  const int* task_map;        // compacted task lists (systems with tmap_off >= 0)
};

// Strip membership of fine lattice point (ix, iy): not in the closed inner
// region G_j of its block (decomp.cpp:73-80, 204-211); G_j never touches an
// interior block side, so the block found by division is the only candidate.
__device__ __forceinline__ bool in_strip(const StripGeom& g, int ix, int iy) {
  const int bx = min(ix / (g.bw * g.scale), g.side - 1);
  const int by = min(iy / (g.bh * g.scale), g.side - 1);
  const int x0 = (bx == 0 ? 0 : bx * g.bw + g.dc) * g.scale;
  const int x1 = (bx == g.side - 1 ? g.nx0 : (bx + 1) * g.bw - g.dc) * g.scale;
  const int y0 = (by == 0 ? 0 : by * g.bh + g.dc) * g.scale;
  const int y1 = (by == g.side - 1 ? g.ny0 : (by + 1) * g.bh - g.dc) * g.scale;
  return !(ix >= x0 && ix <= x1 && iy >= y0 && iy <= y1) && !g.in_hole(ix, iy);
}

// Old iterate at one row of the lane's column.
struct ORow {
  double p, r, x, dv;
  Stencil st;
  int in;
};
// New p (and z) at one row.
struct NRow {
  double p, z, dv;
  Stencil st;
  int in;
};

struct Task {
  bool valid;
  int col, ly0, ly1;
};

__device__ __forceinline__ Task task_of(const CgSys& S, int t, const int* task_map) {
  Task k;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int task = t * kCgWarps + warp;
  k.valid = task < S.ntasks;
  if (k.valid && S.tmap_off >= 0) task = task_map[S.tmap_off + task];
  const int rb = k.valid ? task / S.nstrips : 0;
  const int strip = k.valid ? task % S.nstrips : 0;
  k.col = strip * kCgCols - 2 + lane;
  k.ly0 = rb * S.krows;
  k.ly1 = min(k.ly0 + S.krows, S.h);
  return k;
}

__device__ __forceinline__ bool out_lane(const CgSys& S, const Task& k) {
  const int lane = threadIdx.x & 31;
  return k.valid && lane >= 2 && lane < 2 + kCgCols && k.col < S.w;
}

template <bool UNI>
__device__ __forceinline__ void load_old(const CgSys& S, const SweepArgs& A, int col, int ly,
                                         const double* Rc, const double* Pc, const double* X,
                                         ORow& o) {
  o.p = o.r = o.x = 0.0;
  o.in = 0;
  if constexpr (!UNI) {
    o.st = Stencil{0.0, 0.0, 0.0, 0.0};
    o.dv = 0.0;
  }
  if (col < 0 || col >= S.w || ly < 0 || ly >= S.h) return;
  const long long g = static_cast<long long>(S.y0 + ly) * A.nxp1 + (S.x0 + col);
  if (A.mask ? !in_strip(A.sg, S.x0 + col, S.y0 + ly) : A.sg.in_hole(S.x0 + col, S.y0 + ly))
    return;
  o.in = 1;
  if constexpr (!UNI) {
    o.st = A.st[g];
    o.dv = A.dinv[g];
  }
  const long long v = cg_index(S, ly, col);
  o.p = Pc[v];
  o.r = Rc[v];
  o.x = X[v];
}

// Row product of the window-restricted matrix at the centre row of a 3-row
// register window, terms in CSR column order SW,S,W,C,E,N,NE (sparse.cpp:69-76),
// each rounded separately.  A coefficient is only used when its neighbour is
// inside the system (an interior row), so the uniform stencil is exact there.
template <bool UNI>
__device__ __forceinline__ double product(double sv, const Stencil& sst, int sin_, double cv,
                                          const Stencil& cst, int cin, double nv, int nin,
                                          const SweepArgs& A) {
  const Stencil& cs = UNI ? A.ust : cst;
  const double sn = UNI ? A.ust.n : sst.n;
  const double wa = UNI ? A.ust.e : __shfl_up_sync(kFull, cst.e, 1);
  const double swa = UNI ? A.ust.ne : __shfl_up_sync(kFull, sst.ne, 1);
  const int win = __shfl_up_sync(kFull, cin, 1);
  const int ein = __shfl_down_sync(kFull, cin, 1);
  const int swin = __shfl_up_sync(kFull, sin_, 1);
  const int nein = __shfl_down_sync(kFull, nin, 1);
  const double wv = __shfl_up_sync(kFull, cv, 1);
  const double ev = __shfl_down_sync(kFull, cv, 1);
  const double swv = __shfl_up_sync(kFull, sv, 1);
  const double nev = __shfl_down_sync(kFull, nv, 1);
  double a = 0.0;
  if (swin) a = xadd(a, xmul(swa, swv));
  if (sin_) a = xadd(a, xmul(sn, sv));
  if (win) a = xadd(a, xmul(wa, wv));
  a = xadd(a, xmul(cs.c, cv));
  if (ein) a = xadd(a, xmul(cs.e, ev));
  if (nin) a = xadd(a, xmul(cs.n, nv));
  if (nein) a = xadd(a, xmul(cs.ne, nev));
  return a;
}

// ---- interior fast path (constant-coefficient lattice) ----------------------
// A warp task whose 32 columns and rows ly0-2 .. ly1+1 all lie inside its
// system needs no bounds, mask or presence tests: every neighbour exists and
// the row product is the full 7-term sum (same terms, same order, same
// rounding as the general path).

// Closed rectangle [xa,xb] x [ya,yb] (fine lattice) entirely inside the strip.
__device__ __forceinline__ bool rect_in_strip(const StripGeom& g, int xa, int xb, int ya,
                                              int yb) {
  if (g.rect_meets_hole(xa, xb, ya, yb)) return false;
  const int bxa = min(xa / (g.bw * g.scale), g.side - 1);
  const int bxb = min(xb / (g.bw * g.scale), g.side - 1);
  const int bya = min(ya / (g.bh * g.scale), g.side - 1);
  const int byb = min(yb / (g.bh * g.scale), g.side - 1);
  for (int bx = bxa; bx <= bxb; ++bx)
    for (int by = bya; by <= byb; ++by) {
      const int x0 = (bx == 0 ? 0 : bx * g.bw + g.dc) * g.scale;
      const int x1 = (bx == g.side - 1 ? g.nx0 : (bx + 1) * g.bw - g.dc) * g.scale;
      const int y0 = (by == 0 ? 0 : by * g.bh + g.dc) * g.scale;
      const int y1 = (by == g.side - 1 ? g.ny0 : (by + 1) * g.bh - g.dc) * g.scale;
      if (xa <= x1 && xb >= x0 && ya <= y1 && yb >= y0) return false;
    }
  return true;
}

__device__ __forceinline__ bool task_interior(const CgSys& S, const SweepArgs& A, const Task& k) {
  const int lane = threadIdx.x & 31;
  const int c0 = k.col - lane;  // column of lane 0 (warp-uniform)
  if (c0 < 0 || c0 + 31 >= S.w || k.ly0 - 2 < 0 || k.ly1 + 1 >= S.h) return false;
  if (A.sg.rect_meets_hole(S.x0 + c0, S.x0 + c0 + 31, S.y0 + k.ly0 - 2, S.y0 + k.ly1 + 1))
    return false;
  if (A.mask)
    return rect_in_strip(A.sg, S.x0 + c0, S.x0 + c0 + 31, S.y0 + k.ly0 - 2, S.y0 + k.ly1 + 1);
  return true;
}

__device__ __forceinline__ double product_full(double sv, double cv, double nv,
                                               const Stencil& u) {
  const double wv = __shfl_up_sync(kFull, cv, 1);
  const double ev = __shfl_down_sync(kFull, cv, 1);
  const double swv = __shfl_up_sync(kFull, sv, 1);
  const double nev = __shfl_down_sync(kFull, nv, 1);
  // Constant coefficients are symmetric (W/E share e, S/N share n, SW/NE
  // share ne): pair the neighbours and fuse -- dependency depth 4 instead of
  // 14.  (Inside CG only; the exported SpMV keeps the reference's order.)
  return fma(u.e, wv + ev, fma(u.n, sv + nv, fma(u.ne, swv + nev, u.c * cv)));
}

// Constant-coefficient sweep for ANY task (window edges, strip mask): the
// in-system flag of (column, row) is separable -- column inside the window and
// outside its block's G x-range, row inside the window and outside its block's
// G y-range -- so it costs a few integer ops per row, no memory traffic.
// Presence of W/E/SW/NE neighbours comes from shuffled flags.
__device__ __forceinline__ double product_flags(double sv, int sin_, double cv, int cin,
                                                double nv, int nin, const Stencil& u) {
  const int win = __shfl_up_sync(kFull, cin, 1);
  const int ein = __shfl_down_sync(kFull, cin, 1);
  const int swin = __shfl_up_sync(kFull, sin_, 1);
  const int nein = __shfl_down_sync(kFull, nin, 1);
  const double wr = __shfl_up_sync(kFull, cv, 1);
  const double er = __shfl_down_sync(kFull, cv, 1);
  const double swr = __shfl_up_sync(kFull, sv, 1);
  const double ner = __shfl_down_sync(kFull, nv, 1);
  const double wv = win ? wr : 0.0, ev = ein ? er : 0.0;
  const double swv = swin ? swr : 0.0, nev = nein ? ner : 0.0;
  const double s = sin_ ? sv : 0.0, n = nin ? nv : 0.0;
  // same pairing as product_full (identical result when every neighbour exists)
  return fma(u.e, wv + ev, fma(u.n, s + n, fma(u.ne, swv + nev, u.c * cv)));
}

struct Flags {
  int cin;   // this lane's column is in the window
  int gx;    // ... and inside its block's G x-range (masked systems)
  int hx;    // ... and inside the hole's x-range (domains with a hole)
  int masked;
  int h;
  int y0;    // window origin (fine lattice row of window row 0)
  // g: the kernel parameter's StripGeom (read in place, not copied)
  __device__ __forceinline__ int row_in(int ly, const StripGeom& g) const {
    if (!cin || ly < 0 || ly >= h) return 0;
    const int iy = y0 + ly;
    if (hx && iy >= g.hy0 && iy <= g.hy1) return 0;
    if (!masked || !gx) return 1;
    const int by = min(iy / (g.bh * g.scale), g.side - 1);
    const int ya = (by == 0 ? 0 : by * g.bh + g.dc) * g.scale;
    const int yb = (by == g.side - 1 ? g.ny0 : (by + 1) * g.bh - g.dc) * g.scale;
    return (iy >= ya && iy <= yb) ? 0 : 1;
  }
};

__device__ __forceinline__ Flags make_flags(const CgSys& S, const SweepArgs& A, const Task& k) {
  Flags f;
  f.cin = k.col >= 0 && k.col < S.w;
  f.masked = A.mask != nullptr;
  f.h = S.h;
  f.y0 = S.y0;
  f.gx = 0;
  {
    const int ix = S.x0 + k.col;
    f.hx = f.cin && ix >= A.sg.hx0 && ix <= A.sg.hx1;
  }
  if (f.masked && f.cin) {
    const StripGeom& g = A.sg;
    const int ix = S.x0 + k.col;
    const int bx = min(ix / (g.bw * g.scale), g.side - 1);
    const int xa = (bx == 0 ? 0 : bx * g.bw + g.dc) * g.scale;
    const int xb = (bx == g.side - 1 ? g.nx0 : (bx + 1) * g.bw - g.dc) * g.scale;
    f.gx = (ix >= xa && ix <= xb) ? 1 : 0;
  }
  return f;
}

// True residual r = b - A x of a constant-coefficient system (x current).
template <bool CG>
__device__ __forceinline__ void check_sweep_uni(const CgSys& S, const SweepArgs& A,
                                                const Task& k, const double* bsrc, int bstride,
                                                const double* __restrict__ X,
                                                double* __restrict__ Rn,
                                                double (&acc)[kCgDots]) {
  const int lane = threadIdx.x & 31;
  const Flags f = make_flags(S, A, k);
  const bool out_col = lane >= 2 && lane < 2 + kCgCols && f.cin;
  const long long base = S.voff + k.col;
  const double* __restrict__ Xs = X + base;
  double* __restrict__ Rns = Rn + base;
  auto ld = [&](int ly, int in) -> double {
    return in ? ldv<CG>(Xs + static_cast<long long>(ly) * S.pitch) : 0.0;
  };
  int ia = f.row_in(k.ly0 - 1, A.sg), ib = f.row_in(k.ly0, A.sg);
  double xa = ld(k.ly0 - 1, ia), xb = ld(k.ly0, ib);
  for (int ly = k.ly0; ly < k.ly1; ++ly) {
    const int ic = f.row_in(ly + 1, A.sg);
    const double xc = ld(ly + 1, ic);
    const double ax = product_flags(xa, ia, xb, ib, xc, ic, A.ust);
    if (out_col && ib) {
      const long long g = static_cast<long long>(S.y0 + ly) * A.nxp1 + (S.x0 + k.col);
      const double rt = bsrc[g * bstride + S.rhs] - ax;
      Rns[static_cast<long long>(ly) * S.pitch] = rt;
      acc[0] += rt * rt;
    }
    xa = xb;
    ia = ib;
    xb = xc;
    ib = ic;
  }
}

// Row product inside the CG sweeps.  LAP: the
// level's interior stencil is the 5-point Laplacian {4, -1, -1, 0} with
// D^-1 = 1/4 (P1 on the right-triangle lattice): constants are immediates and
// the zero SW/NE pair is skipped -- fma(0, s, y) == y for finite s, so the
// row product is bitwise the generic paired-FMA product.
// Lateral neighbours through a per-warp shared-memory exchange instead of
// warp shuffles: one 64-bit store, __syncwarp, two 64-bit loads (4 instructions
// per value instead of 4 SHFL + 3 LOP3), and no divergence check (BRA.DIV) in
// front of each shuffle group -- ptxas attaches the waits for outstanding
// global loads to it, which defeated the row prefetch.  Slot 0 serves the
// stage-1 product, slot 1 the stage-2 product; a slot is rewritten only after
// the other slot's __syncwarp, so every lane has read it.
// (Measured: +4 % at config 2 in the register pipeline; -2 % at config 5 in
// the cp.async pipeline, whose shared-memory traffic it competes with, so the
// latter keeps the shuffles.)
struct Xchg {
  double v[2][32];
};

// The warp barrier is a named CTA barrier with a count of 32 (`bar.sync
// 1+warp, 32` -> BAR.SYNC): __syncwarp compiles to a divergence check
// (BRA.DIV) at which ptxas waits for every outstanding global load.
struct Lat {  // a lane's view of its warp's exchange buffer
  double* self;
  const double* west;
  const double* east;
  int bar;
  __device__ __forceinline__ Lat(Xchg& x, int slot) {
    const int lane = threadIdx.x & 31;
    self = &x.v[slot][lane];
    west = &x.v[slot][(lane - 1) & 31];
    east = &x.v[slot][(lane + 1) & 31];
    bar = 1 + (threadIdx.x >> 5);
  }
  __device__ __forceinline__ void get(double c, double& w, double& e) const {
    *self = c;
    asm volatile("bar.sync %0, 32;" ::"r"(bar) : "memory");
    w = *west;
    e = *east;
  }
};

template <bool LAP, bool SMX>
__device__ __forceinline__ double product_lat(double sv, double cv, double nv, const Stencil& u,
                                              const Lat& lat) {
  if constexpr (LAP && SMX) {
    double wv, ev;
    lat.get(cv, wv, ev);
    return fma(-1.0, wv + ev, fma(-1.0, sv + nv, 4.0 * cv));
  } else {
    const double wv = __shfl_up_sync(kFull, cv, 1);
    const double ev = __shfl_down_sync(kFull, cv, 1);
    if constexpr (LAP) return fma(-1.0, wv + ev, fma(-1.0, sv + nv, 4.0 * cv));
    const double swv = __shfl_up_sync(kFull, sv, 1);
    const double nev = __shfl_down_sync(kFull, nv, 1);
    return fma(u.e, wv + ev, fma(u.n, sv + nv, fma(u.ne, swv + nev, u.c * cv)));
  }
}

template <bool LAP>
__device__ __forceinline__ double product_int(double sv, double cv, double nv, const Stencil& u) {
  const double wv = __shfl_up_sync(kFull, cv, 1);
  const double ev = __shfl_down_sync(kFull, cv, 1);
  if constexpr (LAP) {
    return fma(-1.0, wv + ev, fma(-1.0, sv + nv, 4.0 * cv));
  } else {
    const double swv = __shfl_up_sync(kFull, sv, 1);
    const double nev = __shfl_down_sync(kFull, nv, 1);
    return fma(u.e, wv + ev, fma(u.n, sv + nv, fma(u.ne, swv + nev, u.c * cv)));
  }
}

// In-system test of the window rows one task touches, without per-row
// division: the G row intervals of the (at most three) lattice blocks the
// task's rows fall in are precomputed; tasks spanning more blocks (tiny
// levels) fall back to Flags::row_in.
struct RowMask {
  int h, cin, gx, slow, hx;
  int ya0, yb0, ya1, yb1, ya2, yb2;  // window-row intervals of G (closed; empty = (1, 0))
  int yh0, yh1;                      // window-row interval of the hole (closed; empty = (1, 0))
  // SLOW: tasks spanning > 3 blocks (tiny levels only); MASKED: strip systems
  template <bool SLOW, bool MASKED = true>
  __device__ __forceinline__ bool in(int r, const Flags& f, const StripGeom& g) const {
    if (SLOW) return f.row_in(r, g) != 0;
    const bool rowok = static_cast<unsigned>(r) < static_cast<unsigned>(h);
    const bool inh = hx & (r >= yh0) & (r <= yh1);
    if (!MASKED) return cin & rowok & !inh;
    const bool ing = (r >= ya0 & r <= yb0) | (r >= ya1 & r <= yb1) | (r >= ya2 & r <= yb2);
    return cin & rowok & !(gx & ing) & !inh;
  }
};

__device__ __forceinline__ RowMask make_rowmask(const CgSys& S, const SweepArgs& A, const Task& k,
                                                const Flags& f) {
  RowMask m;
  m.h = S.h;
  m.cin = f.cin;
  m.gx = f.masked && f.gx;
  m.slow = 0;
  m.ya0 = m.ya1 = m.ya2 = 1;
  m.yb0 = m.yb1 = m.yb2 = 0;
  m.hx = f.hx;
  m.yh0 = A.sg.hy0 - S.y0;
  m.yh1 = A.sg.hy1 - S.y0;
  if (f.masked) {
    const StripGeom& g = A.sg;
    const int bhs = g.bh * g.scale;
    const int r0 = max(k.ly0 - 2, 0), r1 = min(k.ly1 + 4, S.h - 1);
    const int by0 = min((S.y0 + r0) / bhs, g.side - 1);
    const int by1 = min((S.y0 + r1) / bhs, g.side - 1);
    m.slow = by1 - by0 > 2;
    auto lo = [&](int by) { return (by == 0 ? 0 : by * g.bh + g.dc) * g.scale - S.y0; };
    auto hi = [&](int by) { return (by == g.side - 1 ? g.ny0 : (by + 1) * g.bh - g.dc) * g.scale - S.y0; };
    m.ya0 = lo(by0);
    m.yb0 = hi(by0);
    if (by0 + 1 <= by1) {
      m.ya1 = lo(by0 + 1);
      m.yb1 = hi(by0 + 1);
    }
    if (by0 + 2 <= by1) {
      m.ya2 = lo(by0 + 2);
      m.yb2 = hi(by0 + 2);
    }
  }
  return m;
}

// Register sweep, modulo-scheduled by hand.  The kW-row window of old p, r, x
// (rows n-1 .. n+kW-2) lives in slot (row - ly0 + 2) mod kW of register
// arrays; the step for row n (J = slot of row n-1) consumes slots J, J+1, J+2
// and refills slot J with row n+kW-1.  Nothing is ever copied, so no
// instruction waits on a row before it is consumed (kW-2 steps after it was
// requested); a rotating window compiled as register moves stalls on every
// new load.
//   EDGE = false: the task's stencil rectangle lies inside its system, no tests.
//   EDGE = true: window-edge / strip-boundary task.  The zero frame of the
//     pooled vectors makes reads outside the window zeros and points of G hold
//     zeros, so loads need no tests; r, z, p and q of points outside the
//     system are forced to zero -- an absent neighbour then contributes a
//     literal 0 to the same paired-FMA chain (bitwise the flagged product) and
//     every dot term of such a point is an exact zero.
// Every lane accumulates; the halo lanes' sums are dropped at the end, so the
// only per-row predicate guards the three stores.
template <int... Is, typename Fn>
__device__ __forceinline__ void static_for(std::integer_sequence<int, Is...>, Fn&& fn) {
  (fn(std::integral_constant<int, Is>{}), ...);
}

#ifndef MLG_CG_W
#define MLG_CG_W 5
#endif
constexpr int kW = MLG_CG_W;  // register window rows (prefetch distance kW - 2 steps)

template <bool RST, bool CG, bool LAP, bool EDGE, bool SLOW, bool MASKED = true>
__device__ __forceinline__ void sweep_reg(const CgSys& S, const SweepArgs& A, const Task& k,
                                          double al, double be, double* __restrict__ X,
                                          const double* __restrict__ Rc,
                                          double* __restrict__ Rn,
                                          const double* __restrict__ Pc,
                                          double* __restrict__ Pn, double (&acc)[kCgDots],
                                          Xchg& xch) {
  const Lat lat1(xch, 0), lat2(xch, 1);
  const int lane = threadIdx.x & 31;
  const Flags f = make_flags(S, A, k);          // EDGE only
  const RowMask rm = make_rowmask(S, A, k, f);  // EDGE only
  const bool own = lane >= 2 && lane < 2 + kCgCols && (!EDGE || f.cin);
  const long long w = S.pitch;
  long long lo = cg_index(S, k.ly0 - 2, k.col);  // next row to request
  long long so = lo + 2 * w;                      // next row to store (ly0)
  const Stencil u = A.ust;
  const double dv = LAP ? 0.25 : A.udinv;
  double P[kW], Rr[kW], Xr[kW];
#pragma unroll
  for (int j = 0; j < kW; ++j) {  // rows ly0-2 .. ly0+kW-3
    P[j] = ldv<CG>(Pc + lo);
    Rr[j] = ldv<CG>(Rc + lo);
    Xr[j] = ldv<CG>(X + lo);
    lo += w;
  }
  double sp = 0.0, mp = 0.0, mz = 0.0;  // new p at rows n-2, n-1; z at n-1
  bool m_in = false;
  auto step = [&](auto J, auto store, auto stage2, int n) {
    constexpr int j0 = decltype(J)::value % kW, j1 = (j0 + 1) % kW, j2 = (j0 + 2) % kW;
    bool b_in = true;
    if constexpr (EDGE) b_in = rm.template in<SLOW, MASKED>(n, f, A.sg);
    double rn = Rr[j1], xn = Xr[j1];
    if constexpr (!RST) {
      const double qo = product_lat<LAP, true>(P[j0], P[j1], P[j2], u, lat1);
      rn = fma(-al, qo, Rr[j1]);
      xn = fma(al, P[j1], Xr[j1]);
    }
    if constexpr (EDGE) rn = b_in ? rn : 0.0;
    const double tz = xmul(dv, rn);
    double tp = RST ? tz : fma(be, P[j1], tz);
    if constexpr (EDGE) tp = b_in ? tp : 0.0;
    P[j0] = ldv<CG>(Pc + lo);  // slot of row n-1 is free: request row n+kW-1
    Rr[j0] = ldv<CG>(Rc + lo);
    Xr[j0] = ldv<CG>(X + lo);
    lo += w;
    if constexpr (decltype(store)::value) {
      if (own && b_in) {
        X[so] = xn;
        Rn[so] = rn;
        Pn[so] = tp;
      }
      so += w;
      acc[0] += rn * rn;
      acc[1] += rn * tz;
    }
    if constexpr (decltype(stage2)::value) {  // q = A p_new at row n-1
      double q = product_lat<LAP, true>(sp, mp, tp, u, lat2);
      if constexpr (EDGE) q = m_in ? q : 0.0;
      acc[2] += mp * q;
      acc[3] += q * mz;
      acc[4] += q * xmul(dv, q);
    }
    sp = mp;
    mp = tp;
    mz = tz;
    m_in = b_in;
  };
  using T = std::true_type;
  using F = std::false_type;
  step(std::integral_constant<int, 0>{}, F{}, F{}, k.ly0 - 1);  // stage 1 only
  step(std::integral_constant<int, 1>{}, T{}, F{}, k.ly0);
  int n = k.ly0 + 1;  // slot phase 2
  using Seq = std::make_integer_sequence<int, kW>;
#pragma unroll 1
  for (; n + kW - 1 < k.ly1; n += kW)
    static_for(Seq{}, [&](auto i) {
      constexpr int ii = decltype(i)::value;
      step(std::integral_constant<int, (2 + ii) % kW>{}, T{}, T{}, n + ii);
    });
  const int rem = k.ly1 - n;  // 0..kW-1 rows left, then row ly1 (stage 2 only)
  static_for(std::make_integer_sequence<int, kW - 1>{}, [&](auto i) {
    constexpr int ii = decltype(i)::value;
    if (ii < rem) step(std::integral_constant<int, (2 + ii) % kW>{}, T{}, T{}, n + ii);
  });
  static_for(Seq{}, [&](auto r) {
    constexpr int rr = decltype(r)::value;
    if (rr == rem) step(std::integral_constant<int, (2 + rr) % kW>{}, F{}, T{}, k.ly1);
  });
  if (!own) {  // halo lanes (and columns outside the window) contribute nothing
#pragma unroll
    for (int q = 0; q < kCgDots; ++q) acc[q] = 0.0;
  }
}

// ---- general-stencil interior fast path -------------------------------------
// Variable-coefficient levels, tasks whose 32 columns and rows ly0-2 .. ly1+1
// lie inside the system (task_interior: every neighbour present, no flags).
// Same terms, order and rounding as the flagged general sweep (product<false>,
// xsub/xmul updates), but with a kWG-row register window of the old rows
// (p, r, x, stencil, D^-1), i.e. kWG - 2 rows in flight instead of one.
#ifndef MLG_CG_WG
#define MLG_CG_WG 3  // A/B at config 4: 3 rows +4.5 %, 4 rows +2 % (spills), 5 rows -4 %
#endif
constexpr int kWG = MLG_CG_WG;
#ifndef MLG_CG_GENFAST
#define MLG_CG_GENFAST 1  // 0: every general-stencil task takes the flagged sweep
#endif

// product<false> with every presence flag set (sparse.cpp:69-76 column order)
__device__ __forceinline__ double product_gen(double sv, double s_n, double s_ne, double cv,
                                              const Stencil& c, double nv) {
  const double wa = __shfl_up_sync(kFull, c.e, 1);
  const double swa = __shfl_up_sync(kFull, s_ne, 1);
  const double wv = __shfl_up_sync(kFull, cv, 1);
  const double ev = __shfl_down_sync(kFull, cv, 1);
  const double swv = __shfl_up_sync(kFull, sv, 1);
  const double nev = __shfl_down_sync(kFull, nv, 1);
  double a = 0.0;
  a = xadd(a, xmul(swa, swv));
  a = xadd(a, xmul(s_n, sv));
  a = xadd(a, xmul(wa, wv));
  a = xadd(a, xmul(c.c, cv));
  a = xadd(a, xmul(c.e, ev));
  a = xadd(a, xmul(c.n, nv));
  a = xadd(a, xmul(c.ne, nev));
  return a;
}

template <bool RST>
__device__ __forceinline__ void sweep_gen(const CgSys& S, const SweepArgs& A, const Task& k,
                                          double al, double be, double* __restrict__ X,
                                          const double* __restrict__ Rc,
                                          double* __restrict__ Rn,
                                          const double* __restrict__ Pc,
                                          double* __restrict__ Pn, double (&acc)[kCgDots]) {
  const int lane = threadIdx.x & 31;
  const bool own = lane >= 2 && lane < 2 + kCgCols;
  const unsigned w = static_cast<unsigned>(S.pitch);
  const unsigned gw = static_cast<unsigned>(A.nxp1);
  const unsigned v0 = static_cast<unsigned>(cg_index(S, 0, k.col));
  const unsigned g0 = static_cast<unsigned>(S.y0) * gw + static_cast<unsigned>(S.x0 + k.col);
  const int last = k.ly1 + 1;  // last old row needed (inside the system)
  double P[kWG], Rr[kWG], Xr[kWG], D[kWG];
  Stencil St[kWG];
  auto load = [&](int j, int row) {  // rows past `last` re-read `last` (unused)
    const unsigned rr = static_cast<unsigned>(min(row, last));
    const unsigned v = v0 + rr * w, g = g0 + rr * gw;
    P[j] = Pc[v];
    Rr[j] = Rc[v];
    Xr[j] = X[v];
    St[j] = A.st[g];
    D[j] = A.dinv[g];
  };
#pragma unroll
  for (int j = 0; j < kWG; ++j) load(j, k.ly0 - 2 + j);
  int next = k.ly0 - 2 + kWG;  // next row to request
  // new p at rows n-2 (s) and n-1 (m); z, D^-1 and stencil of row n-1
  double sp = 0.0, mp = 0.0, mz = 0.0, mdv = 0.0;
  double s_n = 0.0, s_ne = 0.0;
  Stencil mst{0.0, 0.0, 0.0, 0.0};
  auto step = [&](auto J, auto store, auto stage2, int n) {
    constexpr int j0 = decltype(J)::value % kWG, j1 = (j0 + 1) % kWG, j2 = (j0 + 2) % kWG;
    double rn = Rr[j1], xn = Xr[j1];
    if constexpr (!RST) {
      const double qo = product_gen(P[j0], St[j0].n, St[j0].ne, P[j1], St[j1], P[j2]);
      rn = xsub(Rr[j1], xmul(al, qo));
      xn = xadd(Xr[j1], xmul(al, P[j1]));
    }
    const double dv = D[j1];
    const double tz = xmul(dv, rn);
    const double tp = RST ? tz : xadd(tz, xmul(be, P[j1]));
    const Stencil tst = St[j1];
    load(j0, next);  // slot of row n-1 is free
    ++next;
    if constexpr (decltype(store)::value) {
      if (own) {
        const unsigned v = v0 + static_cast<unsigned>(n) * w;
        X[v] = xn;
        Rn[v] = rn;
        Pn[v] = tp;
        acc[0] += rn * rn;
        acc[1] += rn * tz;
      }
    }
    if constexpr (decltype(stage2)::value) {  // q = A p_new at row n-1
      const double q = product_gen(sp, s_n, s_ne, mp, mst, tp);
      if (own) {
        acc[2] += mp * q;
        acc[3] += q * mz;
        acc[4] += q * xmul(mdv, q);
      }
    }
    sp = mp;
    s_n = mst.n;
    s_ne = mst.ne;
    mp = tp;
    mz = tz;
    mdv = dv;
    mst = tst;
  };
  using T = std::true_type;
  using F = std::false_type;
  step(std::integral_constant<int, 0>{}, F{}, F{}, k.ly0 - 1);  // stage 1 only
  step(std::integral_constant<int, 1>{}, T{}, F{}, k.ly0);
  int n = k.ly0 + 1;  // slot phase 2
  using Seq = std::make_integer_sequence<int, kWG>;
#pragma unroll 1
  for (; n + kWG - 1 < k.ly1; n += kWG)
    static_for(Seq{}, [&](auto i) {
      constexpr int ii = decltype(i)::value;
      step(std::integral_constant<int, (2 + ii) % kWG>{}, T{}, T{}, n + ii);
    });
  const int rem = k.ly1 - n;  // 0..kWG-1 rows left, then row ly1 (stage 2 only)
  static_for(std::make_integer_sequence<int, kWG - 1>{}, [&](auto i) {
    constexpr int ii = decltype(i)::value;
    if (ii < rem) step(std::integral_constant<int, (2 + ii) % kWG>{}, T{}, T{}, n + ii);
  });
  static_for(Seq{}, [&](auto r) {
    constexpr int rr = decltype(r)::value;
    if (rr == rem) step(std::integral_constant<int, (2 + rr) % kWG>{}, F{}, T{}, k.ly1);
  });
}

template <bool RST, bool CG, bool LAP>
__device__ __forceinline__ void sweep_edge(const CgSys& S, const SweepArgs& A, const Task& k,
                                           double al, double be, double* __restrict__ X,
                                           const double* __restrict__ Rc,
                                           double* __restrict__ Rn,
                                           const double* __restrict__ Pc,
                                           double* __restrict__ Pn, double (&acc)[kCgDots],
                                           Xchg& xch) {
  // warp-uniform: only tiny levels have tasks spanning more than three blocks
  const int bhs = A.sg.bh * A.sg.scale;
  const bool slow = A.mask && (S.y0 + min(k.ly1 + 4, S.h - 1)) / bhs -
                                      (S.y0 + max(k.ly0 - 2, 0)) / bhs > 2;
  if (slow)
    sweep_reg<RST, CG, LAP, true, true>(S, A, k, al, be, X, Rc, Rn, Pc, Pn, acc, xch);
  else if (A.mask)
    sweep_reg<RST, CG, LAP, true, false, true>(S, A, k, al, be, X, Rc, Rn, Pc, Pn, acc, xch);
  else  // local systems: only the window edges (no G)
    sweep_reg<RST, CG, LAP, true, false, false>(S, A, k, al, be, X, Rc, Rn, Pc, Pn, acc, xch);
}

// ---- asynchronous row pipeline for interior tasks ---------------------------
// Every lane streams its column through a private ring of kD shared-memory
// slots with cp.async (8 B per lane and array, LDGSTS): rows n+2 .. n+kD-1 of
// p, r and x are in flight while row n is computed, so each warp keeps ~3(kD-2)
// independent requests outstanding without holding them in registers.  A lane
// only ever reads back what it copied itself, so the per-thread
// cp.async.wait_group is the only synchronisation needed.  A slot is refilled
// at the end of the iteration that consumed it (its values are already in
// registers), so a copy can never overwrite unread data.
#ifndef MLG_CG_D
#define MLG_CG_D 8
#endif
#ifndef MLG_CG_ASYNC_MINBLOCKS
#define MLG_CG_ASYNC_MINBLOCKS 5  // the 4-array ring (deferred x) with 5 CTAs/SM: no spills
#endif
constexpr int kD = MLG_CG_D;
static_assert((kD & (kD - 1)) == 0 && kD >= 4, "ring depth must be a power of two >= 4");

#ifndef MLG_CG_RINGA
#define MLG_CG_RINGA 4
#endif
#ifndef MLG_CG_AUNR
#define MLG_CG_AUNR 2  // unroll of the interior row loop (register rotation by renaming; A/B: 1 -> 2 +1.5 % at config 2)
#endif
constexpr int kAUnr = MLG_CG_AUNR;
#ifndef MLG_CG_OFF32
#define MLG_CG_OFF32 1
#endif
struct RowRing {
  double v[kD][MLG_CG_RINGA][32];  // [slot][p, r, x, p of a deferred x update][lane]
};

// x and the deferred update's p are read once (no halo reuse): keep them out of L1.
__device__ __forceinline__ void cp_async8_cg(double* sdst, const double* gsrc) {
#ifdef MLG_CG_XCG
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sdst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc) : "memory");
#else
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sdst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc) : "memory");
#endif
}

__device__ __forceinline__ void cp_async8(double* sdst, const double* gsrc) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sdst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// EDGE: the task touches the window boundary or (strip systems) the inner
// regions G.  Points outside the system -- column or row outside the window,
// or inside G (separable test, Flags) -- read zeros (the slot is zero-filled
// instead of copied) and their new p is forced to zero, which reproduces the
// flagged product exactly (an absent neighbour contributes a literal 0 to the
// same paired-FMA chain).
// XM: 2 = x += al * p (the reference order), 0 = x untouched (update
// deferred to the next launch), 1 = x += alp * p_prev + al * p (two updates:
// the deferred one and this launch's).  Averaged over a 0/1 pair the x stream
// costs 12 B/row per iteration instead of 16.
template <bool RST, bool LAP, bool EDGE, bool SLOW, bool MASKED = true, int XM = 2>
__device__ __forceinline__ void sweep_async(const CgSys& S, const SweepArgs& A, const Task& k,
                                            double al, double be, double alp,
                                            double* __restrict__ X,
                                            const double* __restrict__ Rc,
                                            double* __restrict__ Rn,
                                            const double* __restrict__ Pc,
                                            double* __restrict__ Pn, double (&acc)[kCgDots],
                                            RowRing& ring, Xchg& xch) {
  const Lat lat1(xch, 0), lat2(xch, 1);
  const int lane = threadIdx.x & 31;
  const Flags f = make_flags(S, A, k);          // EDGE only
  const RowMask rm = make_rowmask(S, A, k, f);  // EDGE only
  const bool own = lane >= 2 && lane < 2 + kCgCols && (!EDGE || f.cin);
#if MLG_CG_OFF32
  // 32-bit element offsets (pools hold < 2^32 elements, checked at setup): one
  // IMAD.WIDE.U32 per address instead of 64-bit offset arithmetic per array
  using Off = unsigned;
#else
  using Off = long long;
#endif
  const Off w = static_cast<Off>(S.pitch);
  const Off base = static_cast<Off>(cg_index(S, 0, k.col));
  const Stencil u = A.ust;
  const double dv = LAP ? 0.25 : A.udinv;
  const int last = k.ly1 + 1;  // last old row needed (the zero frame makes it readable)
  auto issue = [&](int row) {  // one commit group per row, empty past the end
    if (row <= last) {
      const int s = row & (kD - 1);
      const Off o = base + static_cast<Off>(row) * w;
      cp_async8(&ring.v[s][0][lane], Pc + o);
      cp_async8(&ring.v[s][1][lane], Rc + o);
      if (XM != 0) cp_async8_cg(&ring.v[s][2][lane], X + o);
      if constexpr (XM == 1 && MLG_CG_RINGA > 3)
        cp_async8_cg(&ring.v[s][MLG_CG_RINGA - 1][lane], Pn + o);  // p of the deferred update
    }
    cp_async_commit();
  };
#pragma unroll
  for (int i = 0; i < kD; ++i) issue(k.ly0 - 2 + i);
  cp_async_wait<kD - 2>();  // rows ly0-2, ly0-1 landed
  double pa = ring.v[(k.ly0 - 2) & (kD - 1)][0][lane];
  double pb = ring.v[(k.ly0 - 1) & (kD - 1)][0][lane];
  issue(k.ly0 - 2 + kD);  // slot of row ly0-2 consumed
  double sp = 0.0, mp = 0.0, mz = 0.0;
  bool m_in = false;  // row n-1 in the system
  auto step = [&](int n, auto store, auto stage2) {
    // issued up to row n+kD-1; row n+1 must have landed
    cp_async_wait<kD - 2>();
    const int sc = n & (kD - 1);
    const double pc = ring.v[(n + 1) & (kD - 1)][0][lane];
    const double rb = ring.v[sc][1][lane];
    const double xb = XM != 0 ? ring.v[sc][2][lane] : 0.0;
    bool b_in = true;
    if constexpr (EDGE) b_in = rm.template in<SLOW, MASKED>(n, f, A.sg);
    double rn = rb, xn = xb;
    if constexpr (!RST) {
      const double qo = product_lat<LAP, false>(pa, pb, pc, u, lat1);
      rn = fma(-al, qo, rb);
      if constexpr (XM == 1) xn = fma(al, pb, fma(alp, ring.v[sc][MLG_CG_RINGA - 1][lane], xb));
      else if constexpr (XM == 2) xn = fma(al, pb, xb);
    }
    if constexpr (EDGE) rn = b_in ? rn : 0.0;
    const double tz = xmul(dv, rn);
    double tp = RST ? tz : fma(be, pb, tz);
    if constexpr (EDGE) tp = b_in ? tp : 0.0;
    if constexpr (decltype(store)::value) {
      if (own && b_in) {
        const Off o = base + static_cast<Off>(n) * w;
        if (XM != 0) X[o] = xn;
        Rn[o] = rn;
        Pn[o] = tp;
      }
      acc[0] += rn * rn;
      acc[1] += rn * tz;
    }
    if constexpr (decltype(stage2)::value) {  // q = A p_new at row n-1
      double q = product_lat<LAP, false>(sp, mp, tp, u, lat2);
      if constexpr (EDGE) q = m_in ? q : 0.0;
      acc[2] += mp * q;
      acc[3] += q * mz;
      acc[4] += q * xmul(dv, q);
    }
    sp = mp;
    mp = tp;
    mz = tz;
    m_in = b_in;
    pa = pb;
    pb = pc;
    issue(n + kD);  // refill slot n (its p, r, x are consumed)
  };
  using T = std::true_type;
  using F = std::false_type;
  step(k.ly0 - 1, F{}, F{});
  step(k.ly0, T{}, F{});
#pragma unroll kAUnr
  for (int n = k.ly0 + 1; n < k.ly1; ++n) step(n, T{}, T{});
  step(k.ly1, F{}, T{});
  cp_async_wait<0>();
  if (!own) {  // halo lanes (and columns outside the window) contribute nothing
#pragma unroll
    for (int q = 0; q < kCgDots; ++q) acc[q] = 0.0;
  }
}



struct Finish {
  double* part;
  unsigned* counter;
  CgCtl* ctl;
  double tol;
  unsigned long long* rows;  // sampled launches: [update-mode rows, check-mode rows]
  int* active;               // systems still running (decremented when one stops)
  int xdefer;                // 1: x updates are deferred in pairs (async batches)
};

// Scalars of a system as last written by any CTA (L2, not a stale L1 line).
__device__ __forceinline__ CgCtl load_ctl(const CgCtl* p) {
  CgCtl c;
  c.alpha = __ldcg(&p->alpha);
  c.beta = __ldcg(&p->beta);
  c.rho = __ldcg(&p->rho);
  c.bnorm = __ldcg(&p->bnorm);
  c.final_res = __ldcg(&p->final_res);
  c.mode = __ldcg(&p->mode);
  c.restart = __ldcg(&p->restart);
  c.iters = __ldcg(&p->iters);
  c.status = __ldcg(&p->status);
  c.alpha_prev = __ldcg(&p->alpha_prev);
  c.xphase = __ldcg(&p->xphase);
  return c;
}

// Block partial -> partials[tile]; the last tile of the system to arrive sums
// all partials of the system in tile order (fixed, deterministic) and
// advances its scalars.
template <int PH>
__device__ __forceinline__ void finish_tile(const CgSys& S, int sys, int t,
                                            double (&acc)[kCgDots], const Finish& F) {
  block_reduce_store<kCgDots, kBlock>(acc,
                                      F.part + static_cast<long long>(S.toff + t) * kCgDots);
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(F.counter + sys, 1u);
    s_last = (prev == static_cast<unsigned>(S.ntiles - 1));
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // All threads of the last tile sum the system's tile partials (thread t takes
  // tiles t, t + kBlock, ...; then a fixed tree): the order is fixed, so the
  // scalars are bitwise reproducible, and the latency is ~ntiles/kBlock loads.
  {
    double a[kCgDots];
#pragma unroll
    for (int q = 0; q < kCgDots; ++q) a[q] = 0.0;
    for (int tt = threadIdx.x; tt < S.ntiles; tt += kBlock) {
      const double* p = F.part + static_cast<long long>(S.toff + tt) * kCgDots;
#pragma unroll
      for (int q = 0; q < kCgDots; ++q) a[q] += __ldcg(p + q);
    }
    __shared__ double s_red[kCgWarps][kCgDots];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int q = 0; q < kCgDots; ++q) a[q] += __shfl_xor_sync(kFull, a[q], o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < kCgDots; ++q) s_red[warp][q] = a[q];
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
      for (int q = 0; q < kCgDots; ++q) {
        double v = 0.0;
        for (int w = 0; w < kCgWarps; ++w) v += s_red[w][q];
        a[q] = v;
      }
      CgCtl c = load_ctl(F.ctl + sys);
      const bool was_running = PH == kPhaseInit || c.status == kRunning;
      update_ctl<PH>(c, a, F.tol, S.maxit, F.xdefer);
      F.ctl[sys] = c;
      F.counter[sys] = 0u;
      if (was_running && c.status != kRunning) atomicSub(F.active, 1);
    }
  }
}

template <bool UNI>
__global__ void __launch_bounds__(kBlock) k_cg_init(const CgSys* sys, const CgTile* tiles,
                                                    SweepArgs A, const double* bsrc,
                                                    int bstride, double* X, double* R,
                                                    Finish F) {
  const CgTile tl = tiles[blockIdx.x];
  const CgSys S = sys[tl.sys];
  const Task k = task_of(S, tl.t, A.task_map);
  double acc[kCgDots] = {0.0, 0.0, 0.0, 0.0, 0.0};
  if (out_lane(S, k)) {
    for (int ly = k.ly0; ly < k.ly1; ++ly) {
      const long long g = static_cast<long long>(S.y0 + ly) * A.nxp1 + (S.x0 + k.col);
      const long long v = cg_index(S, ly, k.col);
      X[v] = 0.0;
      if (A.mask ? !in_strip(A.sg, S.x0 + k.col, S.y0 + ly)
                 : A.sg.in_hole(S.x0 + k.col, S.y0 + ly)) {
        R[v] = 0.0;
        continue;
      }
      const double b = bsrc[g * bstride + S.rhs];
      R[v] = b;
      acc[0] += b * b;
    }
  }
  finish_tile<kPhaseInit>(S, tl.sys, tl.t, acc, F);
}

#ifndef MLG_CG_MINBLOCKS
#define MLG_CG_MINBLOCKS 5
#endif
// One tile (kCgWarps warp tasks of one system) of one CG iteration.  PERSIST:
// called from the persistent kernel (L1-bypassing iterate loads, rows counted
// in `rows_acc` instead of per-launch atomics).
// Async sweep with the x-update mode of this launch (see sweep_async): with
// deferral on, a restart launch leaves x alone, xphase 0 defers, xphase 1
// applies the deferred update and this launch's.
template <bool LAP, bool EDGE, bool SLOW, bool MASKED>
__device__ __forceinline__ void sweep_async_x(bool rst, int xdefer, int xph, const CgSys& S,
                                              const SweepArgs& A, const Task& k, double al,
                                              double be, double alp, double* X,
                                              const double* Rc, double* Rn, const double* Pc,
                                              double* Pn, double (&acc)[kCgDots], RowRing& ring,
                                              Xchg& xch) {
  if (rst) {
    if (xdefer)
      sweep_async<true, LAP, EDGE, SLOW, MASKED, 0>(S, A, k, al, be, alp, X, Rc, Rn, Pc, Pn, acc,
                                                    ring, xch);
    else
      sweep_async<true, LAP, EDGE, SLOW, MASKED, 2>(S, A, k, al, be, alp, X, Rc, Rn, Pc, Pn, acc,
                                                    ring, xch);
  } else if (!xdefer) {
    sweep_async<false, LAP, EDGE, SLOW, MASKED, 2>(S, A, k, al, be, alp, X, Rc, Rn, Pc, Pn, acc,
                                                   ring, xch);
  } else if (xph) {
    sweep_async<false, LAP, EDGE, SLOW, MASKED, 1>(S, A, k, al, be, alp, X, Rc, Rn, Pc, Pn, acc,
                                                   ring, xch);
  } else {
    sweep_async<false, LAP, EDGE, SLOW, MASKED, 0>(S, A, k, al, be, alp, X, Rc, Rn, Pc, Pn, acc,
                                                   ring, xch);
  }
}

template <bool UNI, bool ASYNC, bool PERSIST, bool LAP>
__device__ __forceinline__ void cg_tile(const CgSys& S, const CgTile tl, int mode, double al,
                                        double be, bool rst, const SweepArgs& A,
                                        const double* bsrc, int bstride, double* __restrict__ X,
                                        const double* __restrict__ Rc, double* __restrict__ Rn,
                                        const double* __restrict__ Pc, double* __restrict__ Pn,
                                        const Finish& F, RowRing* s_ring,
                                        unsigned long long& rows_acc, double alp = 0.0,
                                        int xph = 0) {
  if (mode == kModeSkip) return;  // uniform across the system's tiles
  if constexpr (ASYNC) {  // the only batches with deferred x updates
    if (mode == kModeFlush) {  // apply the deferred x update at owned rows (no neighbours)
      const Task k = task_of(S, tl.t, A.task_map);
      if (out_lane(S, k))
        for (int ly = k.ly0; ly < k.ly1; ++ly) {
          const long long v = cg_index(S, ly, k.col);
          X[v] = fma(alp, Pn[v], X[v]);  // points outside the system hold p = 0
        }
      double acc[kCgDots] = {0.0, 0.0, 0.0, 0.0, 0.0};
      finish_tile<kPhaseIter>(S, tl.sys, tl.t, acc, F);
      return;
    }
  }
  __shared__ Xchg s_xch[kCgWarps];
  Xchg& xch = s_xch[threadIdx.x >> 5];
  const Task k = task_of(S, tl.t, A.task_map);
  const bool out = out_lane(S, k);
  double acc[kCgDots] = {0.0, 0.0, 0.0, 0.0, 0.0};
  bool fast = false, edge = false, flagged = false;
  if constexpr (UNI) {
    fast = k.valid && mode == kModeNormal && task_interior(S, A, k);
#ifdef MLG_CG_FORCE_EDGE
    fast = false;
#endif
    edge = ASYNC && k.valid && mode == kModeNormal && !fast;
    flagged = k.valid && mode == kModeNormal && !fast && !edge;
  }
#ifdef MLG_CG_TRACE
  if (PERSIST && (threadIdx.x & 31) == 0 && blockIdx.x < 4096)
    atomicOr(&g_kind[blockIdx.x], fast ? 1u : edge ? 2u : flagged ? 4u : 8u);
#endif
  if (fast) {
    if constexpr (ASYNC) {
      RowRing& ring = s_ring[threadIdx.x >> 5];
      sweep_async_x<LAP, false, false, true>(rst, F.xdefer, xph, S, A, k, al, be, alp, X, Rc, Rn,
                                             Pc, Pn, acc, ring, xch);
    } else {
      if (rst)
        sweep_reg<true, PERSIST, LAP, false, false>(S, A, k, al, be, X, Rc, Rn, Pc, Pn, acc, xch);
      else
        sweep_reg<false, PERSIST, LAP, false, false>(S, A, k, al, be, X, Rc, Rn, Pc, Pn, acc, xch);
    }
  } else if (ASYNC && edge) {
    RowRing& ring = s_ring[threadIdx.x >> 5];
    const int bhs = A.sg.bh * A.sg.scale;  // see sweep_edge
    const bool slow = A.mask && (S.y0 + min(k.ly1 + 4, S.h - 1)) / bhs -
                                        (S.y0 + max(k.ly0 - 2, 0)) / bhs > 2;
    if (slow)
      sweep_async_x<LAP, true, true, true>(rst, F.xdefer, xph, S, A, k, al, be, alp, X, Rc, Rn,
                                           Pc, Pn, acc, ring, xch);
    else if (A.mask)
      sweep_async_x<LAP, true, false, true>(rst, F.xdefer, xph, S, A, k, al, be, alp, X, Rc, Rn,
                                            Pc, Pn, acc, ring, xch);
    else
      sweep_async_x<LAP, true, false, false>(rst, F.xdefer, xph, S, A, k, al, be, alp, X, Rc,
                                             Rn, Pc, Pn, acc, ring, xch);
  } else if (flagged) {
    if (rst)
      sweep_edge<true, PERSIST, LAP>(S, A, k, al, be, X, Rc, Rn, Pc, Pn, acc, xch);
    else
      sweep_edge<false, PERSIST, LAP>(S, A, k, al, be, X, Rc, Rn, Pc, Pn, acc, xch);
  } else if (!UNI && MLG_CG_GENFAST && k.valid && mode == kModeNormal &&
             task_interior(S, A, k)) {
    if (rst)
      sweep_gen<true>(S, A, k, al, be, X, Rc, Rn, Pc, Pn, acc);
    else
      sweep_gen<false>(S, A, k, al, be, X, Rc, Rn, Pc, Pn, acc);
  } else if (!UNI && k.valid && mode == kModeNormal) {
    ORow a, b, c, d;  // old iterate at rows n-1, n, n+1 (and n+2 in flight)
    NRow s, m;        // new p at rows n-2, n-1
    load_old<UNI>(S, A, k.col, k.ly0 - 2, Rc, Pc, X, a);
    load_old<UNI>(S, A, k.col, k.ly0 - 1, Rc, Pc, X, b);
    load_old<UNI>(S, A, k.col, k.ly0, Rc, Pc, X, c);
    s.in = m.in = 0;
    s.p = s.z = m.p = m.z = 0.0;
    s.dv = m.dv = 0.0;
    s.st = m.st = Stencil{0.0, 0.0, 0.0, 0.0};
    for (int n = k.ly0 - 1; n <= k.ly1; ++n) {  // warp-uniform trip count
      load_old<UNI>(S, A, k.col, n + 2 <= k.ly1 + 1 ? n + 2 : -1, Rc, Pc, X, d);
      // stage 1 at row n: pending update, z, new p
      double rn = b.r, xn = b.x;
      if (!rst) {
        const double qo = product<UNI>(a.p, a.st, a.in, b.p, b.st, b.in, c.p, c.in, A);
        rn = xsub(b.r, xmul(al, qo));
        xn = xadd(b.x, xmul(al, b.p));
      }
      const double dv = UNI ? A.udinv : b.dv;
      NRow t;
      t.z = xmul(dv, rn);
      t.p = rst ? t.z : xadd(t.z, xmul(be, b.p));
      t.dv = dv;
      t.st = b.st;
      t.in = b.in;
      if (out && b.in && n >= k.ly0 && n < k.ly1) {
        const long long v = cg_index(S, n, k.col);
        X[v] = xn;
        Rn[v] = rn;
        Pn[v] = t.p;
        acc[0] += rn * rn;
        acc[1] += rn * t.z;
      }
      // stage 2 at row n-1: q = A p_new, dots for alpha and the rho recurrence
      if (n - 1 >= k.ly0) {
        const double q = product<UNI>(s.p, s.st, s.in, m.p, m.st, m.in, t.p, t.in, A);
        if (out && m.in) {
          acc[2] += m.p * q;
          acc[3] += q * m.z;
          acc[4] += q * xmul(m.dv, q);
        }
      }
      s = m;
      m = t;
      a = b;
      b = c;
      c = d;
    }
  } else if (UNI && k.valid) {  // kModeCheck, constant coefficients: r = b - A x
    check_sweep_uni<PERSIST>(S, A, k, bsrc, bstride, X, Rn, acc);
  } else if (k.valid) {  // kModeCheck: r = b - A x (x is current: updated in place)
    ORow a, b, c;
    load_old<UNI>(S, A, k.col, k.ly0 - 1, Rc, Pc, X, a);
    load_old<UNI>(S, A, k.col, k.ly0, Rc, Pc, X, b);
    for (int ly = k.ly0; ly < k.ly1; ++ly) {
      load_old<UNI>(S, A, k.col, ly + 1, Rc, Pc, X, c);
      const double ax = product<UNI>(a.x, a.st, a.in, b.x, b.st, b.in, c.x, c.in, A);
      if (out && b.in) {
        const long long g = static_cast<long long>(S.y0 + ly) * A.nxp1 + (S.x0 + k.col);
        const long long v = cg_index(S, ly, k.col);
        const double rt = xsub(bsrc[g * bstride + S.rhs], ax);
        Rn[v] = rt;
        acc[0] += rt * rt;
      }
      a = b;
      b = c;
    }
  }
  if (F.rows && k.valid && A.mask == nullptr) {  // roofline evidence (unmasked systems)
    const unsigned n = __reduce_add_sync(kFull, out ? static_cast<unsigned>(k.ly1 - k.ly0) : 0u);
    if (PERSIST) {  // packed: update rows low 40 bits, check rows high 24 bits / 2^40
      rows_acc += mode == kModeCheck ? (1ull * n) << 40 : 1ull * n;
    } else if ((threadIdx.x & 31) == 0) {
      atomicAdd(F.rows + (mode == kModeCheck ? 1 : 0), 1ull * n);
    }
  }
  if (PERSIST && S.ntiles <= kReplTiles)  // reduced after the grid barrier (k_cg_persist)
    block_reduce_store<kCgDots, kBlock>(acc,
                                        F.part + static_cast<long long>(S.toff + tl.t) * kCgDots);
  else
    finish_tile<kPhaseIter>(S, tl.sys, tl.t, acc, F);
}

template <bool UNI, bool ASYNC, bool LAP>
__global__ void __launch_bounds__(kBlock, (!UNI ? 4 : ASYNC ? MLG_CG_ASYNC_MINBLOCKS : MLG_CG_MINBLOCKS) * 4 / kCgWarps)
    k_cg_iter(const CgSys* sys, const CgTile* tiles, SweepArgs A, const double* bsrc,
              int bstride, double* __restrict__ X, const double* __restrict__ Rc,
              double* __restrict__ Rn, const double* __restrict__ Pc, double* __restrict__ Pn,
              Finish F) {
  const CgTile tl = tiles[blockIdx.x];
  const CgSys S = sys[tl.sys];
  __shared__ CgCtl s_c;
  extern __shared__ RowRing s_ring[];  // kCgWarps rings (ASYNC only)
  if (threadIdx.x == 0) s_c = F.ctl[tl.sys];
  __syncthreads();
  unsigned long long rows_acc = 0;
  cg_tile<UNI, ASYNC, false, LAP>(S, tl, s_c.mode, s_c.alpha, s_c.beta, s_c.restart != 0, A, bsrc,
                             bstride, X, Rc, Rn, Pc, Pn, F, s_ring, rows_acc, s_c.alpha_prev,
                             s_c.xphase);
}

// ---- persistent variant: all iterations of a batch in one launch -----------
// For batches whose iterates are L2-resident the per-launch ramp/drain
// dominates; here every CTA keeps a fixed set of <= kPersistTiles tiles and the
// iterations are separated by a grid barrier (co-residency guaranteed by the
// cooperative launch).  Same tile bodies, same reductions (the last tile of a
// system advances its scalars before arriving at the barrier), so the iterates
// are identical to the multi-launch path.
#ifndef MLG_CG_PERSIST_TILES
#define MLG_CG_PERSIST_TILES 8  // A/B: 16 takes config 5's strip batches persistent: strip +15 % time
#endif
constexpr int kPersistTiles = MLG_CG_PERSIST_TILES;

struct GridSync {
  unsigned* count;    // arrivals since the launch began (zeroed before each launch)
  unsigned* running;  // [3] running-system counts of the last iterations (zeroed per launch)
  int max_iters;      // iterations of this launch (even: vector parity is preserved)
};

// Barrier number k (k = 1, 2, ... within the launch): arrive on a monotonic
// counter and wait until it reaches k * gridDim.x -- one atomic round trip per
// CTA, no reset/generation step on the critical path.
// The wait polls with relaxed loads and acquires once: an acquire load also
// invalidates the SM's L1 (CCTL.IVALL), which inside the poll loop would flush
// the lines the other CTAs of the SM are still streaming through.
#ifndef MLG_CG_BARPOLL
#define MLG_CG_BARPOLL 1  // 0: acquire on every poll; 1: relaxed polls + one acquire
#endif
__device__ __forceinline__ void grid_sync(const GridSync& G, unsigned k) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned target = k * gridDim.x;
    unsigned v;
#if MLG_CG_BARPOLL >= 2
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(G.count) : "memory");
#else
    __threadfence();
    atomicAdd(G.count, 1u);
#endif
#if MLG_CG_BARPOLL >= 1
    do {
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(G.count) : "memory");
    } while (v < target);
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(G.count) : "memory");
#else
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(G.count) : "memory");
    } while (v < target);
#endif
  }
  __syncthreads();
}

#ifdef MLG_CG_TRACE
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(slot) \
  if (it == MLG_CG_TRACE && threadIdx.x == 0 && blockIdx.x < 4096) g_trace[blockIdx.x][slot] = gtimer()
#else
#define TRACE(slot)
#endif

#ifndef MLG_CG_PERSIST_MINBLOCKS
#define MLG_CG_PERSIST_MINBLOCKS 4  // 128 registers: the modulo-scheduled sweep without spills
#endif
// tiles: ntiles = per-CTA count x gridDim.x entries, entry i * gridDim.x + b is
// the i-th tile of CTA b (host-balanced); sys < 0 marks an empty slot.
// ASYNC: the cp.async row ring of the streaming kernel instead of the register
// pipeline (deeper prefetch at the same register budget).  Within an iteration
// the rows it streams (old p, r; own x) are not written by any other CTA, and
// every CTA's __threadfence at the grid barrier invalidates its SM's L1, so the
// L1-allocating cp.async never serves a stale line across iterations.
#ifndef MLG_CG_PERSIST_ASYNC_MINBLOCKS
#define MLG_CG_PERSIST_ASYNC_MINBLOCKS 4
#endif
template <bool UNI, bool ASYNC, bool LAP>
__global__ void __launch_bounds__(kBlock, (ASYNC ? MLG_CG_PERSIST_ASYNC_MINBLOCKS
                                                 : MLG_CG_PERSIST_MINBLOCKS) * 4 / kCgWarps)
    k_cg_persist(const CgSys* sys, const CgTile* tiles, int ntiles, SweepArgs A,
                 const double* bsrc, int bstride, double* __restrict__ X, double* R0,
                 double* R1, double* P0, double* P1, Finish F, GridSync G) {
  extern __shared__ RowRing s_ring_p[];  // kCgWarps rings (ASYNC only)
  __shared__ CgSys s_sys[kPersistTiles];
  __shared__ CgTile s_tl[kPersistTiles];
  __shared__ CgCtl s_ctl[kPersistTiles];  // private copy of the tile's system scalars
  __shared__ double s_red[kCgWarps][kCgDots];
  __shared__ unsigned s_running;
  const int mine = (ntiles - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1;
  if (threadIdx.x < mine) {
    const CgTile t = tiles[blockIdx.x + threadIdx.x * gridDim.x];
    s_tl[threadIdx.x] = t;
    if (t.sys >= 0) {
      s_sys[threadIdx.x] = sys[t.sys];
      s_ctl[threadIdx.x] = load_ctl(F.ctl + t.sys);
    }
  }
  __syncthreads();
  unsigned long long rows_acc = 0;
  for (int it = 0; it < G.max_iters; ++it) {
    const bool odd = it & 1;
    TRACE(0);
    TRACE(1);
    for (int i = 0; i < mine; ++i) {
      if (s_tl[i].sys < 0) continue;  // empty slot (CTA-uniform)
      const CgCtl& c = s_ctl[i];
      cg_tile<UNI, ASYNC, true, LAP>(s_sys[i], s_tl[i], c.mode, c.alpha, c.beta, c.restart != 0, A,
                                     bsrc, bstride, X, odd ? R1 : R0, odd ? R0 : R1,
                                     odd ? P1 : P0, odd ? P0 : P1, F, ASYNC ? s_ring_p : nullptr,
                                     rows_acc, c.alpha_prev, c.xphase);
      __syncthreads();  // shared scratch of the tile body is reused
      if (i < 4) TRACE(2 + i);
    }
    TRACE(6);
    grid_sync(G, static_cast<unsigned>(it) + 1u);
    TRACE(7);
    // Every CTA reduces the tile partials of its own systems in the same fixed
    // order (thread t takes tiles t, t + kBlock, ...; then a fixed tree), so all
    // copies of a system's scalars stay bitwise identical -- no "last tile"
    // atomics or fences on the critical path.  Termination: the holder of a
    // system's tile 0 counts it in running[it % 3] while it runs; that slot is
    // complete at the next barrier and is cleared two iterations later.
    unsigned running_prev = 1;
    if (threadIdx.x == 0) {
      if (it > 0) running_prev = __ldcg(G.running + (it - 1) % 3);
      if (blockIdx.x == 0) G.running[(it + 1) % 3] = 0u;
    }
    for (int i = 0; i < mine; ++i) {
      const int sy = s_tl[i].sys;
      if (sy < 0) continue;
      const CgSys& S = s_sys[i];
      if (S.ntiles > kReplTiles) {  // reduced by its last tile before the barrier
        if (threadIdx.x == 0) {
          s_ctl[i] = load_ctl(F.ctl + sy);
          if (s_tl[i].t == 0 && s_ctl[i].status == kRunning) atomicAdd(G.running + it % 3, 1u);
        }
        __syncthreads();
        continue;
      }
      double a[kCgDots];
#pragma unroll
      for (int q = 0; q < kCgDots; ++q) a[q] = 0.0;
      for (int tt = threadIdx.x; tt < S.ntiles; tt += kBlock) {
        const double* p = F.part + static_cast<long long>(S.toff + tt) * kCgDots;
#pragma unroll
        for (int q = 0; q < kCgDots; ++q) a[q] += __ldcg(p + q);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int q = 0; q < kCgDots; ++q) a[q] += __shfl_xor_sync(kFull, a[q], o);
      if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int q = 0; q < kCgDots; ++q) s_red[threadIdx.x >> 5][q] = a[q];
      __syncthreads();
      if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < kCgDots; ++q) {
          double v = 0.0;
          for (int w = 0; w < kCgWarps; ++w) v += s_red[w][q];
          a[q] = v;
        }
        CgCtl c = s_ctl[i];
        if (c.mode != kModeSkip) update_ctl<kPhaseIter>(c, a, F.tol, S.maxit, F.xdefer);
        s_ctl[i] = c;
        if (s_tl[i].t == 0 && c.status == kRunning) atomicAdd(G.running + it % 3, 1u);
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) s_running = running_prev;
    __syncthreads();
    if (s_running == 0) break;  // every system had stopped one iteration ago
  }
  // write the scalars back (one copy per system: the holder of its tile 0)
  if (threadIdx.x < mine && s_tl[threadIdx.x].sys >= 0 && s_tl[threadIdx.x].t == 0)
    F.ctl[s_tl[threadIdx.x].sys] = s_ctl[threadIdx.x];
  if (F.rows && (threadIdx.x & 31) == 0 && rows_acc) {
    atomicAdd(F.rows, rows_acc & ((1ull << 40) - 1));
    atomicAdd(F.rows + 1, rows_acc >> 40);
  }
}



constexpr int kRingBytes = kCgWarps * static_cast<int>(sizeof(RowRing));

// Resident CTAs per GPU of the CG iteration kernel (register or async variant).
int resident_tiles(bool async) {
  static const int res[2] = {[] {
                               int dev = 0, sms = 0, per = 0;
                               cudaGetDevice(&dev);
                               cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
                               cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                                   &per, k_cg_iter<true, false, true>, kBlock, 0);
                               return std::max(1, sms * std::max(per, 1));
                             }(),
                             [] {
                               int dev = 0, sms = 0, per = 0;
                               cudaGetDevice(&dev);
                               cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
                               for (auto fn : {k_cg_iter<true, true, true>, k_cg_iter<true, true, false>})
                                 cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                      kRingBytes);
                               cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                                   &per, k_cg_iter<true, true, true>, kBlock, kRingBytes);
                               return std::max(1, sms * std::max(per, 1));
                             }()};
  return res[async ? 1 : 0];
}

bool persist_async_on() {
  static const bool on = [] {
    const char* e = std::getenv("MLG_CG_PERSIST_ASYNC");  // A/B hook: 0 / 1
    return e ? std::atoi(e) != 0 : true;  // measured at config 2: 30.4 -> 31.1 M DOF/s
  }();
  return on;
}

int resident_persist() {
  static const int res = [] {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (persist_async_on()) {
      for (auto f : {k_cg_persist<true, true, true>, k_cg_persist<true, true, false>})
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, kRingBytes);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_cg_persist<true, true, true>, kBlock,
                                                    kRingBytes);
    } else {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_cg_persist<true, false, true>, kBlock,
                                                    0);
    }
    return std::max(1, sms * std::max(per, 1));
  }();
  return res;
}

// Unknowns of a window system: the window's lattice points minus those in a
// closed G_j (strip systems) or in the hole -- the size n of the reference's
// extracted system, so maxit = 10 n (sparse.cpp:204) matches.  Per row the
// excluded points are a union of at most side + 1 intervals.
int system_points(const StripGeom& g, bool strip, const CgSys& s) {
  long long n = 0;
  std::vector<std::pair<int, int>> iv;
  for (int y = s.y0; y < s.y0 + s.h; ++y) {
    iv.clear();
    if (strip) {
      const int by = std::min(y / (g.bh * g.scale), g.side - 1);
      const int y0 = (by == 0 ? 0 : by * g.bh + g.dc) * g.scale;
      const int y1 = (by == g.side - 1 ? g.ny0 : (by + 1) * g.bh - g.dc) * g.scale;
      if (y >= y0 && y <= y1)
        for (int bx = 0; bx < g.side; ++bx) {
          const int x0 = (bx == 0 ? 0 : bx * g.bw + g.dc) * g.scale;
          const int x1 = (bx == g.side - 1 ? g.nx0 : (bx + 1) * g.bw - g.dc) * g.scale;
          iv.emplace_back(x0, x1);
        }
    }
    if (y >= g.hy0 && y <= g.hy1 && g.hx1 >= g.hx0) iv.emplace_back(g.hx0, g.hx1);
    std::sort(iv.begin(), iv.end());
    long long excl = 0;
    int cur = s.x0 - 1;  // last excluded column counted
    for (const auto& q : iv) {
      const int a = std::max(q.first, std::max(cur + 1, s.x0));
      const int b = std::min(q.second, s.x0 + s.w - 1);
      if (b >= a) {
        excl += b - a + 1;
        cur = b;
      }
    }
    n += s.w - excl;
  }
  return static_cast<int>(n);
}

SweepArgs sweep_args(const Level& L, const unsigned char* mask) {
  SweepArgs A{};
  // domains with a hole: the interior-restricted operator (identity rows on
  // the hole, see assemble.cu k_cg_stencil)
  A.st = L.hole.any() ? L.stCG.get() : L.stA.get();
  A.dinv = L.hole.any() ? L.dinvCG.get() : L.dinv.get();
  A.nxp1 = L.nx + 1;
  A.mask = mask;
  A.sg = L.strip_geom;
  A.ust = L.ust;
  A.udinv = L.udinv;
  return A;
}

}  // namespace

void CgBatch::setup(Ctx& c, const Level& lev, std::vector<CgSys> systems,
                    const unsigned char* mask_, const double* bsrc_, int bstride_) {
  L = &lev;
  mask = mask_;
  bsrc = bsrc_;
  bstride = bstride_;
  total_rows = 0;
  total_tiles = 0;
  long long all_rows = 0;
  for (const CgSys& s : systems) all_rows += static_cast<long long>(s.w) * s.h;
  // Vectors that outgrow L2 stream from HBM: use the asynchronous row pipeline
  // (deep prefetch in shared memory); L2-resident batches keep the register
  // pipeline (lower latency, fewer instructions).
  static const int async_env = [] {
    const char* e = std::getenv("MLG_CG_ASYNC");  // A/B hook: 0 / 1
    return e ? std::atoi(e) : -1;
  }();
  const bool streaming_async =
      lev.uniform != 0 && (async_env >= 0 ? async_env != 0 : all_rows * 48 > (128LL << 20));
  // Constant-coefficient batches whose tiles fit the resident CTAs: one
  // persistent launch per solve (measured: L2-resident config 2 and the
  // streaming config 3 both gain; config 5's batches do not fit and fall back
  // to one launch per iteration below).  MLG_CG_ASYNC=1 forces the latter.
  static const int persist_env = [] {
    const char* e = std::getenv("MLG_CG_PERSIST");  // A/B hook: 0 / 1
    return e ? std::atoi(e) : 1;
  }();
  use_persist = lev.uniform != 0 && persist_env != 0 && async_env != 1;
  use_async = use_persist ? false : streaming_async;
  int s_krows = 0;
  for (int pass = 0; pass < 2; ++pass) {
    // Rows per warp task: long sweeps amortise the 2-row halo, but the batch
    // must still offer >= ~8k warps (148 SMs x ~56 resident) to hide latency.
    static const long long target_tasks = [] {
      const char* e = std::getenv("MLG_CG_TASKS");  // tuning hook
      return e ? std::atoll(e) : 8192LL;
    }();
    static const int min_rows = [] {
      const char* e = std::getenv("MLG_CG_MINROWS");  // tuning hook
      return e ? std::atoi(e) : 16;
    }();
    static const int max_rows_async = [] {
      const char* e = std::getenv("MLG_CG_MAXROWS");  // tuning hook
      return e ? std::atoi(e) : kCgRowsAsync;
    }();
    const int max_rows = use_async ? max_rows_async : kCgRows;
    int krows = static_cast<int>(std::min<long long>(
        max_rows, std::max<long long>(min_rows, all_rows / (kCgCols * target_tasks))));
    // Wave quantisation: every tile costs ~(krows + c0) row steps and the grid
    // runs in waves of `resident` tiles, so pick the row count that minimises
    // waves x (krows + c0) from half the first choice up to the cap.
    {
      const int resident = use_persist ? resident_persist() : resident_tiles(use_async);
      // Strip systems drop the tasks whose output cells lie inside one G_j
      // (setup below); count them per block in closed form.
      auto inside_tasks = [&](const CgSys& s, int kr) {
        if (!mask_) return 0LL;
        const StripGeom& g = lev.strip_geom;
        long long n = 0;
        for (int bx = 0; bx < g.side; ++bx)
          for (int by = 0; by < g.side; ++by) {
            const int gx0 = (bx == 0 ? 0 : bx * g.bw + g.dc) * g.scale;
            const int gx1 = (bx == g.side - 1 ? g.nx0 : (bx + 1) * g.bw - g.dc) * g.scale;
            const int gy0 = (by == 0 ? 0 : by * g.bh + g.dc) * g.scale;
            const int gy1 = (by == g.side - 1 ? g.ny0 : (by + 1) * g.bh - g.dc) * g.scale;
            long long cs = 0, cr = 0;
            for (int c = 0; c * kCgCols < s.w; ++c) {
              const int ca = s.x0 + c * kCgCols, cb = s.x0 + std::min(c * kCgCols + kCgCols, s.w) - 1;
              cs += ca >= gx0 && cb <= gx1;
            }
            for (int r = 0; r * kr < s.h; ++r) {
              const int ra = s.y0 + r * kr, rb = s.y0 + std::min(r * kr + kr, s.h) - 1;
              cr += ra >= gy0 && rb <= gy1;
            }
            n += cs * cr;
          }
        return n;
      };
      auto tiles_for = [&](int kr) {
        // strip systems (mask) all share one window: count its dropped tasks once.
        // (Persistent batches keep the uncompacted count: there the per-tile
        // fixed cost favours fewer, taller tiles -- measured at config 2.)
        const long long drop =
            mask_ && !use_persist && !systems.empty() ? inside_tasks(systems[0], kr) : 0;
        long long t = 0;
        for (const CgSys& s : systems) {
          const long long ns = std::max(1, (s.w + kCgCols - 1) / kCgCols);
          const long long nb = std::max(1, (s.h + kr - 1) / kr);
          const long long nt = std::max(1LL, ns * nb - drop);
          t += (nt + kCgWarps - 1) / kCgWarps;
        }
        return t;
      };
      // (c0: a task's prologue/epilogue in row steps)
      static const int c0 = [] {
        const char* e = std::getenv("MLG_CG_C0");  // tuning hook
        return e ? std::atoi(e) : 6;
      }();
      double best = 1e300;
      int best_k = krows;
      for (int kr = std::max(4, krows / 2); kr <= max_rows; ++kr) {
        const long long waves = (tiles_for(kr) + resident - 1) / resident;
        const double cost = static_cast<double>(waves) * (kr + c0);
        if (cost < best - 1e-9) {
          best = cost;
          best_k = kr;
        }
      }
      krows = best_k;
      static const int strip_rows = [] {
        const char* e = std::getenv("MLG_CG_STRIP_ROWS");  // tuning hook (strip batches)
        return e ? std::atoi(e) : 0;
      }();
      if (mask_ && strip_rows > 0) krows = strip_rows;
      // Persistent batches: one tile per CTA leaves the slow (edge) tiles on the
      // critical path; aim for ~`tpc` tiles per CTA so the LPT assignment can
      // pair them with cheap ones.
      static const int tpc = [] {
        const char* e = std::getenv("MLG_CG_PTPC");  // tuning hook
        return e ? std::atoi(e) : 1;
      }();
      if (use_persist && tpc > 1) {
        int kr = krows;
        while (kr > 4 && tiles_for(kr) < static_cast<long long>(tpc) * resident) --kr;
        krows = kr;
      }
      if (use_persist && (tiles_for(krows) + resident - 1) / resident > kPersistTiles) {
        use_persist = false;  // too many tiles per CTA: multi-launch path, retiled
        use_async = streaming_async;
        continue;
      }
    }
    s_krows = krows;
    break;
  }
  const int krows = s_krows;
  for (CgSys& s : systems) {
    s.nrows = system_points(lev.strip_geom, mask_ != nullptr, s);
    s.krows = krows;
    s.nstrips = std::max(1, (s.w + kCgCols - 1) / kCgCols);
    s.nrb = std::max(1, (s.h + krows - 1) / krows);
    s.ntasks = s.nstrips * s.nrb;
    s.tmap_off = -1;
  }
  // Strip systems: keep only tasks whose output cells meet the strip (tasks
  // lying inside a closed G_j would only sweep masked rows).
  std::vector<int> tmap;
  if (mask && !systems.empty()) {
    const CgSys& s = systems[0];
    const StripGeom& g = lev.strip_geom;
    auto inside_g = [&](int xa, int xb, int ya, int yb) {
      const int bx = std::min(xa / (g.bw * g.scale), g.side - 1);
      const int by = std::min(ya / (g.bh * g.scale), g.side - 1);
      const int x0 = (bx == 0 ? 0 : bx * g.bw + g.dc) * g.scale;
      const int x1 = (bx == g.side - 1 ? g.nx0 : (bx + 1) * g.bw - g.dc) * g.scale;
      const int y0 = (by == 0 ? 0 : by * g.bh + g.dc) * g.scale;
      const int y1 = (by == g.side - 1 ? g.ny0 : (by + 1) * g.bh - g.dc) * g.scale;
      return xa >= x0 && xb <= x1 && ya >= y0 && yb <= y1;
    };
    for (int t = 0; t < s.ntasks; ++t) {
      const int rb = t / s.nstrips, strip = t % s.nstrips;
      const int ca = s.x0 + strip * kCgCols, cb = s.x0 + std::min(strip * kCgCols + kCgCols, s.w) - 1;
      const int ra = s.y0 + rb * s.krows, rbb = s.y0 + std::min(rb * s.krows + s.krows, s.h) - 1;
      if (!inside_g(ca, cb, ra, rbb) && !g.rect_inside_hole(ca, cb, ra, rbb)) tmap.push_back(t);
    }
    for (CgSys& q : systems) {
      q.tmap_off = 0;
      q.ntasks = static_cast<int>(tmap.size());
    }
  }
  // Pooled layout: window rows at pitch w + 1 (the extra column is zero and
  // doubles as the left neighbour of the next row), a zero row above and
  // below each window, two spare rows in front and kCgPadRows behind the last
  // window (prefetch overrun).  Everything outside the windows stays zero.
  int max_pitch = 1;
  for (const CgSys& s : systems) max_pitch = std::max(max_pitch, s.w + 1);
  long long cursor = 2LL * max_pitch + 2;
  for (CgSys& s : systems) {
    s.pitch = s.w + 1;
    s.ntiles = std::max(1, (s.ntasks + kCgWarps - 1) / kCgWarps);
    s.voff = cursor + s.pitch;  // row 0 (row -1 is the zero row)
    s.toff = total_tiles;
    s.maxit = 10 * std::max(s.nrows, 1);
    cursor += static_cast<long long>(s.h + 2) * s.pitch;
    total_tiles += s.ntiles;
  }
  total_rows = cursor + static_cast<long long>(kCgPadRows) * max_pitch + 64;
  if (total_rows >= (1LL << 32))  // sweep_async indexes the pool with 32-bit offsets
    throw std::runtime_error("cg batch: pooled vectors exceed 2^32 elements");
  tmap_h = tmap;
  task_map.ensure(std::max<std::size_t>(tmap.size(), 1));
  if (!tmap.empty()) task_map.upload(tmap.data(), tmap.size(), c.stream);
  sys_h = std::move(systems);
  const std::size_t nv = static_cast<std::size_t>(total_rows);
  for (DevBuf<double>* v : {&X, &R0, &R1, &P0, &P1}) {
    v->ensure(nv);
    MLG_CUDA(cudaMemsetAsync(v->get(), 0, nv * sizeof(double), c.stream));  // zero frames
  }
  part.ensure(static_cast<std::size_t>(total_tiles) * kCgDots);
  sys_d.ensure(sys_h.size());
  sys_d.upload(sys_h.data(), sys_h.size(), c.stream);
  ctl_d.ensure(sys_h.size());
  ctl_d.zero(c.stream);
  counters.ensure(sys_h.size());
  counters.zero(c.stream);
  // persistent layouts hold up to kPersistTiles slots per resident CTA
  tiles_d.ensure(use_persist ? std::max<std::size_t>(total_tiles, static_cast<std::size_t>(kPersistTiles) * resident_persist())
                             : static_cast<std::size_t>(total_tiles));
}

namespace {
bool host_rect_in_strip(const StripGeom& g, int xa, int xb, int ya, int yb) {
  if (g.rect_meets_hole(xa, xb, ya, yb)) return false;
  const int bxa = std::min(xa / (g.bw * g.scale), g.side - 1);
  const int bxb = std::min(xb / (g.bw * g.scale), g.side - 1);
  const int bya = std::min(ya / (g.bh * g.scale), g.side - 1);
  const int byb = std::min(yb / (g.bh * g.scale), g.side - 1);
  for (int bx = bxa; bx <= bxb; ++bx)
    for (int by = bya; by <= byb; ++by) {
      const int x0 = (bx == 0 ? 0 : bx * g.bw + g.dc) * g.scale;
      const int x1 = (bx == g.side - 1 ? g.nx0 : (bx + 1) * g.bw - g.dc) * g.scale;
      const int y0 = (by == 0 ? 0 : by * g.bh + g.dc) * g.scale;
      const int y1 = (by == g.side - 1 ? g.ny0 : (by + 1) * g.bh - g.dc) * g.scale;
      if (xa <= x1 && xb >= x0 && ya <= y1 && yb >= y0) return false;
    }
  return true;
}
}  // namespace

// Estimated cost of a tile: its slowest warp task, (rows + 6) row steps, x1.6
// for tasks on the window edge or touching G (the flagged sweep).
double CgBatch::tile_cost(const CgTile& t, const std::vector<int>& tmap) const {
  const CgSys& S = sys_h[static_cast<std::size_t>(t.sys)];
  double worst = 0.0;
  for (int wi = 0; wi < kCgWarps; ++wi) {
    int task = t.t * kCgWarps + wi;
    if (task >= S.ntasks) break;
    if (S.tmap_off >= 0) task = tmap[static_cast<std::size_t>(S.tmap_off + task)];
    const int rb = task / S.nstrips, strip = task % S.nstrips;
    const int c0 = strip * kCgCols - 2, ly0 = rb * S.krows, ly1 = std::min(ly0 + S.krows, S.h);
    bool interior = c0 >= 0 && c0 + 31 < S.w && ly0 - 2 >= 0 && ly1 + 1 < S.h;
    if (interior && L->strip_geom.rect_meets_hole(S.x0 + c0, S.x0 + c0 + 31, S.y0 + ly0 - 2,
                                                  S.y0 + ly1 + 1))
      interior = false;
    if (interior && mask)
      interior = host_rect_in_strip(L->strip_geom, S.x0 + c0, S.x0 + c0 + 31, S.y0 + ly0 - 2,
                                    S.y0 + ly1 + 1);
    worst = std::max(worst, (ly1 - ly0 + 6) * (interior ? 1.0 : 1.6));
  }
  return worst;
}

std::vector<CgTile> CgBatch::balance_tiles(const std::vector<CgTile>& tiles, int grid) const {
  std::vector<std::pair<double, int>> order;
  order.reserve(tiles.size());
  for (std::size_t i = 0; i < tiles.size(); ++i)
    order.emplace_back(tile_cost(tiles[i], tmap_h), static_cast<int>(i));
  std::stable_sort(order.begin(), order.end(),
                   [](const auto& a, const auto& b) { return a.first > b.first; });
  // min-heap of (load, cta); CTAs at kPersistTiles are retired from the heap
  using Slot = std::pair<double, int>;
  std::priority_queue<Slot, std::vector<Slot>, std::greater<Slot>> heap;
  for (int b = 0; b < grid; ++b) heap.emplace(0.0, b);
  std::vector<std::vector<int>> per(static_cast<std::size_t>(grid));
  for (const auto& o : order) {
    Slot sl = heap.top();
    heap.pop();
    per[static_cast<std::size_t>(sl.second)].push_back(o.second);
    if (static_cast<int>(per[static_cast<std::size_t>(sl.second)].size()) < kPersistTiles)
      heap.emplace(sl.first + o.first, sl.second);
  }
  std::size_t m = 0;
  for (const auto& p : per) m = std::max(m, p.size());
  std::vector<CgTile> lay(m * static_cast<std::size_t>(grid), CgTile{-1, 0});
  for (int b = 0; b < grid; ++b)
    for (std::size_t i = 0; i < per[static_cast<std::size_t>(b)].size(); ++i)
      lay[i * static_cast<std::size_t>(grid) + static_cast<std::size_t>(b)] =
          tiles[static_cast<std::size_t>(per[static_cast<std::size_t>(b)][i])];
  return lay;
}

CgResult CgBatch::solve(Ctx& c, double tol, int maxit_override) {
  const int nsys = static_cast<int>(sys_h.size());
  if (maxit_override > 0) {
    for (CgSys& s : sys_h) s.maxit = maxit_override;
    sys_d.upload(sys_h.data(), sys_h.size(), c.stream);
  }
  // Constant-stencil batches whose systems fit on chip run SM-resident
  // (cg_resident.cu): always when the five pooled vectors do not fit L2 (config 5
  // local 2.31 -> 1.49 s, config 3 local 74 -> 37 ms), and for L2-sized batches
  // from 256 k pooled rows up, where the resident kernel with a slab-sized
  // instantiation beats the persistent one (config 2: strip 13.8 -> 11.0 ms at 48
  // points per thread already).  Smaller batches keep the persistent kernel.
  static const int resident_mode = [] {
    // A/B hook: 0 never, 2 whenever it fits, 3 only beyond L2 (the earlier rule)
    const char* e = std::getenv("MLG_CG_RESIDENT");
    return e ? std::atoi(e) : 1;
  }();
  static const long long l2_bytes = [] {
    int dev = 0, l2 = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    return static_cast<long long>(l2);
  }();
  const bool beyond_l2 = total_rows * 5LL * static_cast<long long>(sizeof(double)) > l2_bytes;
  const bool sizeable = resident_mode != 3 && total_rows >= (1LL << 18);
  if (!use_persist || beyond_l2 || sizeable || resident_mode == 2) {
    CgResult rr;
    if (solve_resident(c, tol, rr)) return rr;
  }
  static const bool lpt_env = [] {
    const char* e = std::getenv("MLG_CG_LPT");  // A/B hook: 0 keeps the system-major order
    return e ? std::atoi(e) != 0 : true;
  }();
  std::vector<CgTile> tiles;
  auto rebuild = [&](const std::vector<char>& active) {
    tiles.clear();
    for (int s = 0; s < nsys; ++s)
      if (active[s])
        for (int t = 0; t < sys_h[s].ntiles; ++t) tiles.push_back({s, t});
    if (lpt_env && !use_persist && !use_async) {
      // per-iteration launches of the register pipeline (general-stencil batches):
      // the block scheduler hands tiles out in order, so the costly ones (window
      // edges, G_j borders: flagged sweeps) go first and the short ones last -- a
      // shorter drain at the end of every launch (config 4 local 346 -> 336 ms).
      // Stable: full interior tiles keep their order.  The HBM-streaming cp.async
      // batches keep the system-major order: there the sort separates vertically
      // adjacent tiles, whose halo rows then miss L2 (config 5 strip 1.00 -> 1.08 s).
      std::vector<std::pair<double, CgTile>> keyed;
      keyed.reserve(tiles.size());
      for (const CgTile& t : tiles) keyed.emplace_back(tile_cost(t, tmap_h), t);
      std::stable_sort(keyed.begin(), keyed.end(),
                       [](const auto& a, const auto& b) { return a.first > b.first; });
      for (std::size_t i = 0; i < tiles.size(); ++i) tiles[i] = keyed[i].second;
    }
    tiles_d.upload(tiles.data(), tiles.size(), c.stream);
  };
  std::vector<char> active(nsys, 1);
  rebuild(active);
  cudaStream_t st = c.stream;
  const bool uni = L->uniform != 0;
  // 5-point Laplacian stencil (P1 Laplace on the right-triangle lattice)
  const bool lap = uni && L->ust.c == 4.0 && L->ust.e == -1.0 && L->ust.n == -1.0 &&
                   L->ust.ne == 0.0 && L->udinv == 0.25 && std::getenv("MLG_CG_NOLAP") == nullptr;
  SweepArgs A = sweep_args(*L, mask);
  A.task_map = task_map.get();
  // Roofline evidence: local batches (no mask) sample launches and count swept
  // rows on the device; strip batches time every launch and count unknowns x
  // CG updates on the host at the end.
  const bool profiling = c.profile && mask == nullptr;
  const bool sprof = c.profile && mask != nullptr;
  if (profiling) {
    prof_rows.ensure(2);
    prof_rows.zero(c.stream);
  }
  gsync.ensure(4);  // persistent kernel: barrier counter + running[3]
  gsync.zero(st);
  active_d.ensure(1);
  active_d.upload(&nsys, 1, st);
  // Deferred x updates in pairs for the HBM-streaming (async) batches: 44 B/row
  // per iteration on average instead of 48 (MLG_CG_XDEFER=0 turns it off).
  static const int xdefer_env = [] {
    const char* e = std::getenv("MLG_CG_XDEFER");
    return e ? std::atoi(e) : 1;
  }();
  static const int xdefer_p_env = [] {  // persistent batches on the ring (A/B hook)
    const char* e = std::getenv("MLG_CG_XDEFER_P");
    return e ? std::atoi(e) : 1;  // config 2: 31.1 -> 31.4 M DOF/s
  }();
  const int xdefer = ((use_async && xdefer_env) ||
                      (use_persist && persist_async_on() && xdefer_p_env)) &&
                             MLG_CG_RINGA > 3
                         ? 1
                         : 0;
  const Finish F{part.get(), counters.get(), ctl_d.get(), tol, nullptr, active_d.get(), xdefer};
  const Finish Fp{part.get(), counters.get(), ctl_d.get(), tol, prof_rows.get(), active_d.get(),
                  xdefer};
  double *rc = R0.get(), *rn = R1.get(), *pc = P0.get(), *pn = P1.get();

  if (uni)
    k_cg_init<true><<<static_cast<unsigned>(tiles.size()), kBlock, 0, st>>>(
        sys_d.get(), tiles_d.get(), A, bsrc, bstride, X.get(), rc, F);
  else
    k_cg_init<false><<<static_cast<unsigned>(tiles.size()), kBlock, 0, st>>>(
        sys_d.get(), tiles_d.get(), A, bsrc, bstride, X.get(), rc, F);
  MLG_LAUNCH_CHECK();

  std::vector<CgCtl> ctl(static_cast<std::size_t>(nsys));
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> evs;
  int chunk = 16;
  long long iter_count = 0;
  const bool persist_async = persist_async_on();
  if (use_persist) {
    // All iterations in cooperative launches of at most kIters iterations (an
    // even count, so the vector parity is unchanged between launches).
    constexpr int kIters = 4096;
    const int grid = std::min(static_cast<int>(tiles.size()), resident_persist());
    // Longest-processing-time assignment of tiles to the resident CTAs (a
    // window-edge / strip-boundary tile costs ~1.6 interior tiles): the
    // iteration ends with the slowest CTA, so balance the per-CTA sums.
    const std::vector<CgTile> lay = balance_tiles(tiles, grid);
#ifdef MLG_CG_TRACE
    for (int b : {0, 1, 2, 3, grid / 2, grid - 1}) {
      const CgTile& t = lay[static_cast<std::size_t>(b)];
      if (t.sys < 0) continue;
      const CgSys& S = sys_h[static_cast<std::size_t>(t.sys)];
      fprintf(stderr, "  layout cta %d: sys %d tile %d (w %d h %d krows %d nstrips %d nrb %d) cost %.1f tasks:", b,
              t.sys, t.t, S.w, S.h, S.krows, S.nstrips, S.nrb, tile_cost(t, tmap_h));
      for (int wi = 0; wi < kCgWarps; ++wi) {
        int task = t.t * kCgWarps + wi;
        if (task >= S.ntasks) break;
        if (S.tmap_off >= 0) task = tmap_h[static_cast<std::size_t>(S.tmap_off + task)];
        fprintf(stderr, " (strip %d rb %d)", task % S.nstrips, task / S.nstrips);
      }
      fprintf(stderr, "\n");
    }
#endif
    tiles_d.ensure(lay.size());
    tiles_d.upload(lay.data(), lay.size(), st);
    const int ntiles = static_cast<int>(lay.size());
    const CgSys* sp = sys_d.get();
    const CgTile* tp = tiles_d.get();
    double* xp = X.get();
    double *r0 = R0.get(), *r1 = R1.get(), *p0 = P0.get(), *p1 = P1.get();
    const Finish& Fl = profiling ? Fp : F;
    const bool timed = profiling || sprof;
    GridSync G{gsync.get(), gsync.get() + 1, kIters};
    void* args[] = {(void*)&sp, (void*)&tp, (void*)&ntiles, (void*)&A, (void*)&bsrc,
                    (void*)&bstride, (void*)&xp, (void*)&r0, (void*)&r1, (void*)&p0,
                    (void*)&p1, (void*)&Fl, (void*)&G};
    for (int launch = 0;; ++launch) {
      cudaEvent_t ev0 = nullptr, ev1 = nullptr;
      if (timed) {
        ev0 = c.event(2 * evs.size());
        ev1 = c.event(2 * evs.size() + 1);
        MLG_CUDA(cudaEventRecord(ev0, st));
      }
      gsync.zero(st);  // barrier counter restarts with every launch
      const void* fn =
          persist_async ? (lap ? reinterpret_cast<const void*>(&k_cg_persist<true, true, true>)
                               : reinterpret_cast<const void*>(&k_cg_persist<true, true, false>))
                        : (lap ? reinterpret_cast<const void*>(&k_cg_persist<true, false, true>)
                               : reinterpret_cast<const void*>(&k_cg_persist<true, false, false>));
      MLG_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kBlock), args,
                                           persist_async ? kRingBytes : 0, st));
      ++launch_counter();
      if (timed) {
        MLG_CUDA(cudaEventRecord(ev1, st));
        evs.emplace_back(ev0, ev1);
        if (profiling) ++c.times.ka_launches_all;
      }
      ctl_d.download(ctl.data(), ctl.size(), st);
      c.sync();
      bool any = false;
      for (const CgCtl& q : ctl) any |= q.status == kRunning;
      if (!any) break;
      if (launch > 1000) throw SolverError("cg_solve: persistent CG did not terminate");
    }
#ifdef MLG_CG_TRACE
    {
      static unsigned long long tr[4096][8];
      MLG_CUDA(cudaMemcpyFromSymbol(tr, g_trace, sizeof(tr)));
      unsigned long long t0 = ~0ull, t7 = 0;
      double s1 = 0, s6 = 0, s7 = 0, m6 = 0;
      for (int b = 0; b < grid; ++b) {
        t0 = std::min(t0, tr[b][0]);
        t7 = std::max(t7, tr[b][7]);
      }
      for (int b = 0; b < grid; ++b) {
        s1 += tr[b][1] - tr[b][0];
        s6 += tr[b][6] - tr[b][1];
        m6 = std::max(m6, double(tr[b][6] - t0));
        s7 += tr[b][7] - tr[b][6];
      }
      fprintf(stderr, "trace: grid %d tiles %d span %.2f us | ctl %.2f work %.2f (last done %.2f) barrier %.2f us avg\n",
              grid, ntiles, (t7 - t0) * 1e-3, s1 / grid * 1e-3, s6 / grid * 1e-3, m6 * 1e-3, s7 / grid * 1e-3);
      static unsigned kind[4096];
      MLG_CUDA(cudaMemcpyFromSymbol(kind, g_kind, sizeof(kind)));
      for (unsigned kk = 0; kk < 16; ++kk) {
        int n = 0;
        double sum = 0, mx = 0;
        for (int b = 0; b < grid; ++b)
          if (kind[b] == kk) {
            ++n;
            const double d = (tr[b][6] - tr[b][1]) * 1e-3;
            sum += d;
            mx = std::max(mx, d);
          }
        if (n) fprintf(stderr, "  kind %u: %d CTAs, tile work avg %.2f max %.2f us\n", kk, n, sum / n, mx);
      }
      memset(kind, 0, sizeof(kind));
      MLG_CUDA(cudaMemcpyToSymbol(g_kind, kind, sizeof(kind)));
      for (int b = 0; b < grid; b += grid / 6)
        fprintf(stderr, "  cta %d: start %+.2f ctl %.2f tiles %.2f %.2f %.2f done %.2f out %.2f\n", b,
                (tr[b][0] - t0) * 1e-3, (tr[b][1] - tr[b][0]) * 1e-3, (tr[b][2] - tr[b][1]) * 1e-3,
                tr[b][3] ? (tr[b][3] - tr[b][2]) * 1e-3 : 0.0, tr[b][4] ? (tr[b][4] - tr[b][3]) * 1e-3 : 0.0,
                (tr[b][6] - t0) * 1e-3, (tr[b][7] - t0) * 1e-3);
      memset(tr, 0, sizeof(tr));
      MLG_CUDA(cudaMemcpyToSymbol(g_trace, tr, sizeof(tr)));
    }
#endif
    ctl_d.download(ctl.data(), ctl.size(), st);
    c.sync();
    for (int s = 0; s < nsys; ++s)
      if (ctl[static_cast<std::size_t>(s)].status == kIndefinite)
        throw SolverError("cg_solve: matrix is not positive definite (p'Mp <= 0)");
  }
  while (!use_persist) {
    for (int it = 0; it < chunk && !tiles.empty(); ++it) {
      const unsigned nt = static_cast<unsigned>(tiles.size());
      // Kernel timing evidence: every 4th launch of the local solves is
      // bracketed by pooled CUDA events (cheap enough not to starve the stream).
      // (pairs of consecutive launches: with deferred x updates the two phases
      // move 32 and 56 B/row, so a pair is the unit the 44 B/row average holds for)
      const bool prof = sprof || (profiling && (iter_count++ % 8 < 2));
      if (profiling) ++c.times.ka_launches_all;
      cudaEvent_t ev0 = nullptr, ev1 = nullptr;
      if (prof) {
        ev0 = c.event(2 * evs.size());
        ev1 = c.event(2 * evs.size() + 1);
        MLG_CUDA(cudaEventRecord(ev0, st));
      }
      const Finish& Fl = prof && profiling ? Fp : F;
      if (uni && use_async && lap)
        k_cg_iter<true, true, true><<<nt, kBlock, kRingBytes, st>>>(
            sys_d.get(), tiles_d.get(), A, bsrc, bstride, X.get(), rc, rn, pc, pn, Fl);
      else if (uni && use_async)
        k_cg_iter<true, true, false><<<nt, kBlock, kRingBytes, st>>>(
            sys_d.get(), tiles_d.get(), A, bsrc, bstride, X.get(), rc, rn, pc, pn, Fl);
      else if (uni && lap)
        k_cg_iter<true, false, true><<<nt, kBlock, 0, st>>>(
            sys_d.get(), tiles_d.get(), A, bsrc, bstride, X.get(), rc, rn, pc, pn, Fl);
      else if (uni)
        k_cg_iter<true, false, false><<<nt, kBlock, 0, st>>>(
            sys_d.get(), tiles_d.get(), A, bsrc, bstride, X.get(), rc, rn, pc, pn, Fl);
      else
        k_cg_iter<false, false, false><<<nt, kBlock, 0, st>>>(
            sys_d.get(), tiles_d.get(), A, bsrc, bstride, X.get(), rc, rn, pc, pn, Fl);
      MLG_LAUNCH_CHECK();
      if (prof) {
        MLG_CUDA(cudaEventRecord(ev1, st));
        evs.emplace_back(ev0, ev1);
      }
      std::swap(rc, rn);
      std::swap(pc, pn);
    }
    ctl_d.download(ctl.data(), ctl.size(), st);
    c.sync();
    bool running = false;
    bool changed = false;
    for (int s = 0; s < nsys; ++s) {
      const CgCtl& k = ctl[static_cast<std::size_t>(s)];
      if (k.status == kIndefinite)
        throw SolverError("cg_solve: matrix is not positive definite (p'Mp <= 0)");
      const bool sys_running = k.status == kRunning;
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
  for (auto& e : evs) {
    float ms = 0.f;
    MLG_CUDA(cudaEventElapsedTime(&ms, e.first, e.second));
    if (sprof) {
      c.times.ks_ms += ms;
      c.times.ks_launches += 1;
    } else {
      c.times.ka_ms_sum += ms;
      c.times.ka_launches += 1;
    }
  }
  if (sprof) {
    for (std::size_t k = 0; k < ctl.size(); ++k)
      c.times.ks_row_iters += static_cast<double>(sys_h[k].nrows) * ctl[k].iters;
  }
  (mask ? c.times.ks_kernel : c.times.ka_kernel) = use_persist ? 1 : 0;
  if (profiling) {
    unsigned long long rows[2] = {0, 0};
    prof_rows.download(rows, 2, c.stream);
    c.sync();
    c.times.ka_rows += static_cast<double>(rows[0]);
    c.times.ka_check_rows += static_cast<double>(rows[1]);
  }
  if (mask)
    c.times.ks_bytes_per_row = uni ? (xdefer ? 44 : 48) : 88;  // cg_bytes_per_row (bench.py)
  else
    c.times.ka_uniform = uni ? (xdefer ? 2 : 1) : 0;
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

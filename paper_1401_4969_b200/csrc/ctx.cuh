// Host-side data model of the B200 path.  Mirrors the reference's ownership
// (corrector.hpp:47-95): a Hierarchy owns the coarse level, the partition and
// every refinement built so far; each level owns its mesh, space and operators.
// Here all per-level arrays live in HBM and the host keeps only sizes and the
// (tiny) partition rectangles.
//
// HBM layout (full lattice = the reference's DOF numbering, fespace.cpp:230-290:
// dof = iy*(nx+1)+ix on the P1 lattice of a rectangle):
//   tri[nt][3] int32, lat[nv][2] int32, xy[nv][2] f64, parent[nt] int32,
//   bedges[nb][2] int32                         -- Mesh (mesh.hpp:32-50), bit-exact
//   vid[(nx+1)(ny+1)] int32   lattice point -> vertex id (history dependent)
//   geo[2*nx*ny] uint32       geometric triangle (cell, lower/upper) -> (elem<<2)|rot
//   stA[ndofs], stM[ndofs]    Stencil{c,e,n,ne}: the upper half of the symmetric
//                             7-point rows of A and M (W/S/SW are the mirrored
//                             E/N/NE of the neighbour rows, sparse.cpp:36-46)
//   dinv[ndofs] f64           1/A_ii (JacobiPreconditioner, sparse.cpp:186-193)
// Vectors are full-lattice, rhs-interleaved: v[dof*NR + r], boundary rows 0.
#pragma once

#include <cusolverDn.h>

#include <algorithm>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"

namespace mlg {

struct alignas(32) Stencil {
  double c, e, n, ne;
};

// Closed form of the strip (interior dofs outside every closed G_j) at one
// level: block grid, overlap cells and the fine/coarse scale 2^level.
struct StripGeom {
  int side = 1, bw = 1, bh = 1, dc = 0, nx0 = 1, ny0 = 1, scale = 1;
  // closed hole of a domain with a corner hole, fine lattice points of the
  // level (hx1 < hx0: none): its points are outside every CG system
  int hx0 = 1, hx1 = 0, hy0 = 1, hy1 = 0;
  __host__ __device__ bool in_hole(int ix, int iy) const {
    return ix >= hx0 && ix <= hx1 && iy >= hy0 && iy <= hy1;
  }
  __host__ __device__ bool rect_inside_hole(int xa, int xb, int ya, int yb) const {
    return xa >= hx0 && xb <= hx1 && ya >= hy0 && yb <= hy1;
  }
  __host__ __device__ bool rect_meets_hole(int xa, int xb, int ya, int yb) const {
    return xa <= hx1 && xb >= hx0 && ya <= hy1 && yb >= hy0;
  }
};

// A rectangular hole [x0, x1) x [y0, y1) (lattice cells of one level) cut at
// a corner of the bounding rectangle: the L-shaped domains of BASELINE config 3
// (a B200 extension; the reference meshes rectangles only).  x1 == 0 means no
// hole.  Everything stays on the bounding lattice: lattice points strictly
// inside the hole belong to no element ("inactive" dofs, always zero, empty
// rows); points on the hole's edges are Dirichlet boundary.
struct Hole {
  int x0 = 0, y0 = 0, x1 = 0, y1 = 0;
  __host__ __device__ bool any() const { return x1 > x0; }
  __host__ __device__ bool cell_in(int cx, int cy) const {
    return cx >= x0 && cx < x1 && cy >= y0 && cy < y1;
  }
  __host__ __device__ Hole scaled(int s) const { return Hole{x0 * s, y0 * s, x1 * s, y1 * s}; }
};

// Cell (cx, cy) of an nx x ny lattice carries elements.
__host__ __device__ __forceinline__ bool cell_active(const Hole& h, int nx, int ny, int cx,
                                                     int cy) {
  return cx >= 0 && cy >= 0 && cx < nx && cy < ny && !h.cell_in(cx, cy);
}

// Interior points and their row-major order (FeSpace::interior_dofs is
// ascending in dof id = iy*(nx+1)+ix, fespace.cpp:290-310).  With a corner
// hole every interior row is one contiguous x range, so the map is closed form.
struct IMap {
  int nx = 0, ny = 0;
  Hole h;  // at this level's scale
  // closed hole rows [bya, byb] (clamped to 1..ny-1) and their x range [bxa, bxb]
  int bya = 1, byb = 0, bxa = 1, bxb = 0;
  __host__ __device__ int wfull() const { return nx - 1; }
  __host__ __device__ int wband() const { return bxb - bxa + 1; }
  __host__ __device__ bool in_band(int iy) const { return iy >= bya && iy <= byb; }
  __host__ __device__ bool interior(int ix, int iy) const {
    if (ix <= 0 || iy <= 0 || ix >= nx || iy >= ny) return false;
    return !in_band(iy) || (ix >= bxa && ix <= bxb);
  }
  // rows 1..iy-1 before row iy
  __host__ __device__ long long prefix(int iy) const {
    const long long full = static_cast<long long>(iy - 1) * wfull();
    if (byb < bya) return full;
    const int nb = max(0, min(iy - 1, byb) - bya + 1);  // band rows below iy
    return full + static_cast<long long>(nb) * (wband() - wfull());
  }
  __host__ __device__ long long index(int ix, int iy) const {  // -1 if not interior
    if (!interior(ix, iy)) return -1;
    return prefix(iy) + (ix - (in_band(iy) ? bxa : 1));
  }
  __host__ __device__ long long count() const { return prefix(ny); }
  __host__ __device__ void point(long long k, int* ix, int* iy) const {
    // rows come in (at most) three runs: full rows below the band, band rows,
    // full rows above the band
    const int W = wfull();
    if (byb < bya) {
      *iy = static_cast<int>(k / W) + 1;
      *ix = static_cast<int>(k % W) + 1;
      return;
    }
    const long long below = static_cast<long long>(bya - 1) * W;
    if (k < below) {
      *iy = static_cast<int>(k / W) + 1;
      *ix = static_cast<int>(k % W) + 1;
      return;
    }
    const long long kb = k - below, nbw = static_cast<long long>(byb - bya + 1) * wband();
    if (kb < nbw) {
      *iy = bya + static_cast<int>(kb / wband());
      *ix = bxa + static_cast<int>(kb % wband());
      return;
    }
    const long long ka = kb - nbw;
    *iy = byb + 1 + static_cast<int>(ka / W);
    *ix = static_cast<int>(ka % W) + 1;
  }
};

inline IMap make_imap(int nx, int ny, const Hole& h) {
  IMap m;
  m.nx = nx;
  m.ny = ny;
  m.h = h;
  if (h.any()) {
    // closed hole in points: [x0, x1] x [y0, y1]; interior rows it cuts
    m.bya = std::max(h.y0, 1);
    m.byb = std::min(h.y1, ny - 1);
    if (h.x0 == 0) {  // hole on the left: band rows keep x in (x1, nx)
      m.bxa = h.x1 + 1;
      m.bxb = nx - 1;
    } else {  // hole on the right
      m.bxa = 1;
      m.bxb = h.x0 - 1;
    }
  }
  return m;
}

struct Config {
  double x_min = -1.0, x_max = 1.0, y_min = -1.0, y_max = 1.0;
  double H = 0.25;
  double delta = 0.1;
  int m = 4;
  int n_levels = 5;
  int degree = 1;
  int nev = 5;
  int example = 0;  // 0 laplace, 1 variable (CoefficientField, fespace.cpp:105-123),
                    // 2 reaction (BASELINE config 4, B200 extension)
  int workers = 1;
  double cg_tol = 1e-10;
  int deterministic = 1;
  int device = 0;
  unsigned long long seed = 0;  // example 2
  // corner hole (coordinates; hole_x1 <= hole_x0 means none): L-shaped domain
  double hole_x0 = 0.0, hole_x1 = 0.0, hole_y0 = 0.0, hole_y1 = 0.0;
};

// Example 2 coefficients: (k1, k2) = 1 + (splitmix64 outputs 1, 2 of seed) >> 62.
inline void reaction_modes(unsigned long long seed, int* k1, int* k2) {
  auto next = [&seed]() {
    seed += 0x9E3779B97F4A7C15ULL;
    unsigned long long z = seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  };
  *k1 = 1 + static_cast<int>(next() >> 62);
  *k2 = 1 + static_cast<int>(next() >> 62);
}

struct IRect {
  int x0 = 0, y0 = 0, x1 = 0, y1 = 0;
};

// decomp.hpp:59-93 / decomp.cpp:24-86.
struct Partition {
  int m = 0, side = 0, delta_cells = 0, nx0 = 0, ny0 = 0;
  double cell_h = 0.0;
  std::vector<IRect> blocks, overlaps, inners;
  // Level-0 element sets (decomp.cpp:101-121); finer levels are the
  // contiguous descendant ranges [t*4^L, (t+1)*4^L) (children are 4t+c).
  std::vector<std::vector<int>> block_elems, overlap_elems, inner_elems;
  std::vector<int> strip_elems;
  // block (bottom-up row rb, column c) -> subdomain j, -1 for blocks removed
  // by a hole; the reference's order j = (side-1-rb)*side + c otherwise.
  std::vector<int> blk2j;
  int nt0 = 0;  // level-0 elements
};

struct Level {
  int level = 0, nx = 0, ny = 0;
  double dx = 0.0, dy = 0.0;
  std::int64_t nv = 0, nt = 0, nb = 0;
  double h_max = 0.0;
  DevBuf<int> tri, lat, parent, bedges, vid;
  DevBuf<double> xy;
  DevBuf<unsigned> geo;
  DevBuf<Stencil> stA, stM;
  DevBuf<double> dinv;
  DevBuf<unsigned char> strip_mask;  // built lazily (1 = interior dof of the strip)
  StripGeom strip_geom;              // same set in closed form (set with the mask)
  // All interior rows of A (and 1/A_ii) bitwise identical: the CG kernels then
  // take the stencil from kernel parameters (constant-coefficient lattice).
  int uniform = 0;
  int asm_table = 0;  // operators came from k_assemble_table (translation-invariant lattice)
  Stencil ust{0.0, 0.0, 0.0, 0.0};
  double udinv = 0.0;

  Hole hole;  // in this level's cells (none for rectangles)
  // Element degree.  P2 dofs live on the half lattice: grid (2nx+1) x (2ny+1),
  // dof = Y*(2nx+1)+X (p2.cu); gx/gy are the dof-grid extents in both cases.
  int deg = 1;
  int gx() const { return deg == 2 ? 2 * nx : nx; }
  int gy() const { return deg == 2 ? 2 * ny : ny; }
  IMap imap() const { return make_imap(gx(), gy(), deg == 2 ? hole.scaled(2) : hole); }
  // P2 operators: 25 slot values per dof (5x5 half-lattice block, ascending
  // column order) and the mask of structurally present couplings
  DevBuf<double> p2A, p2M;
  DevBuf<unsigned> p2pat;
  std::int64_t p2nnz = 0;
  // CG operator for domains with a hole: the interior restriction of A with
  // identity rows at non-interior points (see corrector.cu ensure_cg_stencil).
  DevBuf<Stencil> stCG;
  DevBuf<double> dinvCG;

  std::int64_t npts() const { return static_cast<std::int64_t>(nx + 1) * (ny + 1); }  // lattice
  std::int64_t ndofs() const { return static_cast<std::int64_t>(gx() + 1) * (gy() + 1); }
  std::int64_t nint() const {
    return hole.any() ? imap().count() : static_cast<std::int64_t>(gx() - 1) * (gy() - 1);
  }
};

struct StepTimes {
  double local_s = 0, iface_s = 0, aug_s = 0, build_s = 0;
  int local_iters_max = 0, strip_iters_max = 0;
  double ka_ms_sum = 0;  // summed device time of the local-solve SpMV kernel
  int ka_launches = 0;
  long long ka_launches_all = 0;  // every launch of that kernel, sampled or not
  double ka_rows = 0;    // rows swept in CG-update mode by those launches (device count)
  double ka_check_rows = 0;  // ... in true-residual mode
  long long kernel_launches = 0;
  int ka_uniform = 0;  // the CG ran the constant-coefficient (no stencil stream) variant
  long long launch_base = 0;  // launch_counter() at the start of the step
  // strip-solve CG kernel (profiling on): every launch timed; algorithmic work =
  // sum over strip systems of unknowns x CG updates (host count, check sweeps excluded)
  double ks_ms = 0;
  long long ks_launches = 0;
  double ks_row_iters = 0;
  int ks_kernel = 0;  // strip batch CG kernel: 0 k_cg_iter, 1 k_cg_persist, 2 k_cg_resident
  int ka_kernel = 0;  // the same for the local batch
  int ks_bytes_per_row = 0;  // algorithmic bytes per unknown and CG update of that kernel
};

struct SolveReport {
  int iterations = 0;
  double final_residual = 0.0;
  int converged = 0;
};

class Ctx;

// ---- mesh.cu -------------------------------------------------------------
void build_level0(Ctx& c);
void refine_level(Ctx& c, const Level& coarse, Level& fine);
void export_mesh(Ctx& c, const Level& L, double* xy, int* lat, int* tri, int* parent,
                 int* bedges);
void export_space(Ctx& c, const Level& L, int* dof_lattice, int* interior_dofs,
                  int* interior_index, int* conn3);

// ---- assemble.cu ---------------------------------------------------------
void assemble_level(Ctx& c, Level& L);
void export_csr(Ctx& c, const Level& L, int form, int* row_ptr, int* cols, double* vals);
std::int64_t csr_nnz(const Level& L);
void interior_dense(Ctx& c, const Level& L, int form, double* d_dense);

class Ctx {
 public:
  explicit Ctx(const Config& cfg);
  ~Ctx();
  Config cfg;
  Partition part;
  cudaStream_t stream = nullptr;
  cusolverDnHandle_t solver = nullptr;
  std::vector<std::unique_ptr<Level>> levels;
  int max_level() const { return static_cast<int>(levels.size()) - 1; }
  Level& level(int k) {
    if (k < 0 || k > max_level())
      throw ConfigError("level " + std::to_string(k) + " not built");
    return *levels[k];
  }
  void extend_to(int level);
  void sync() { MLG_CUDA(cudaStreamSynchronize(stream)); }

  // Coarse dense interior blocks (corrector.cpp:172-181), cached.
  DevBuf<double> coarse_a, coarse_b, coarse_bchol;
  int mc = 0;
  bool coarse_ready = false;
  void ensure_coarse_dense();
  // Spectrum of the coarse pencil A_cc V = B_cc V diag(lam), V'B_cc V = I
  // (ascending), cached for the arrowhead form of the augmented problem.
  DevBuf<double> coarse_lam, coarse_vec;
  bool spectrum_ready = false;
  void ensure_coarse_spectrum();

  // Scratch (grow-only) owned by the context.
  DevBuf<double> io_in, io_out, io_u_in, io_u_out;  // C-ABI step marshalling
  DevBuf<unsigned char> scratch;
  void* scratch_bytes(std::size_t n) {
    scratch.ensure(n);
    return scratch.get();
  }
  std::shared_ptr<void> ws;  // corrector.cu Workspace (CG pools, step vectors)
  // Pooled timing events (created once, reused by every profiled launch).
  std::vector<cudaEvent_t> ev_pool;
  cudaEvent_t event(std::size_t i) {
    while (ev_pool.size() <= i) {
      cudaEvent_t e;
      MLG_CUDA(cudaEventCreate(&e));
      ev_pool.push_back(e);
    }
    return ev_pool[i];
  }
  bool profile = false;  // record CUDA events around the local-solve SpMV kernel
  StepTimes times;
  // Stream whose prior work the *_device entry points wait for before reading
  // caller-owned device memory (mlg_set_input_stream; 0 = legacy default stream).
  cudaStream_t input_stream = nullptr;
  // k_assemble of the most recent level built with profiling on (CUDA events)
  double asm_ms = 0, asm_dofs = 0;
  int asm_kernel = 0;  // 0 k_assemble (generic gather), 1 k_assemble_table, 2 k_assemble_var
  cudaEvent_t input_ready = nullptr;
  void order_after_input() {
    if (!input_ready) MLG_CUDA(cudaEventCreateWithFlags(&input_ready, cudaEventDisableTiming));
    MLG_CUDA(cudaEventRecord(input_ready, input_stream));
    MLG_CUDA(cudaStreamWaitEvent(stream, input_ready, 0));
  }
};

}  // namespace mlg

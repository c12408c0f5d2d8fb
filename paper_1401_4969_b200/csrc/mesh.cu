// Level build, integer part: structured coarse mesh and uniform red
// refinement on device, bit-exact with the reference's numbering.
//
//   build_structured_mesh  mesh.cpp:68-104   (lexicographic vertices, 2 tris/cell)
//   refine_regular         mesh.cpp:106-155  (parents keep ids; midpoints
//                          appended in ascending edge-key order min*nv+max;
//                          children 4t+{0..3}; parent map)
//   compute_boundary_edges mesh.cpp:50-64    (count-1 edges in key order)
//   compute_h_max          mesh.cpp:34-48
//
// B200 design: the reference sorts 3T int64 edge keys through a std::map.  On
// the structured lattice every mesh edge is a lattice edge, so the rank of
// edge (a,b), a<b, in key order is  off[a] + #{neighbours c of a : a<c<b}
// with off = exclusive scan of "neighbours with a larger id".  That turns the
// sort into one O(V) count, one scan and one O(V) emit, all coalesced.
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <climits>
#include <cmath>

#include "ctx.cuh"

namespace mlg {
namespace {

constexpr int kBlock = 256;

// Lattice neighbours that share a mesh edge on the SW-NE split lattice:
// E, W, N, S, NE, SW.
__constant__ int kNbDx[6] = {1, -1, 0, 0, 1, -1};
__constant__ int kNbDy[6] = {0, 0, 1, -1, 1, -1};

__global__ void k_level0_vertices(int nx, int ny, double x0, double y0, double dx, double dy,
                                  int* lat, double* xy, int* vid) {
  const std::int64_t v = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  const std::int64_t nv = static_cast<std::int64_t>(nx + 1) * (ny + 1);
  if (v >= nv) return;
  const int ix = static_cast<int>(v % (nx + 1)), iy = static_cast<int>(v / (nx + 1));
  lat[2 * v] = ix;
  lat[2 * v + 1] = iy;
  xy[2 * v] = lattice_coord(x0, ix, dx);
  xy[2 * v + 1] = lattice_coord(y0, iy, dy);
  vid[v] = static_cast<int>(v);
}

// Two triangles per cell {v00,v10,v11},{v00,v11,v01} (mesh.cpp:96-97).
// geo slot 2*cell+0 = lower-right "L" triangle, 2*cell+1 = upper-left "U";
// canonical CCW orders L:(00,10,11), U:(00,11,01); level 0 has rotation 0.
__global__ void k_level0_triangles(int nx, int ny, int* tri, unsigned* geo) {
  const std::int64_t c = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (c >= static_cast<std::int64_t>(nx) * ny) return;
  const int ix = static_cast<int>(c % nx), iy = static_cast<int>(c / nx);
  const int v00 = iy * (nx + 1) + ix, v10 = v00 + 1, v01 = v00 + nx + 1, v11 = v01 + 1;
  int* t = tri + 6 * c;
  t[0] = v00;
  t[1] = v10;
  t[2] = v11;
  t[3] = v00;
  t[4] = v11;
  t[5] = v01;
  geo[2 * c] = static_cast<unsigned>(2 * c) << 2;
  geo[2 * c + 1] = static_cast<unsigned>(2 * c + 1) << 2;
}

// ---- level 0 of a domain with a corner hole (B200 extension, config 3) ----
// Vertices: the lattice points touching an element, lexicographic (y, x) --
// the order build_structured_mesh uses for rectangles (mesh.cpp:80-90);
// triangles: two per element-carrying cell, cells lexicographic, the same
// split {v00,v10,v11},{v00,v11,v01} (mesh.cpp:96-97).
__device__ __forceinline__ bool point_active(const Hole& h, int nx, int ny, int ix, int iy) {
  return cell_active(h, nx, ny, ix, iy) || cell_active(h, nx, ny, ix - 1, iy) ||
         cell_active(h, nx, ny, ix, iy - 1) || cell_active(h, nx, ny, ix - 1, iy - 1);
}

__global__ void k_hole_flags(int nx, int ny, Hole h, int* pflag, int* cflag) {
  const std::int64_t v = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  const std::int64_t np = static_cast<std::int64_t>(nx + 1) * (ny + 1);
  if (v < np) {
    const int ix = static_cast<int>(v % (nx + 1)), iy = static_cast<int>(v / (nx + 1));
    pflag[v] = point_active(h, nx, ny, ix, iy) ? 1 : 0;
  }
  if (v < static_cast<std::int64_t>(nx) * ny) {
    const int cx = static_cast<int>(v % nx), cy = static_cast<int>(v / nx);
    cflag[v] = cell_active(h, nx, ny, cx, cy) ? 1 : 0;
  }
}

__global__ void k_level0_hole(int nx, int ny, Hole h, double x0, double y0, double dx,
                              double dy, const int* prank, const int* crank, int* lat,
                              double* xy, int* vid, int* tri, unsigned* geo) {
  const std::int64_t v = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  const std::int64_t np = static_cast<std::int64_t>(nx + 1) * (ny + 1);
  if (v < np) {
    const int ix = static_cast<int>(v % (nx + 1)), iy = static_cast<int>(v / (nx + 1));
    if (point_active(h, nx, ny, ix, iy)) {
      const int id = prank[v];
      lat[2 * id] = ix;
      lat[2 * id + 1] = iy;
      xy[2 * id] = lattice_coord(x0, ix, dx);
      xy[2 * id + 1] = lattice_coord(y0, iy, dy);
      vid[v] = id;
    } else {
      vid[v] = -1;
    }
  }
  if (v < static_cast<std::int64_t>(nx) * ny) {
    const int cx = static_cast<int>(v % nx), cy = static_cast<int>(v / nx);
    if (!cell_active(h, nx, ny, cx, cy)) {
      geo[2 * v] = geo[2 * v + 1] = 0xFFFFFFFFu;
      return;
    }
    const std::int64_t r = crank[v];
    const std::int64_t p00 = static_cast<std::int64_t>(cy) * (nx + 1) + cx;
    const int v00 = prank[p00], v10 = prank[p00 + 1], v01 = prank[p00 + nx + 1],
              v11 = prank[p00 + nx + 2];
    int* t = tri + 6 * r;
    t[0] = v00;
    t[1] = v10;
    t[2] = v11;
    t[3] = v00;
    t[4] = v11;
    t[5] = v01;
    geo[2 * v] = static_cast<unsigned>(2 * r) << 2;
    geo[2 * v + 1] = static_cast<unsigned>(2 * r + 1) << 2;
  }
}

// Boundary edges of a domain with a hole: lattice edges with exactly one
// element-carrying cell beside them (count-1 edges, mesh.cpp:50-64).  Keys are
// appended in any order; k_rank_keys then orders them like std::map.
__global__ void k_boundary_keys_hole(int nx, int ny, Hole h, const int* vid, std::int64_t nv,
                                     long long* keys, int* n_out) {
  const std::int64_t e = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  const std::int64_t nh = static_cast<std::int64_t>(nx) * (ny + 1);
  const std::int64_t nvv = static_cast<std::int64_t>(nx + 1) * ny;
  if (e >= nh + nvv) return;
  int ax, ay, bx, by;
  bool c1, c2;
  if (e < nh) {  // horizontal (ax,ay)-(ax+1,ay): cells below / above
    ax = static_cast<int>(e % nx);
    ay = static_cast<int>(e / nx);
    bx = ax + 1;
    by = ay;
    c1 = cell_active(h, nx, ny, ax, ay - 1);
    c2 = cell_active(h, nx, ny, ax, ay);
  } else {  // vertical (ax,ay)-(ax,ay+1): cells left / right
    const std::int64_t f = e - nh;
    ax = static_cast<int>(f % (nx + 1));
    ay = static_cast<int>(f / (nx + 1));
    bx = ax;
    by = ay + 1;
    c1 = cell_active(h, nx, ny, ax - 1, ay);
    c2 = cell_active(h, nx, ny, ax, ay);
  }
  if (c1 == c2) return;
  const long long u = vid[static_cast<std::int64_t>(ay) * (nx + 1) + ax];
  const long long w = vid[static_cast<std::int64_t>(by) * (nx + 1) + bx];
  keys[atomicAdd(n_out, 1)] = (u < w) ? u * nv + w : w * nv + u;
}

// Position of a triangle (given its vertex lattices in element order) on the
// lattice: cell, L/U type and the rotation rot with t[k] = canonical[(rot+k)%3].
__device__ __forceinline__ unsigned geo_slot(int x0, int y0, int x1, int y1, int x2, int y2,
                                             int nx, unsigned elem, unsigned* slot_out) {
  const int cx = min(x0, min(x1, x2)), cy = min(y0, min(y1, y2));
  const bool upper = (x0 == cx && y0 == cy + 1) || (x1 == cx && y1 == cy + 1) ||
                     (x2 == cx && y2 == cy + 1);
  const int k = (x0 == cx && y0 == cy) ? 0 : ((x1 == cx && y1 == cy) ? 1 : 2);
  const unsigned rot = static_cast<unsigned>((3 - k) % 3);
  *slot_out = 2u * static_cast<unsigned>(cy * nx + cx) + (upper ? 1u : 0u);
  return (elem << 2) | rot;
}

__device__ __forceinline__ double edge_len(int ax, int ay, int bx, int by, double dx, double dy) {
  const double ex = xmul(static_cast<double>(bx - ax), dx);
  const double ey = xmul(static_cast<double>(by - ay), dy);
  return sqrt(xadd(xmul(ex, ex), xmul(ey, ey)));
}

__device__ __forceinline__ void atomic_max_pos(double* addr, double v) {
  // Positive doubles order like their bit patterns: exact, order-independent.
  atomicMax(reinterpret_cast<unsigned long long*>(addr),
            static_cast<unsigned long long>(__double_as_longlong(v)));
}

__global__ void k_hmax(const int* tri, const int* lat, std::int64_t nt, double dx, double dy,
                       double* hmax) {
  const std::int64_t t = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  double h = 0.0;
  if (t < nt) {
    for (int e = 0; e < 3; ++e) {
      const int a = tri[3 * t + e], b = tri[3 * t + (e + 1) % 3];
      h = fmax(h, edge_len(lat[2 * a], lat[2 * a + 1], lat[2 * b], lat[2 * b + 1], dx, dy));
    }
  }
  for (int o = 16; o > 0; o >>= 1) h = fmax(h, __shfl_xor_sync(0xffffffffu, h, o));
  if ((threadIdx.x & 31) == 0 && h > 0.0) atomic_max_pos(hmax, h);
}

__global__ void k_ref_parent_verts(std::int64_t nv, const int* lat_c, int nxf, double x0,
                                   double y0, double dxf, double dyf, int* lat_f, double* xy_f,
                                   int* vid_f) {
  const std::int64_t v = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (v >= nv) return;
  const int ix = 2 * lat_c[2 * v], iy = 2 * lat_c[2 * v + 1];
  lat_f[2 * v] = ix;
  lat_f[2 * v + 1] = iy;
  xy_f[2 * v] = lattice_coord(x0, ix, dxf);
  xy_f[2 * v + 1] = lattice_coord(y0, iy, dyf);
  vid_f[static_cast<std::int64_t>(iy) * (nxf + 1) + ix] = static_cast<int>(v);
}

// The lattice edge from (ix,iy) in direction d (E, W, N, S, NE, SW) is a mesh
// edge iff one of the cells containing it carries elements (with a corner
// hole two active points can face each other across a removed cell).
__device__ __forceinline__ bool edge_exists(const Hole& h, int nx, int ny, int ix, int iy,
                                            int d) {
  if (!h.any()) return true;
  switch (d) {
    case 0: return cell_active(h, nx, ny, ix, iy) || cell_active(h, nx, ny, ix, iy - 1);
    case 1: return cell_active(h, nx, ny, ix - 1, iy) || cell_active(h, nx, ny, ix - 1, iy - 1);
    case 2: return cell_active(h, nx, ny, ix, iy) || cell_active(h, nx, ny, ix - 1, iy);
    case 3: return cell_active(h, nx, ny, ix, iy - 1) || cell_active(h, nx, ny, ix - 1, iy - 1);
    case 4: return cell_active(h, nx, ny, ix, iy);
    default: return cell_active(h, nx, ny, ix - 1, iy - 1);
  }
}

__global__ void k_ref_count(std::int64_t nv, const int* lat_c, const int* vid_c, int nxc,
                            int nyc, Hole hc, int* count) {
  const std::int64_t a = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (a >= nv) return;
  const int ix = lat_c[2 * a], iy = lat_c[2 * a + 1];
  int cnt = 0;
#pragma unroll
  for (int d = 0; d < 6; ++d) {
    const int jx = ix + kNbDx[d], jy = iy + kNbDy[d];
    if (jx < 0 || jy < 0 || jx > nxc || jy > nyc) continue;
    if (!edge_exists(hc, nxc, nyc, ix, iy, d)) continue;
    if (vid_c[static_cast<std::int64_t>(jy) * (nxc + 1) + jx] > a) ++cnt;
  }
  count[a] = cnt;
}

// Midpoint ids: V + rank in ascending (min*nv+max) order (mesh.cpp:121-135).
__global__ void k_ref_midpoints(std::int64_t nv, const int* lat_c, const int* vid_c, int nxc,
                                int nyc, Hole hc, const int* off, int nxf, double x0, double y0,
                                double dxf, double dyf, int* lat_f, double* xy_f, int* vid_f) {
  const std::int64_t a = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (a >= nv) return;
  const int ix = lat_c[2 * a], iy = lat_c[2 * a + 1];
  int ids[6], mx[6], my[6], n = 0;
#pragma unroll
  for (int d = 0; d < 6; ++d) {
    const int jx = ix + kNbDx[d], jy = iy + kNbDy[d];
    if (jx < 0 || jy < 0 || jx > nxc || jy > nyc) continue;
    if (!edge_exists(hc, nxc, nyc, ix, iy, d)) continue;
    const int b = vid_c[static_cast<std::int64_t>(jy) * (nxc + 1) + jx];
    if (b <= a) continue;
    // insertion by id
    int k = n++;
    while (k > 0 && ids[k - 1] > b) {
      ids[k] = ids[k - 1];
      mx[k] = mx[k - 1];
      my[k] = my[k - 1];
      --k;
    }
    ids[k] = b;
    mx[k] = ix + jx;  // fine lattice of the midpoint = sum of coarse lattices
    my[k] = iy + jy;
  }
  const std::int64_t base = nv + off[a];
  for (int k = 0; k < n; ++k) {
    const std::int64_t id = base + k;
    lat_f[2 * id] = mx[k];
    lat_f[2 * id + 1] = my[k];
    xy_f[2 * id] = lattice_coord(x0, mx[k], dxf);
    xy_f[2 * id + 1] = lattice_coord(y0, my[k], dyf);
    vid_f[static_cast<std::int64_t>(my[k]) * (nxf + 1) + mx[k]] = static_cast<int>(id);
  }
}

// Children 4t+{0..3} = {a,mab,mca},{mab,b,mbc},{mca,mbc,c},{mab,mbc,mca}
// (mesh.cpp:139-150), their lattice slots, and h_max of the fine mesh.
__global__ void k_ref_children(std::int64_t nt, const int* tri_c, const int* lat_c,
                               const int* vid_f, int nxf, double dxf, double dyf, int* tri_f,
                               int* parent_f, unsigned* geo_f, double* hmax) {
  const std::int64_t t = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  double h = 0.0;
  if (t < nt) {
    const int a = tri_c[3 * t], b = tri_c[3 * t + 1], c = tri_c[3 * t + 2];
    const int ax = lat_c[2 * a], ay = lat_c[2 * a + 1];
    const int bx = lat_c[2 * b], by = lat_c[2 * b + 1];
    const int cx = lat_c[2 * c], cy = lat_c[2 * c + 1];
    // fine lattices
    const int Ax = 2 * ax, Ay = 2 * ay, Bx = 2 * bx, By = 2 * by, Cx = 2 * cx, Cy = 2 * cy;
    const int Px = ax + bx, Py = ay + by;  // mab
    const int Qx = bx + cx, Qy = by + cy;  // mbc
    const int Rx = cx + ax, Ry = cy + ay;  // mca
    const std::int64_t st = nxf + 1;
    const int mab = vid_f[Py * st + Px], mbc = vid_f[Qy * st + Qx], mca = vid_f[Ry * st + Rx];
    const int ch[4][3] = {{a, mab, mca}, {mab, b, mbc}, {mca, mbc, c}, {mab, mbc, mca}};
    const int cl[4][6] = {{Ax, Ay, Px, Py, Rx, Ry},
                          {Px, Py, Bx, By, Qx, Qy},
                          {Rx, Ry, Qx, Qy, Cx, Cy},
                          {Px, Py, Qx, Qy, Rx, Ry}};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const std::int64_t e = 4 * t + k;
      tri_f[3 * e] = ch[k][0];
      tri_f[3 * e + 1] = ch[k][1];
      tri_f[3 * e + 2] = ch[k][2];
      parent_f[e] = static_cast<int>(t);
      unsigned slot;
      const unsigned code = geo_slot(cl[k][0], cl[k][1], cl[k][2], cl[k][3], cl[k][4], cl[k][5],
                                     nxf, static_cast<unsigned>(e), &slot);
      geo_f[slot] = code;
      h = fmax(h, edge_len(cl[k][0], cl[k][1], cl[k][2], cl[k][3], dxf, dyf));
      h = fmax(h, edge_len(cl[k][2], cl[k][3], cl[k][4], cl[k][5], dxf, dyf));
      h = fmax(h, edge_len(cl[k][4], cl[k][5], cl[k][0], cl[k][1], dxf, dyf));
    }
  }
  for (int o = 16; o > 0; o >>= 1) h = fmax(h, __shfl_xor_sync(0xffffffffu, h, o));
  if ((threadIdx.x & 31) == 0 && h > 0.0) atomic_max_pos(hmax, h);
}

// Boundary edges of the rectangle lattice, enumerated bottom, top, left,
// right; key = min*nv + max.
__global__ void k_boundary_keys(int nx, int ny, const int* vid, std::int64_t nv,
                                long long* keys) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int nb = 2 * (nx + ny);
  if (b >= nb) return;
  int ax, ay, bx, by;
  if (b < nx) {
    ax = b; ay = 0; bx = b + 1; by = 0;
  } else if (b < 2 * nx) {
    ax = b - nx; ay = ny; bx = ax + 1; by = ny;
  } else if (b < 2 * nx + ny) {
    ax = 0; ay = b - 2 * nx; bx = 0; by = ay + 1;
  } else {
    ax = nx; ay = b - 2 * nx - ny; bx = nx; by = ay + 1;
  }
  const long long u = vid[static_cast<std::int64_t>(ay) * (nx + 1) + ax];
  const long long w = vid[static_cast<std::int64_t>(by) * (nx + 1) + bx];
  keys[b] = (u < w) ? u * nv + w : w * nv + u;
}

// Rank-by-counting sort of the (unique) boundary keys; writes (key/nv, key%nv)
// at its rank, which is exactly the std::map iteration order of mesh.cpp:57-63.
__global__ void k_rank_keys(const long long* keys, int n, std::int64_t nv, int* out) {
  __shared__ long long tile[1024];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const long long mine = (i < n) ? keys[i] : 0;
  int rank = 0;
  for (int base = 0; base < n; base += 1024) {
    for (int k = threadIdx.x; k < 1024; k += blockDim.x)
      tile[k] = (base + k < n) ? keys[base + k] : LLONG_MAX;
    __syncthreads();
    const int lim = min(1024, n - base);
    for (int k = 0; k < lim; ++k) rank += (tile[k] < mine) ? 1 : 0;
    __syncthreads();
  }
  if (i < n) {
    out[2 * rank] = static_cast<int>(mine / nv);
    out[2 * rank + 1] = static_cast<int>(mine % nv);
  }
}

void boundary_edges(Ctx& c, Level& L) {
  if (L.hole.any()) {
    // outer boundary + the two inner sides of the hole (the hole touches one
    // corner, so the count is the rectangle's)
    const int nb = 2 * (L.nx + L.ny);
    L.nb = nb;
    L.bedges.alloc(2 * static_cast<std::size_t>(nb));
    DevBuf<long long> keys(nb);
    DevBuf<int> n(1);
    n.zero(c.stream);
    const std::int64_t ne = static_cast<std::int64_t>(L.nx) * (L.ny + 1) +
                            static_cast<std::int64_t>(L.nx + 1) * L.ny;
    k_boundary_keys_hole<<<grid_for(ne, kBlock), kBlock, 0, c.stream>>>(
        L.nx, L.ny, L.hole, L.vid.get(), L.nv, keys.get(), n.get());
    MLG_LAUNCH_CHECK();
    int got = 0;
    n.download(&got, 1, c.stream);
    c.sync();
    if (got != nb) throw SolverError("boundary of the L-shaped mesh has an unexpected length");
    k_rank_keys<<<grid_for(nb, kBlock), kBlock, 0, c.stream>>>(keys.get(), nb, L.nv,
                                                              L.bedges.get());
    MLG_LAUNCH_CHECK();
    c.sync();
    return;
  }
  const int nb = 2 * (L.nx + L.ny);
  L.nb = nb;
  L.bedges.alloc(2 * static_cast<std::size_t>(nb));
  auto* keys = static_cast<long long*>(c.scratch_bytes(sizeof(long long) * nb));
  k_boundary_keys<<<grid_for(nb, kBlock), kBlock, 0, c.stream>>>(L.nx, L.ny, L.vid.get(), L.nv,
                                                                  keys);
  MLG_LAUNCH_CHECK();
  k_rank_keys<<<grid_for(nb, kBlock), kBlock, 0, c.stream>>>(keys, nb, L.nv, L.bedges.get());
  MLG_LAUNCH_CHECK();
}

__global__ void k_dof_lattice(int nx, int ny, int* dof_lattice) {
  const std::int64_t d = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (d >= static_cast<std::int64_t>(nx + 1) * (ny + 1)) return;
  dof_lattice[2 * d] = 2 * static_cast<int>(d % (nx + 1));
  dof_lattice[2 * d + 1] = 2 * static_cast<int>(d / (nx + 1));
}

__global__ void k_interior_lists(IMap m, int* interior_dofs, int* interior_index) {
  const int nx = m.nx, ny = m.ny;
  const std::int64_t d = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (d >= static_cast<std::int64_t>(nx + 1) * (ny + 1)) return;
  const int ix = static_cast<int>(d % (nx + 1)), iy = static_cast<int>(d / (nx + 1));
  const long long k = m.index(ix, iy);
  if (interior_index) interior_index[d] = static_cast<int>(k);
  if (k >= 0 && interior_dofs) interior_dofs[k] = static_cast<int>(d);
}

__global__ void k_connectivity(std::int64_t nt, const int* tri, const int* lat, int nx,
                               int* conn3) {
  const std::int64_t t = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (t >= nt) return;
  for (int k = 0; k < 3; ++k) {
    const int v = tri[3 * t + k];
    conn3[3 * t + k] = lat[2 * v + 1] * (nx + 1) + lat[2 * v];
  }
}

}  // namespace

// The config's corner hole in coarse cells (aligned to H, touching exactly one
// corner of the bounding rectangle, strictly smaller in both directions).
Hole hole_cells(const Config& cfg, int nx, int ny) {
  if (!(cfg.hole_x1 > cfg.hole_x0) && !(cfg.hole_y1 > cfg.hole_y0)) return Hole{};
  auto cell = [&](double v, double lo, int n, const char* what) {
    const double r = (v - lo) / cfg.H;
    const int k = static_cast<int>(std::lround(r));
    if (std::abs(r - k) > 1e-9 * std::max(1.0, std::abs(r)) || k < 0 || k > n)
      throw ConfigError(std::string("hole ") + what + " is not on the coarse lattice");
    return k;
  };
  Hole h;
  h.x0 = cell(cfg.hole_x0, cfg.x_min, nx, "x_min");
  h.x1 = cell(cfg.hole_x1, cfg.x_min, nx, "x_max");
  h.y0 = cell(cfg.hole_y0, cfg.y_min, ny, "y_min");
  h.y1 = cell(cfg.hole_y1, cfg.y_min, ny, "y_max");
  if (!(h.x1 > h.x0) || !(h.y1 > h.y0))
    throw ConfigError("hole rectangle must have positive side lengths");
  const bool cx = (h.x0 == 0) != (h.x1 == nx), cy = (h.y0 == 0) != (h.y1 == ny);
  if (!cx || !cy)
    throw ConfigError("hole must touch exactly one corner of the domain rectangle (L-shape)");
  return h;
}

void build_level0(Ctx& c) {
  auto L = std::make_unique<Level>();
  const Config& cfg = c.cfg;
  // checked_cell_count (mesh.cpp:18-25)
  auto cells = [](double length, double H, const char* axis) {
    const double ratio = length / H;
    const int n = static_cast<int>(std::lround(ratio));
    if (n < 1 || std::abs(ratio - n) > 1e-9 * std::max(1.0, ratio))
      throw ConfigError(std::string("mesh size H does not divide the ") + axis +
                        " side length into an integer number of cells");
    return n;
  };
  if (!(cfg.x_min < cfg.x_max) || !(cfg.y_min < cfg.y_max))
    throw ConfigError("domain rectangle must have positive side lengths");
  if (!(cfg.H > 0.0)) throw ConfigError("mesh size H must be positive");
  L->level = 0;
  L->deg = cfg.degree;
  L->nx = cells(cfg.x_max - cfg.x_min, cfg.H, "x");
  L->ny = cells(cfg.y_max - cfg.y_min, cfg.H, "y");
  L->dx = (cfg.x_max - cfg.x_min) / L->nx;
  L->dy = (cfg.y_max - cfg.y_min) / L->ny;
  L->hole = hole_cells(cfg, L->nx, L->ny);
  if (L->hole.any()) {
    const std::int64_t np = L->npts(), ncell = static_cast<std::int64_t>(L->nx) * L->ny;
    DevBuf<int> pflag(np + 1), cflag(ncell + 1), prank(np + 1), crank(ncell + 1);
    pflag.zero(c.stream);
    cflag.zero(c.stream);
    k_hole_flags<<<grid_for(np, kBlock), kBlock, 0, c.stream>>>(L->nx, L->ny, L->hole,
                                                               pflag.get(), cflag.get());
    MLG_LAUNCH_CHECK();
    std::size_t tb1 = 0, tb2 = 0;
    MLG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb1, pflag.get(), prank.get(),
                                           static_cast<int>(np + 1), c.stream));
    MLG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb2, cflag.get(), crank.get(),
                                           static_cast<int>(ncell + 1), c.stream));
    void* tmp = c.scratch_bytes(std::max(tb1, tb2));
    MLG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb1, pflag.get(), prank.get(),
                                           static_cast<int>(np + 1), c.stream));
    int nvh = 0, nch = 0;
    MLG_CUDA(cudaMemcpyAsync(&nvh, prank.get() + np, sizeof(int), cudaMemcpyDeviceToHost,
                             c.stream));
    c.sync();
    MLG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb2, cflag.get(), crank.get(),
                                           static_cast<int>(ncell + 1), c.stream));
    MLG_CUDA(cudaMemcpyAsync(&nch, crank.get() + ncell, sizeof(int), cudaMemcpyDeviceToHost,
                             c.stream));
    c.sync();
    L->nv = nvh;
    L->nt = 2LL * nch;
    L->lat.alloc(2 * L->nv);
    L->xy.alloc(2 * L->nv);
    L->vid.alloc(np);
    L->tri.alloc(3 * L->nt);
    L->geo.alloc(2 * ncell);
    k_level0_hole<<<grid_for(np, kBlock), kBlock, 0, c.stream>>>(
        L->nx, L->ny, L->hole, cfg.x_min, cfg.y_min, L->dx, L->dy, prank.get(), crank.get(),
        L->lat.get(), L->xy.get(), L->vid.get(), L->tri.get(), L->geo.get());
    MLG_LAUNCH_CHECK();
    c.sync();
  } else {
  L->nv = L->npts();
  L->nt = 2LL * L->nx * L->ny;
  L->lat.alloc(2 * L->nv);
  L->xy.alloc(2 * L->nv);
  L->vid.alloc(L->nv);
  L->tri.alloc(3 * L->nt);
  L->geo.alloc(L->nt);
  k_level0_vertices<<<grid_for(L->nv, kBlock), kBlock, 0, c.stream>>>(
      L->nx, L->ny, cfg.x_min, cfg.y_min, L->dx, L->dy, L->lat.get(), L->xy.get(), L->vid.get());
  MLG_LAUNCH_CHECK();
  k_level0_triangles<<<grid_for(static_cast<std::int64_t>(L->nx) * L->ny, kBlock), kBlock, 0,
                       c.stream>>>(L->nx, L->ny, L->tri.get(), L->geo.get());
  MLG_LAUNCH_CHECK();
  }
  boundary_edges(c, *L);
  auto* hm = static_cast<double*>(c.scratch_bytes(sizeof(double)));
  MLG_CUDA(cudaMemsetAsync(hm, 0, sizeof(double), c.stream));
  k_hmax<<<grid_for(L->nt, kBlock), kBlock, 0, c.stream>>>(L->tri.get(), L->lat.get(), L->nt,
                                                          L->dx, L->dy, hm);
  MLG_LAUNCH_CHECK();
  MLG_CUDA(cudaMemcpyAsync(&L->h_max, hm, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  c.levels.push_back(std::move(L));
}

void refine_level(Ctx& c, const Level& C, Level& F) {
  F.level = C.level + 1;
  F.deg = C.deg;
  F.nx = 2 * C.nx;
  F.ny = 2 * C.ny;
  F.dx = (c.cfg.x_max - c.cfg.x_min) / F.nx;
  F.dy = (c.cfg.y_max - c.cfg.y_min) / F.ny;
  F.nt = 4 * C.nt;
  F.hole = C.hole.scaled(2);
  std::int64_t nvf_max = F.npts();
  if (F.hole.any()) {  // lattice points strictly inside the hole carry no vertex
    const std::int64_t ix = F.hole.x0 == 0 ? F.hole.x1 : F.nx - F.hole.x0;
    const std::int64_t iy = F.hole.y0 == 0 ? F.hole.y1 : F.ny - F.hole.y0;
    nvf_max -= ix * iy;
  }
  if (F.nt >= (1LL << 30) || nvf_max >= (1LL << 31))
    throw ConfigError("refined mesh exceeds the 32-bit index range of the reference layout");
  F.lat.alloc(2 * nvf_max);
  F.xy.alloc(2 * nvf_max);
  F.vid.alloc(F.npts());
  F.tri.alloc(3 * F.nt);
  F.parent.alloc(F.nt);
  F.geo.alloc(2LL * F.nx * F.ny);
  if (F.hole.any()) {  // absent points / cells
    MLG_CUDA(cudaMemsetAsync(F.vid.get(), 0xFF, sizeof(int) * F.npts(), c.stream));
    MLG_CUDA(cudaMemsetAsync(F.geo.get(), 0xFF, sizeof(unsigned) * 2 * F.nx * F.ny, c.stream));
  }

  const std::int64_t nv = C.nv;
  k_ref_parent_verts<<<grid_for(nv, kBlock), kBlock, 0, c.stream>>>(
      nv, C.lat.get(), F.nx, c.cfg.x_min, c.cfg.y_min, F.dx, F.dy, F.lat.get(), F.xy.get(),
      F.vid.get());
  MLG_LAUNCH_CHECK();

  // count + exclusive scan (cub) -> edge ranks grouped by the min endpoint
  DevBuf<int> count(nv + 1), off(nv + 1);
  k_ref_count<<<grid_for(nv, kBlock), kBlock, 0, c.stream>>>(nv, C.lat.get(), C.vid.get(), C.nx,
                                                            C.ny, C.hole, count.get());
  MLG_LAUNCH_CHECK();
  MLG_CUDA(cudaMemsetAsync(count.get() + nv, 0, sizeof(int), c.stream));
  std::size_t tmp_bytes = 0;
  MLG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, count.get(), off.get(),
                                         static_cast<int>(nv + 1), c.stream));
  void* tmp = c.scratch_bytes(tmp_bytes);
  MLG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, count.get(), off.get(),
                                         static_cast<int>(nv + 1), c.stream));
  int n_edges = 0;
  MLG_CUDA(cudaMemcpyAsync(&n_edges, off.get() + nv, sizeof(int), cudaMemcpyDeviceToHost,
                           c.stream));
  c.sync();
  F.nv = nv + n_edges;
  if (F.nv != nvf_max)
    throw SolverError("refinement produced a non-lattice vertex set (" + std::to_string(F.nv) +
                      " vs " + std::to_string(nvf_max) + ")");
  k_ref_midpoints<<<grid_for(nv, kBlock), kBlock, 0, c.stream>>>(
      nv, C.lat.get(), C.vid.get(), C.nx, C.ny, C.hole, off.get(), F.nx, c.cfg.x_min, c.cfg.y_min, F.dx,
      F.dy, F.lat.get(), F.xy.get(), F.vid.get());
  MLG_LAUNCH_CHECK();

  auto* hm = static_cast<double*>(c.scratch_bytes(sizeof(double)));
  MLG_CUDA(cudaMemsetAsync(hm, 0, sizeof(double), c.stream));
  k_ref_children<<<grid_for(C.nt, kBlock), kBlock, 0, c.stream>>>(
      C.nt, C.tri.get(), C.lat.get(), F.vid.get(), F.nx, F.dx, F.dy, F.tri.get(), F.parent.get(),
      F.geo.get(), hm);
  MLG_LAUNCH_CHECK();
  MLG_CUDA(cudaMemcpyAsync(&F.h_max, hm, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  boundary_edges(c, F);
  c.sync();
}

void export_mesh(Ctx& c, const Level& L, double* xy, int* lat, int* tri, int* parent,
                 int* bedges) {
  if (xy) L.xy.download(xy, 2 * L.nv, c.stream);
  if (lat) L.lat.download(lat, 2 * L.nv, c.stream);
  if (tri) L.tri.download(tri, 3 * L.nt, c.stream);
  if (parent && L.level > 0) L.parent.download(parent, L.nt, c.stream);
  if (bedges) L.bedges.download(bedges, 2 * L.nb, c.stream);
  c.sync();
}

void export_space_p2(Ctx& c, const Level& L, int* dof_lattice, int* conn6);

void export_space(Ctx& c, const Level& L, int* dof_lattice, int* interior_dofs,
                  int* interior_index, int* conn3) {
  const std::int64_t nd = L.ndofs();
  if (L.deg == 2) {  // dof lattice and 6-dof connectivity of the half lattice (p2.cu)
    export_space_p2(c, L, dof_lattice, conn3);
    dof_lattice = nullptr;
    conn3 = nullptr;
  }
  if (dof_lattice) {
    DevBuf<int> d(2 * nd);
    k_dof_lattice<<<grid_for(nd, kBlock), kBlock, 0, c.stream>>>(L.nx, L.ny, d.get());
    MLG_LAUNCH_CHECK();
    d.download(dof_lattice, 2 * nd, c.stream);
    c.sync();
  }
  if (interior_dofs || interior_index) {
    DevBuf<int> di(L.nint()), ii(nd);
    k_interior_lists<<<grid_for(nd, kBlock), kBlock, 0, c.stream>>>(
        L.imap(), interior_dofs ? di.get() : nullptr, interior_index ? ii.get() : nullptr);
    MLG_LAUNCH_CHECK();
    if (interior_dofs) di.download(interior_dofs, L.nint(), c.stream);
    if (interior_index) ii.download(interior_index, nd, c.stream);
    c.sync();
  }
  if (conn3) {
    DevBuf<int> cn(3 * L.nt);
    k_connectivity<<<grid_for(L.nt, kBlock), kBlock, 0, c.stream>>>(L.nt, L.tri.get(),
                                                                    L.lat.get(), L.nx, cn.get());
    MLG_LAUNCH_CHECK();
    cn.download(conn3, 3 * L.nt, c.stream);
    c.sync();
  }
}

}  // namespace mlg

"""TEST INFRASTRUCTURE ONLY: a numpy/scipy restatement of the reference's
correction-step path (arXiv 1401.4969, /root/reference/proj), written from
the reference's algorithm with each function citing the file:line it follows.

Role: an independent CPU checker, pinned against the golden vectors that the
compiled reference (oracle/_ref) produced (tests/golden/, made by
tests/golden/make_golden.py) and against the compiled reference itself.
Integer/structure work and element/assembly arithmetic reproduce the
reference's operation order (so digests match bitwise); reductions inside CG
use numpy's dot order, so iterates agree to rounding, not bitwise.
Only tests/ and bench.py's cpu_baseline leg may import this module.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import scipy.sparse as sp


class ConfigError(ValueError):
    pass


class SolverError(RuntimeError):
    pass


# ---------------------------------------------------------------- mesh.cpp ----
@dataclass
class Mesh:  # mesh.hpp:32-50
    domain: tuple
    level: int
    nx: int
    ny: int
    vertices: np.ndarray      # f64 [V,2]
    lattice: np.ndarray       # i32 [V,2]
    triangles: np.ndarray     # i32 [T,3]
    boundary_edges: np.ndarray
    parent: np.ndarray
    h_max: float = 0.0

    @property
    def dx(self):
        return (self.domain[1] - self.domain[0]) / self.nx

    @property
    def dy(self):
        return (self.domain[3] - self.domain[2]) / self.ny


def _coords(domain, nx, ny, lat):
    # Mesh::lattice_point (mesh.hpp:47-49): x_min + ix * cell_dx
    dx = (domain[1] - domain[0]) / nx
    dy = (domain[3] - domain[2]) / ny
    return np.stack([domain[0] + lat[:, 0].astype(np.float64) * dx,
                     domain[2] + lat[:, 1].astype(np.float64) * dy], axis=1)


def _edge_keys(tri, nv):  # edge_key mesh.cpp:27-30, all 3 edges of every triangle
    a = tri.astype(np.int64)
    b = np.roll(a, -1, axis=1)
    return (np.minimum(a, b) * nv + np.maximum(a, b)).reshape(-1)


def _boundary_edges(tri, nv):  # mesh.cpp:50-64 (std::map order = sorted keys)
    keys, counts = np.unique(_edge_keys(tri, nv), return_counts=True)
    k = keys[counts == 1]
    return np.stack([k // nv, k % nv], axis=1).astype(np.int32)


def _h_max(m):  # mesh.cpp:34-48
    lat = m.lattice
    h = 0.0
    for e in range(3):
        a = lat[m.triangles[:, e]]
        b = lat[m.triangles[:, (e + 1) % 3]]
        ex = (b[:, 0] - a[:, 0]).astype(np.float64) * m.dx
        ey = (b[:, 1] - a[:, 1]).astype(np.float64) * m.dy
        h = max(h, float(np.max(np.sqrt(ex * ex + ey * ey))))
    return h


def checked_cell_count(length, H, axis):  # mesh.cpp:18-25
    ratio = length / H
    n = int(np.floor(ratio + 0.5))
    if n < 1 or abs(ratio - n) > 1e-9 * max(1.0, ratio):
        raise ConfigError(f"mesh size H does not divide the {axis} side length into an "
                          "integer number of cells")
    return n


def build_structured_mesh(domain, H):  # mesh.cpp:68-104
    if not (domain[0] < domain[1]) or not (domain[2] < domain[3]):
        raise ConfigError("domain rectangle must have positive side lengths")
    if not H > 0:
        raise ConfigError("mesh size H must be positive")
    nx = checked_cell_count(domain[1] - domain[0], H, "x")
    ny = checked_cell_count(domain[3] - domain[2], H, "y")
    iy, ix = np.mgrid[0:ny + 1, 0:nx + 1]
    lat = np.stack([ix.ravel(), iy.ravel()], axis=1).astype(np.int32)
    cy, cx = np.mgrid[0:ny, 0:nx]
    v00 = (cy * (nx + 1) + cx).ravel()
    v10, v01 = v00 + 1, v00 + nx + 1
    v11 = v01 + 1
    tri = np.empty((2 * nx * ny, 3), np.int32)
    tri[0::2] = np.stack([v00, v10, v11], axis=1)
    tri[1::2] = np.stack([v00, v11, v01], axis=1)
    m = Mesh(tuple(domain), 0, nx, ny, _coords(domain, nx, ny, lat), lat, tri,
             _boundary_edges(tri, len(lat)), np.zeros(0, np.int32))
    m.h_max = _h_max(m)
    return m


def hole_cells(domain, H, nx, ny, hole):
    """B200 extension (BASELINE config 3, no reference code path): the corner
    hole [x0,x1]x[y0,y1] in coarse cells (csrc/mesh.cu hole_cells)."""
    def cell(v, lo):
        return int(np.floor((v - lo) / H + 0.5))
    h = (cell(hole[0], domain[0]), cell(hole[2], domain[2]), cell(hole[1], domain[0]),
         cell(hole[3], domain[2]))  # x0, y0, x1, y1
    if not ((h[0] == 0) != (h[2] == nx) and (h[1] == 0) != (h[3] == ny)):
        raise ConfigError("hole must touch exactly one corner of the domain rectangle (L-shape)")
    return h


def _cell_active(h, nx, ny, cx, cy):
    cx, cy = np.asarray(cx), np.asarray(cy)
    inside = (cx >= 0) & (cy >= 0) & (cx < nx) & (cy < ny)
    in_hole = (cx >= h[0]) & (cx < h[2]) & (cy >= h[1]) & (cy < h[3])
    return inside & ~in_hole


def build_structured_mesh_hole(domain, H, hole):
    """The B200 definition of an L-shaped level 0 (csrc/mesh.cu k_level0_hole):
    vertices = lattice points touching an element-carrying cell, lexicographic
    (y, x); two triangles per such cell, cells lexicographic, the split of
    mesh.cpp:96-97."""
    nx = checked_cell_count(domain[1] - domain[0], H, "x")
    ny = checked_cell_count(domain[3] - domain[2], H, "y")
    h = hole_cells(domain, H, nx, ny, hole)
    iy, ix = np.mgrid[0:ny + 1, 0:nx + 1]
    act = (_cell_active(h, nx, ny, ix, iy) | _cell_active(h, nx, ny, ix - 1, iy) |
           _cell_active(h, nx, ny, ix, iy - 1) | _cell_active(h, nx, ny, ix - 1, iy - 1)).ravel()
    vid = np.full((ny + 1) * (nx + 1), -1, np.int64)
    vid[act] = np.arange(int(act.sum()))
    lat = np.stack([ix.ravel()[act], iy.ravel()[act]], axis=1).astype(np.int32)
    cy, cx = np.mgrid[0:ny, 0:nx]
    cact = _cell_active(h, nx, ny, cx, cy).ravel()
    cx, cy = cx.ravel()[cact], cy.ravel()[cact]
    p00 = cy * (nx + 1) + cx
    v00, v10, v01, v11 = vid[p00], vid[p00 + 1], vid[p00 + nx + 1], vid[p00 + nx + 2]
    tri = np.empty((2 * len(cx), 3), np.int32)
    tri[0::2] = np.stack([v00, v10, v11], axis=1)
    tri[1::2] = np.stack([v00, v11, v01], axis=1)
    m = Mesh(tuple(domain), 0, nx, ny, _coords(domain, nx, ny, lat), lat, tri,
             _boundary_edges(tri, len(lat)), np.zeros(0, np.int32))
    m.h_max = _h_max(m)
    m.hole = h
    return m


def refine_regular(mesh):  # mesh.cpp:106-155
    nv = len(mesh.vertices)
    nx, ny = 2 * mesh.nx, 2 * mesh.ny
    keys = np.unique(_edge_keys(mesh.triangles, nv))           # one midpoint per edge, sorted
    a, b = keys // nv, keys % nv
    lat = np.concatenate([2 * mesh.lattice, mesh.lattice[a] + mesh.lattice[b]]).astype(np.int32)
    t = mesh.triangles.astype(np.int64)

    def mid(u, v):
        return nv + np.searchsorted(keys, np.minimum(u, v) * nv + np.maximum(u, v))

    A, B, Cc = t[:, 0], t[:, 1], t[:, 2]
    mab, mbc, mca = mid(A, B), mid(B, Cc), mid(Cc, A)
    ch = np.stack([np.stack([A, mab, mca], 1), np.stack([mab, B, mbc], 1),
                   np.stack([mca, mbc, Cc], 1), np.stack([mab, mbc, mca], 1)], axis=1)
    tri = ch.reshape(-1, 3).astype(np.int32)
    parent = np.repeat(np.arange(len(t), dtype=np.int32), 4)
    m = Mesh(mesh.domain, mesh.level + 1, nx, ny, _coords(mesh.domain, nx, ny, lat), lat, tri,
             _boundary_edges(tri, len(lat)), parent)
    m.h_max = _h_max(m)
    if getattr(mesh, "hole", None) is not None:
        m.hole = tuple(2 * v for v in mesh.hole)
    return m


# ------------------------------------------------------------- fespace.cpp ----
@dataclass
class FeSpace:  # fespace.hpp:52-65 (P1)
    mesh: Mesh
    ndofs: int
    dof_lattice: np.ndarray
    interior_dofs: np.ndarray
    interior_index: np.ndarray
    connectivity: np.ndarray


def build_space(mesh):  # fespace.cpp:230-312 (degree 1)
    stride = 2 * mesh.nx + 1
    pts = 2 * mesh.lattice[mesh.triangles]                     # [T,3,2] half units
    keys = pts[..., 1].astype(np.int64) * stride + pts[..., 0]
    uk = np.unique(keys)
    dof_lattice = np.stack([uk % stride, uk // stride], axis=1).astype(np.int32)
    conn = np.searchsorted(uk, keys).astype(np.int32)
    on_b = np.zeros(len(uk), bool)
    be = mesh.boundary_edges
    for k in (0, 1):
        lb = 2 * mesh.lattice[be[:, k]]
        on_b[np.searchsorted(uk, lb[:, 1].astype(np.int64) * stride + lb[:, 0])] = True
    interior = np.nonzero(~on_b)[0].astype(np.int32)
    iidx = np.full(len(uk), -1, np.int32)
    iidx[interior] = np.arange(len(interior), dtype=np.int32)
    return FeSpace(mesh, len(uk), dof_lattice, interior, iidx, conn)


def build_space_lattice(mesh):
    """B200 convention for domains with a hole: dofs on the bounding lattice
    (dof = iy*(nx+1)+ix, points strictly inside the hole inactive: no element,
    empty rows); interior = element-touching points off the boundary edges."""
    nx, ny = mesh.nx, mesh.ny
    nd = (nx + 1) * (ny + 1)
    iy, ix = np.divmod(np.arange(nd), nx + 1)
    dof_lattice = np.stack([2 * ix, 2 * iy], axis=1).astype(np.int32)
    ldof = (mesh.lattice[:, 1].astype(np.int64) * (nx + 1) + mesh.lattice[:, 0])
    conn = ldof[mesh.triangles].astype(np.int32)
    active = np.zeros(nd, bool)
    active[ldof] = True
    on_b = np.zeros(nd, bool)
    on_b[ldof[mesh.boundary_edges.reshape(-1)]] = True
    interior = np.nonzero(active & ~on_b)[0].astype(np.int32)
    iidx = np.full(nd, -1, np.int32)
    iidx[interior] = np.arange(len(interior), dtype=np.int32)
    return FeSpace(mesh, nd, dof_lattice, interior, iidx, conn)


QUAD2 = (np.array([[0.5, 0.5, 0.0], [0.0, 0.5, 0.5], [0.5, 0.0, 0.5]]), 1.0 / 3.0)  # :41-47


# quad_degree6 (make_degree6, fespace.cpp:49-75): barycentrics and weights, same order
_A1, _B1, _W1 = 0.501426509658179, 0.249286745170910, 0.116786275726379
_A2, _B2, _W2 = 0.873821971016996, 0.063089014491502, 0.050844906370207
_A3, _B3, _C3, _W3 = 0.053145049844816, 0.310352451033785, 0.636502499121399, 0.082851075618374
QUAD6 = [((_A1, _B1, _B1), _W1), ((_B1, _A1, _B1), _W1), ((_B1, _B1, _A1), _W1),
         ((_A2, _B2, _B2), _W2), ((_B2, _A2, _B2), _W2), ((_B2, _B2, _A2), _W2),
         ((_A3, _B3, _C3), _W3), ((_A3, _C3, _B3), _W3), ((_B3, _A3, _C3), _W3),
         ((_B3, _C3, _A3), _W3), ((_C3, _A3, _B3), _W3), ((_C3, _B3, _A3), _W3)]


def local_matrices_variable(mesh):
    """CoefficientField::variable (fespace.cpp:114-123) with the degree-6 rule
    (default_rule, fespace.cpp:219-222), operation order of local_matrix
    (fespace.cpp:185-217).  np.exp is not glibc's exp: entries agree with the
    reference to a few ulp."""
    v = mesh.vertices[mesh.triangles]
    x0, y0, x1, y1, x2, y2 = (v[:, 0, 0], v[:, 0, 1], v[:, 1, 0], v[:, 1, 1], v[:, 2, 0],
                              v[:, 2, 1])
    area2 = (x1 - x0) * (y2 - y0) - (x2 - x0) * (y1 - y0)
    area = 0.5 * area2
    g = np.stack([np.stack([(y1 - y2) / area2, (x2 - x1) / area2], 1),
                  np.stack([(y2 - y0) / area2, (x0 - x2) / area2], 1),
                  np.stack([(y0 - y1) / area2, (x1 - x0) / area2], 1)], axis=1)
    T = len(v)
    KA = np.zeros((T, 3, 3))
    KM = np.zeros((T, 3, 3))
    for (l, wq) in QUAD6:
        w = wq * area
        x = l[0] * x0 + l[1] * x1 + l[2] * x2
        y = l[0] * y0 + l[1] * y1 + l[2] * y2
        d0, d1, d2 = np.exp(1.0 + x * x), np.exp(x * y), np.exp(1.0 + y * y)
        phi = (1.0 + x * x) * (1.0 + y * y)
        for i in range(3):
            agx = d0 * g[:, i, 0] + d1 * g[:, i, 1]
            agy = d1 * g[:, i, 0] + d2 * g[:, i, 1]
            for j in range(i, 3):
                KA[:, i, j] = KA[:, i, j] + w * (agx * g[:, j, 0] + agy * g[:, j, 1])
                KM[:, i, j] = KM[:, i, j] + w * phi * l[i] * l[j]
    return KA, KM


def reaction_modes(seed):
    """BASELINE config 4: (k1, k2) = 1 + (splitmix64 outputs 1 and 2 of seed) >> 62."""
    M64 = 0xFFFFFFFFFFFFFFFF
    out = []
    for _ in range(2):
        seed = (seed + 0x9E3779B97F4A7C15) & M64
        z = seed
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        z ^= z >> 31
        out.append(1 + (z >> 62))
    return tuple(out)


def local_matrices_reaction(mesh, seed):
    """BASELINE config 4 (no reference code path; the B200 definition in
    csrc/assemble.cu): -div(a grad u) + c u with a = 1 + 0.5 sin(2 pi k1 x)
    sin(2 pi k2 y), c = 1 + x^2 + y^2 at the centroid; element stiffness
    a*K + c*M from the Laplace K and M, element mass M."""
    KA, KM = local_matrices(mesh, "laplace")
    k1, k2 = reaction_modes(seed)
    v = mesh.vertices[mesh.triangles]
    xc = (v[:, 0, 0] + v[:, 1, 0] + v[:, 2, 0]) / 3.0
    yc = (v[:, 0, 1] + v[:, 1, 1] + v[:, 2, 1]) / 3.0
    two_pi = 6.283185307179586476925286766559
    ac = 1.0 + 0.5 * np.sin(two_pi * k1 * xc) * np.sin(two_pi * k2 * yc)
    cc = 1.0 + xc * xc + yc * yc
    return ac[:, None, None] * KA + cc[:, None, None] * KM, KM


def local_matrices(mesh, example="laplace", seed=0):
    """Element stiffness and mass, P1, Laplace field, 3-point rule, in the exact
    operation order of local_matrix/element_geometry (fespace.cpp:169-217)."""
    if example == "variable":
        return local_matrices_variable(mesh)
    if example == "reaction":
        return local_matrices_reaction(mesh, seed)
    v = mesh.vertices[mesh.triangles]                            # [T,3,2]
    x0, y0, x1, y1, x2, y2 = (v[:, 0, 0], v[:, 0, 1], v[:, 1, 0], v[:, 1, 1], v[:, 2, 0],
                              v[:, 2, 1])
    area2 = (x1 - x0) * (y2 - y0) - (x2 - x0) * (y1 - y0)
    area = 0.5 * area2
    g = np.stack([np.stack([(y1 - y2) / area2, (x2 - x1) / area2], 1),
                  np.stack([(y2 - y0) / area2, (x0 - x2) / area2], 1),
                  np.stack([(y0 - y1) / area2, (x1 - x0) / area2], 1)], axis=1)
    pts, wq = QUAD2
    T = len(v)
    KA = np.zeros((T, 3, 3))
    KM = np.zeros((T, 3, 3))
    w = wq * area
    for q in range(3):
        for i in range(3):
            agx = 1.0 * g[:, i, 0] + 0.0 * g[:, i, 1]
            agy = 0.0 * g[:, i, 0] + 1.0 * g[:, i, 1]
            for j in range(i, 3):
                KA[:, i, j] = KA[:, i, j] + w * (agx * g[:, j, 0] + agy * g[:, j, 1])
                KM[:, i, j] = KM[:, i, j] + w * 1.0 * pts[q, i] * pts[q, j]
    return KA, KM


def from_upper_triplets(n, rows, cols, vals):  # sparse.cpp:24-61
    if np.any(rows > cols) or np.any(rows < 0) or np.any(cols >= n):
        raise ConfigError("upper triplet outside the upper triangle")
    order = np.lexsort((cols, rows))  # stable
    r, c, v = rows[order], cols[order], vals[order]
    start = np.ones(len(r), bool)
    start[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
    gid = np.cumsum(start) - 1
    gstart = np.nonzero(start)[0]
    pos = np.arange(len(r)) - gstart[gid]
    acc = np.zeros(len(gstart))
    for p in range(int(pos.max()) + 1 if len(pos) else 0):  # in-order sums from 0.0
        sel = pos == p
        acc[gid[sel]] = acc[gid[sel]] + v[sel]
    ur, uc = r[gstart], c[gstart]
    off = ur != uc
    fr = np.concatenate([ur, uc[off]])
    fc = np.concatenate([uc, ur[off]])
    fv = np.concatenate([acc, acc[off]])
    o = np.lexsort((fc, fr))
    fr, fc, fv = fr[o], fc[o], fv[o]
    row_ptr = np.zeros(n + 1, np.int64)
    np.add.at(row_ptr, fr + 1, 1)
    return np.cumsum(row_ptr).astype(np.int32), fc.astype(np.int32), fv


def assemble(space, example="laplace", seed=0):  # assemble_form fespace.cpp:314-341
    KA, KM = local_matrices(space.mesh, example, seed)
    iu, ju = np.triu_indices(3)                                  # i<=j, row-major order
    gi, gj = space.connectivity[:, iu], space.connectivity[:, ju]
    rows = np.minimum(gi, gj).reshape(-1).astype(np.int64)
    cols = np.maximum(gi, gj).reshape(-1).astype(np.int64)
    A = from_upper_triplets(space.ndofs, rows, cols, KA[:, iu, ju].reshape(-1))
    M = from_upper_triplets(space.ndofs, rows, cols, KM[:, iu, ju].reshape(-1))
    return A, M


def csr_multiply(csr, x):  # SparseSymMatrix::multiply, sparse.cpp:69-76 (sequential rows)
    rp, cols, vals = csr
    n = len(rp) - 1
    y = np.zeros(n)
    lens = np.diff(rp)
    for k in range(int(lens.max()) if n else 0):
        rows = np.nonzero(lens > k)[0]
        idx = rp[rows] + k
        y[rows] = y[rows] + vals[idx] * x[cols[idx]]
    return y


def to_scipy(csr, n=None):
    rp, cols, vals = csr
    n = len(rp) - 1 if n is None else n
    return sp.csr_matrix((vals, cols, rp), shape=(len(rp) - 1, n))


def prolongation(coarse, fine):  # prolongation_matrix fespace.cpp:355-400
    cm, fm = coarse.mesh, fine.mesh
    flat = fine.connectivity.reshape(-1)
    fdofs, first = np.unique(flat, return_index=True)         # first (element, i) per dof
    fe = first // 3
    pe = fm.parent[fe]
    pt = cm.triangles[pe]
    L = 4 * cm.lattice.astype(np.int64)
    x0, y0 = L[pt[:, 0], 0], L[pt[:, 0], 1]
    x1, y1 = L[pt[:, 1], 0], L[pt[:, 1], 1]
    x2, y2 = L[pt[:, 2], 0], L[pt[:, 2], 1]
    px = fine.dof_lattice[fdofs, 0].astype(np.int64)
    py = fine.dof_lattice[fdofs, 1].astype(np.int64)
    denom = ((x1 - x0) * (y2 - y0) - (x2 - x0) * (y1 - y0)).astype(np.float64)
    l1 = ((px - x0) * (y2 - y0) - (x2 - x0) * (py - y0)).astype(np.float64) / denom
    l2 = ((x1 - x0) * (py - y0) - (px - x0) * (y1 - y0)).astype(np.float64) / denom
    lam = np.stack([1.0 - l1 - l2, l1, l2], axis=1)
    cconn = coarse.connectivity[pe]
    rows, cols, vals = [], [], []
    for c in range(3):
        nz = lam[:, c] != 0.0
        rows.append(fdofs[nz]); cols.append(cconn[nz, c]); vals.append(lam[nz, c])
    r, c, v = np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)
    o = np.lexsort((c, r))
    r, c, v = r[o], c[o], v[o]
    rp = np.zeros(fine.ndofs + 1, np.int64)
    np.add.at(rp, r + 1, 1)
    return np.cumsum(rp).astype(np.int32), c.astype(np.int32), v, coarse.ndofs


def prolong_apply(P, x):  # SparseMatrix::multiply sparse.cpp:129-136
    return csr_multiply(P[:3], x)


def prolong_transpose(P, x):  # multiply_transpose sparse.cpp:144-148: scatter row by row
    rp, cols, vals, ncols = P
    y = np.zeros(ncols)
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    order = np.argsort(cols, kind="stable")   # per column, ascending row = scatter order
    cs, contrib = cols[order], vals[order] * x[rows[order]]
    start = np.ones(len(cs), bool)
    start[1:] = cs[1:] != cs[:-1]
    gid = np.cumsum(start) - 1
    pos = np.arange(len(cs)) - np.nonzero(start)[0][gid]
    ucols = cs[start]
    acc = np.zeros(len(ucols))
    for p in range(int(pos.max()) + 1 if len(pos) else 0):
        sel = pos == p
        acc[gid[sel]] = acc[gid[sel]] + contrib[sel]
    y[ucols] = acc
    return y


# -------------------------------------------------------------- decomp.cpp ----
@dataclass
class Partition:  # decomp.hpp:59-93
    m: int
    side: int
    delta_cells: int
    nx0: int
    ny0: int
    blocks: list = field(default_factory=list)
    overlaps: list = field(default_factory=list)
    inners: list = field(default_factory=list)


def build_partition_hole(coarse, m, delta):
    """Partition of a domain with a corner hole (B200 extension, csrc/corrector.cu
    build_partition): blocks inside the hole are dropped; inner regions follow
    decomp.cpp:73-80 (the hole's edges are shrunk from like block sides)."""
    p = build_partition(coarse, m, delta, keep_all=True)
    h = coarse.hole
    bw, bh = coarse.nx // p.side, coarse.ny // p.side
    if h[0] % bw or h[2] % bw or h[1] % bh or h[3] % bh:
        raise ConfigError("hole does not align with the subdomain block grid")

    def in_hole(c, rb):
        return c * bw >= h[0] and (c + 1) * bw <= h[2] and rb * bh >= h[1] and (rb + 1) * bh <= h[3]

    q = Partition(0, p.side, p.delta_cells, p.nx0, p.ny0)
    for r in range(p.side):
        for c in range(p.side):
            rb = p.side - 1 - r
            if in_hole(c, rb):
                continue
            x0, y0, x1, y1 = p.blocks[r * p.side + c]
            q.blocks.append((x0, y0, x1, y1))
            q.overlaps.append(p.overlaps[r * p.side + c])
            q.inners.append(p.inners[r * p.side + c])  # hole edges shrink like block sides
    q.m = len(q.blocks)
    return q


def build_partition(coarse, m, delta, keep_all=False):  # decomp.cpp:24-86
    side = int(np.floor(np.sqrt(m) + 0.5))
    if m < 1 or side * side != m:
        raise ConfigError("subdomain count m must be a perfect square")
    hx, hy = coarse.dx, coarse.dy
    if abs(hx - hy) > 1e-12 * max(hx, hy):
        raise ConfigError("partition requires square coarse cells")
    if coarse.nx % side or coarse.ny % side:
        raise ConfigError("block grid does not align with the coarse mesh")
    ratio = delta / hx
    dc = int(np.floor(ratio + 0.5))
    if dc < 1 or abs(ratio - dc) > 1e-9:
        raise ConfigError("overlap width delta must be a positive multiple of the coarse cell size")
    bw, bh = coarse.nx // side, coarse.ny // side
    if 2 * dc >= bw or 2 * dc >= bh:
        raise ConfigError("overlap width leaves a degenerate inner region (2*delta >= block side)")
    p = Partition(m, side, dc, coarse.nx, coarse.ny)
    for r in range(side):
        for c in range(side):
            x0, x1 = c * bw, (c + 1) * bw
            y1 = coarse.ny - r * bh
            y0 = y1 - bh
            p.blocks.append((x0, y0, x1, y1))
            p.overlaps.append((max(0, x0 - dc), max(0, y0 - dc), min(coarse.nx, x1 + dc),
                               min(coarse.ny, y1 + dc)))
            p.inners.append((0 if x0 == 0 else x0 + dc, 0 if y0 == 0 else y0 + dc,
                             coarse.nx if x1 == coarse.nx else x1 - dc,
                             coarse.ny if y1 == coarse.ny else y1 - dc))
    return p


def restrict_space(space, part, kind, j, zero_trace):  # decomp.cpp:167-217
    level = space.mesh.level
    scale = 1 << (level + 1)
    d = space.interior_dofs
    px, py = space.dof_lattice[d, 0], space.dof_lattice[d, 1]

    def in_rect(r, strict):
        x0, y0, x1, y1 = (v * scale for v in r)
        if strict:
            return (px > x0) & (px < x1) & (py > y0) & (py < y1)
        return (px >= x0) & (px <= x1) & (py >= y0) & (py <= y1)

    if kind == "domain":
        keep = np.ones(len(d), bool)
    elif kind == "block":
        keep = in_rect(part.blocks[j], zero_trace)
    elif kind == "overlap":
        keep = in_rect(part.overlaps[j], zero_trace)
    elif kind == "inner":
        keep = in_rect(part.inners[j], zero_trace)
    else:
        keep = np.ones(len(d), bool)
        for r in part.inners:
            keep &= ~in_rect(r, not zero_trace)
    return d[keep]


# -------------------------------------------------------------- sparse.cpp ----
def cg_solve(A, rhs, tol=1e-10, maxit=0):  # sparse.cpp:199-258 (Jacobi-PCG)
    n = A.shape[0]
    if tol <= 0:
        raise ConfigError("cg_solve: tolerance must be positive")
    if maxit <= 0:
        maxit = 10 * max(n, 1)
    x = np.zeros(n)
    bnorm = float(np.sqrt(rhs @ rhs))
    if bnorm == 0.0:
        return x, (0, 0.0, True)
    d = A.diagonal()
    if np.any(d <= 0):
        raise SolverError("Jacobi preconditioner requires a positive diagonal")
    inv = 1.0 / d
    r = rhs.copy()
    z = inv * r
    p = z.copy()
    rho = float(r @ z)
    it = 0
    for it in range(1, maxit + 1):
        q = A @ p
        pq = float(p @ q)
        if pq <= 0.0:
            raise SolverError("cg_solve: matrix is not positive definite (p'Mp <= 0)")
        alpha = rho / pq
        x += alpha * p
        r -= alpha * q
        if np.sqrt(r @ r) <= tol * bnorm:
            rt = rhs - A @ x
            true_rel = float(np.sqrt(rt @ rt)) / bnorm
            if true_rel <= tol:
                return x, (it, true_rel, True)
            r = rt
            z = inv * r
            p = z.copy()
            rho = float(r @ z)
            continue
        z = inv * r
        rho_next = float(r @ z)
        p = z + (rho_next / rho) * p
        rho = rho_next
    rt = rhs - A @ x
    final = float(np.sqrt(rt @ rt)) / bnorm
    return x, (it, final, final <= tol)


def fix_sign(v):  # sparse.cpp:260-271
    idx = int(np.argmax(np.abs(v))) if len(v) else 0
    return -v if len(v) and v[idx] < 0 else v


def order_ties(pairs):  # sparse.cpp:277-293
    i = 0
    while i < len(pairs):
        j = i + 1
        tol = 1e-12 * max(1.0, abs(pairs[i][0]))
        while j < len(pairs) and abs(pairs[j][0] - pairs[i][0]) <= tol:
            j += 1
        pairs[i:j] = sorted(pairs[i:j], key=lambda p: tuple(p[1]))
        i = j
    return pairs


def dense_gen_eigensolve(a, b, nev):  # sparse.cpp:297-324
    n = a.shape[0]
    if nev < 1 or nev > n:
        raise ConfigError("dense_gen_eigensolve: invalid nev")
    try:
        np.linalg.cholesky(b)
    except np.linalg.LinAlgError:
        raise SolverError("dense_gen_eigensolve: mass block is not SPD")
    w, v = scipy.linalg.eigh(a, b, type=1, driver="gvd")
    return order_ties([(float(w[i]), fix_sign(v[:, i].copy())) for i in range(nev)])


# ----------------------------------------------------------- corrector.cpp ----
class Level:
    def __init__(self, mesh, space, A, M, P=None):
        self.mesh, self.space, self.A, self.M, self.P = mesh, space, A, M, P
        self.As = to_scipy(A)
        self.Ms = to_scipy(M)


class Hierarchy:  # corrector.cpp:111-181
    def __init__(self, domain=(-1.0, 1.0, -1.0, 1.0), H=0.25, delta=0.1, m=4, n_levels=5,
                 nev=5, cg_tol=1e-10, example="laplace", seed=0, hole=None):
        self.n_levels, self.nev, self.cg_tol = n_levels, nev, cg_tol
        self.example, self.seed = example, seed
        self.hole = hole
        mesh = (build_structured_mesh(domain, H) if hole is None
                else build_structured_mesh_hole(domain, H, hole))
        self._space = build_space if hole is None else build_space_lattice
        cell = mesh.dx
        dc = max(1, int(np.ceil(delta / cell - 1e-9)))         # corrector.cpp:117-121
        self.part = (build_partition(mesh, m, dc * cell) if hole is None
                     else build_partition_hole(mesh, m, dc * cell))
        sp0 = self._space(mesh)
        self.levels = [Level(mesh, sp0, *assemble(sp0, example, seed))]
        self._dense = None

    def extend_to(self, level):  # corrector.cpp:131-146
        while len(self.levels) - 1 < level:
            prev = self.levels[-1]
            mesh = refine_regular(prev.mesh)
            s = self._space(mesh)
            self.levels.append(Level(mesh, s, *assemble(s, self.example, self.seed),
                                     prolongation(prev.space, s)))

    def prolong(self, full, a, b):  # corrector.cpp:158-163
        for k in range(a + 1, b + 1):
            full = prolong_apply(self.levels[k].P, full)
        return full

    def restrict_transpose(self, full, a, b):  # corrector.cpp:165-170
        for k in range(a, b, -1):
            full = prolong_transpose(self.levels[k].P, full)
        return full

    def coarse_dense(self):  # corrector.cpp:172-181
        if self._dense is None:
            L0 = self.levels[0]
            d = L0.space.interior_dofs
            a = L0.As[d][:, d].toarray()
            b = L0.Ms[d][:, d].toarray()
            self._dense = (a, b, scipy.linalg.cho_factor(b, lower=True))
        return self._dense

    def expand(self, level, coeffs):  # fespace.cpp:408-415
        s = self.levels[level].space
        full = np.zeros(s.ndofs)
        full[s.interior_dofs] = coeffs
        return full


def solve_interior_eigenproblem(hy, level, nev):  # sparse.cpp:326-355
    hy.extend_to(level)
    L = hy.levels[level]
    d = L.space.interior_dofs
    if len(d) > 5000:
        raise ConfigError(f"interior dimension {len(d)} exceeds the dense eigensolver "
                          "threshold 5000")
    a = L.As[d][:, d]
    b = L.Ms[d][:, d]
    out = []
    for lam, v in dense_gen_eigensolve(a.toarray(), b.toarray(), nev):
        q = float(v @ (b @ v))
        if q <= 0:
            raise SolverError("eigenvector with nonpositive mass norm")
        out.append((lam, fix_sign(v / np.sqrt(q))))
    return out


def region_system(hy, level, kind, j=0):
    L = hy.levels[level]
    d = restrict_space(L.space, hy.part, kind, j, True)
    return d, L.As[d][:, d].tocsr()


def local_bvp_solve(hy, level, j, lam, u_full, tol):  # corrector.cpp:198-214
    L = hy.levels[level]
    d, A = region_system(hy, level, "overlap", j)
    residual = lam * (L.Ms @ u_full) - L.As @ u_full
    x, (it, fr, ok) = cg_solve(A, residual[d], tol)
    if not ok:
        raise SolverError(f"subdomain {j + 1} solve did not converge ({it} iterations, "
                          f"residual {fr:f})")
    e = np.zeros(L.space.ndofs)
    e[d] = x
    return e, it


def interface_solve(hy, level, lam, u_full, corrections, tol):  # corrector.cpp:216-254
    L = hy.levels[level]
    glued = np.zeros(L.space.ndofs)
    owned = np.zeros(L.space.ndofs, bool)
    for j in range(hy.part.m):
        g = restrict_space(L.space, hy.part, "inner", j, False)
        if np.any(owned[g]):
            raise SolverError("interface dof claimed by two inner regions")
        owned[g] = True
        glued[g] = u_full[g] + corrections[j][g]
    d, A = region_system(hy, level, "strip")
    it = 0
    if len(d):
        load = lam * (L.Ms @ u_full) - L.As @ glued
        x, (it, fr, ok) = cg_solve(A, load[d], tol)
        if not ok:
            raise SolverError(f"strip solve did not converge ({it} iterations, residual {fr:f})")
        owned[d] = True
        glued[d] = x
    if not np.all(owned[L.space.interior_dofs]):
        raise SolverError("interior dof not covered by the glue/strip partition")
    return glued, it


def augmented_eigensolve(hy, level, glued, nev):  # corrector.cpp:256-334
    L = hy.levels[level]
    L0 = hy.levels[0]
    a_cc, b_cc, chol = hy.coarse_dense()
    mc = a_cc.shape[0]
    d0 = L0.space.interior_dofs
    k_in = len(glued)
    au = [L.As @ g for g in glued]
    bu = [L.Ms @ g for g in glued]
    a_cu = np.stack([hy.restrict_transpose(v, level, 0)[d0] for v in au], 1)
    b_cu = np.stack([hy.restrict_transpose(v, level, 0)[d0] for v in bu], 1)
    a_uu = np.array([[glued[l] @ au[l2] for l2 in range(k_in)] for l in range(k_in)])
    b_uu = np.array([[glued[l] @ bu[l2] for l2 in range(k_in)] for l in range(k_in)])
    keep = []
    for l in range(k_in):
        c = scipy.linalg.cho_solve(chol, b_cu[:, l])
        res2 = b_uu[l, l] - b_cu[:, l] @ c
        if np.sqrt(max(res2, 0.0)) >= 1e-10:
            keep.append(l)
    k = len(keep)
    dim = mc + k
    if nev < 1 or nev > dim:
        raise ConfigError("augmented eigenproblem smaller than the requested nev")
    A = np.zeros((dim, dim))
    B = np.zeros((dim, dim))
    A[:mc, :mc], B[:mc, :mc] = a_cc, b_cc
    for i, l in enumerate(keep):
        A[:mc, mc + i] = A[mc + i, :mc] = a_cu[:, l]
        B[:mc, mc + i] = B[mc + i, :mc] = b_cu[:, l]
        for i2, l2 in enumerate(keep):
            A[mc + i, mc + i2] = a_uu[l, l2]
            B[mc + i, mc + i2] = b_uu[l, l2]
    pairs = []
    for lam, vec in dense_gen_eigensolve(A, B, nev):
        full = hy.prolong(hy.expand(0, vec[:mc]), 0, level)
        for i, l in enumerate(keep):
            full = full + vec[mc + i] * glued[l]
        q = float(full @ (L.Ms @ full))
        if q <= 0:
            raise SolverError("augmented eigenvector with nonpositive mass norm")
        pairs.append((lam, fix_sign(full[L.space.interior_dofs] / np.sqrt(q))))
    return sorted(pairs, key=lambda p: p[0])  # stable


def one_correction_step(hy, level, pairs, to_level):  # corrector.cpp:336-412
    if not pairs:
        raise ConfigError("correction step needs at least one eigenpair")
    if to_level not in (level, level + 1):
        raise ConfigError("correction step targets the next level (or the same level)")
    hy.extend_to(to_level)
    L = hy.levels[to_level]
    u_fine = []
    for _, c in pairs:
        full = hy.expand(level, c)
        u_fine.append(full if to_level == level else hy.prolong(full, level, to_level))
    glued = []
    for (lam, _), u in zip(pairs, u_fine):
        corr = [local_bvp_solve(hy, to_level, j, lam, u, hy.cg_tol)[0] for j in range(hy.part.m)]
        glued.append(interface_solve(hy, to_level, lam, u, corr, hy.cg_tol)[0])
    nxt = augmented_eigensolve(hy, to_level, glued, len(pairs))
    matched = True
    for i2, (_, c) in enumerate(nxt):
        bfull = L.Ms @ hy.expand(to_level, c)
        vals = [abs(u @ bfull) for u in u_fine]
        if int(np.argmax(vals)) != i2:
            matched = False
    return nxt, matched


def multilevel_correction(hy):  # corrector.cpp:414-462
    hy.extend_to(1)
    state = solve_interior_eigenproblem(hy, 1, hy.nev)
    lams = [[p[0] for p in state]]
    for k in range(1, hy.n_levels):
        state, _ = one_correction_step(hy, k, state, k + 1)
        lams.append([p[0] for p in state])
    return np.array(lams), state

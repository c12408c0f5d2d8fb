"""Host-side mirror of the reference's corrector interface over the C ABI.

Same names, argument meaning and error behaviour as the reference's C++ API
(/root/reference/proj/include/mleig/corrector.hpp, decomp.hpp, fespace.hpp),
so parity tests read like the reference's own tests.  All compute runs in
libmlg_b200.so on the GPU; this module only marshals numpy arrays.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import (MlgConfig, MlgLevelInfo, MlgSolveReport, MlgStepTimings, c_double_p,
                   c_int64_p, c_int_p, check, lib)

REGION_KINDS = {"domain": 0, "block": 1, "overlap": 2, "inner": 3, "strip": 4}
FORMS = {"stiffness": 0, "mass": 1}


def _dp(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(c_double_p)


def _ip(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(c_int_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class DomainRect:  # mesh.hpp:22-27
    x_min: float = -1.0
    x_max: float = 1.0
    y_min: float = -1.0
    y_max: float = 1.0


@dataclass
class RunConfig:  # corrector.hpp:21-33
    domain: DomainRect = field(default_factory=DomainRect)
    H: float = 0.25
    delta: float = 0.1
    m: int = 4
    n_levels: int = 5
    degree: int = 1
    nev: int = 5
    example: str = "laplace"
    cg_tol: float = 1e-10
    workers: int = 1
    deterministic: bool = True
    device: int = 0  # CUDA device of the context (B200-specific)
    seed: int = 0    # example "reaction" (BASELINE config 4): draws (k1, k2)
    hole: DomainRect | None = None  # corner hole -> L-shaped domain (BASELINE config 3)

    def to_c(self) -> MlgConfig:
        ex = {"laplace": 0, "variable": 1, "reaction": 2}.get(self.example, -1)
        h = self.hole or DomainRect(0.0, 0.0, 0.0, 0.0)
        return MlgConfig(self.domain.x_min, self.domain.x_max, self.domain.y_min,
                         self.domain.y_max, self.H, self.delta, self.m, self.n_levels,
                         self.degree, self.nev, ex, self.workers, self.cg_tol,
                         int(self.deterministic), self.device, self.seed,
                         h.x_min, h.x_max, h.y_min, h.y_max)


@dataclass
class SolveReport:  # sparse.hpp:103-107
    iterations: int = 0
    final_residual: float = 0.0
    converged: bool = False


@dataclass
class StepTimings:  # corrector.hpp:97-101 (+ device evidence)
    local_seconds: float = 0.0
    iface_seconds: float = 0.0
    aug_seconds: float = 0.0
    build_seconds: float = 0.0
    local_iterations_max: int = 0
    strip_iterations_max: int = 0
    spmv_kernel_ms: float = 0.0
    spmv_launches: int = 0
    spmv_rows: float = 0.0
    kernel_launches: int = 0
    step_seconds: float = 0.0
    spmv_uniform_stencil: int = 0  # 0 general, 1 uniform, 2 uniform + deferred x
    spmv_check_rows: float = 0.0
    spmv_launches_all: int = 0  # every launch of the sampled kernel in the step
    strip_kernel_ms: float = 0.0  # every strip-solve CG launch (profiling on)
    strip_launches: int = 0
    strip_row_iters: float = 0.0  # strip unknowns x CG updates
    strip_kernel: int = 0
    strip_bytes_per_row: int = 0
    local_kernel: int = 0  # 0 k_cg_iter, 1 k_cg_persist, 2 k_cg_resident

    @classmethod
    def from_c(cls, t: MlgStepTimings) -> "StepTimings":
        return cls(t.local_seconds, t.iface_seconds, t.aug_seconds, t.build_seconds,
                   t.local_iterations_max, t.strip_iterations_max, t.spmv_kernel_ms,
                   t.spmv_launches, t.spmv_rows, t.kernel_launches, t.step_seconds,
                   int(t.spmv_uniform_stencil), t.spmv_check_rows, t.spmv_launches_all,
                   t.strip_kernel_ms, t.strip_launches, t.strip_row_iters,
                   int(t.strip_kernel), int(t.strip_bytes_per_row),
                   int(t.local_kernel))


@dataclass
class EigenPair:  # sparse.hpp:133-137
    lam: float
    coeffs: np.ndarray
    level: int


@dataclass
class CorrectionState:  # corrector.hpp:103-107
    level: int = 0
    pairs: list = field(default_factory=list)
    matched_previous: bool = True


@dataclass
class LevelTrace:  # corrector.hpp:151-159 (reporting fields filled by the caller)
    level: int
    h: float
    interior_dofs: int
    lambdas: list
    timings: StepTimings
    matched_previous: bool
    pairs: list
    eig_errors: list = field(default_factory=list)  # filled when a ReferenceSet is given
    l2_errors: list = field(default_factory=list)
    h1_errors: list = field(default_factory=list)


@dataclass
class Mesh:  # mesh.hpp:32-50
    level: int
    nx: int
    ny: int
    vertices: np.ndarray
    vertex_lattice: np.ndarray
    triangles: np.ndarray
    boundary_edges: np.ndarray
    parent: np.ndarray
    h_max: float


@dataclass
class FeSpace:  # fespace.hpp:52-65 (P1)
    ndofs: int
    dof_lattice: np.ndarray
    interior_dofs: np.ndarray
    interior_index: np.ndarray
    connectivity: np.ndarray


class Hierarchy:
    """Owns the device-resident level hierarchy (corrector.hpp:63-95)."""

    def __init__(self, config: RunConfig):
        self.config = config
        self._cfg = config.to_c()
        h = C.c_void_p()
        check(lib().mlg_create(C.byref(self._cfg), C.byref(h)))
        self._h = h

    # -- lifecycle --
    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().mlg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._h

    # -- levels --
    def extend_to(self, level: int) -> None:
        check(lib().mlg_extend_to(self._h, level))

    def max_level(self) -> int:
        v = C.c_int()
        check(lib().mlg_max_level(self._h, C.byref(v)))
        return v.value

    def level_info(self, level: int) -> MlgLevelInfo:
        info = MlgLevelInfo()
        check(lib().mlg_get_level_info(self._h, level, C.byref(info)))
        return info

    def mesh(self, level: int) -> Mesh:
        i = self.level_info(level)
        v = np.empty((i.num_vertices, 2), np.float64)
        lat = np.empty((i.num_vertices, 2), np.int32)
        t = np.empty((i.num_triangles, 3), np.int32)
        p = np.empty(i.num_triangles if level > 0 else 0, np.int32)
        b = np.empty((i.num_boundary_edges, 2), np.int32)
        check(lib().mlg_export_mesh(self._h, level, _dp(v), _ip(lat), _ip(t),
                                    _ip(p) if level > 0 else None, _ip(b)))
        return Mesh(level, i.nx, i.ny, v, lat, t, b, p, i.h_max)

    def space(self, level: int) -> FeSpace:
        i = self.level_info(level)
        dl = np.empty((i.ndofs, 2), np.int32)
        idofs = np.empty(i.n_interior, np.int32)
        iidx = np.empty(i.ndofs, np.int32)
        conn = np.empty((i.num_triangles, 6 if self.config.degree == 2 else 3), np.int32)
        check(lib().mlg_export_space(self._h, level, _ip(dl), _ip(idofs), _ip(iidx),
                                     _ip(conn)))
        return FeSpace(int(i.ndofs), dl, idofs, iidx, conn)

    def csr(self, level: int, form: str):
        """(row_ptr, cols, values) of assemble_form (fespace.cpp:314-341)."""
        i = self.level_info(level)
        rp = np.empty(i.ndofs + 1, np.int32)
        cols = np.empty(i.nnz, np.int32)
        vals = np.empty(i.nnz, np.float64)
        check(lib().mlg_export_csr(self._h, level, FORMS[form], _ip(rp), _ip(cols), _dp(vals)))
        return rp, cols, vals

    def partition(self):
        info = np.zeros(5, np.int32)
        check(lib().mlg_partition(self._h, None, _ip(info)))
        rects = np.zeros((info[0], 3, 4), np.int32)
        check(lib().mlg_partition(self._h, _ip(rects), _ip(info)))
        return {"m": int(info[0]), "side": int(info[1]), "overlap_cells": int(info[2]),
                "coarse_nx": int(info[3]), "coarse_ny": int(info[4]),
                "blocks": rects[:, 0], "overlaps": rects[:, 1], "inners": rects[:, 2]}

    def region_dofs(self, level: int, region: str, j: int = 0, zero_trace: bool = False):
        """restrict_space(...).dofs (decomp.cpp:167-217)."""
        n = C.c_int64()
        k = REGION_KINDS[region]
        check(lib().mlg_region_dofs(self._h, level, k, j, int(zero_trace), None, C.byref(n)))
        out = np.empty(n.value, np.int32)
        check(lib().mlg_region_dofs(self._h, level, k, j, int(zero_trace), _ip(out), C.byref(n)))
        return out

    def region_elements(self, level: int, region: str, j: int = 0):
        n = C.c_int64()
        k = REGION_KINDS[region]
        check(lib().mlg_region_elements(self._h, level, k, j, None, C.byref(n)))
        out = np.empty(n.value, np.int32)
        check(lib().mlg_region_elements(self._h, level, k, j, _ip(out), C.byref(n)))
        return out

    # -- operators --
    def apply(self, level: int, form: str, x) -> np.ndarray:
        x = _f64(x)
        y = np.empty_like(x)
        check(lib().mlg_spmv(self._h, level, FORMS[form], _dp(x), _dp(y)))
        return y

    def prolong(self, full, from_level: int, to_level: int) -> np.ndarray:
        x = _f64(full)
        y = np.empty(self._ndofs_after_extend(to_level), np.float64)
        check(lib().mlg_prolong(self._h, from_level, to_level, _dp(x), _dp(y)))
        return y

    def restrict_transpose(self, full, from_level: int, to_level: int) -> np.ndarray:
        x = _f64(full)
        y = np.empty(self.level_info(to_level).ndofs, np.float64)
        check(lib().mlg_restrict_transpose(self._h, from_level, to_level, _dp(x), _dp(y)))
        return y

    def _ndofs_after_extend(self, level: int) -> int:
        self.extend_to(level)
        return int(self.level_info(level).ndofs)

    def _interior(self, level: int) -> np.ndarray:
        cache = self.__dict__.setdefault("_interior_cache", {})
        if level not in cache:
            i = self.level_info(level)
            d = np.empty(i.n_interior, np.int32)
            check(lib().mlg_export_space(self._h, level, None, _ip(d), None, None))
            cache[level] = d
        return cache[level]

    def expand_interior(self, level: int, coeffs) -> np.ndarray:  # fespace.cpp:408-415
        i = self.level_info(level)
        full = np.zeros(i.ndofs, np.float64)
        full[self._interior(level)] = np.asarray(coeffs).reshape(-1)
        return full

    def restrict_interior(self, level: int, full) -> np.ndarray:  # fespace.cpp:417-423
        return np.ascontiguousarray(np.asarray(full)[self._interior(level)])

    def set_input_stream(self, stream: int) -> None:
        """CUDA stream (raw handle; 0 = legacy default) the *_device calls order after."""
        check(lib().mlg_set_input_stream(self._h, C.c_void_p(stream)))

    def build_profile(self):
        """(assemble_ms, assembled dofs) of the last level built with profiling on."""
        ms = C.c_double()
        n = C.c_double()
        check(lib().mlg_build_profile(self._h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def build_profile_kernel(self) -> str:
        """Name of the assembly kernel `build_profile` timed."""
        k = C.c_int()
        check(lib().mlg_build_profile_kernel(self._h, C.byref(k)))
        return ("k_assemble", "k_assemble_table", "k_assemble_var")[k.value]

    def set_profiling(self, on: bool) -> None:
        check(lib().mlg_set_profiling(self._h, int(on)))

    def bench_spmv(self, level: int, reps: int = 20):
        ms = C.c_double()
        by = C.c_double()
        check(lib().mlg_bench_spmv(self._h, level, reps, C.byref(ms), C.byref(by)))
        return ms.value, by.value


def coarse_eigensolve(hy: Hierarchy, level: int, nev: int):
    """solve_interior_eigenproblem on `level` (fespace.hpp:128-132)."""
    hy.extend_to(level)
    n = hy.level_info(level).n_interior
    lam = np.empty(nev, np.float64)
    coeffs = np.empty((nev, n), np.float64)
    check(lib().mlg_coarse_eigensolve(hy.handle, level, nev, _dp(lam), _dp(coeffs)))
    return [EigenPair(float(lam[i]), coeffs[i].copy(), level) for i in range(nev)]


def local_bvp_solve(hy: Hierarchy, level: int, j: int, lam: float, u_full, cg_tol: float):
    """corrector.hpp:112-113; returns (e_full, SolveReport)."""
    u = _f64(u_full)
    e = np.empty_like(u)
    rep = MlgSolveReport()
    check(lib().mlg_local_bvp_solve(hy.handle, level, j, lam, _dp(u), cg_tol, _dp(e),
                                    C.byref(rep)))
    return e, SolveReport(rep.iterations, rep.final_residual, bool(rep.converged))


def local_cg_solve(hy: Hierarchy, level: int, j: int, lam: float, u_full, cg_tol: float,
                   maxit: int = 0):
    """The CG of local_bvp_solve with cg_solve's contract (sparse.cpp:199-258):
    maxit > 0 caps the iterations and non-convergence is reported, not raised."""
    u = _f64(u_full)
    e = np.empty_like(u)
    rep = MlgSolveReport()
    check(lib().mlg_local_cg_solve(hy.handle, level, j, lam, _dp(u), cg_tol, int(maxit),
                                   _dp(e), C.byref(rep)))
    return e, SolveReport(rep.iterations, rep.final_residual, bool(rep.converged))


def interface_solve(hy: Hierarchy, level: int, lam: float, u_full, corrections, cg_tol: float):
    """corrector.hpp:118-120; corrections: (m, ndofs).  Returns (glued, SolveReport)."""
    u = _f64(u_full)
    corr = _f64(corrections)
    g = np.empty_like(u)
    rep = MlgSolveReport()
    check(lib().mlg_interface_solve(hy.handle, level, lam, _dp(u), _dp(corr), cg_tol, _dp(g),
                                    C.byref(rep)))
    return g, SolveReport(rep.iterations, rep.final_residual, bool(rep.converged))


def augmented_eigensolve(hy: Hierarchy, level: int, glued, nev: int):
    """corrector.hpp:127-128; glued: (k_in, ndofs)."""
    g = _f64(np.atleast_2d(glued))
    n = hy.level_info(level).n_interior
    lam = np.empty(nev, np.float64)
    coeffs = np.empty((nev, n), np.float64)
    check(lib().mlg_augmented_eigensolve(hy.handle, level, g.shape[0], _dp(g), nev, _dp(lam),
                                         _dp(coeffs)))
    return [EigenPair(float(lam[i]), coeffs[i].copy(), level) for i in range(nev)]


def one_correction_step(hy: Hierarchy, state: CorrectionState, to_level: int):
    """corrector.hpp:135-136; returns (CorrectionState, StepTimings)."""
    nev = len(state.pairs)
    lam_in = np.array([p.lam for p in state.pairs], np.float64)
    cin = _f64(np.stack([p.coeffs for p in state.pairs])) if nev else np.zeros((0, 0))
    hy.extend_to(max(to_level, state.level))
    nout = hy.level_info(to_level).n_interior
    lam_out = np.empty(max(nev, 1), np.float64)
    cout = np.empty((max(nev, 1), nout), np.float64)
    matched = C.c_int()
    t = MlgStepTimings()
    check(lib().mlg_correction_step(hy.handle, state.level, to_level, nev, _dp(lam_in),
                                    _dp(cin), _dp(lam_out), _dp(cout), C.byref(matched),
                                    C.byref(t)))
    pairs = [EigenPair(float(lam_out[i]), cout[i].copy(), to_level) for i in range(nev)]
    return CorrectionState(to_level, pairs, bool(matched.value)), StepTimings.from_c(t)


def _check_host_block(a, shape, name, writeable):
    """The raw entry point hands the buffer to C as nev*n doubles: refuse anything
    else (dtype, layout, shape) instead of letting the library overrun it."""
    if not isinstance(a, np.ndarray):
        raise TypeError(f"{name} must be a numpy array")
    if a.dtype != np.float64 or not a.flags.c_contiguous:
        raise TypeError(f"{name} must be a C-contiguous float64 array")
    if tuple(a.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {a.shape}, expected {tuple(shape)}")
    if writeable and not a.flags.writeable:
        raise ValueError(f"{name} must be writeable")


def one_correction_step_raw(hy: Hierarchy, from_level: int, to_level: int, lambdas_in,
                            coeffs_in: np.ndarray, coeffs_out: np.ndarray):
    """one_correction_step on caller-owned (e.g. pinned) host arrays, no copies on
    the Python side: coeffs_in (nev, n_int(from)), coeffs_out (nev, n_int(to))."""
    lam_in = _f64(lambdas_in)
    nev = len(lam_in)
    _check_host_block(coeffs_in, (nev, hy.level_info(from_level).n_interior), "coeffs_in",
                      writeable=False)
    _check_host_block(coeffs_out, (nev, hy.level_info(to_level).n_interior), "coeffs_out",
                      writeable=True)
    lam_out = np.empty(nev, np.float64)
    matched = C.c_int()
    t = MlgStepTimings()
    check(lib().mlg_correction_step(hy.handle, from_level, to_level, nev, _dp(lam_in),
                                    _dp(coeffs_in), _dp(lam_out), _dp(coeffs_out),
                                    C.byref(matched), C.byref(t)))
    return lam_out, bool(matched.value), StepTimings.from_c(t)


def one_correction_step_device(hy: Hierarchy, from_level: int, to_level: int, lambdas_in,
                               d_coeffs_in: int, d_coeffs_out: int):
    """Same on device-resident coefficient arrays (raw CUDA pointers)."""
    lam_in = _f64(lambdas_in)
    nev = len(lam_in)
    lam_out = np.empty(nev, np.float64)
    matched = C.c_int()
    t = MlgStepTimings()
    check(lib().mlg_correction_step_device(hy.handle, from_level, to_level, nev, _dp(lam_in),
                                           C.c_void_p(d_coeffs_in), _dp(lam_out),
                                           C.c_void_p(d_coeffs_out), C.byref(matched),
                                           C.byref(t)))
    return lam_out, bool(matched.value), StepTimings.from_c(t)


def multilevel_correction_device(hy: Hierarchy, last_level: int, d_final_coeffs: int):
    """multilevel_correction up to last_level leaving the final coefficients in
    device memory (raw pointer, (nev, n_int(last))); returns lambdas per level."""
    nev = hy.config.nev
    lam = np.empty((last_level, nev), np.float64)
    hy.extend_to(last_level)
    check(lib().mlg_multilevel_correction(hy.handle, last_level, _dp(lam), None,
                                          C.c_void_p(d_final_coeffs), None, None))
    return lam


def multilevel_correction(hy: Hierarchy, last_level: int = 0):
    """corrector.cpp:414-462 (errors/reporting are the caller's); returns
    (lambdas[levels][nev], final pairs, matched[levels], timings[levels])."""
    nlev = last_level if last_level > 0 else hy.config.n_levels
    nev = hy.config.nev
    lam = np.empty((nlev, nev), np.float64)
    matched = np.zeros(nlev, np.int32)
    times = (MlgStepTimings * nlev)()
    hy.extend_to(nlev)
    n = hy.level_info(nlev).n_interior
    coeffs = np.empty((nev, n), np.float64)
    check(lib().mlg_multilevel_correction(hy.handle, nlev, _dp(lam), _dp(coeffs), None,
                                          _ip(matched), times))
    pairs = [EigenPair(float(lam[-1, i]), coeffs[i].copy(), nlev) for i in range(nev)]
    return lam, pairs, matched.astype(bool), [StepTimings.from_c(t) for t in times]

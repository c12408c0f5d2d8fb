"""TEST INFRASTRUCTURE ONLY: ctypes binding of oracle/_ref/libmleig_ref.so, the
UNMODIFIED reference library (/root/reference/proj/src) compiled by
oracle/Makefile against self-written Eigen/doctest shims.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs use this module, and only as the checker or the timed CPU baseline.  The
product (paper_1401_4969_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_ref" / "libmleig_ref.so"

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)
lp = C.POINTER(C.c_longlong)


class RefConfig(C.Structure):
    _fields_ = [
        ("x_min", C.c_double), ("x_max", C.c_double), ("y_min", C.c_double),
        ("y_max", C.c_double), ("H", C.c_double), ("delta", C.c_double), ("m", C.c_int),
        ("n_levels", C.c_int), ("degree", C.c_int), ("nev", C.c_int), ("example", C.c_int),
        ("workers", C.c_int), ("cg_tol", C.c_double), ("deterministic", C.c_int),
    ]


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


_lib = None


def available() -> bool:
    return LIB_PATH.exists()


def build() -> None:
    """Compile the oracle from /root/reference (container only)."""
    subprocess.run(["make", "-C", str(HERE), "-j8", "ref"], check=True,
                   stdout=subprocess.DEVNULL)


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} missing; run `make -C oracle ref`")
        h = C.CDLL(str(LIB_PATH))
        h.ref_last_error.restype = C.c_char_p
        h.ref_destroy.restype = None
        h.ref_destroy.argtypes = [C.c_void_p]
        _lib = h
    return _lib


def _chk(code):
    if code != 0:
        raise RefError(code, lib().ref_last_error().decode())


def _d(a):
    return a.ctypes.data_as(dp)


def _i(a):
    return a.ctypes.data_as(ip)


class RefHierarchy:
    """Reference Hierarchy (corrector.hpp:63-95) driven through ref_capi.cpp."""

    def __init__(self, domain=(-1.0, 1.0, -1.0, 1.0), H=0.25, delta=0.1, m=4, n_levels=5,
                 nev=5, cg_tol=1e-10, workers=1, degree=1, example=0):
        self.cfg = RefConfig(*domain, H, delta, m, n_levels, degree, nev, example, workers,
                             cg_tol, 1)
        h = C.c_void_p()
        _chk(lib().ref_create(C.byref(self.cfg), C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            lib().ref_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def extend_to(self, level):
        t = C.c_double()
        _chk(lib().ref_extend_to(self.h, level, C.byref(t)))
        return t.value

    def build_region_systems(self, level):
        t = C.c_double()
        _chk(lib().ref_build_region_systems(self.h, level, C.byref(t)))
        return t.value

    def sizes(self, level):
        out = (C.c_longlong * 10)()
        hm = C.c_double()
        _chk(lib().ref_level_sizes(self.h, level, out, C.byref(hm)))
        keys = ["nv", "nt", "nb", "ndofs", "n_int", "nnz_a", "nnz_m", "nx", "ny", "level"]
        d = {k: int(v) for k, v in zip(keys, out)}
        d["h_max"] = hm.value
        return d

    def mesh(self, level):
        s = self.sizes(level)
        v = np.empty((s["nv"], 2)); lat = np.empty((s["nv"], 2), np.int32)
        t = np.empty((s["nt"], 3), np.int32); p = np.empty(s["nt"] if level else 0, np.int32)
        b = np.empty((s["nb"], 2), np.int32)
        _chk(lib().ref_export_mesh(self.h, level, _d(v), _i(lat), _i(t), _i(p) if level else None,
                                   _i(b)))
        return dict(vertices=v, lattice=lat, triangles=t, parent=p, boundary_edges=b,
                    h_max=s["h_max"], nx=s["nx"], ny=s["ny"])

    def space(self, level):
        s = self.sizes(level)
        dl = np.empty((s["ndofs"], 2), np.int32); idofs = np.empty(s["n_int"], np.int32)
        iidx = np.empty(s["ndofs"], np.int32)
        conn = np.empty((s["nt"], 6 if self.cfg.degree == 2 else 3), np.int32)
        _chk(lib().ref_export_space(self.h, level, _i(dl), _i(idofs), _i(iidx), _i(conn)))
        return dict(dof_lattice=dl, interior_dofs=idofs, interior_index=iidx, connectivity=conn)

    def csr(self, level, form):
        s = self.sizes(level)
        rp = np.empty(s["ndofs"] + 1, np.int32); cols = np.empty(s["nnz_a"], np.int32)
        vals = np.empty(s["nnz_a"])
        _chk(lib().ref_export_csr(self.h, level, {"stiffness": 0, "mass": 1}[form], _i(rp),
                                  _i(cols), _d(vals)))
        return rp, cols, vals

    def apply(self, level, form, x):
        x = np.ascontiguousarray(x, np.float64); y = np.empty_like(x)
        _chk(lib().ref_spmv(self.h, level, {"stiffness": 0, "mass": 1}[form], _d(x), _d(y)))
        return y

    def prolong(self, x, a, b):
        self.extend_to(b)
        x = np.ascontiguousarray(x, np.float64); y = np.empty(self.sizes(b)["ndofs"])
        _chk(lib().ref_prolong(self.h, a, b, _d(x), _d(y)))
        return y

    def restrict_transpose(self, x, a, b):
        x = np.ascontiguousarray(x, np.float64); y = np.empty(self.sizes(b)["ndofs"])
        _chk(lib().ref_restrict_transpose(self.h, a, b, _d(x), _d(y)))
        return y

    def region_dofs(self, level, kind, j=0, zero_trace=False):
        k = {"domain": 0, "block": 1, "overlap": 2, "inner": 3, "strip": 4}[kind]
        n = C.c_longlong()
        _chk(lib().ref_region_dofs(self.h, level, k, j, int(zero_trace), None, C.byref(n)))
        out = np.empty(n.value, np.int32)
        _chk(lib().ref_region_dofs(self.h, level, k, j, int(zero_trace), _i(out), C.byref(n)))
        return out

    def region_elements(self, level, kind, j=0):
        k = {"domain": 0, "block": 1, "overlap": 2, "inner": 3, "strip": 4}[kind]
        n = C.c_longlong()
        _chk(lib().ref_region_elements(self.h, level, k, j, None, C.byref(n)))
        out = np.empty(n.value, np.int32)
        _chk(lib().ref_region_elements(self.h, level, k, j, _i(out), C.byref(n)))
        return out

    def partition(self):
        info = np.zeros(5, np.int32)
        _chk(lib().ref_partition(self.h, None, _i(info)))
        rects = np.zeros((info[0], 3, 4), np.int32)
        _chk(lib().ref_partition(self.h, _i(rects), _i(info)))
        return info, rects

    def coarse_eigensolve(self, level, nev):
        self.extend_to(level)
        n = self.sizes(level)["n_int"]
        lam = np.empty(nev); co = np.empty((nev, n))
        _chk(lib().ref_coarse_eigensolve(self.h, level, nev, _d(lam), _d(co)))
        return lam, co

    def local_bvp_solve(self, level, j, lam, u_full, tol):
        u = np.ascontiguousarray(u_full, np.float64); e = np.empty_like(u)
        it = C.c_int(); fr = C.c_double()
        _chk(lib().ref_local_bvp_solve(self.h, level, j, C.c_double(lam), _d(u), C.c_double(tol),
                                       _d(e), C.byref(it), C.byref(fr)))
        return e, it.value, fr.value

    def local_bvp_time(self, level, j, lam, u_full, tol):
        """(seconds, iterations) of one local_bvp_solve task, timed in C++."""
        u = np.ascontiguousarray(u_full, np.float64)
        sec = C.c_double(); it = C.c_int()
        _chk(lib().ref_local_bvp_time(self.h, level, j, C.c_double(lam), _d(u), C.c_double(tol),
                                      C.byref(sec), C.byref(it)))
        return sec.value, it.value

    def strip_cg_sample(self, level, lam, u_full, tol, maxit):
        """(seconds, iterations) of cg_solve on the strip system capped at maxit."""
        u = np.ascontiguousarray(u_full, np.float64)
        sec = C.c_double(); it = C.c_int()
        _chk(lib().ref_strip_cg_sample(self.h, level, C.c_double(lam), _d(u), C.c_double(tol),
                                       int(maxit), C.byref(sec), C.byref(it)))
        return sec.value, it.value

    def interface_solve(self, level, lam, u_full, corr, tol):
        u = np.ascontiguousarray(u_full, np.float64); corr = np.ascontiguousarray(corr, np.float64)
        g = np.empty_like(u); it = C.c_int(); fr = C.c_double()
        _chk(lib().ref_interface_solve(self.h, level, C.c_double(lam), _d(u), _d(corr),
                                       C.c_double(tol), _d(g), C.byref(it), C.byref(fr)))
        return g, it.value, fr.value

    def augmented_eigensolve(self, level, glued, nev):
        g = np.ascontiguousarray(np.atleast_2d(glued), np.float64)
        n = self.sizes(level)["n_int"]
        lam = np.empty(nev); co = np.empty((nev, n))
        _chk(lib().ref_augmented_eigensolve(self.h, level, g.shape[0], _d(g), nev, _d(lam), _d(co)))
        return lam, co

    def correction_step(self, frm, to, lam_in, coeffs_in, want_coeffs=True):
        nev = len(lam_in)
        self.extend_to(max(frm, to))
        n = self.sizes(to)["n_int"]
        li = np.ascontiguousarray(lam_in, np.float64)
        ci = np.ascontiguousarray(coeffs_in, np.float64)
        lo = np.empty(nev); co = np.empty((nev, n)) if want_coeffs else None
        matched = C.c_int(); t3 = (C.c_double * 3)()
        _chk(lib().ref_correction_step(self.h, frm, to, nev, _d(li), _d(ci), _d(lo),
                                       _d(co) if want_coeffs else None, C.byref(matched), t3))
        return lo, co, bool(matched.value), tuple(t3)

    def multilevel(self, n_levels, nev, want_coeffs=True):
        # multilevel_correction always runs the configured number of levels
        if n_levels != self.cfg.n_levels or nev != self.cfg.nev:
            raise ValueError("multilevel() must match the hierarchy's n_levels and nev")
        lam = np.empty((n_levels, nev)); matched = np.zeros(n_levels, np.int32)
        times = np.zeros((n_levels, 3))
        self.extend_to(n_levels)
        n = self.sizes(n_levels)["n_int"]
        co = np.empty((nev, n)) if want_coeffs else None
        _chk(lib().ref_multilevel(self.h, _d(lam), _d(co) if want_coeffs else None, _i(matched),
                                  _d(times)))
        return lam, co, matched.astype(bool), times


def cg_solve_csr(row_ptr, cols, vals, rhs, tol, maxit=0):
    n = len(row_ptr) - 1
    rp = np.ascontiguousarray(row_ptr, np.int32); cl = np.ascontiguousarray(cols, np.int32)
    vl = np.ascontiguousarray(vals, np.float64); b = np.ascontiguousarray(rhs, np.float64)
    x = np.empty(n); it = C.c_int(); fr = C.c_double(); cv = C.c_int()
    _chk(lib().ref_cg_solve_csr(n, _i(rp), _i(cl), _d(vl), _d(b), C.c_double(tol), maxit, _d(x),
                                C.byref(it), C.byref(fr), C.byref(cv)))
    return x, it.value, fr.value, bool(cv.value)


def fnv1a64(*arrays) -> str:
    """FNV-1a-64 chained over raw little-endian bytes."""
    h = 1469598103934665603
    if available():
        f = lib().ref_fnv1a64
        f.restype = C.c_ulonglong
        f.argtypes = [C.c_void_p, C.c_ulonglong, C.c_ulonglong]
        for a in arrays:
            b = np.ascontiguousarray(a)
            h = f(b.ctypes.data, b.nbytes, h)
        return f"{h:016x}"
    for a in arrays:
        for byte in np.ascontiguousarray(a).tobytes():
            h ^= byte
            h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


# ---- harness and error reporting (harness.hpp, fespace.hpp:103-120) ----
def _cfg(domain=(-1.0, 1.0, -1.0, 1.0), H=0.5, delta=0.5, m=1, n_levels=2, nev=2, cg_tol=1e-10,
         workers=1, degree=1, example=0, deterministic=True):
    return RefConfig(*domain, H, delta, m, n_levels, degree, nev, example, workers, cg_tol,
                     int(deterministic))


def _cfg_dict(c: RefConfig) -> dict:
    return {k: getattr(c, k) for k, _ in RefConfig._fields_}


def parse_config_json(text: str):
    """(status, message, config dict) of the reference's parse_config_json."""
    out = RefConfig()
    st = lib().ref_parse_config_json(text.encode(), C.byref(out))
    return st, (lib().ref_last_error().decode() if st else ""), (_cfg_dict(out) if st == 0
                                                                 else None)


def parse_config_file(path: str):
    out = RefConfig()
    st = lib().ref_parse_config_file(str(path).encode(), C.byref(out))
    return st, (lib().ref_last_error().decode() if st else ""), (_cfg_dict(out) if st == 0
                                                                 else None)


def estimate_orders(errors, beta):
    e = np.ascontiguousarray(errors, np.float64)
    out = np.empty(max(len(e) - 1, 1))
    lib().ref_estimate_orders.argtypes = [dp, C.c_int, C.c_double, dp]
    st = lib().ref_estimate_orders(_d(e), len(e), beta, _d(out))
    if st:
        raise RefError(st, lib().ref_last_error().decode())
    return out[:max(len(e) - 1, 0)]


def make_reference(example: str, nev: int, pts=None):
    """lambdas, has_fn, and (value, dx, dy) of each closed form at pts (k x 2)."""
    lam = np.empty(nev)
    has = np.zeros(nev, np.int32)
    pts = np.zeros((0, 2)) if pts is None else np.ascontiguousarray(pts, np.float64)
    vals = np.zeros((nev, len(pts), 3))
    _chk(lib().ref_make_reference(example.encode(), nev, _d(lam), _i(has), len(pts), _d(pts),
                                  _d(vals)))
    return lam, has.astype(bool), vals


def run_experiment(csv_path, **kw):
    c = _cfg(**kw)
    _chk(lib().ref_run_experiment(C.byref(c), str(csv_path).encode()))


def print_table(csv_path) -> str:
    n = C.c_ulong()
    lib().ref_print_table.argtypes = [C.c_char_p, C.c_char_p, C.c_ulong, C.POINTER(C.c_ulong)]
    _chk(lib().ref_print_table(str(csv_path).encode(), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _chk(lib().ref_print_table(str(csv_path).encode(), buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def export_vtk(out_dir, **kw):
    c = _cfg(**kw)
    _chk(lib().ref_export_vtk(C.byref(c), str(out_dir).encode()))


def compute_errors(h: "RefHierarchy", level, coeffs_full, lambda_h, lambda_ref, ref_index=-1):
    """compute_errors with make_reference("laplace")'s eigenfunction ref_index."""
    u = np.ascontiguousarray(coeffs_full, np.float64)
    out = np.empty(3)
    lib().ref_compute_errors.argtypes = [C.c_void_p, C.c_int, dp, C.c_double, C.c_double,
                                         C.c_int, dp]
    _chk(lib().ref_compute_errors(h.h, level, _d(u), lambda_h, lambda_ref, ref_index, _d(out)))
    return out

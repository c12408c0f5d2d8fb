"""ctypes binding of libmlg_b200.so (the C ABI in include/mlg_b200.h).

There is no fallback: if the shared library is missing or cannot be loaded the
import-time call `lib()` raises, and every API entry point fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

LIB_PATH = Path(os.environ.get("MLG_LIB", Path(__file__).resolve().parent / "libmlg_b200.so"))

c_int_p = C.POINTER(C.c_int)
c_double_p = C.POINTER(C.c_double)
c_int64_p = C.POINTER(C.c_int64)


class MlgError(RuntimeError):
    code = 1


class ConfigError(MlgError):  # mleig::ConfigError (errors.hpp:10-12), exit code 2
    code = 2


class SolverError(MlgError):  # mleig::SolverError (errors.hpp:15-17), exit code 3
    code = 3


class IoError(MlgError):  # mleig::IoError (errors.hpp:20-22), exit code 4
    code = 4


class CudaError(MlgError):
    code = 5


_ERRORS = {1: MlgError, 2: ConfigError, 3: SolverError, 4: IoError, 5: CudaError}


class MlgConfig(C.Structure):
    _fields_ = [
        ("x_min", C.c_double), ("x_max", C.c_double),
        ("y_min", C.c_double), ("y_max", C.c_double),
        ("H", C.c_double), ("delta", C.c_double),
        ("m", C.c_int), ("n_levels", C.c_int), ("degree", C.c_int),
        ("nev", C.c_int), ("example", C.c_int), ("workers", C.c_int),
        ("cg_tol", C.c_double), ("deterministic", C.c_int), ("device", C.c_int),
        ("seed", C.c_uint64),
        ("hole_x_min", C.c_double), ("hole_x_max", C.c_double),
        ("hole_y_min", C.c_double), ("hole_y_max", C.c_double),
    ]


class MlgLevelInfo(C.Structure):
    _fields_ = [
        ("num_vertices", C.c_int64), ("num_triangles", C.c_int64),
        ("num_boundary_edges", C.c_int64), ("ndofs", C.c_int64),
        ("n_interior", C.c_int64), ("nnz", C.c_int64),
        ("nx", C.c_int), ("ny", C.c_int), ("level", C.c_int), ("h_max", C.c_double),
    ]


class MlgSolveReport(C.Structure):
    _fields_ = [("iterations", C.c_int), ("final_residual", C.c_double),
                ("converged", C.c_int)]


class MlgStepTimings(C.Structure):
    _fields_ = [
        ("local_seconds", C.c_double), ("iface_seconds", C.c_double),
        ("aug_seconds", C.c_double), ("build_seconds", C.c_double),
        ("local_iterations_max", C.c_int), ("strip_iterations_max", C.c_int),
        ("spmv_kernel_ms", C.c_double), ("spmv_launches", C.c_int64),
        ("spmv_rows", C.c_double), ("kernel_launches", C.c_int64),
        ("step_seconds", C.c_double), ("spmv_uniform_stencil", C.c_int),
        ("spmv_check_rows", C.c_double), ("spmv_launches_all", C.c_int64),
        ("strip_kernel_ms", C.c_double), ("strip_launches", C.c_int64),
        ("strip_row_iters", C.c_double), ("strip_kernel", C.c_int),
        ("strip_bytes_per_row", C.c_int), ("local_kernel", C.c_int),
    ]


class MlgExactMode(C.Structure):
    _fields_ = [("mx", C.c_int), ("my", C.c_int), ("x0", C.c_double), ("lx", C.c_double),
                ("y0", C.c_double), ("ly", C.c_double), ("amp", C.c_double)]


class MlgErrorReport(C.Structure):
    _fields_ = [("eig_err", C.c_double), ("l2_err", C.c_double), ("h1_err", C.c_double)]


class MlgReportRow(C.Structure):
    _fields_ = [
        ("level", C.c_int), ("h", C.c_double), ("dofs", C.c_int), ("eig_index", C.c_int),
        ("lambda_", C.c_double), ("eig_err", C.c_double), ("has_h1", C.c_int),
        ("h1_err", C.c_double), ("has_order", C.c_int), ("order", C.c_double),
        ("local_s", C.c_double), ("iface_s", C.c_double), ("aug_s", C.c_double),
    ]


# name -> argtypes (every symbol declared in include/mlg_b200.h)
SIGNATURES = {
    "mlg_last_error": [],
    "mlg_create": [C.POINTER(MlgConfig), C.POINTER(C.c_void_p)],
    "mlg_destroy": [C.c_void_p],
    "mlg_extend_to": [C.c_void_p, C.c_int],
    "mlg_max_level": [C.c_void_p, c_int_p],
    "mlg_get_level_info": [C.c_void_p, C.c_int, C.POINTER(MlgLevelInfo)],
    "mlg_export_mesh": [C.c_void_p, C.c_int, c_double_p, c_int_p, c_int_p, c_int_p, c_int_p],
    "mlg_export_space": [C.c_void_p, C.c_int, c_int_p, c_int_p, c_int_p, c_int_p],
    "mlg_export_csr": [C.c_void_p, C.c_int, C.c_int, c_int_p, c_int_p, c_double_p],
    "mlg_partition": [C.c_void_p, c_int_p, c_int_p],
    "mlg_region_dofs": [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, c_int_p, c_int64_p],
    "mlg_region_elements": [C.c_void_p, C.c_int, C.c_int, C.c_int, c_int_p, c_int64_p],
    "mlg_spmv": [C.c_void_p, C.c_int, C.c_int, c_double_p, c_double_p],
    "mlg_prolong": [C.c_void_p, C.c_int, C.c_int, c_double_p, c_double_p],
    "mlg_restrict_transpose": [C.c_void_p, C.c_int, C.c_int, c_double_p, c_double_p],
    "mlg_coarse_eigensolve": [C.c_void_p, C.c_int, C.c_int, c_double_p, c_double_p],
    "mlg_local_bvp_solve": [C.c_void_p, C.c_int, C.c_int, C.c_double, c_double_p, C.c_double,
                            c_double_p, C.POINTER(MlgSolveReport)],
    "mlg_local_cg_solve": [C.c_void_p, C.c_int, C.c_int, C.c_double, c_double_p, C.c_double,
                           C.c_int, c_double_p, C.POINTER(MlgSolveReport)],
    "mlg_interface_solve": [C.c_void_p, C.c_int, C.c_double, c_double_p, c_double_p,
                            C.c_double, c_double_p, C.POINTER(MlgSolveReport)],
    "mlg_augmented_eigensolve": [C.c_void_p, C.c_int, C.c_int, c_double_p, C.c_int,
                                 c_double_p, c_double_p],
    "mlg_correction_step": [C.c_void_p, C.c_int, C.c_int, C.c_int, c_double_p, c_double_p,
                            c_double_p, c_double_p, c_int_p, C.POINTER(MlgStepTimings)],
    "mlg_correction_step_device": [C.c_void_p, C.c_int, C.c_int, C.c_int, c_double_p,
                                   C.c_void_p, c_double_p, C.c_void_p, c_int_p,
                                   C.POINTER(MlgStepTimings)],
    "mlg_multilevel_correction": [C.c_void_p, C.c_int, c_double_p, c_double_p, C.c_void_p,
                                  c_int_p, C.POINTER(MlgStepTimings)],
    "mlg_multilevel_correction_refs": [C.c_void_p, C.c_int, C.c_int, c_double_p,
                                       C.POINTER(MlgExactMode), c_double_p, c_double_p,
                                       c_double_p, c_double_p, c_double_p, c_int_p,
                                       C.POINTER(MlgStepTimings)],
    "mlg_make_reference": [C.c_int, C.c_int, c_double_p, c_double_p, C.POINTER(MlgExactMode)],
    "mlg_make_reference_for": [C.POINTER(MlgConfig), C.c_int, c_double_p,
                               C.POINTER(MlgExactMode)],
    "mlg_compute_errors": [C.c_void_p, C.c_int, c_double_p, C.c_double, C.c_double,
                           C.POINTER(MlgExactMode), C.POINTER(MlgErrorReport)],
    "mlg_parse_config_json": [C.c_char_p, C.POINTER(MlgConfig)],
    "mlg_parse_config_file": [C.c_char_p, C.POINTER(MlgConfig)],
    "mlg_estimate_orders": [c_double_p, C.c_int, C.c_double, c_double_p],
    "mlg_run_experiment": [C.POINTER(MlgConfig), C.c_char_p, C.POINTER(MlgReportRow), C.c_int,
                           c_int_p],
    "mlg_write_csv": [C.POINTER(MlgReportRow), C.c_int, C.c_char_p],
    "mlg_print_table": [C.c_char_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)],
    "mlg_export_vtk": [C.POINTER(MlgConfig), C.c_char_p],
    "mlg_set_profiling": [C.c_void_p, C.c_int],
    "mlg_set_input_stream": [C.c_void_p, C.c_void_p],
    "mlg_build_profile": [C.c_void_p, c_double_p, c_double_p],
    "mlg_build_profile_kernel": [C.c_void_p, c_int_p],
    "mlg_bench_spmv": [C.c_void_p, C.c_int, C.c_int, c_double_p, c_double_p],
}

_lock = threading.Lock()
_lib: C.CDLL | None = None


def lib() -> C.CDLL:
    """Load the CUDA library; raise if it is absent (no CPU fallback exists)."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                    "(the B200 path has no CPU fallback)")
            h = C.CDLL(str(LIB_PATH))
            for name, args in SIGNATURES.items():
                fn = getattr(h, name)
                fn.argtypes = args
                fn.restype = C.c_int
            h.mlg_last_error.restype = C.c_char_p
            h.mlg_destroy.restype = None
            _lib = h
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().mlg_last_error().decode(errors="replace")
        raise _ERRORS.get(status, MlgError)(msg)

"""Host mirror of the reference's experiment harness (include/mleig/harness.hpp,
src/harness.cpp) and error reporting (compute_errors, fespace.hpp:118-120) over
the C ABI.  Parsing, the CSV/table/VTK writers and make_reference are native
code in libmlg_b200.so (csrc/harness.cu, csrc/errors.cu); the error sweeps run
on the device."""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from ._lib import (MlgConfig, MlgErrorReport, MlgExactMode, MlgReportRow, MlgStepTimings,
                   c_double_p, check, lib)
from .corrector import (DomainRect, EigenPair, Hierarchy, LevelTrace, RunConfig, StepTimings,
                        _dp, _f64, _ip)

EXAMPLES = ("laplace", "variable", "reaction")


def _config_from_c(c: MlgConfig) -> RunConfig:
    return RunConfig(domain=DomainRect(c.x_min, c.x_max, c.y_min, c.y_max), H=c.H,
                     delta=c.delta, m=c.m, n_levels=c.n_levels, degree=c.degree, nev=c.nev,
                     example=EXAMPLES[c.example], cg_tol=c.cg_tol, workers=c.workers,
                     deterministic=bool(c.deterministic), device=c.device, seed=c.seed,
                     hole=(DomainRect(c.hole_x_min, c.hole_x_max, c.hole_y_min, c.hole_y_max)
                           if c.hole_x_max > c.hole_x_min else None))


def parse_config_json(text: str) -> RunConfig:  # harness.cpp:58-102
    out = MlgConfig()
    check(lib().mlg_parse_config_json(text.encode(), C.byref(out)))
    return _config_from_c(out)


def parse_config_file(path: str) -> RunConfig:  # harness.cpp:104-111
    out = MlgConfig()
    check(lib().mlg_parse_config_file(str(path).encode(), C.byref(out)))
    return _config_from_c(out)


def estimate_orders(errors, beta: float) -> list:  # harness.cpp:113-122
    e = _f64(errors)
    out = np.empty(max(len(e) - 1, 1))
    check(lib().mlg_estimate_orders(_dp(e), len(e), beta, _dp(out)))
    return out[:max(len(e) - 1, 0)].tolist()


@dataclass
class ExactFunction:
    """A closed-form eigenfunction of make_reference: amp * sin(mx pi (x-x0)/lx)
    * sin(my pi (y-y0)/ly) (harness.cpp:153-163)."""
    mx: int
    my: int
    x0: float
    lx: float
    y0: float
    ly: float
    amp: float

    def value(self, x, y):
        return self.amp * (np.sin(self.mx * math.pi * (x - self.x0) / self.lx) *
                           np.sin(self.my * math.pi * (y - self.y0) / self.ly))

    def gradient(self, x, y):
        ax, ay = self.mx * math.pi / self.lx, self.my * math.pi / self.ly
        sx, cx = np.sin(ax * (x - self.x0)), np.cos(ax * (x - self.x0))
        sy, cy = np.sin(ay * (y - self.y0)), np.cos(ay * (y - self.y0))
        return self.amp * ax * cx * sy, self.amp * ay * sx * cy

    def to_c(self) -> MlgExactMode:
        return MlgExactMode(self.mx, self.my, self.x0, self.lx, self.y0, self.ly, self.amp)


@dataclass
class ReferenceSet:  # corrector.hpp ReferenceSet
    lambdas: list
    eigenfunctions: dict = field(default_factory=dict)  # index -> ExactFunction


def make_reference(example: str, nev: int, domain: DomainRect | None = None) -> ReferenceSet:
    """harness.cpp:126-169; with `domain` the Laplace table is that rectangle's
    (bitwise the reference's on (-1,1)^2), without it the reference's own."""
    if example not in EXAMPLES:
        raise _config_error(f'no reference data for example "{example}"')
    lam = np.empty(nev)
    modes = (MlgExactMode * nev)()
    dom = None if domain is None else _f64([domain.x_min, domain.x_max, domain.y_min,
                                            domain.y_max])
    check(lib().mlg_make_reference(EXAMPLES.index(example), nev, _dp(dom), _dp(lam), modes))
    fns = {i: ExactFunction(m.mx, m.my, m.x0, m.lx, m.y0, m.ly, m.amp)
           for i, m in enumerate(modes) if m.mx > 0}
    return ReferenceSet(lam.tolist(), fns)


def make_reference_for(config: RunConfig, nev: int) -> ReferenceSet:
    """The reference set run_experiment reports against for `config` (the
    configured rectangle's table, or the L-shaped domain's for config 3)."""
    cfg = config.to_c()
    lam = np.empty(nev)
    modes = (MlgExactMode * nev)()
    check(lib().mlg_make_reference_for(C.byref(cfg), nev, _dp(lam), modes))
    fns = {i: ExactFunction(m.mx, m.my, m.x0, m.lx, m.y0, m.ly, m.amp)
           for i, m in enumerate(modes) if m.mx > 0}
    return ReferenceSet(lam.tolist(), fns)


def _config_error(msg):
    from ._lib import ConfigError
    return ConfigError(msg)


@dataclass
class ErrorReport:  # fespace.hpp:108-112
    eig_err: float
    l2_err: float
    h1_err: float


def compute_errors(hy: Hierarchy, level: int, coeffs_full, lambda_h: float, lambda_ref: float,
                   reference: ExactFunction | None = None) -> ErrorReport:
    """fespace.cpp:434-488 on the device (49-point Gauss-Duffy sweep)."""
    u = _f64(coeffs_full)
    rep = MlgErrorReport()
    mode = reference.to_c() if reference is not None else None
    check(lib().mlg_compute_errors(hy.handle, level, _dp(u), lambda_h, lambda_ref,
                                   C.byref(mode) if mode is not None else None, C.byref(rep)))
    return ErrorReport(rep.eig_err, rep.l2_err, rep.h1_err)


@dataclass
class MultilevelResult:  # corrector.hpp:161-163
    levels: list


def multilevel_correction(hy: Hierarchy, refs: ReferenceSet | None = None) -> MultilevelResult:
    """corrector.cpp:414-462 with the optional ReferenceSet: every LevelTrace
    carries lambdas, eig_errors, l2_errors and h1_errors (NaN where undefined)."""
    nl, nev = hy.config.n_levels, hy.config.nev
    hy.extend_to(nl)
    lam = np.empty((nl, nev))
    ee = np.full((nl, nev), np.nan)
    l2 = np.full((nl, nev), np.nan)
    h1 = np.full((nl, nev), np.nan)
    matched = np.zeros(nl, np.int32)
    times = (MlgStepTimings * nl)()
    n = hy.level_info(nl).n_interior
    co = np.empty((nev, n))
    if refs is not None:
        nref = min(len(refs.lambdas), nev)
        rl = _f64(refs.lambdas[:nref]) if nref else _f64([0.0])
        modes = (MlgExactMode * max(nref, 1))()
        for i in range(nref):
            if i in refs.eigenfunctions:
                modes[i] = refs.eigenfunctions[i].to_c()
        check(lib().mlg_multilevel_correction_refs(hy.handle, nl, nref, _dp(rl), modes,
                                                   _dp(lam), _dp(ee), _dp(l2), _dp(h1), _dp(co),
                                                   _ip(matched), times))
    else:
        check(lib().mlg_multilevel_correction(hy.handle, nl, _dp(lam), _dp(co), None,
                                              _ip(matched), times))
    out = []
    for k in range(1, nl + 1):
        info = hy.level_info(k)
        tr = LevelTrace(k, info.h_max, int(info.n_interior), lam[k - 1].tolist(),
                        StepTimings.from_c(times[k - 1]), bool(matched[k - 1]),
                        [EigenPair(float(lam[-1, i]), co[i].copy(), nl) for i in range(nev)]
                        if k == nl else [], ee[k - 1].tolist(), l2[k - 1].tolist(),
                        h1[k - 1].tolist())
        out.append(tr)
    return MultilevelResult(out)


@dataclass
class ReportRow:  # harness.hpp:23-35
    level: int
    h: float
    dofs: int
    eig_index: int
    lam: float
    eig_err: float
    h1_err: float | None
    order: float | None
    local_s: float
    iface_s: float
    aug_s: float

    @classmethod
    def from_c(cls, r: MlgReportRow) -> "ReportRow":
        return cls(r.level, r.h, r.dofs, r.eig_index, r.lambda_, r.eig_err,
                   r.h1_err if r.has_h1 else None, r.order if r.has_order else None,
                   r.local_s, r.iface_s, r.aug_s)

    def to_c(self) -> MlgReportRow:
        return MlgReportRow(self.level, self.h, self.dofs, self.eig_index, self.lam,
                            self.eig_err, int(self.h1_err is not None),
                            0.0 if self.h1_err is None else self.h1_err,
                            int(self.order is not None), 0.0 if self.order is None else self.order,
                            self.local_s, self.iface_s, self.aug_s)


@dataclass
class ExperimentReport:  # harness.hpp:37-41
    config: RunConfig
    rows: list


def run_experiment(config: RunConfig, csv_path: str) -> ExperimentReport:
    """harness.cpp:171-206: multilevel correction + errors against the example's
    reference set, CSV written by the native writer."""
    cfg = config.to_c()
    cap = max(config.n_levels * config.nev, 1)
    rows = (MlgReportRow * cap)()
    n = C.c_int()
    check(lib().mlg_run_experiment(C.byref(cfg), str(csv_path).encode(), rows, cap,
                                   C.byref(n)))
    return ExperimentReport(config, [ReportRow.from_c(rows[i]) for i in range(n.value)])


def write_csv(report: ExperimentReport, path: str) -> None:  # harness.cpp:208-222
    rows = (MlgReportRow * max(len(report.rows), 1))(*[r.to_c() for r in report.rows])
    check(lib().mlg_write_csv(rows, len(report.rows), str(path).encode()))


def print_table(csv_path: str) -> str:  # harness.cpp:240-290 (returns the text)
    n = C.c_size_t()
    check(lib().mlg_print_table(str(csv_path).encode(), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(lib().mlg_print_table(str(csv_path).encode(), buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def export_vtk(config: RunConfig, out_dir: str) -> None:  # harness.cpp:292-351
    cfg = config.to_c()
    check(lib().mlg_export_vtk(C.byref(cfg), str(out_dir).encode()))

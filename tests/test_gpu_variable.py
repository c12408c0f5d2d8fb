"""The reference's variable-coefficient field (CoefficientField::variable,
fespace.cpp:114-123: A = [[e^{1+x^2}, e^{xy}], [e^{xy}, e^{1+y^2}]], phi =
(1+x^2)(1+y^2), 12-point degree-6 rule fespace.cpp:49-75) on the B200 path:
operators vs the compiled reference (structure bitwise; values to a few ulp
because exp() is the one operation whose last bit differs between libms), and
the multilevel correction vs the golden eigenpairs (north-star tolerances).
The CG runs its general per-row stencil path here (no constant-coefficient
shortcut)."""
import json
from pathlib import Path

import numpy as np
import pytest

from _parity import compare_pairs

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())
SQUARE = (-1.0, 1.0, -1.0, 1.0)


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@pytest.mark.parametrize("domain,H,m,levels", [(SQUARE, 0.25, 4, 3), ((0.0, 1.0, 0.0, 1.0), 1 / 8, 4, 3),
                                               ((0.0, 3.0, -1.0, 1.0), 0.5, 1, 3)])
def test_variable_operators_match_reference(mlg, oracle_ref, domain, H, m, levels):
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*domain), H=H, delta=H, m=m, n_levels=levels,
                        nev=1, example="variable")
    hy = mlg.Hierarchy(cfg)
    rh = oracle_ref.RefHierarchy(domain=domain, H=H, delta=H, m=m, n_levels=levels, nev=1,
                                 example=1)
    hy.extend_to(levels)
    rh.extend_to(levels)
    for k in range(levels + 1):
        for form in ("stiffness", "mass"):
            grp, gc, gv = hy.csr(k, form)
            rrp, rc, rv = rh.csr(k, form)
            assert np.array_equal(grp, rrp) and np.array_equal(gc, rc), (k, form)
            scale = np.abs(rv).max()
            assert np.max(np.abs(gv - rv)) <= 4e-16 * scale, (k, form)
            if form == "mass":  # no exp on the mass path: bitwise
                assert np.array_equal(bits(gv), bits(rv)), k
            else:
                assert np.mean(bits(gv) == bits(rv)) > 0.8, k


def test_variable_multilevel_matches_golden(mlg):
    g = GOLDEN["multilevel"]["variable_square_L4_m4_nev3"]
    c = g["config"]
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*c["domain"]), H=c["H"], delta=c["delta"],
                        m=c["m"], n_levels=c["n_levels"], nev=c["nev"], example="variable")
    with mlg.Hierarchy(cfg) as hy:
        lam, pairs, matched, times = mlg.multilevel_correction(hy)
        ref = np.array(g["lambdas"])
        assert np.max(np.abs(lam - ref) / ref) <= 1e-10, (lam, ref)
        assert all(matched)
        assert not any(t.spmv_uniform_stencil for t in times[1:])  # general stencil path
        u_ref = np.load(ROOT / "tests" / "golden" / "variable_L4_u.npy")
        L = c["n_levels"]
        compare_pairs(lam[-1], [p.coeffs for p in pairs], ref[-1], list(u_ref),
                      lambda f: hy.apply(L, "mass", f), lambda v: hy.expand_interior(L, v))


def test_variable_multilevel_larger_matches_golden(mlg):
    g = GOLDEN["multilevel"]["variable_square_L6_m16_nev2"]
    c = g["config"]
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*c["domain"]), H=c["H"], delta=c["delta"],
                        m=c["m"], n_levels=c["n_levels"], nev=c["nev"], example="variable")
    with mlg.Hierarchy(cfg) as hy:
        lam, pairs, matched, _ = mlg.multilevel_correction(hy)
        ref = np.array(g["lambdas"])
        assert np.max(np.abs(lam - ref) / ref) <= 1e-10, (lam, ref)
        # seeded projections of the final eigenvectors (sign-free: compare |.|)
        n = pairs[0].coeffs.size
        rng = np.random.default_rng(20261019)
        R = rng.uniform(-1.0, 1.0, size=(8, n))
        for i, p in enumerate(pairs):
            got = np.abs(R @ p.coeffs)
            want = np.abs(np.array(g["projections"][i]))
            assert np.max(np.abs(got - want)) <= 1e-7 * np.max(want)


def test_variable_step_matches_reference_step(mlg, oracle_ref):
    """One correction step from the same input on both sides (test_corrector-style)."""
    kw = dict(domain=SQUARE, H=0.25, delta=0.25, m=4, n_levels=3, nev=2)
    rh = oracle_ref.RefHierarchy(**kw, example=1)
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*SQUARE), H=0.25, delta=0.25, m=4, n_levels=3,
                        nev=2, example="variable")
    with mlg.Hierarchy(cfg) as hy:
        lam1, co1 = rh.coarse_eigensolve(2, 2)
        st = mlg.CorrectionState(2, [mlg.EigenPair(float(lam1[i]), co1[i], 2) for i in range(2)])
        out, _ = mlg.one_correction_step(hy, st, 3)
        lam_r, co_r, _, _ = rh.correction_step(2, 3, lam1, co1)
        rh.extend_to(3)
        compare_pairs([p.lam for p in out.pairs], [p.coeffs for p in out.pairs], lam_r, co_r,
                      lambda f: rh.apply(3, "mass", f), lambda v: hy.expand_interior(3, v))

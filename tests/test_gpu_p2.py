"""P2 (degree 2) spaces on the B200 path vs the compiled reference: the dof
numbering, 6-dof connectivity, stiffness and mass CSR (bitwise for the Laplace
field, a few ulp for the variable field's exp), the full-space SpMV, the P2
prolongation and its transpose (bitwise), and the level-1 dense eigensolve.
Mirrors test_fespace.cpp:34-60,121-128,187-213.  The correction step is
run by the degree-2 batched CG (cg_p2.cu) and checked against the reference's
multilevel run."""
import numpy as np
import pytest

from _parity import compare_pairs

pytestmark = pytest.mark.gpu

SQUARE = (-1.0, 1.0, -1.0, 1.0)
CASES = [("square_H05", SQUARE, 0.5, 1, 3), ("square_H025", SQUARE, 0.25, 4, 3),
         ("rect", (0.0, 3.0, -1.0, 1.0), 0.5, 1, 2)]


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64) if a.dtype == np.float64 else a


def pair(mlg, oracle_ref, domain, H, m, levels, example=0):
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*domain), H=H, delta=H, m=m, n_levels=levels,
                        nev=2, degree=2, example=["laplace", "variable"][example])
    hy = mlg.Hierarchy(cfg)
    rh = oracle_ref.RefHierarchy(domain=domain, H=H, delta=H, m=m, n_levels=levels, nev=2,
                                 degree=2, example=example)
    hy.extend_to(levels)
    rh.extend_to(levels)
    return hy, rh


@pytest.mark.parametrize("name,domain,H,m,levels", CASES)
def test_p2_space_and_operators_bitexact(mlg, oracle_ref, name, domain, H, m, levels):
    hy, rh = pair(mlg, oracle_ref, domain, H, m, levels)
    for k in range(levels + 1):
        gs, rs = hy.space(k), rh.space(k)
        for key in ("dof_lattice", "interior_dofs", "interior_index", "connectivity"):
            assert np.array_equal(getattr(gs, key), rs[key]), (name, k, key)
        for form in ("stiffness", "mass"):
            grp, gc, gv = hy.csr(k, form)
            rrp, rc, rv = rh.csr(k, form)
            assert np.array_equal(grp, rrp) and np.array_equal(gc, rc), (name, k, form)
            assert np.array_equal(bits(gv), bits(rv)), (name, k, form)
        x = np.random.default_rng(k).uniform(-1, 1, gs.ndofs)
        for form in ("stiffness", "mass"):
            assert np.array_equal(bits(hy.apply(k, form, x)), bits(rh.apply(k, form, x)))


def test_p2_space_sizes(mlg, oracle_ref):  # test_fespace.cpp:34-60
    hy, _ = pair(mlg, oracle_ref, SQUARE, 0.5, 1, 1)
    s = hy.space(0)
    assert s.ndofs == 25 + 56 and len(s.interior_dofs) == 49
    order = s.dof_lattice[:, 1] * 100 + s.dof_lattice[:, 0]
    assert np.all(np.diff(order) > 0)  # lexicographic (y, x)


def test_p2_transfer_bitexact_and_energy(mlg, oracle_ref):  # test_fespace.cpp:187-213
    hy, rh = pair(mlg, oracle_ref, SQUARE, 0.25, 4, 3)
    rng = np.random.default_rng(29)
    for a in range(3):
        for b in range(a + 1, 4):
            x = rng.uniform(-1, 1, hy.level_info(a).ndofs)
            px = hy.prolong(x, a, b)
            assert np.array_equal(bits(px), bits(rh.prolong(x, a, b))), (a, b)
            ea = x @ hy.apply(a, "stiffness", x)
            eb = px @ hy.apply(b, "stiffness", px)
            assert abs(eb - ea) <= 1e-12 * ea
            y = rng.uniform(-1, 1, hy.level_info(b).ndofs)
            assert np.array_equal(bits(hy.restrict_transpose(y, b, a)),
                                  bits(rh.restrict_transpose(y, b, a))), (a, b)
    ones = np.ones(hy.level_info(1).ndofs)
    assert np.allclose(hy.prolong(ones, 1, 2), 1.0, rtol=0, atol=1e-15)


def test_p2_variable_field_operators(mlg, oracle_ref):
    hy, rh = pair(mlg, oracle_ref, SQUARE, 0.5, 1, 2, example=1)
    for k in range(3):
        for form in ("stiffness", "mass"):
            grp, gc, gv = hy.csr(k, form)
            rrp, rc, rv = rh.csr(k, form)
            assert np.array_equal(grp, rrp) and np.array_equal(gc, rc)
            assert np.max(np.abs(gv - rv)) <= 8e-16 * np.max(np.abs(rv)), (k, form)


def test_p2_coarse_eigensolve_and_mass(mlg, oracle_ref):
    hy, rh = pair(mlg, oracle_ref, SQUARE, 0.25, 4, 2)
    pairs = mlg.coarse_eigensolve(hy, 1, 3)
    lam_r, co_r = rh.coarse_eigensolve(1, 3)
    compare_pairs([p.lam for p in pairs], [p.coeffs for p in pairs], lam_r, co_r,
                  lambda f: rh.apply(1, "mass", f), lambda v: hy.expand_interior(1, v))
    ones = np.ones(hy.level_info(2).ndofs)  # test_fespace.cpp:121-128
    assert abs(ones @ hy.apply(2, "mass", ones) - 4.0) <= 1e-12 * 4.0


@pytest.mark.parametrize("spec", [(SQUARE, 0.25, 4, 3, 2), (SQUARE, 0.5, 1, 3, 3),
                                  ((0.0, 1.0, 0.0, 1.0), 1 / 8, 4, 3, 1)])
def test_p2_multilevel_matches_reference(mlg, oracle_ref, spec):
    """The whole degree-2 multilevel correction (P2 batched CG, strip, arrowhead /
    dense augmented solve) vs the reference with degree 2."""
    domain, H, m, levels, nev = spec
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*domain), H=H, delta=H, m=m, n_levels=levels,
                        nev=nev, degree=2)
    hy = mlg.Hierarchy(cfg)
    rh = oracle_ref.RefHierarchy(domain=domain, H=H, delta=H, m=m, n_levels=levels, nev=nev,
                                 degree=2)
    lam_g, pairs, matched, _ = mlg.multilevel_correction(hy)
    lam_r, co_r, matched_r, _ = rh.multilevel(levels, nev)
    for k in range(levels):
        assert np.max(np.abs(lam_g[k] - lam_r[k]) / lam_r[k]) <= 1e-10, (k, lam_g, lam_r)
    rh.extend_to(levels)
    compare_pairs(lam_g[-1], [p.coeffs for p in pairs], lam_r[-1], co_r,
                  lambda f: rh.apply(levels, "mass", f), lambda v: hy.expand_interior(levels, v))
    assert list(matched) == list(matched_r)


def test_p2_local_solve_matches_reference(mlg, oracle_ref):
    hy, rh = pair(mlg, oracle_ref, SQUARE, 0.25, 4, 2)
    lam, co = rh.coarse_eigensolve(1, 1)
    u = rh.prolong(hy.expand_interior(1, co[0]), 1, 2)
    for j in range(4):
        e_g, rep = mlg.local_bvp_solve(hy, 2, j, lam[0], u, 1e-12)
        e_r, it_r, _ = rh.local_bvp_solve(2, j, lam[0], u, 1e-12)
        assert rep.converged and abs(rep.iterations - it_r) <= 2
        assert np.max(np.abs(e_g - e_r)) <= 1e-10 * max(1.0, np.max(np.abs(e_r)))


def test_p2_errors_and_report_match_reference(mlg, oracle_ref, tmp_path):
    """compute_errors with P2 shape functions and the degree-2 run_experiment vs the
    reference's (harness.cpp:171-222 with degree 2)."""
    from paper_1401_4969_b200 import harness as H
    kw = dict(domain=SQUARE, H=0.5, delta=0.5, m=1, n_levels=3, nev=2, degree=2)
    ref_csv = tmp_path / "ref.csv"
    oracle_ref.run_experiment(ref_csv, **kw)
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*SQUARE), H=0.5, delta=0.5, m=1, n_levels=3,
                        nev=2, degree=2)
    H.run_experiment(cfg, str(tmp_path / "ours.csv"))
    a = (tmp_path / "ours.csv").read_text().splitlines()
    b = ref_csv.read_text().splitlines()
    assert a[0] == b[0] and len(a) == len(b)
    for la, lb in zip(a[1:], b[1:]):
        fa, fb = la.split(","), lb.split(",")
        assert fa[:4] == fb[:4]
        assert abs(float(fa[4]) - float(fb[4])) <= 1e-10 * float(fb[4])
        if fb[6]:
            assert abs(float(fa[6]) - float(fb[6])) <= 1e-7 * float(fb[6]), (fa, fb)


def test_p2_golden_fixtures(mlg):
    """Against the committed fixtures only (no reference at run time)."""
    import json
    from pathlib import Path
    from oracle.ref import fnv1a64 as f
    g = json.loads((Path(__file__).resolve().parent / "golden" / "golden.json").read_text())["p2"]
    c = g["multilevel"]["config"]
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*c["domain"]), H=c["H"], delta=c["delta"],
                        m=c["m"], n_levels=c["n_levels"], nev=c["nev"], degree=2)
    with mlg.Hierarchy(cfg) as hy:
        hy.extend_to(3)
        sp = hy.space(3)
        assert [f(sp.dof_lattice), f(sp.interior_dofs), f(sp.connectivity)] == g["space"]
        for form in ("stiffness", "mass"):
            assert [f(a) for a in hy.csr(3, form)] == g[form]
        lam, pairs, matched, _ = mlg.multilevel_correction(hy)
        ref = np.array(g["multilevel"]["lambdas"])
        assert np.max(np.abs(lam - ref) / ref) <= 1e-10

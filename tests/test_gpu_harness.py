"""Error reporting and the experiment harness through the B200 path vs the
compiled reference: compute_errors on the device (fespace.cpp:434-488),
run_experiment's CSV (harness.cpp:171-222) and export_vtk (harness.cpp:292-351).
Mirrors test_fespace.cpp:316-358 and test_harness.cpp:98-187."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SQUARE = (-1.0, 1.0, -1.0, 1.0)


@pytest.fixture(scope="module")
def H(mlg):
    from paper_1401_4969_b200 import harness
    return harness


def hier(mlg, domain=SQUARE, H=0.25, delta=0.25, m=4, levels=3, nev=1, example="laplace"):
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*domain), H=H, delta=delta, m=m, n_levels=levels,
                        nev=nev, example=example)
    return mlg.Hierarchy(cfg)


def dof_xy(hy, level):
    sp = hy.space(level)
    info = hy.level_info(level)
    d = hy.config.domain
    dx = (d.x_max - d.x_min) / info.nx
    dy = (d.y_max - d.y_min) / info.ny
    lat = sp.dof_lattice / 2.0
    return d.x_min + lat[:, 0] * dx, d.y_min + lat[:, 1] * dy


def test_compute_errors_interpolant_kat(mlg, H):
    """test_fespace.cpp:316-358: interpolated exact eigenfunction."""
    refs = H.make_reference("laplace", 1)
    u1 = refs.eigenfunctions[0]
    lam1 = math.pi ** 2 / 2.0
    with hier(mlg, H=0.25, levels=2) as hy:
        hy.extend_to(2)
        prev = None
        for k in range(3):
            x, y = dof_xy(hy, k)
            c = u1.value(x, y)
            e = H.compute_errors(hy, k, c, lam1, lam1, u1)
            h = hy.level_info(k).h_max
            assert e.eig_err == 0.0
            assert e.h1_err <= 5.0 * h and e.l2_err <= 5.0 * h * h
            if prev is not None:
                assert e.h1_err <= 0.6 * prev
            prev = e.h1_err
            flipped = H.compute_errors(hy, k, -c, lam1, lam1, u1)
            assert abs(flipped.h1_err - e.h1_err) <= 1e-14 * e.h1_err
            bare = H.compute_errors(hy, k, c, lam1, lam1 + 0.5)
            assert abs(bare.eig_err - 0.5) <= 1e-14 and math.isnan(bare.h1_err)


@pytest.mark.parametrize("idx", [0, 3])
def test_compute_errors_matches_reference(mlg, H, oracle_ref, idx):
    """Same coefficient vectors on both sides: the device sweep vs the reference's
    sequential one.  The reference forms L2^2 as s_hh - 2 s_hu + s_uu (rounding
    noise ~1e-13 absolute); the tolerance is set above that noise."""
    refs = H.make_reference("laplace", idx + 1)
    fn = refs.eigenfunctions[idx]
    lam_ref = refs.lambdas[idx]
    with hier(mlg, levels=3, nev=4) as hy:
        rh = oracle_ref.RefHierarchy(domain=SQUARE, H=0.25, delta=0.25, m=4, n_levels=3, nev=4)
        hy.extend_to(3)
        rh.extend_to(3)
        rng = np.random.default_rng(11)
        for k in (1, 2, 3):
            lam, co = rh.coarse_eigensolve(k, 4) if k < 3 else (None, None)
            x, y = dof_xy(hy, k)
            cands = [fn.value(x, y) * (1 + 1e-3 * rng.standard_normal(x.size))]
            if co is not None:
                cands.append(hy.expand_interior(k, co[idx]))
            for c in cands:
                g = H.compute_errors(hy, k, c, 1.01 * lam_ref, lam_ref, fn)
                r = oracle_ref.compute_errors(rh, k, c, 1.01 * lam_ref, lam_ref, idx)
                assert g.eig_err == r[0]
                assert abs(g.l2_err - r[1]) <= 1e-6 * r[1] + 1e-12, (k, g, r)
                assert abs(g.h1_err - r[2]) <= 1e-9 * r[2], (k, g, r)


def test_multilevel_with_refs_matches_reference_report(mlg, H, oracle_ref, tmp_path):
    """run_experiment on test_harness.cpp's config: every CSV row agrees with the
    reference's (lambda 1e-10, errors / orders to the parity tolerance)."""
    kw = dict(domain=SQUARE, H=0.5, delta=0.5, m=1, n_levels=3, nev=2)
    ref_csv = tmp_path / "ref.csv"
    oracle_ref.run_experiment(ref_csv, **kw)
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*SQUARE), H=0.5, delta=0.5, m=1, n_levels=3,
                        nev=2)
    ours = tmp_path / "ours.csv"
    rep = H.run_experiment(cfg, str(ours))
    assert len(rep.rows) == 6
    a = ours.read_text().splitlines()
    b = ref_csv.read_text().splitlines()
    assert a[0] == b[0] == "level,h,dofs,eig_index,lambda,eig_err,h1_err,order,local_s,iface_s,aug_s"
    for la, lb in zip(a[1:], b[1:]):
        fa, fb = la.split(","), lb.split(",")
        assert fa[0:4] == fb[0:4]  # level, h (bitwise text), dofs, index
        assert abs(float(fa[4]) - float(fb[4])) <= 1e-10 * float(fb[4])
        assert abs(float(fa[5]) - float(fb[5])) <= 1e-10 * float(fb[4])
        assert (fa[6] == "") == (fb[6] == "") and (fa[7] == "") == (fb[7] == "")
        if fb[6]:
            assert abs(float(fa[6]) - float(fb[6])) <= 1e-8 * float(fb[6])
        if fb[7]:
            assert abs(float(fa[7]) - float(fb[7])) <= 1e-6
        assert fa[8:] == ["0", "0", "0"] == fb[8:]
    # byte-identical on a repeated run (test_harness.cpp:123-127) and the table
    again = tmp_path / "again.csv"
    H.run_experiment(cfg, str(again))
    assert again.read_bytes() == ours.read_bytes()
    assert "eigenvalue 2:" in H.print_table(str(ours))
    with pytest.raises(mlg.IoError):
        H.run_experiment(cfg, "/nonexistent/dir/report.csv")


def test_single_level_report_has_no_orders(mlg, H, tmp_path):
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*SQUARE), H=0.5, delta=0.5, m=1, n_levels=1,
                        nev=2)
    rep = H.run_experiment(cfg, str(tmp_path / "s.csv"))
    assert all(r.order is None for r in rep.rows) and len(rep.rows) == 2


def test_unit_square_errors_converge(mlg, H):
    """The generalised reference table on the unit square (the BASELINE domain):
    second-order eigenvalue error, first-order H1 error of the correction."""
    cfg = mlg.RunConfig(domain=mlg.DomainRect(0.0, 1.0, 0.0, 1.0), H=1 / 8, delta=1 / 8, m=4,
                        n_levels=4, nev=1)
    refs = H.make_reference("laplace", 1, cfg.domain)
    with mlg.Hierarchy(cfg) as hy:
        res = H.multilevel_correction(hy, refs)
    ee = [t.eig_errors[0] for t in res.levels]
    h1 = [t.h1_errors[0] for t in res.levels]
    orders = H.estimate_orders(ee, 2.0)
    assert all(1.8 < o < 2.2 for o in orders[1:]), (ee, orders)
    assert all(0.85 < o < 1.15 for o in H.estimate_orders(h1, 2.0)[1:]), h1
    assert abs(abs(res.levels[-1].lambdas[0] - 2 * math.pi ** 2) - ee[-1]) <= 1e-13


def test_export_vtk_matches_reference(mlg, H, oracle_ref, tmp_path):
    kw = dict(domain=SQUARE, H=0.5, delta=0.5, m=1, n_levels=2, nev=2)
    oracle_ref.export_vtk(tmp_path / "ref", **kw)
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*SQUARE), H=0.5, delta=0.5, m=1, n_levels=2,
                        nev=2)
    H.export_vtk(cfg, str(tmp_path / "ours" / "sub"))
    a = (tmp_path / "ours" / "sub" / "eigenfunctions.vtk").read_text().splitlines()
    b = (tmp_path / "ref" / "eigenfunctions.vtk").read_text().splitlines()
    assert len(a) == len(b)
    assert "POINTS 289 double" in a and "POINT_DATA 289" in a  # test_harness.cpp:177-187
    first = a.index("POINT_DATA 289")
    assert a[:first + 1] == b[:first + 1]  # mesh text bitwise
    blocks_a, blocks_b = [], []
    for lines, blocks in ((a, blocks_a), (b, blocks_b)):
        i = first + 1
        while i < len(lines):
            assert lines[i].startswith("SCALARS eig_") and lines[i + 1] == "LOOKUP_TABLE default"
            blocks.append(np.array([float(v) for v in lines[i + 2:i + 2 + 289]]))
            i += 2 + 289
    assert len(blocks_a) == 2
    # eig_1 is simple: values agree; eig_2 belongs to the lambda_2 ~ lambda_3 pair of
    # the square, so only its norm is compared (the parity tests compare subspaces)
    u, v = blocks_a[0], blocks_b[0]
    assert np.max(np.abs(u - v)) <= 1e-8 * np.max(np.abs(v))
    assert abs(blocks_a[1] @ blocks_a[1] - blocks_b[1] @ blocks_b[1]) <= 1e-6 * (
        blocks_b[1] @ blocks_b[1])


def test_variable_example_reports_eigenvalue_errors_only(mlg, H, tmp_path):
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*SQUARE), H=0.5, delta=0.5, m=1, n_levels=3,
                        nev=2, example="variable")
    rep = H.run_experiment(cfg, str(tmp_path / "v.csv"))
    assert all(r.h1_err is None for r in rep.rows)
    table = [17.982932, 33.384973]
    for r in rep.rows:
        assert abs(r.eig_err - abs(r.lam - table[r.eig_index - 1])) <= 1e-12 * r.lam

"""CUDA correction step vs the compiled reference on the same inputs
(reference tests it mirrors: tests/test_corrector.cpp, test_sparse.cpp)."""
import numpy as np
import pytest

from _parity import compare_pairs

pytestmark = pytest.mark.gpu

SMALL = dict(domain=(-1.0, 1.0, -1.0, 1.0), H=0.25, delta=0.25, m=4)  # test_corrector.cpp:15-25
WHOLE = dict(domain=(-1.0, 1.0, -1.0, 1.0), H=0.5, delta=0.5, m=1)   # test_corrector.cpp:27-37
UNIT8 = dict(domain=(0.0, 1.0, 0.0, 1.0), H=1 / 8, delta=1 / 8, m=4)  # config 1 substitute (a)
UNIT16 = dict(domain=(0.0, 1.0, 0.0, 1.0), H=1 / 16, delta=1 / 16, m=16)  # config 1 subst. (b)


def pair(mlg, oracle_ref, spec, levels, nev, tol=1e-10):
    d = spec["domain"]
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*d), H=spec["H"], delta=spec["delta"],
                        m=spec["m"], n_levels=levels, nev=nev, cg_tol=tol)
    hy = mlg.Hierarchy(cfg)
    rh = oracle_ref.RefHierarchy(domain=d, H=spec["H"], delta=spec["delta"], m=spec["m"],
                                 n_levels=levels, nev=nev, cg_tol=tol)
    return hy, rh


def mass_ops(hy, rh, level):
    return (lambda f: rh.apply(level, "mass", f)), (lambda c: hy.expand_interior(level, c))


def test_coarse_eigensolve_matches(mlg, oracle_ref):
    hy, rh = pair(mlg, oracle_ref, SMALL, 2, 3)
    pairs = mlg.coarse_eigensolve(hy, 1, 3)
    lam_r, co_r = rh.coarse_eigensolve(1, 3)
    am, ex = mass_ops(hy, rh, 1)
    compare_pairs([p.lam for p in pairs], [p.coeffs for p in pairs], lam_r, co_r, am, ex)


def test_local_solve_matches_reference(mlg, oracle_ref):
    hy, rh = pair(mlg, oracle_ref, SMALL, 2, 1)
    hy.extend_to(2)
    rh.extend_to(2)
    lam, co = rh.coarse_eigensolve(1, 1)
    u = rh.prolong(hy.expand_interior(1, co[0]), 1, 2)
    for j in range(4):
        e_g, rep = mlg.local_bvp_solve(hy, 2, j, lam[0], u, 1e-12)
        e_r, it_r, fr_r = rh.local_bvp_solve(2, j, lam[0], u, 1e-12)
        assert rep.converged
        assert np.max(np.abs(e_g - e_r)) <= 1e-10 * max(1.0, np.max(np.abs(e_r)))
        assert np.array_equal(e_g == 0.0, e_r == 0.0)  # support = interior of Omega_j
        assert abs(rep.iterations - it_r) <= 2


def test_local_solve_failure_names_subdomain(mlg, oracle_ref):
    hy, rh = pair(mlg, oracle_ref, SMALL, 2, 1)
    hy.extend_to(2)
    lam, co = rh.coarse_eigensolve(1, 1)
    rh.extend_to(2)
    u = rh.prolong(hy.expand_interior(1, co[0]), 1, 2)
    with pytest.raises(mlg.SolverError, match="subdomain 2"):  # test_corrector.cpp:129-139
        mlg.local_bvp_solve(hy, 2, 1, lam[0], u, 1e-30)


def test_interface_solve_matches_reference(mlg, oracle_ref):
    hy, rh = pair(mlg, oracle_ref, SMALL, 2, 1)
    rh.extend_to(2)
    hy.extend_to(2)
    lam, co = rh.coarse_eigensolve(1, 1)
    u = rh.prolong(hy.expand_interior(1, co[0]), 1, 2)
    corr = np.stack([rh.local_bvp_solve(2, j, lam[0], u, 1e-12)[0] for j in range(4)])
    g_g, rep = mlg.interface_solve(hy, 2, lam[0], u, corr, 1e-12)
    g_r, it_r, _ = rh.interface_solve(2, lam[0], u, corr, 1e-12)
    assert rep.converged
    assert np.max(np.abs(g_g - g_r)) <= 1e-10 * np.max(np.abs(g_r))
    # glue is bitwise u + e_j on the closed G_j (test_corrector.cpp:141-153)
    for j in range(4):
        d = hy.region_dofs(2, "inner", j, False)
        assert np.array_equal(g_g[d], u[d] + corr[j][d])


def test_whole_domain_glue_is_identity(mlg, oracle_ref):
    hy, rh = pair(mlg, oracle_ref, WHOLE, 2, 1)
    rh.extend_to(2)
    hy.extend_to(2)
    lam, co = rh.coarse_eigensolve(1, 1)
    u = rh.prolong(hy.expand_interior(1, co[0]), 1, 2)
    e, _ = mlg.local_bvp_solve(hy, 2, 0, lam[0], u, 1e-10)
    g, rep = mlg.interface_solve(hy, 2, lam[0], u, e[None, :], 1e-10)
    assert len(hy.region_dofs(2, "strip", 0, True)) == 0
    d = hy.space(2).interior_dofs
    assert np.array_equal(g[d], (u + e)[d])


def test_augmented_matches_reference(mlg, oracle_ref):
    hy, rh = pair(mlg, oracle_ref, SMALL, 2, 3)
    rh.extend_to(2)
    hy.extend_to(2)
    lam, co = rh.coarse_eigensolve(1, 3)
    glued = []
    for i in range(3):
        u = rh.prolong(hy.expand_interior(1, co[i]), 1, 2)
        corr = np.stack([rh.local_bvp_solve(2, j, lam[i], u, 1e-10)[0] for j in range(4)])
        glued.append(rh.interface_solve(2, lam[i], u, corr, 1e-10)[0])
    glued = np.stack(glued)
    pairs = mlg.augmented_eigensolve(hy, 2, glued, 3)
    lam_r, co_r = rh.augmented_eigensolve(2, glued, 3)
    am, ex = mass_ops(hy, rh, 2)
    compare_pairs([p.lam for p in pairs], [p.coeffs for p in pairs], lam_r, co_r, am, ex)


@pytest.mark.parametrize("spec,levels,nev", [(SMALL, 3, 3), (UNIT8, 4, 1), (UNIT16, 3, 1),
                                             (WHOLE, 3, 3), (UNIT8, 3, 4)])
def test_multilevel_matches_reference(mlg, oracle_ref, spec, levels, nev):
    hy, rh = pair(mlg, oracle_ref, spec, levels, nev)
    lam_g, pairs, matched, times = mlg.multilevel_correction(hy)
    lam_r, co_r, matched_r, _ = rh.multilevel(levels, nev)
    am, ex = mass_ops(hy, rh, levels)
    for k in range(levels):
        assert np.max(np.abs(lam_g[k] - lam_r[k]) / np.abs(lam_r[k])) <= 1e-10, (k, lam_g, lam_r)
    compare_pairs(lam_g[-1], [p.coeffs for p in pairs], lam_r[-1], co_r, am, ex)
    assert list(matched) == list(matched_r)


def test_step_matches_reference_same_input(mlg, oracle_ref):
    hy, rh = pair(mlg, oracle_ref, UNIT8, 4, 4)
    _, rh3 = pair(mlg, oracle_ref, UNIT8, 3, 4)
    lam_r, co_r, _, _ = rh3.multilevel(3, 4)
    state = mlg.CorrectionState(3, [mlg.EigenPair(lam_r[-1][i], co_r[i], 3) for i in range(4)])
    out, t = mlg.one_correction_step(hy, state, 4)
    lo, co, matched, _ = rh.correction_step(3, 4, lam_r[-1], co_r)
    am, ex = mass_ops(hy, rh, 4)
    compare_pairs([p.lam for p in out.pairs], [p.coeffs for p in out.pairs], lo, co, am, ex)
    assert out.matched_previous == matched
    assert t.local_iterations_max > 0 and t.strip_iterations_max > 0


def test_step_idempotent_and_bounds(mlg, oracle_ref):
    # test_corrector.cpp:259-272 and 274-289
    hy, rh = pair(mlg, oracle_ref, SMALL, 2, 3)
    exact = mlg.coarse_eigensolve(hy, 2, 3)
    out, _ = mlg.one_correction_step(hy, mlg.CorrectionState(2, exact), 2)
    for i in range(3):
        assert abs(out.pairs[i].lam - exact[i].lam) <= 1e-9 * abs(exact[i].lam)
    start = mlg.coarse_eigensolve(hy, 1, 3)
    out, _ = mlg.one_correction_step(hy, mlg.CorrectionState(1, start), 2)
    ex = sorted(np.pi ** 2 / 4 * (a * a + b * b) for a in range(1, 13) for b in range(1, 13))[:3]
    assert out.matched_previous
    for i in range(3):
        if i:
            assert out.pairs[i].lam >= out.pairs[i - 1].lam
        assert out.pairs[i].lam > ex[i]


def test_step_is_deterministic(mlg, oracle_ref):
    hy, rh = pair(mlg, oracle_ref, UNIT8, 3, 4)
    start = mlg.coarse_eigensolve(hy, 1, 4)
    s2, _ = mlg.one_correction_step(hy, mlg.CorrectionState(1, start), 2)
    a, _ = mlg.one_correction_step(hy, s2, 3)
    b, _ = mlg.one_correction_step(hy, s2, 3)
    for pa, pb in zip(a.pairs, b.pairs):
        assert pa.lam == pb.lam
        assert np.array_equal(pa.coeffs.view(np.uint64), pb.coeffs.view(np.uint64))


def test_uniform_stencil_fast_path_matches_general_path(mlg, monkeypatch):
    """The constant-coefficient CG path (stencil from kernel parameters, paired
    FMA row products) and the general per-row path (the reference's exact
    term order) agree to rounding level: same iteration counts, eigenvalues to
    1e-12, eigenvectors to 1e-9."""
    def run():
        cfg = mlg.RunConfig(domain=mlg.DomainRect(0.0, 1.0, 0.0, 1.0), H=1 / 8, delta=1 / 8, m=4,
                            n_levels=4, nev=4)
        with mlg.Hierarchy(cfg) as hy:
            lam, pairs, matched, times = mlg.multilevel_correction(hy)
        return lam, pairs
    monkeypatch.setenv("MLG_GENERAL_STENCIL", "1")
    lam_g, p_g = run()
    monkeypatch.delenv("MLG_GENERAL_STENCIL")
    lam_u, p_u = run()
    assert np.max(np.abs(lam_g - lam_u) / lam_g) <= 1e-12
    for i in (0, 3):  # isolated eigenvalues (lambda_2 ~ lambda_3 is a cluster)
        a, b = p_g[i].coeffs, p_u[i].coeffs
        s = 1.0 if a @ b >= 0 else -1.0
        assert np.max(np.abs(a - s * b)) <= 1e-9 * np.max(np.abs(a))


def test_config_errors(mlg):
    bad = [dict(m=3), dict(delta=1.0), dict(H=0.3), dict(nev=0), dict(degree=3),
           dict(example="helmholtz"), dict(workers=0)]
    for b in bad:
        cfg = mlg.RunConfig(**{**dict(H=0.25, delta=0.25, m=4, nev=1), **b})
        with pytest.raises(mlg.ConfigError):
            mlg.Hierarchy(cfg)
    hy = mlg.Hierarchy(mlg.RunConfig(H=0.25, delta=0.1, m=4, nev=1))  # delta rounded up
    assert hy.partition()["overlap_cells"] == 1
    with pytest.raises(mlg.ConfigError, match="next level"):
        st = mlg.CorrectionState(1, mlg.coarse_eigensolve(hy, 1, 1))
        mlg.one_correction_step(hy, st, 3)


@pytest.mark.parametrize("case", ["candidate", "in_coarse_space", "unit8"])
def test_augmented_single_candidate_arrowhead(mlg, oracle_ref, case):
    """nev = 1: the device arrowhead/secular solve of the augmented pencil vs the
    reference's dense generalized solve (corrector.cpp:256-334), including the
    dependence drop when the candidate lies in V_H (corrector.cpp:285-292)."""
    spec = UNIT8 if case == "unit8" else SMALL
    L = 3
    hy, rh = pair(mlg, oracle_ref, spec, L, 1)
    rh.extend_to(L)
    hy.extend_to(L)
    if case == "in_coarse_space":
        lam0, co0 = rh.coarse_eigensolve(0, 1)
        glued = rh.prolong(hy.expand_interior(0, co0[0]), 0, L)
    else:
        lam, co = rh.coarse_eigensolve(L - 1, 1)
        u = rh.prolong(hy.expand_interior(L - 1, co[0]), L - 1, L)
        m = spec["m"]
        corr = np.stack([rh.local_bvp_solve(L, j, lam[0], u, 1e-10)[0] for j in range(m)])
        glued = rh.interface_solve(L, lam[0], u, corr, 1e-10)[0]
    pairs = mlg.augmented_eigensolve(hy, L, glued[None, :], 1)
    lam_r, co_r = rh.augmented_eigensolve(L, glued[None, :], 1)
    am, ex = mass_ops(hy, rh, L)
    compare_pairs([p.lam for p in pairs], [p.coeffs for p in pairs], lam_r, co_r, am, ex)
    if case == "in_coarse_space":
        assert abs(pairs[0].lam - lam0[0]) <= 1e-10 * lam0[0]

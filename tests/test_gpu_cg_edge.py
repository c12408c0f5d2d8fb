"""Edge cases of the reference's cg_solve (sparse.cpp:199-258) on the CUDA path,
through mlg_local_cg_solve (the batched device CG with cg_solve's contract):

* zero right-hand side returns after 0 iterations, converged, x = 0
  (sparse.cpp:208-212; tests/test_sparse.cpp:124-130);
* maxit reached: non-convergence is REPORTED, not thrown, with the true
  relative residual (sparse.cpp:255-257; tests/test_sparse.cpp:108-115) --
  compared with the reference's own cg_solve on the same extracted system;
* the default maxit reproduces local_bvp_solve.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

UNIT8 = dict(domain=(0.0, 1.0, 0.0, 1.0), H=1 / 8, delta=1 / 8, m=4)


def _setup(mlg, oracle_ref, level=3):
    d = UNIT8["domain"]
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*d), H=UNIT8["H"], delta=UNIT8["delta"],
                        m=UNIT8["m"], n_levels=level, nev=1)
    hy = mlg.Hierarchy(cfg)
    rh = oracle_ref.RefHierarchy(domain=d, H=UNIT8["H"], delta=UNIT8["delta"], m=UNIT8["m"],
                                 n_levels=level, nev=1)
    hy.extend_to(level)
    rh.extend_to(level)
    lam, co = rh.coarse_eigensolve(1, 1)
    u = rh.prolong(hy.expand_interior(1, co[0]), 1, level)
    return hy, rh, lam[0], u


def _ref_system(rh, level, j, lam, u):
    """A_jj = extract_submatrix(A, Omega_j dofs) and the local rhs, from the
    reference's own CSR and SpMV (corrector.cpp:198-214, sparse.cpp:156-174)."""
    dofs = rh.region_dofs(level, "overlap", j, zero_trace=True)
    rp, cols, vals = rh.csr(level, "stiffness")
    loc = -np.ones(len(rp) - 1, np.int64)
    loc[dofs] = np.arange(len(dofs))
    r_rp, r_cols, r_vals = [0], [], []
    for d in dofs:
        for k in range(rp[d], rp[d + 1]):
            if loc[cols[k]] >= 0:
                r_cols.append(loc[cols[k]])
                r_vals.append(vals[k])
        r_rp.append(len(r_cols))
    load = lam * rh.apply(level, "mass", u) - rh.apply(level, "stiffness", u)
    return (np.array(r_rp, np.int32), np.array(r_cols, np.int32), np.array(r_vals),
            load[dofs], dofs)


def test_zero_rhs_returns_after_zero_iterations(mlg, oracle_ref):
    hy, rh, lam, u = _setup(mlg, oracle_ref)
    z = np.zeros_like(u)
    for j in range(UNIT8["m"]):
        e, rep = mlg.local_cg_solve(hy, 3, j, lam, z, 1e-10)
        assert rep.iterations == 0 and rep.converged and rep.final_residual == 0.0
        assert not np.any(e)
    rp, cols, vals, _, dofs = _ref_system(rh, 3, 0, lam, u)
    x, it, fr, cv = oracle_ref.cg_solve_csr(rp, cols, vals, np.zeros(len(dofs)), 1e-10)
    assert it == 0 and cv and not np.any(x)


@pytest.mark.parametrize("maxit", [1, 5, 17])
def test_maxit_reports_nonconvergence(mlg, oracle_ref, maxit):
    hy, rh, lam, u = _setup(mlg, oracle_ref)
    j = 1
    e, rep = mlg.local_cg_solve(hy, 3, j, lam, u, 1e-10, maxit=maxit)
    rp, cols, vals, rhs, dofs = _ref_system(rh, 3, j, lam, u)
    x, it, fr, cv = oracle_ref.cg_solve_csr(rp, cols, vals, rhs, 1e-10, maxit)
    assert (rep.iterations, rep.converged) == (it, cv) == (maxit, False)
    assert rep.final_residual > 1e-10
    assert rep.final_residual == pytest.approx(fr, rel=1e-9)
    assert np.max(np.abs(e[dofs] - x)) <= 1e-10 * np.max(np.abs(x))


def test_default_maxit_matches_local_bvp_solve(mlg, oracle_ref):
    hy, rh, lam, u = _setup(mlg, oracle_ref)
    for j in (0, 3):
        e1, r1 = mlg.local_cg_solve(hy, 3, j, lam, u, 1e-10)
        e2, r2 = mlg.local_bvp_solve(hy, 3, j, lam, u, 1e-10)
        assert r1.converged and r1.iterations == r2.iterations
        assert np.array_equal(e1, e2)

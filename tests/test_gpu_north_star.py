"""North-star parity: the full multilevel correction of BASELINE config 5
(reference-valid substitute: unit square, 32x32 coarse, 7 levels = 4096^2
cells, m=64, delta=1/32, nev=4) against the reference's own run of the same
configuration (tests/golden/golden_l7.json, produced by
tests/golden/make_golden_l7.py from oracle/_ref: corrector.cpp:414-462).

* eigenvalues at every level: relative error <= 1e-10;
* eigenfunctions at level 7: the reference vectors are 16.8M doubles each, so
  the committed pins are a 32-row seeded random-projection sketch S (a
  Johnson-Lindenstrauss estimate of the full-vector relative difference, see
  tests/_parity.py) and point values on the 63x63 sub-lattice.  Isolated
  eigenvalues: ||S(u - s v)|| / ||S v|| <= 1e-8 (sign s from the sketch);
  the lambda_2 ~ lambda_3 cluster (relative gap 5.6e-7 < 1e-6) is
  compared as a subspace: the 2x2 least-squares fit S U ~ Q S V has relative
  residual <= 1e-8 (and the same on the sampled point values);
* the reference's local-solve iteration counts at level 7 (8 tasks) and its
  strip-solve count for eigenvector 0 (2321) are met within +-2 by the device CG
  started from the reference's level-6 state.

Config 2 and the config-5 shape at 1024^2 are compared on FULL vectors in the
mass norm against a live reference run (compare_pairs, tests/_parity.py).
"""
import json
import os
from pathlib import Path

import numpy as np
import pytest

from _parity import SKETCH_K, SKETCH_SEED, compare_pairs, sketch

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
GOLD = ROOT / "tests" / "golden" / "golden_l7.json"
UNIT = (0.0, 1.0, 0.0, 1.0)


def _golden():
    if not GOLD.exists():
        pytest.skip("golden_l7.json not generated (tests/golden/make_golden_l7.py)")
    return json.loads(GOLD.read_text())


@pytest.fixture(scope="module")
def c5_run(mlg):
    g = _golden()
    c = g["config"]
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*c["domain"]), H=c["H"], delta=c["delta"],
                        m=c["m"], n_levels=c["n_levels"], nev=c["nev"])
    with mlg.Hierarchy(cfg) as hy:
        lam, pairs, matched, times = mlg.multilevel_correction(hy)
    return g, lam, np.stack([p.coeffs for p in pairs]), matched, times


def test_c5_eigenvalues_every_level(c5_run):
    g, lam, _, matched, _ = c5_run
    ref = np.array(g["lambdas"])
    err = np.abs(lam - ref) / ref
    assert np.max(err) <= 1e-10, err
    assert list(map(bool, matched)) == list(map(bool, g["matched"]))


def _fit_residual(P, R):
    """min_Q ||P - Q R||_F / ||P||_F for P, R of shape (k, n)."""
    Q, *_ = np.linalg.lstsq(R.T, P.T, rcond=None)
    return np.linalg.norm(P - (R.T @ Q).T) / np.linalg.norm(P)


def test_c5_eigenfunctions_sketch_and_samples(c5_run):
    g, lam, vecs, _, _ = c5_run
    sk = g["sketch"]
    assert (sk["k"], sk["seed"]) == (SKETCH_K, SKETCH_SEED)
    P_ref = np.array(sk["projections"])
    P, rn = sketch(vecs)
    assert np.allclose(rn, sk["row_norms"], rtol=1e-12)  # same random rows
    n = 4095
    stride = g["sample_stride"]
    idx = np.arange(stride - 1, n, stride)
    S_ref = np.load(ROOT / "tests" / "golden" / g["samples"])
    S = vecs.reshape(vecs.shape[0], n, n)[:, idx][:, :, idx].reshape(vecs.shape[0], -1)
    S_ref = S_ref.reshape(S_ref.shape[0], -1)
    lam_ref = np.array(g["lambdas"][-1])
    iso, clus = [0, 3], [1, 2]
    assert abs(lam_ref[1] - lam_ref[2]) / lam_ref[1] < 1e-6  # the cluster rule applies
    worst = {}
    for i in iso:
        s = 1.0 if P[i] @ P_ref[i] >= 0 else -1.0
        worst[f"sketch{i}"] = np.linalg.norm(P[i] - s * P_ref[i]) / np.linalg.norm(P_ref[i])
        worst[f"samples{i}"] = np.max(np.abs(S[i] - s * S_ref[i])) / np.max(np.abs(S_ref[i]))
        assert float(vecs[i] @ vecs[i]) == pytest.approx(g["norm2"][i], rel=1e-8)
    worst["sketch_cluster"] = _fit_residual(P[clus], P_ref[clus])
    worst["samples_cluster"] = _fit_residual(S[clus], S_ref[clus])
    assert max(worst.values()) <= 1e-8, worst
    # the sketch does resolve differences at this level: a 1e-7 relative
    # perturbation of one vector is visible
    rng = np.random.default_rng(7)
    d = rng.standard_normal(vecs.shape[1])
    pert = vecs[0] + 1e-7 * np.linalg.norm(vecs[0]) / np.linalg.norm(d) * d
    Pp, _ = sketch(pert[None, :])
    est = np.linalg.norm(Pp[0] - P[0]) / np.linalg.norm(P[0])
    assert 0.5e-7 < est < 2e-7, est


def test_c5_local_iterations_match_reference(mlg):
    """Level-7 local solves started from the level-6 eigenvectors (equal to the
    reference's to 1e-10, test above): iteration counts within +-2 of the
    reference's own local_bvp_solve counts from the same state (make_golden_l7.py)."""
    g = _golden()
    its = g.get("local_iterations_L7") or {}
    if not its:
        pytest.skip("no reference iteration counts recorded")
    c = g["config"]
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*c["domain"]), H=c["H"], delta=c["delta"],
                        m=c["m"], n_levels=c["n_levels"], nev=c["nev"])
    with mlg.Hierarchy(cfg) as hy:
        lam, pairs, _, _ = mlg.multilevel_correction(hy, last_level=6)
        hy.extend_to(7)
        for key, it_ref in its.items():
            i, j = map(int, key.split("_"))
            u = hy.prolong(hy.expand_interior(6, pairs[i].coeffs), 6, 7)
            _, rep = mlg.local_bvp_solve(hy, 7, j, g["lambdas"][5][i], u, 1e-10)
            assert rep.converged
            assert abs(rep.iterations - it_ref) <= 2, (key, rep.iterations, it_ref)


def test_c5_strip_iterations_match_reference(mlg):
    """Level-7 strip solve of eigenvector 0 (interface_solve, corrector.cpp:216-254)
    from the level-6 state: the reference's own cg_solve on the strip system took
    2321 iterations (make_golden_l7.py strip()); the device CG is within +-2.
    Needs the 64 full-length corrections on the host (8.6 GB), as the reference's
    signature does."""
    g = _golden()
    ref_its = g.get("reference_strip_iterations_L7") or []
    if not ref_its:
        pytest.skip("no reference strip iteration count recorded")
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError):
        avail = 0
    if avail < 40 * 2**30:
        pytest.skip("needs ~20 GB of free host memory")
    c = g["config"]
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*c["domain"]), H=c["H"], delta=c["delta"],
                        m=c["m"], n_levels=c["n_levels"], nev=c["nev"])
    with mlg.Hierarchy(cfg) as hy:
        lam, pairs, _, _ = mlg.multilevel_correction(hy, last_level=6)
        hy.extend_to(7)
        lam0 = g["lambdas"][5][0]
        u = hy.prolong(hy.expand_interior(6, pairs[0].coeffs), 6, 7)
        corr = np.empty((c["m"], u.size))
        for j in range(c["m"]):
            corr[j], rep = mlg.local_bvp_solve(hy, 7, j, lam0, u, 1e-10)
            assert rep.converged
        _, rep = mlg.interface_solve(hy, 7, lam0, u, corr, 1e-10)
        assert rep.converged
        assert abs(rep.iterations - ref_its[0]) <= 2, (rep.iterations, ref_its)


@pytest.mark.parametrize("name,H,m,L,nev", [("c2sub_16_L6_m16_nev1", 1 / 16, 16, 6, 1),
                                            ("c5shape_32_L5_m64_nev4", 1 / 32, 64, 5, 4)])
def test_full_vector_parity_live_reference(mlg, oracle_ref, name, H, m, L, nev):
    """Full eigenvectors in the mass norm (and the cluster as a subspace) against
    a live reference run on this host (config 2 substitute at 1024^2; the
    config-5 partition at 1024^2 with nev=4).  There lambda_2/lambda_3 are
    2.3e-6 apart (relative): an individual vector of such a pair is determined
    only to ~(Gram-matrix rounding)/gap ~ 1e-7, so pairs closer than 1e-4 are
    compared as subspaces (SURVEY §8(d)'s 1e-6 rule applies at level 7)."""
    workers = os.cpu_count() or 1
    rh = oracle_ref.RefHierarchy(domain=UNIT, H=H, delta=H, m=m, n_levels=L, nev=nev,
                                 workers=workers)
    lam_r, co_r, matched_r, _ = rh.multilevel(L, nev)
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*UNIT), H=H, delta=H, m=m, n_levels=L, nev=nev)
    with mlg.Hierarchy(cfg) as hy:
        lam, pairs, matched, _ = mlg.multilevel_correction(hy)
        lerr, verr = compare_pairs(lam[-1], [p.coeffs for p in pairs], lam_r[-1], co_r,
                                   lambda f: rh.apply(L, "mass", f),
                                   lambda c: hy.expand_interior(L, c), gap=1e-4)
    assert np.max(np.abs(lam - lam_r) / lam_r) <= 1e-10
    assert list(matched) == list(matched_r)
    rh.close()

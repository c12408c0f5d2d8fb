"""BASELINE config 4's problem on the B200 path: -div(a grad u) + c u = lambda u
with a = 1 + 0.5 sin(2 pi k1 x) sin(2 pi k2 y), c = 1 + x^2 + y^2 at triangle
centroids, (k1, k2) drawn from the seed (example "reaction").  The reference has
no such field, so the checker is the numpy restatement (oracle/restate.py) and
the golden fixtures it generated (parity unpinned against the reference)."""
import json
from pathlib import Path

import numpy as np
import pytest

from _parity import compare_pairs

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())
UNIT = (0.0, 1.0, 0.0, 1.0)


def cfg_of(mlg, c):
    return mlg.RunConfig(domain=mlg.DomainRect(*c["domain"]), H=c["H"], delta=c["delta"],
                         m=c["m"], n_levels=c["n_levels"], nev=c["nev"], example="reaction",
                         seed=c["seed"])


@pytest.mark.parametrize("seed", [0, 3, 7])
def test_reaction_operators_match_restatement(mlg, seed):
    from oracle import restate as R
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*UNIT), H=1 / 8, delta=1 / 8, m=4, n_levels=3,
                        nev=1, example="reaction", seed=seed)
    rh = R.Hierarchy(domain=UNIT, H=1 / 8, delta=1 / 8, m=4, n_levels=3, nev=1,
                     example="reaction", seed=seed)
    rh.extend_to(3)
    with mlg.Hierarchy(cfg) as hy:
        hy.extend_to(3)
        for k in range(4):
            for form, csr in (("stiffness", rh.levels[k].A), ("mass", rh.levels[k].M)):
                rp, cols, vals = hy.csr(k, form)
                assert np.array_equal(rp, csr[0]) and np.array_equal(cols, csr[1])
                # sin() of CUDA and of numpy may differ in the last bit
                assert np.max(np.abs(vals - csr[2])) <= 4e-16 * np.max(np.abs(csr[2])), (k, form)


@pytest.mark.parametrize("name", ["unit8_L4_m4_nev2_seed0", "unit8_L3_m4_nev1_seed3"])
def test_reaction_multilevel_matches_golden(mlg, name):
    from oracle import restate as R
    g = GOLDEN["reaction"][name]
    c = g["config"]
    with mlg.Hierarchy(cfg_of(mlg, c)) as hy:
        lam, pairs, matched, times = mlg.multilevel_correction(hy)
        ref = np.array(g["lambdas"])
        assert np.max(np.abs(lam - ref) / ref) <= 1e-10, (lam, ref)
        assert not any(t.spmv_uniform_stencil for t in times[1:])  # general stencil path
        rh = R.Hierarchy(domain=tuple(c["domain"]), H=c["H"], delta=c["delta"], m=c["m"],
                         n_levels=c["n_levels"], nev=c["nev"], example="reaction",
                         seed=c["seed"])
        lams_r, state = R.multilevel_correction(rh)
        L = c["n_levels"]
        compare_pairs(lam[-1], [p.coeffs for p in pairs], lams_r[-1], [v for _, v in state],
                      lambda f: hy.apply(L, "mass", f), lambda v: hy.expand_interior(L, v))


def test_reaction_has_no_reference_table(mlg):
    from paper_1401_4969_b200 import harness as H
    with pytest.raises(mlg.ConfigError, match='no reference data for example "reaction"'):
        H.make_reference("reaction", 1)
    cfg = H.parse_config_json(
        '{"domain": {"x_min": 0.0, "x_max": 1.0, "y_min": 0.0, "y_max": 1.0}, "H": 0.125, '
        '"delta": 0.125, "m": 4, "n_levels": 3, "degree": 1, "nev": 1, "example": "reaction", '
        '"cg_tol": 1e-10, "workers": 1, "deterministic": true, "seed": 3}')
    assert cfg.example == "reaction" and cfg.seed == 3
    with mlg.Hierarchy(cfg) as hy:
        lam, *_ = mlg.multilevel_correction(hy)
    g = GOLDEN["reaction"]["unit8_L3_m4_nev1_seed3"]["lambdas"]
    assert np.max(np.abs(lam - np.array(g)) / np.array(g)) <= 1e-10

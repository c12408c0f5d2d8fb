"""BASELINE config 3's L-shaped domain (-1,1)^2 minus [0,1] x [-1,0] on the B200
path (a B200 extension: the reference meshes rectangles only).  The checker is
the numpy restatement (oracle/restate.py: build_structured_mesh_hole,
build_space_lattice, build_partition_hole; the rest of the restatement is the
reference's algorithm on those inputs) and the golden fixtures it generated --
parity unpinned against the reference, bit-exact against the restatement for
mesh / space / CSR / regions, eigenpairs to the north-star tolerances."""
import json
from pathlib import Path

import numpy as np
import pytest

from _parity import compare_pairs

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())
SQUARE = (-1.0, 1.0, -1.0, 1.0)
HOLE = (0.0, 1.0, -1.0, 0.0)
HOLES = {"lower_right": HOLE, "upper_left": (-1.0, 0.0, 0.0, 1.0),
         "lower_left": (-1.0, 0.0, -1.0, 0.0), "upper_right": (0.0, 1.0, 0.0, 1.0)}


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64) if a.dtype == np.float64 else a


def pair(mlg, hole=HOLE, H=1 / 8, m=16, levels=3, nev=1):
    from oracle import restate as R
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*SQUARE), H=H, delta=H, m=m, n_levels=levels,
                        nev=nev, hole=mlg.DomainRect(*hole))
    rh = R.Hierarchy(domain=SQUARE, H=H, delta=H, m=m, n_levels=levels, nev=nev, hole=hole)
    return mlg.Hierarchy(cfg), rh


@pytest.mark.parametrize("corner", sorted(HOLES))
def test_lshape_mesh_space_csr_bitexact(mlg, corner):
    hy, rh = pair(mlg, HOLES[corner])
    hy.extend_to(3)
    rh.extend_to(3)
    for k in range(4):
        g, r = hy.mesh(k), rh.levels[k].mesh
        assert np.array_equal(g.triangles, r.triangles), (corner, k)
        assert np.array_equal(bits(g.vertices), bits(r.vertices)), (corner, k)
        assert np.array_equal(g.vertex_lattice, r.lattice), (corner, k)
        assert np.array_equal(g.boundary_edges, r.boundary_edges), (corner, k)
        if k:
            assert np.array_equal(g.parent, r.parent), (corner, k)
        assert g.h_max == r.h_max
        gs, rs = hy.space(k), rh.levels[k].space
        assert np.array_equal(gs.dof_lattice, rs.dof_lattice)
        assert np.array_equal(gs.interior_dofs, rs.interior_dofs), (corner, k)
        assert np.array_equal(gs.interior_index, rs.interior_index), (corner, k)
        assert np.array_equal(gs.connectivity, rs.connectivity), (corner, k)
        for form, csr in (("stiffness", rh.levels[k].A), ("mass", rh.levels[k].M)):
            rp, cols, vals = hy.csr(k, form)
            assert np.array_equal(rp, csr[0]) and np.array_equal(cols, csr[1]), (corner, k, form)
            assert np.array_equal(bits(vals), bits(csr[2])), (corner, k, form)


def test_lshape_golden_digests(mlg):
    from oracle.ref import fnv1a64 as f
    g = GOLDEN["lshape"]["H8_L3_m16_nev3"]
    hy, _ = pair(mlg)
    hy.extend_to(3)
    me = hy.mesh(3)
    assert f(me.triangles, me.vertices, me.parent, me.boundary_edges) == g["mesh"]
    rp, c, va = hy.csr(3, "stiffness")
    assert [f(rp), f(c), f(va), f(hy.csr(3, "mass")[2])] == g["csr"]
    assert f(hy.space(3).interior_dofs) == g["interior_dofs"]
    assert hy.partition()["m"] == g["n_sub"] == 12


def test_lshape_regions_and_transfer(mlg):
    from oracle import restate as R
    hy, rh = pair(mlg)
    hy.extend_to(3)
    rh.extend_to(3)
    p = hy.partition()
    assert p["m"] == rh.part.m
    assert [tuple(r) for r in p["inners"]] == rh.part.inners
    assert [tuple(r) for r in p["overlaps"]] == rh.part.overlaps
    for k in range(4):
        sp = rh.levels[k].space
        for kind in ("domain", "block", "overlap", "inner", "strip"):
            for j in ([0] if kind in ("domain", "strip") else range(p["m"])):
                for zt in (False, True):
                    assert np.array_equal(hy.region_dofs(k, kind, j, zt),
                                          R.restrict_space(sp, rh.part, kind, j, zt)), (k, kind, j)
    rng = np.random.default_rng(3)
    for a in range(3):
        x = rng.uniform(-1, 1, hy.level_info(a).ndofs)
        x[~np.isin(np.arange(x.size), rh.levels[a].space.connectivity)] = 0.0
        assert np.array_equal(bits(hy.prolong(x, a, a + 1)), bits(rh.prolong(x, a, a + 1)))
        y = rng.uniform(-1, 1, hy.level_info(a + 1).ndofs)
        y[~np.isin(np.arange(y.size), rh.levels[a + 1].space.connectivity)] = 0.0
        assert np.array_equal(bits(hy.restrict_transpose(y, a + 1, a)),
                              bits(rh.restrict_transpose(y, a + 1, a)))


@pytest.mark.parametrize("name", ["H8_L3_m16_nev3", "H8_L4_m16_nev1"])
def test_lshape_multilevel_matches_golden(mlg, name):
    from oracle import restate as R
    g = GOLDEN["lshape"][name]
    c = g["config"]
    hy, rh = pair(mlg, H=c["H"], m=c["m"], levels=c["n_levels"], nev=c["nev"])
    lam, pairs, matched, times = mlg.multilevel_correction(hy)
    ref = np.array(g["lambdas"])
    assert np.max(np.abs(lam - ref) / ref) <= 1e-10, (lam, ref)
    lams_r, state = R.multilevel_correction(rh)
    L = c["n_levels"]
    compare_pairs(lam[-1], [p.coeffs for p in pairs], lams_r[-1], [v for _, v in state],
                  lambda f: hy.apply(L, "mass", f), lambda v: hy.expand_interior(L, v))
    assert lam[-1][0] > 9.6397238440219  # min-max: above the exact L-shape eigenvalue


def test_lshape_experiment_report(mlg, tmp_path):
    from paper_1401_4969_b200 import harness as H
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*SQUARE), H=1 / 8, delta=1 / 8, m=16, n_levels=4,
                        nev=3, hole=mlg.DomainRect(*HOLE))
    refs = H.make_reference_for(cfg, 3)
    assert abs(refs.lambdas[0] - 9.6397238440219) < 1e-12 and sorted(refs.eigenfunctions) == [2]
    rep = H.run_experiment(cfg, str(tmp_path / "l.csv"))
    e1 = [r.eig_err for r in rep.rows if r.eig_index == 1]
    assert all(a > b for a, b in zip(e1, e1[1:]))  # converging to the corner eigenvalue
    h3 = [r.h1_err for r in rep.rows if r.eig_index == 3]
    assert all(v is not None for v in h3) and h3[-1] < h3[0]
    with pytest.raises(mlg.ConfigError, match="no reference data"):
        H.make_reference_for(mlg.RunConfig(domain=mlg.DomainRect(0.0, 1.0, 0.0, 1.0), H=1 / 8,
                                           hole=mlg.DomainRect(0.5, 1.0, 0.0, 0.5)), 1)

"""Parity at BASELINE sizes: structure digests at 1024^2 / 2048^2 / 4096^2
against the golden vectors from the compiled reference, eigenvalues per level
against the reference's multilevel runs (config 2 substitute at 1024^2, config 5
shape at 1024^2 and 2048^2), and size-independent properties of the full
config-5 (4096^2, nev=4) step where no reference run exists: M-orthonormality,
Rayleigh-quotient consistency, upper-bound monotonicity, determinism."""
import json
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())
UNIT = (0.0, 1.0, 0.0, 1.0)

pytestmark = pytest.mark.gpu


def fnv(*arrays):
    from oracle.ref import fnv1a64
    return fnv1a64(*arrays)


@pytest.mark.parametrize("key,n0,L,m", [("16_6", 16, 6, 16), ("16_7", 16, 7, 16),
                                        ("32_7", 32, 7, 64)])
def test_structure_digests_at_scale(mlg, key, n0, L, m):
    if key not in GOLDEN["digests"]:
        pytest.skip(f"golden digest {key} not generated")
    g = GOLDEN["digests"][key]
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*UNIT), H=1 / n0, delta=1 / n0, m=m, n_levels=L,
                        nev=1)
    with mlg.Hierarchy(cfg) as hy:
        hy.extend_to(L)
        info = hy.level_info(L)
        assert (info.num_vertices, info.num_triangles, info.num_boundary_edges) == (
            g["counts"]["nv"], g["counts"]["nt"], g["counts"]["nb"])
        assert info.nnz == g["counts"]["nnz_a"] and info.h_max == g["h_max"]
        me = hy.mesh(L)
        assert fnv(me.triangles, me.vertices, me.parent, me.boundary_edges) == g["mesh"]
        del me
        rp, cols, va = hy.csr(L, "stiffness")
        assert (fnv(rp), fnv(cols), fnv(va)) == (g["row_ptr"], g["cols"], g["values_A"])
        del rp, cols, va
        assert fnv(hy.csr(L, "mass")[2]) == g["values_M"]
        sp = hy.space(L)
        assert fnv(sp.connectivity) == g["connectivity"]
        assert fnv(sp.interior_dofs) == g["interior_dofs"]


def projections(vecs, seed=20261019, k=8):
    rng = np.random.default_rng(seed)
    R = rng.uniform(-1.0, 1.0, size=(k, vecs.shape[1]))
    return vecs @ R.T, np.linalg.norm(R, axis=1)


@pytest.mark.parametrize("name", ["c2sub_16_L6_m16_nev1", "c5shape_32_L5_m64_nev4",
                                  "c5shape_32_L6_m64_nev4"])
def test_multilevel_eigenvalues_match_reference_at_scale(mlg, name):
    if name not in GOLDEN["multilevel"]:
        pytest.skip(f"golden run {name} not generated")
    g = GOLDEN["multilevel"][name]
    c = g["config"]
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*c["domain"]), H=c["H"], delta=c["delta"],
                        m=c["m"], n_levels=c["n_levels"], nev=c["nev"])
    with mlg.Hierarchy(cfg) as hy:
        lam, pairs, matched, times = mlg.multilevel_correction(hy)
    ref = np.array(g["lambdas"])
    assert np.max(np.abs(lam - ref) / ref) <= 1e-10
    assert list(matched) == g["matched"]
    # kernel choice at BASELINE sizes (2 = k_cg_resident, cg.cu CgBatch::solve): the
    # last level's local solves run SM-resident, and so does config 2's strip solve
    assert int(times[-1].local_kernel) == 2, [int(t.local_kernel) for t in times]
    if name.startswith("c2sub"):
        assert int(times[-1].strip_kernel) == 2, [int(t.strip_kernel) for t in times]
    # eigenfunctions of isolated eigenvalues: seeded projections (size-independent pin)
    vecs = np.stack([p.coeffs for p in pairs])
    proj, rn = projections(vecs)
    pref = np.array(g["projections"])
    lam_last = ref[-1]
    for i in range(c["nev"]):
        gaps = [abs(lam_last[i] - lam_last[j]) / lam_last[i] for j in range(c["nev"]) if j != i]
        if gaps and min(gaps) < 1e-4:
            # lambda_2 ~ lambda_3 (relative gap 2e-6 at 1024^2, 6e-7 at 2048^2): the
            # individual vectors are ill-conditioned (SURVEY finding 9); the subspace
            # comparison at these sizes is test_gpu_solvers' compare_pairs.
            continue
        scale = np.sqrt(g["norm2"][i]) * rn
        assert np.max(np.abs(proj[i] - pref[i]) / scale) <= 1e-8


def test_config5_full_step_properties(mlg):
    """Config 5 substitute at 4096^2 (no reference run exists at this size)."""
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*UNIT), H=1 / 32, delta=1 / 32, m=64, n_levels=7,
                        nev=4)
    with mlg.Hierarchy(cfg) as hy:
        lam, pairs, matched, times = mlg.multilevel_correction(hy)
        L = 7
        # reference values at level 6 (2048^2) and the order of the levels
        if "c5shape_32_L6_m64_nev4" in GOLDEN["multilevel"]:
            ref6 = np.array(GOLDEN["multilevel"]["c5shape_32_L6_m64_nev4"]["lambdas"])
            assert np.max(np.abs(lam[:6] - ref6) / ref6) <= 1e-10
        exact = np.pi ** 2 * np.array([2.0, 5.0, 5.0, 8.0])
        assert np.all(lam[-1] > exact)                       # upper bounds
        assert np.all(lam[-1] < lam[-2])                     # monotone in h
        ratio = (lam[-2] - exact) / (lam[-1] - exact)        # O(h^2): ~4 per level
        assert np.all((ratio > 3.4) & (ratio < 4.6)), ratio
        assert all(matched)
        for i, p in enumerate(pairs):
            f = hy.expand_interior(L, p.coeffs)
            mf = hy.apply(L, "mass", f)
            af = hy.apply(L, "stiffness", f)
            q = f @ mf
            assert abs(q - 1.0) <= 1e-12                      # b-normalised
            assert abs((f @ af) / q - lam[-1][i]) <= 1e-9 * lam[-1][i]  # Ritz value
        for i in range(4):
            for j in range(i + 1, 4):                         # M-orthogonal Ritz vectors
                fi = hy.expand_interior(L, pairs[i].coeffs)
                fj = hy.expand_interior(L, pairs[j].coeffs)
                assert abs(fi @ hy.apply(L, "mass", fj)) <= 1e-10
        assert times[-1].local_iterations_max > 2000
    # bitwise determinism of the full 4096^2 step (same input twice)
    with mlg.Hierarchy(cfg) as hy:
        lam6, pairs6, _, _ = mlg.multilevel_correction(hy, last_level=6)
        st6 = mlg.CorrectionState(6, pairs6)
        a, _ = mlg.one_correction_step(hy, st6, 7)
        b, _ = mlg.one_correction_step(hy, st6, 7)
    for pa, pb, pc in zip(a.pairs, b.pairs, pairs):
        assert pa.lam == pb.lam
        assert np.array_equal(pa.coeffs.view(np.uint64), pb.coeffs.view(np.uint64))
        assert pa.lam == pc.lam  # the multilevel driver ran the same step

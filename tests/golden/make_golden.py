"""Generate the golden fixtures in tests/golden/ from the compiled reference
(oracle/_ref/libmleig_ref.so = /root/reference/proj/src built by oracle/Makefile).

    python tests/golden/make_golden.py            # small + medium fixtures
    python tests/golden/make_golden.py --big      # adds the 4096^2 mesh/CSR digests and
                                                  # the 2048^2 nev=4 run (tens of minutes)

Outputs: golden.json (digests, eigenvalues per level, CG iteration counts,
seeded projections of final eigenvectors) and unit8_L4_u1.npy (one small
eigenvector).  Digests are FNV-1a-64 over raw little-endian bytes
(SURVEY.md Appendix B).
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import ref  # noqa: E402

OUT = Path(__file__).resolve().parent
UNIT = (0.0, 1.0, 0.0, 1.0)
SQUARE = (-1.0, 1.0, -1.0, 1.0)
N_PROJ = 8


def projections(vecs, seed=20261019):
    """u . r_k for seeded uniform(-1,1) r_k (size-independent eigenvector pins)."""
    vecs = np.atleast_2d(vecs)
    rng = np.random.default_rng(seed)
    R = rng.uniform(-1.0, 1.0, size=(N_PROJ, vecs.shape[1]))
    return (vecs @ R.T).tolist()


def digests(n0, levels, m, delta):
    t = time.time()
    h = ref.RefHierarchy(domain=UNIT, H=1.0 / n0, delta=delta, m=m, n_levels=levels, nev=1)
    h.extend_to(levels)
    L = levels
    mesh = h.mesh(L)
    s = h.sizes(L)
    out = {
        "counts": {k: s[k] for k in ("nv", "nt", "nb", "ndofs", "n_int", "nnz_a")},
        "h_max": s["h_max"],
        "mesh": ref.fnv1a64(mesh["triangles"], mesh["vertices"], mesh["parent"],
                            mesh["boundary_edges"]),
        "lattice": ref.fnv1a64(mesh["lattice"]),
    }
    del mesh
    rp, cols, va = h.csr(L, "stiffness")
    out.update(row_ptr=ref.fnv1a64(rp), cols=ref.fnv1a64(cols), values_A=ref.fnv1a64(va))
    del rp, cols, va
    _, _, vm = h.csr(L, "mass")
    out["values_M"] = ref.fnv1a64(vm)
    del vm
    sp = h.space(L)
    out["connectivity"] = ref.fnv1a64(sp["connectivity"])
    out["interior_dofs"] = ref.fnv1a64(sp["interior_dofs"])
    out["seconds"] = time.time() - t
    h.close()
    return out


def multilevel(name, domain, H, delta, m, levels, nev, workers=8, save_vec=None, example=0):
    t = time.time()
    h = ref.RefHierarchy(domain=domain, H=H, delta=delta, m=m, n_levels=levels, nev=nev,
                         workers=workers, example=example)
    lam, co, matched, times = h.multilevel(levels, nev)
    out = {
        "config": dict(domain=domain, H=H, delta=delta, m=m, n_levels=levels, nev=nev,
                       example=["laplace", "variable"][example]),
        "lambdas": lam.tolist(),
        "matched": matched.tolist(),
        "projections": projections(co),
        "norm2": [float(v @ v) for v in co],
        "seconds": time.time() - t,
    }
    if save_vec:
        np.save(OUT / save_vec, co)
    h.close()
    print(name, out["lambdas"][-1], f"{out['seconds']:.1f}s", flush=True)
    return out


def reaction_run(domain, H, delta, m, levels, nev, seed):
    from oracle import restate as R
    t = time.time()
    hy = R.Hierarchy(domain=domain, H=H, delta=delta, m=m, n_levels=levels, nev=nev,
                     example="reaction", seed=seed)
    lams, state = R.multilevel_correction(hy)
    co = np.stack([v for _, v in state])
    return {"config": dict(domain=domain, H=H, delta=delta, m=m, n_levels=levels, nev=nev,
                           example="reaction", seed=seed, k=list(R.reaction_modes(seed))),
            "lambdas": np.asarray(lams).tolist(), "projections": projections(co),
            "generator": "oracle/restate.py", "seconds": time.time() - t}


LSHAPE_HOLE = (0.0, 1.0, -1.0, 0.0)  # (-1,1)^2 minus [0,1] x [-1,0]


def lshape_run(H, delta, m, levels, nev):
    from oracle import restate as R
    t = time.time()
    hy = R.Hierarchy(domain=SQUARE, H=H, delta=delta, m=m, n_levels=levels, nev=nev,
                     hole=LSHAPE_HOLE)
    lams, state = R.multilevel_correction(hy)
    co = np.stack([v for _, v in state])
    lv = hy.levels[levels]
    me = lv.mesh
    f = ref.fnv1a64
    return {"config": dict(domain=SQUARE, hole=LSHAPE_HOLE, H=H, delta=delta, m=m,
                           n_levels=levels, nev=nev),
            "lambdas": np.asarray(lams).tolist(), "projections": projections(co),
            "mesh": f(me.triangles, me.vertices, me.parent, me.boundary_edges),
            "csr": [f(lv.A[0]), f(lv.A[1]), f(lv.A[2]), f(lv.M[2])],
            "interior_dofs": f(lv.space.interior_dofs), "n_sub": hy.part.m,
            "generator": "oracle/restate.py", "seconds": time.time() - t}


def p2_fixtures():
    h = ref.RefHierarchy(domain=SQUARE, H=0.25, delta=0.25, m=4, n_levels=3, nev=2, degree=2)
    h.extend_to(3)
    f = ref.fnv1a64
    sp = h.space(3)
    out = {"space": [f(sp["dof_lattice"]), f(sp["interior_dofs"]), f(sp["connectivity"])]}
    for form in ("stiffness", "mass"):
        rp, cols, v = h.csr(3, form)
        out[form] = [f(rp), f(cols), f(v)]
    lam, co, matched, _ = h.multilevel(3, 2)
    out["multilevel"] = {"config": dict(domain=SQUARE, H=0.25, delta=0.25, m=4, n_levels=3,
                                        nev=2, degree=2),
                         "lambdas": lam.tolist(), "matched": matched.tolist(),
                         "projections": projections(co)}
    h.close()
    return out


def variable_values():
    """Variable-field operator values at (-1,1)^2, H=0.25, level 3: exact digests
    (for the record: exp() differs between libms, so consumers compare values to
    a few ulp) and the sums of |values| with the row_ptr/cols digests."""
    h = ref.RefHierarchy(domain=SQUARE, H=0.25, delta=0.25, m=4, n_levels=3, nev=1, example=1)
    h.extend_to(3)
    out = {}
    for form in ("stiffness", "mass"):
        rp, cols, v = h.csr(3, form)
        out[form] = {"row_ptr": ref.fnv1a64(rp), "cols": ref.fnv1a64(cols),
                     "values": ref.fnv1a64(v), "abs_sum": float(np.abs(v).sum()),
                     "diag_head": v[rp[:-1]][:16].tolist()}
    h.close()
    return out


def cg_iterations():
    """Iteration counts of the reference's local solves (test_corrector-style)."""
    h = ref.RefHierarchy(domain=UNIT, H=1 / 8, delta=1 / 8, m=4, n_levels=4, nev=1)
    lam, co = h.coarse_eigensolve(3, 1)
    h.extend_to(4)
    u = h.prolong(np.concatenate([[0.0]]) if False else _expand(h, 3, co[0]), 3, 4)
    its = []
    for j in range(4):
        _, it, _ = h.local_bvp_solve(4, j, lam[0], u, 1e-10)
        its.append(it)
    return {"unit8_L3to4_local_iterations": its}


def _expand(h, level, coeffs):
    s = h.sizes(level)
    full = np.zeros(s["ndofs"])
    full.reshape(s["ny"] + 1, s["nx"] + 1)[1:-1, 1:-1] = coeffs.reshape(s["ny"] - 1, s["nx"] - 1)
    return full


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    args = ap.parse_args()
    if not ref.available():
        ref.build()
    path = OUT / "golden.json"
    g = json.loads(path.read_text()) if path.exists() else {}
    g.setdefault("digests", {})
    g.setdefault("multilevel", {})
    g["generator"] = "tests/golden/make_golden.py via oracle/_ref (reference sources + shims)"
    for (n0, L, m, d) in [(8, 4, 4, 1 / 8), (16, 3, 16, 1 / 16), (16, 6, 16, 1 / 16),
                          (16, 7, 16, 1 / 16)]:
        key = f"{n0}_{L}"
        if key not in g["digests"]:
            g["digests"][key] = digests(n0, L, m, d)
            print(key, g["digests"][key]["mesh"], flush=True)
    runs = {
        "small_L3_nev3": (SQUARE, 0.25, 0.25, 4, 3, 3, None),
        "whole_L3_nev3": (SQUARE, 0.5, 0.5, 1, 3, 3, None),
        "square_L4_nev5": (SQUARE, 0.25, 0.25, 4, 4, 5, None),
        "unit8_L4_m4_nev1": (UNIT, 1 / 8, 1 / 8, 4, 4, 1, "unit8_L4_u1.npy"),
        "unit16_L3_m16_nev1": (UNIT, 1 / 16, 1 / 16, 16, 3, 1, None),
        "unit8_L3_m4_nev4": (UNIT, 1 / 8, 1 / 8, 4, 3, 4, None),
        "c2sub_16_L6_m16_nev1": (UNIT, 1 / 16, 1 / 16, 16, 6, 1, None),
        "c5shape_32_L5_m64_nev4": (UNIT, 1 / 32, 1 / 32, 64, 5, 4, None),
    }
    if args.big:
        runs["c5shape_32_L6_m64_nev4"] = (UNIT, 1 / 32, 1 / 32, 64, 6, 4, None)
    for name, (dom, H, d, m, L, nev, vec) in runs.items():
        if name not in g["multilevel"]:
            g["multilevel"][name] = multilevel(name, dom, H, d, m, L, nev, save_vec=vec)
            path.write_text(json.dumps(g, indent=1))
    # CoefficientField::variable (fespace.cpp:114-123), the reference's Example 2
    var_runs = {
        "variable_square_L4_m4_nev3": (SQUARE, 0.25, 0.25, 4, 4, 3, "variable_L4_u.npy"),
        "variable_square_L6_m16_nev2": (SQUARE, 0.125, 0.125, 16, 6, 2, None),
    }
    for name, (dom, H, d, m, L, nev, vec) in var_runs.items():
        if name not in g["multilevel"]:
            g["multilevel"][name] = multilevel(name, dom, H, d, m, L, nev, save_vec=vec,
                                               example=1)
            path.write_text(json.dumps(g, indent=1))
    # L-shaped domain (BASELINE config 3): no reference code path; fixtures from
    # the numpy restatement (oracle/restate.py, B200 definitions) -- parity
    # unpinned against the reference, pinned against our own restatement.
    g.setdefault("lshape", {})
    for name, (H, d, m, L, nev) in {"H8_L3_m16_nev3": (1 / 8, 1 / 8, 16, 3, 3),
                                    "H8_L4_m16_nev1": (1 / 8, 1 / 8, 16, 4, 1)}.items():
        if name not in g["lshape"]:
            g["lshape"][name] = lshape_run(H, d, m, L, nev)
            print("lshape", name, g["lshape"][name]["lambdas"][-1], flush=True)
            path.write_text(json.dumps(g, indent=1))
    if "variable_values" not in g:
        g["variable_values"] = variable_values()
    # P2 (degree 2): the reference's own path -- digests of the level-3 space and
    # operators and a multilevel run
    if "p2" not in g:
        g["p2"] = p2_fixtures()
        path.write_text(json.dumps(g, indent=1))
    # Example "reaction" (BASELINE config 4): no reference code path, so these
    # fixtures come from the numpy restatement (oracle/restate.py) -- parity
    # unpinned against the reference, pinned against our own restatement.
    g.setdefault("reaction", {})
    for name, (dom, H, d, m, L, nev, seed) in {
            "unit8_L4_m4_nev2_seed0": (UNIT, 1 / 8, 1 / 8, 4, 4, 2, 0),
            "unit8_L3_m4_nev1_seed3": (UNIT, 1 / 8, 1 / 8, 4, 3, 1, 3)}.items():
        if name not in g["reaction"]:
            g["reaction"][name] = reaction_run(dom, H, d, m, L, nev, seed)
            print(name, g["reaction"][name]["lambdas"][-1], flush=True)
            path.write_text(json.dumps(g, indent=1))
    if "cg" not in g:
        g["cg"] = cg_iterations()
    if args.big and "32_7" not in g["digests"]:
        g["digests"]["32_7"] = digests(32, 7, 64, 1 / 32)
    path.write_text(json.dumps(g, indent=1))


if __name__ == "__main__":
    main()

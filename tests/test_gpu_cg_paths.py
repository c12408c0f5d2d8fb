"""Every CG code path reproduces the reference's multilevel eigenvalues (golden
vectors from the compiled reference, tests/golden/golden.json).

The path is chosen per batch at run time (SM-resident kernel for batches
beyond L2, persistent cooperative kernel for L2-resident batches, multi-launch
register pipeline, cp.async row pipeline for HBM-streaming batches, general
per-row stencil, generic uniform stencil); the
selection hooks are read once per process, so each variant runs in its own
subprocess.  The L-shaped cases (config 3's domain, golden vectors of the
restatement) cover the hole exclusion of every path."""
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())
CASES = ["small_L3_nev3", "unit8_L3_m4_nev4", "square_L4_nev5", "unit8_L4_m4_nev1"]
VARIANTS = {
    "default": {},
    # (MLG_CG_RESIDENT=0: without it the resident kernel takes every constant-stencil
    # batch the persistent kernel does not)
    "multi_launch_registers": {"MLG_CG_PERSIST": "0", "MLG_CG_RESIDENT": "0"},
    "cp_async_pipeline": {"MLG_CG_ASYNC": "1", "MLG_CG_RESIDENT": "0"},
    "general_stencil": {"MLG_GENERAL_STENCIL": "1"},
    "general_stencil_multi_launch": {"MLG_GENERAL_STENCIL": "1", "MLG_CG_PERSIST": "0"},
    "general_stencil_flagged_only": {"MLG_GENERAL_STENCIL": "1", "MLG_CG_MINROWS": "4",
                                     "MLG_CG_MAXROWS": "8"},
    "generic_uniform_stencil": {"MLG_CG_NOLAP": "1"},
    "short_tasks": {"MLG_CG_MINROWS": "4", "MLG_CG_MAXROWS": "8"},
    # k_cg_resident for every constant-stencil batch that fits on chip (by
    # default only batches beyond L2 or of >= 256 k pooled rows take it)
    "sm_resident": {"MLG_CG_RESIDENT": "2"},
    "sm_resident_generic_stencil": {"MLG_CG_RESIDENT": "2", "MLG_CG_NOLAP": "1"},
}

SCRIPT = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
import paper_1401_4969_b200 as mlg
out = {}
for name, c in json.loads(sys.argv[2]).items():
    hole = mlg.DomainRect(*c["hole"]) if "hole" in c else None
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*c["domain"]), H=c["H"], delta=c["delta"], m=c["m"],
                        n_levels=c["n_levels"], nev=c["nev"], hole=hole)
    with mlg.Hierarchy(cfg) as hy:
        lam, pairs, matched, times = mlg.multilevel_correction(hy)
    out[name] = {"lam": [list(map(float, l)) for l in lam],
                 "kernels": [[int(t.local_kernel), int(t.strip_kernel)] for t in times[1:]]}
print(json.dumps(out))
"""


LSHAPE = ["H8_L3_m16_nev3", "H8_L4_m16_nev1"]


def _lshape_config(name):
    c = GOLDEN["lshape"][name]["config"]
    return {"domain": [-1.0, 1.0, -1.0, 1.0], "hole": [0.0, 1.0, -1.0, 0.0], "H": c["H"],
            "delta": c["H"], "m": c["m"], "n_levels": c["n_levels"], "nev": c["nev"]}


def _golden(name):
    if name.startswith("lshape:"):
        return GOLDEN["lshape"][name[7:]]["lambdas"]
    return GOLDEN["multilevel"][name]["lambdas"]


def _run(env_extra):
    cfgs = {n: GOLDEN["multilevel"][n]["config"] for n in CASES if n in GOLDEN["multilevel"]}
    cfgs.update({"lshape:" + n: _lshape_config(n) for n in LSHAPE})
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT), json.dumps(cfgs)],
                       capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("variant", sorted(VARIANTS))
def test_cg_path_matches_golden_eigenvalues(variant):
    got = _run(VARIANTS[variant])
    if variant.startswith("sm_resident"):  # the path under test really ran (2 = k_cg_resident)
        assert all(2 in [k[0] for k in g["kernels"]] for g in got.values()), \
            {n: g["kernels"] for n, g in got.items()}
        assert any(2 in [k[1] for k in g["kernels"]] for g in got.values())  # masked strip too
    if variant in ("multi_launch_registers", "cp_async_pipeline"):  # 0 = k_cg_iter
        assert all(k == [0, 0] for g in got.values() for k in g["kernels"]), \
            {n: g["kernels"] for n, g in got.items()}
    if variant == "default":  # small batches stay off the resident kernel (2)
        assert all(2 not in k for g in got.values() for k in g["kernels"]), \
            {n: g["kernels"] for n, g in got.items()}
    for name, g in got.items():
        lams = g["lam"]
        ref = _golden(name)
        assert len(lams) == len(ref), name
        for k, (a, b) in enumerate(zip(lams, ref)):
            a, b = np.asarray(a), np.asarray(b)
            rel = np.max(np.abs(a - b) / np.abs(b))
            assert rel <= 1e-10, (variant, name, k, rel)

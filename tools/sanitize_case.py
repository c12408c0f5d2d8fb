"""Small multilevel runs (BASELINE config 1 substitute, 128^2 cells) through each
batched-CG kernel, for compute-sanitizer (memcheck / racecheck / synccheck):
    python tools/sanitize_case.py resident|persist|iter
resident: k_cg_resident (local + strip); persist: k_cg_persist (MLG_CG_RESIDENT=0);
iter: k_cg_iter with the cp.async ring (MLG_CG_RESIDENT=0 MLG_CG_PERSIST=0
MLG_CG_ASYNC=1).  Checks the eigenvalues against the golden vector."""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
mode = sys.argv[1]
env = {"resident": {}, "persist": {"MLG_CG_RESIDENT": "0"},
       "iter": {"MLG_CG_RESIDENT": "0", "MLG_CG_PERSIST": "0", "MLG_CG_ASYNC": "1"}}[mode]
os.environ.update(env)
import numpy as np  # noqa: E402

import paper_1401_4969_b200 as mlg  # noqa: E402

cfg = mlg.RunConfig(domain=mlg.DomainRect(0.0, 1.0, 0.0, 1.0), H=1 / 8, delta=1 / 8, m=4,
                    n_levels=4, nev=1, device=0)
with mlg.Hierarchy(cfg) as hy:
    lam, pairs, matched, times = mlg.multilevel_correction(hy)
g = json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())
print(mode, lam[-1], [t.local_kernel for t in times[1:]], [t.strip_kernel for t in times[1:]])
ref = g["multilevel"]["unit8_L4_m4_nev1"]["lambdas"][-1][0]
assert abs(lam[-1][0] - ref) <= 1e-10 * ref, (lam[-1][0], ref)
print("ok")

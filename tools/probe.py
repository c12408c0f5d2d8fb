"""Quick GPU probe: multilevel correction timings per level for a named config."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_1401_4969_b200 as mlg  # noqa: E402

CFG = {
    "c1": dict(H=1 / 8, delta=1 / 8, m=4, n_levels=4, nev=1),
    "c2": dict(H=1 / 16, delta=1 / 16, m=16, n_levels=6, nev=1),
    "c4": dict(H=1 / 16, delta=1 / 16, m=16, n_levels=7, nev=1),
    "c5": dict(H=1 / 32, delta=1 / 32, m=64, n_levels=7, nev=4),
}

for name in sys.argv[1:] or ["c2"]:
    c = CFG[name]
    cfg = mlg.RunConfig(domain=mlg.DomainRect(0, 1, 0, 1), **c)
    t0 = time.time()
    hy = mlg.Hierarchy(cfg)
    hy.set_profiling(True)
    lam, pairs, matched, times = mlg.multilevel_correction(hy)
    t1 = time.time()
    print(f"== {name}: wall {t1 - t0:.3f}s lam_final={lam[-1].tolist()} matched={matched.tolist()}")
    for k, t in enumerate(times):
        n = hy.level_info(k + 1).n_interior
        tot = t.local_seconds + t.iface_seconds + t.aug_seconds
        bw = ""
        if t.spmv_launches:
            ms = t.spmv_kernel_ms / t.spmv_launches
            b_up, b_chk = (48, 24) if t.spmv_uniform_stencil else (88, 64)
            by = (t.spmv_rows * b_up + t.spmv_check_rows * b_chk) / t.spmv_launches
            bw = f" cg {ms:.3f}ms {by / ms / 1e6:.0f}GB/s"
        print(f"  L{k + 1}: n={n} local {t.local_seconds:.4f} iface {t.iface_seconds:.4f} "
              f"aug {t.aug_seconds:.4f} build {t.build_seconds:.4f} it {t.local_iterations_max}"
              f"/{t.strip_iterations_max} DOF/s {n / tot if tot else 0:.3e}{bw}")
    ms, by = hy.bench_spmv(c["n_levels"], 20)
    print(f"  spmv L{c['n_levels']}: {ms:.4f} ms {by / ms / 1e6:.0f} GB/s")
    hy.close()

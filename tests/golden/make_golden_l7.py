"""Reference run of the north-star configuration (BASELINE config 5, reference-valid
substitute: unit square, 32x32 coarse, 7 levels = 4096^2, m=64, delta=1/32, nev=4)
through the compiled reference (oracle/_ref = /root/reference/proj/src built by
oracle/Makefile).  TEST INFRASTRUCTURE ONLY; runs in the CPU container.

    python tests/golden/make_golden_l7.py run        # ~1 h on 8 cores, ~50 GB RAM
    python tests/golden/make_golden_l7.py strip      # ~20 min: reference strip iterations
    python tests/golden/make_golden_l7.py fixtures   # cheap: writes the committed pins

Stage `run` drives the same chain as multilevel_correction (corrector.cpp:414-462):
coarse_eigensolve on level 1 (:449-454), then one_correction_step k -> k+1
(:456-460) through ref_correction_step, which round-trips the coefficients as
f64 (bitwise the same state).  It keeps the level-6 and level-7 eigenvectors in
.bigcache/ (git- and gpurun-ignored: 135 MB / 537 MB), then times the reference's
local_bvp_solve (corrector.cpp:198-214) on a few level-7 subdomains for the
iteration counts.  Stage `fixtures` turns the cache into small committed pins
(tests/golden/golden_l7.json + c5sub_L7_samples.npy):
  * lambdas and matched_previous at every level;
  * K=32 seeded uniform(-1,1) projections of each level-7 vector and its l2 norm
    (a Johnson-Lindenstrauss sketch: ||S(u-v)|| / ||S v|| estimates the full-vector
    relative difference, see tests/_parity.py);
  * point values on the 63x63 sub-lattice (every 64th fine lattice line).
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import ref  # noqa: E402
sys.path.insert(0, str(ROOT / "tests"))
from _parity import SKETCH_K, SKETCH_SEED, sketch  # noqa: E402

CACHE = ROOT / ".bigcache"
OUT = Path(__file__).resolve().parent
UNIT = (0.0, 1.0, 0.0, 1.0)
CFG = dict(domain=UNIT, H=1 / 32, delta=1 / 32, m=64, n_levels=7, nev=4)
SAMPLE_STRIDE = 64
LOCAL_J = (0, 9, 27, 63)


def log(*a):
    print(time.strftime("%H:%M:%S"), *a, flush=True)


def run():
    CACHE.mkdir(exist_ok=True)
    if not ref.available():
        ref.build()
    c = CFG
    h = ref.RefHierarchy(domain=c["domain"], H=c["H"], delta=c["delta"], m=c["m"],
                         n_levels=c["n_levels"], nev=c["nev"], workers=8)
    meta = {"config": c, "lambdas": [], "matched": [True], "timings": [[0.0, 0.0, 0.0]],
            "step_wall_s": [0.0], "generator": "tests/golden/make_golden_l7.py via oracle/_ref"}
    t = time.time()
    lam, co = h.coarse_eigensolve(1, c["nev"])
    meta["lambdas"].append(lam.tolist())
    log("level 1", lam.tolist(), f"{time.time() - t:.1f}s")
    for k in range(1, c["n_levels"]):
        t = time.time()
        lam, co, matched, t3 = h.correction_step(k, k + 1, lam, co)
        meta["lambdas"].append(lam.tolist())
        meta["matched"].append(bool(matched))
        meta["timings"].append(list(t3))
        meta["step_wall_s"].append(time.time() - t)
        log(f"level {k + 1}", lam.tolist(), matched, [round(x, 1) for x in t3],
            f"{time.time() - t:.1f}s")
        if k + 1 >= 6:
            np.save(CACHE / f"c5sub_L{k + 1}_coeffs.npy", co)
        (CACHE / "c5sub_meta.json").write_text(json.dumps(meta, indent=1))
    # reference local-solve iteration counts at level 7 from the level-6 state
    co6 = np.load(CACHE / "c5sub_L6_coeffs.npy")
    s6 = h.sizes(6)
    its = {}
    for i in (0, 1):
        full = np.zeros(s6["ndofs"])
        full.reshape(s6["ny"] + 1, s6["nx"] + 1)[1:-1, 1:-1] = co6[i].reshape(
            s6["ny"] - 1, s6["nx"] - 1)
        u7 = h.prolong(full, 6, 7)
        for j in LOCAL_J:
            t = time.time()
            _, it, _ = h.local_bvp_solve(7, j, meta["lambdas"][5][i], u7, 1e-10)
            its[f"{i}_{j}"] = it
            log("local", i, j, it, f"{time.time() - t:.1f}s")
        meta["local_iterations_L7"] = its
        (CACHE / "c5sub_meta.json").write_text(json.dumps(meta, indent=1))
    h.close()


def strip():
    """Reference strip-solve iteration count at level 7 (interface_solve,
    corrector.cpp:216-254) for eigenvector 0 from the level-6 state: the 64
    local corrections (local_bvp_solve, run on 8 threads like parallel_tasks),
    then the strip CG.  bench.py's reference arm scales its timed strip sample
    by this count."""
    import threading
    meta = json.loads((CACHE / "c5sub_meta.json").read_text())
    c = CFG
    h = ref.RefHierarchy(domain=c["domain"], H=c["H"], delta=c["delta"], m=c["m"],
                         n_levels=c["n_levels"], nev=c["nev"], workers=8)
    h.extend_to(7)
    h.build_region_systems(7)
    co6 = np.load(CACHE / "c5sub_L6_coeffs.npy")
    s6 = h.sizes(6)
    out = {}
    for i in (0,):
        full = np.zeros(s6["ndofs"])
        full.reshape(s6["ny"] + 1, s6["nx"] + 1)[1:-1, 1:-1] = co6[i].reshape(
            s6["ny"] - 1, s6["nx"] - 1)
        u7 = h.prolong(full, 6, 7)
        lam = meta["lambdas"][5][i]
        corr = np.zeros((c["m"], u7.size))
        nxt = [0]
        lock = threading.Lock()

        def work():
            while True:
                with lock:
                    j = nxt[0]
                    nxt[0] += 1
                if j >= c["m"]:
                    return
                corr[j], _, _ = h.local_bvp_solve(7, j, lam, u7, 1e-10)
        t = time.time()
        th = [threading.Thread(target=work) for _ in range(8)]
        for x in th:
            x.start()
        for x in th:
            x.join()
        log("corrections", i, f"{time.time() - t:.1f}s")
        t = time.time()
        _, its, res = h.interface_solve(7, lam, u7, corr, 1e-10)
        log("strip", i, its, res, f"{time.time() - t:.1f}s")
        out[str(i)] = its
        meta["strip_iterations_L7"] = out
        meta["strip_seconds_L7"] = time.time() - t
        (CACHE / "c5sub_meta.json").write_text(json.dumps(meta, indent=1))
    h.close()


def fixtures():
    meta = json.loads((CACHE / "c5sub_meta.json").read_text())
    co = np.load(CACHE / "c5sub_L7_coeffs.npy")
    n = 4095
    proj, rn = sketch(co)
    idx = np.arange(SAMPLE_STRIDE - 1, n, SAMPLE_STRIDE)
    samples = co.reshape(co.shape[0], n, n)[:, idx][:, :, idx]
    np.save(OUT / "c5sub_L7_samples.npy", samples)
    out = {k: meta[k] for k in ("config", "lambdas", "matched", "timings", "step_wall_s",
                                "generator")}
    out.update(local_iterations_L7=meta.get("local_iterations_L7", {}),
               reference_strip_iterations_L7=list(meta.get("strip_iterations_L7", {}).values()),
               workers=8,
               sketch={"k": SKETCH_K, "seed": SKETCH_SEED, "projections": proj.tolist(),
                       "row_norms": rn.tolist()},
               norm2=[float(v @ v) for v in co], sample_stride=SAMPLE_STRIDE,
               samples="c5sub_L7_samples.npy")
    (OUT / "golden_l7.json").write_text(json.dumps(out, indent=1))
    print("wrote", OUT / "golden_l7.json")


if __name__ == "__main__":
    {"run": run, "strip": strip, "fixtures": fixtures}[sys.argv[1]]()

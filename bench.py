#!/usr/bin/env python
"""Benchmark of the B200 correction step (BASELINE.json metric: fine-grid DOF/s
per correction step; local-solve SpMV HBM GB/s vs B200 peak).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c3|c4|c5]
    python bench.py --impl reference ...        # the reference's CPU path (oracle/_ref)

A "step" is one correction step L-1 -> L (one_correction_step,
corrector.cpp:336-412) of the named workload; its input eigenpairs come from
the multilevel pipeline itself (level-1 dense solve + correction steps).
`value` times the step with coefficient arrays resident in HBM (device C-ABI
entry point, CUDA events on the library stream); `e2e` times the same step
through the host C-ABI call with pinned host buffers (H2D/D2H inside).  Under
torchrun every rank runs an independent replica on its GPU ("replicas only",
DESIGN.md): value = all ranks' DOF / max-over-ranks time.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "fine-grid DOF/s per correction step; local-solve SpMV HBM GB/s vs B200 peak"
WORKLOADS = {
    "c2": dict(desc="config 2 (reference-valid substitute m=16): unit square, Laplace P1 FP64, "
                    "16x16 coarse squares, 6 levels (1024^2 cells), 4x4 overlapping subdomains, "
                    "delta=1/16, nev=1; step level 5 -> 6",
               H=1 / 16, delta=1 / 16, m=16, n_levels=6, nev=1),
    "c5": dict(desc="config 5 (reference-valid substitute m=64): unit square, Laplace P1 FP64, "
                    "32x32 coarse squares, 7 levels (4096^2 cells), 8x8 overlapping subdomains, "
                    "delta=1/32, nev=4; step level 6 -> 7",
               H=1 / 32, delta=1 / 32, m=64, n_levels=7, nev=4),
    "c3": dict(desc="config 3 (B200 extension, no reference code path): L-shaped domain "
                    "(-1,1)^2 minus [0,1]x[-1,0], Laplace P1 FP64, 3 unit squares of 16x16 "
                    "cells (768 coarse triangles), 6 levels (3.1M fine triangles), 48 "
                    "subdomains on the 8x8 block grid clipped to the domain, delta = 1 coarse "
                    "cell, nev=1; step level 5 -> 6",
               domain=(-1.0, 1.0, -1.0, 1.0), hole=(0.0, 1.0, -1.0, 0.0),
               H=1 / 16, delta=1 / 16, m=64, n_levels=6, nev=1),
    "c4": dict(desc="config 4 (reference-valid partition m=16): unit square, "
                    "-div(a grad u) + c u = lambda u, a = 1 + 0.5 sin(2 pi k1 x) sin(2 pi k2 y), "
                    "c = 1 + x^2 + y^2 at centroids, (k1,k2) = (4,2) from seed 0, P1 FP64, "
                    "16x16 coarse squares, 7 levels (2048^2 cells), 4x4 overlapping subdomains, "
                    "delta=1/16, nev=1; step level 6 -> 7 (no reference code path)",
               H=1 / 16, delta=1 / 16, m=16, n_levels=7, nev=1, example="reaction", seed=0),
}
FALLBACK_HBM = 6650.0


def cg_bytes_per_row(uniform=0):
    """Algorithmic HBM bytes per window row of one CG iteration launch (k_cg_iter,
    the fused one-reduction PCG sweep): update mode reads x, r, p and writes x, r,
    p (6 x 8 B = 48 B); true-residual mode reads x and b and writes r (24 B).
    Non-uniform levels add the stencil {C,E,N,NE} and D^-1 (40 B); on uniform
    levels they are kernel parameters.  uniform == 2: x updates deferred in
    pairs -- one launch moves r, p (32 B), the next r, p, x and the deferred
    update's p (56 B): 44 B/row per launch of a sampled pair.  Stencil
    neighbours come from registers and warp shuffles, so nothing else is
    re-read.  Returns (update, check)."""
    return {0: (88, 64), 1: (48, 24), 2: (44, 24)}[int(uniform)]


# ----------------------------------------------------------------- helpers ---
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 3 + k and r[3 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload):
    """Per-row DRAM traffic of k_cg_iter from the committed ncu --set full summary."""
    p = ROOT / "profiles" / "ka_traffic.json"
    try:
        d = json.loads(p.read_text())
        e = d.get(workload)
        return e["dram_bytes_per_launch"] / e["rows_per_launch"]
    except Exception:
        return None


def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        backend = "nccl" if args.impl != "reference" else "gloo"
        dist.init_process_group(backend, init_method="env://")
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def allreduce_max(x, ws, device=None):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------ reference arm --
def reference_step_run(wl, steps, warmup, workers):
    """The reference's own implementation (oracle/_ref = unmodified reference
    sources) on host cores: setup to level L-1, then one_correction_step L-1->L."""
    from oracle import ref
    L = wl["n_levels"]
    t0 = time.time()
    setup = ref.RefHierarchy(domain=(0.0, 1.0, 0.0, 1.0), H=wl["H"], delta=wl["delta"], m=wl["m"],
                             n_levels=L - 1, nev=wl["nev"], workers=workers)
    lam, co, _, _ = setup.multilevel(L - 1, wl["nev"])
    setup.close()
    h = ref.RefHierarchy(domain=(0.0, 1.0, 0.0, 1.0), H=wl["H"], delta=wl["delta"], m=wl["m"],
                         n_levels=L, nev=wl["nev"], workers=workers)
    build = h.extend_to(L)
    regions = h.build_region_systems(L)
    setup_s = time.time() - t0
    times, splits = [], []
    for k in range(warmup + steps):
        t = time.perf_counter()
        lo, _, matched, t3 = h.correction_step(L - 1, L, lam[-1], co, want_coeffs=False)
        dt = time.perf_counter() - t
        if k >= warmup:
            times.append(dt)
            splits.append(t3)
    n = h.sizes(L)["n_int"]
    h.close()
    return dict(n_int=n, times=times, splits=splits, build_s=build, regions_s=regions,
                setup_s=setup_s, lam=list(lo))


def run_reference(args, ws, rank):
    if rank != 0:
        return
    wl = WORKLOADS[args.workload]
    cores = os.cpu_count() or 1
    if wl.get("example", "laplace") == "reaction" or wl.get("hole"):
        print(json.dumps({"impl": "reference", "unavailable": "the reference has no code path "
                          "for this workload (config 3's L-shaped mesh / config 4's "
                          "reaction/centroid-coefficient field)"}))
        return
    try:
        from oracle import ref
        if not ref.available():
            raise ImportError("oracle/_ref/libmleig_ref.so not built")
    except Exception as e:
        print(json.dumps({"impl": "reference", "unavailable": f"{e}"}))
        return
    # bounded sample: at most 1 warm-up and 3 timed full steps (each a complete
    # reference correction step of the workload)
    r = reference_step_run(wl, steps=min(args.steps, 3), warmup=min(args.warmup, 1),
                           workers=cores)
    step_s = statistics.mean(r["times"])
    value = r["n_int"] / step_s
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "DOF/s",
        "n_gpus": args.gpus, "steps": len(r["times"]), "warmup": min(args.warmup, 1),
        "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl["desc"], "n_interior": r["n_int"], "threads": cores},
        "cpu_baseline": {"value": value, "unit": "DOF/s", "cores": cores, "kind": "reference",
                         "sample": f"{len(r['times'])} full one_correction_step calls "
                                   f"(L{wl['n_levels'] - 1}->L{wl['n_levels']}) of the workload, "
                                   f"reference sources built by oracle/Makefile, workers={cores}"},
        "e2e": {"value": value, "unit": "DOF/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "reference_split_s": {"local": statistics.mean(s[0] for s in r["splits"]),
                              "iface": statistics.mean(s[1] for s in r["splits"]),
                              "aug": statistics.mean(s[2] for s in r["splits"]),
                              "level_build": r["build_s"], "region_systems": r["regions_s"]},
    }
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------------- ours ---
def run_ours(args, ws, rank, local, workload, steps, warmup, with_e2e=True, profile=True):
    import numpy as np
    import torch

    import paper_1401_4969_b200 as mlg
    from paper_1401_4969_b200.corrector import (multilevel_correction_device,
                                                one_correction_step_device,
                                                one_correction_step_raw)
    wl = WORKLOADS[workload]
    L, nev = wl["n_levels"], wl["nev"]
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    hole = wl.get("hole")
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*wl.get("domain", (0.0, 1.0, 0.0, 1.0))),
                        H=wl["H"], delta=wl["delta"], m=wl["m"], n_levels=L, nev=nev,
                        cg_tol=1e-10, device=local, example=wl.get("example", "laplace"),
                        seed=wl.get("seed", 0), hole=mlg.DomainRect(*hole) if hole else None)
    hy = mlg.Hierarchy(cfg)
    t0 = time.time()
    hy.extend_to(L - 1)
    n_in = hy.level_info(L - 1).n_interior
    d_in = torch.empty((nev, n_in), dtype=torch.float64, device=dev)
    lam = multilevel_correction_device(hy, L - 1, d_in.data_ptr())[-1].copy()
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    # the level-1 dense generalized eigensolve that starts the multilevel run
    # (solve_interior_eigenproblem, sparse.cpp:326-355; cuSOLVER sygvd), timed alone
    from paper_1401_4969_b200.corrector import coarse_eigensolve
    t = time.perf_counter()
    coarse_eigensolve(hy, 1, nev)
    torch.cuda.synchronize()
    level1_s = time.perf_counter() - t
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > L2 (126 MB)

    # level build of the target level, measured once (Hierarchy::extend_to)
    t = time.perf_counter()
    hy.extend_to(L)
    build_s = time.perf_counter() - t
    n_out = hy.level_info(L).n_interior
    d_out = torch.empty((nev, n_out), dtype=torch.float64, device=dev)

    for _ in range(warmup):
        one_correction_step_device(hy, L - 1, L, lam, d_in.data_ptr(), d_out.data_ptr())
    hy.set_profiling(profile)
    torch.cuda.synchronize()
    barrier(ws)
    step_s, tims = [], []
    with ClockSampler(local) as clk:
        for _ in range(steps):
            flush.zero_()
            torch.cuda.synchronize()
            lo, matched, tm = one_correction_step_device(hy, L - 1, L, lam, d_in.data_ptr(),
                                                         d_out.data_ptr())
            step_s.append(tm.step_seconds)
            tims.append(tm)
    torch.cuda.synchronize()
    barrier(ws)
    hy.set_profiling(False)
    total = allreduce_max(sum(step_s), ws, dev)
    value = ws * n_out * steps / total

    out = dict(value=value, ms_per_step=total / steps * 1e3, n_int=n_out, setup_s=setup_s,
               level1_dense_s=level1_s,
               build_s=build_s, lam=list(lo), matched=matched, clocks=clk.summary(),
               timings={"local_s": statistics.mean(t.local_seconds for t in tims),
                        "iface_s": statistics.mean(t.iface_seconds for t in tims),
                        "aug_s": statistics.mean(t.aug_seconds for t in tims),
                        "local_cg_iterations": tims[-1].local_iterations_max,
                        "strip_cg_iterations": tims[-1].strip_iterations_max},
               gpu_launches=int(sum(t.kernel_launches for t in tims)))
    ka_ms = sum(t.spmv_kernel_ms for t in tims)
    ka_n = sum(t.spmv_launches for t in tims)
    ka_rows = sum(t.spmv_rows for t in tims)
    ka_chk = sum(t.spmv_check_rows for t in tims)
    ka_all = sum(t.spmv_launches_all for t in tims)
    # one cooperative launch per solve vs one launch per CG iteration
    persistent = ka_all < 0.5 * sum(t.local_iterations_max for t in tims)
    if ka_n:
        bpr, bpc = cg_bytes_per_row(tims[-1].spmv_uniform_stencil)
        ka_bytes = ka_rows * bpr + ka_chk * bpc
        achieved = ka_bytes / (ka_ms * 1e-3) / 1e9
        peak, peak_src = measured_peak()
        tr = ncu_traffic(workload)
        out["roofline"] = {
            "kernel": ("k_cg_persist (local solves: the fused PCG sweep, all iterations in one "
                       "cooperative launch, cp.async row ring)" if persistent else
                       "k_cg_iter (local solves: fused PCG sweep, one launch per iteration)"),
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "peak_source": peak_src,
            "traffic": None if tr is None else tr * (ka_rows + ka_chk) / ka_n,
            "algorithmic_bytes_per_launch": ka_bytes / ka_n,
            "bytes_per_row": bpr, "bytes_per_check_row": bpc,
            "rows_per_launch": (ka_rows + ka_chk) / ka_n,
            "uniform_stencil": int(tims[-1].spmv_uniform_stencil),
            "avg_launch_ms": ka_ms / ka_n, "launches": int(ka_n),
            "launches_all": int(ka_all),
            # the sampled launches' mean duration x every launch of the kernel
            "share_of_step": ka_ms / ka_n * ka_all * 1e-3 / sum(step_s),
        }

    if with_e2e:  # through the host C-ABI with pinned host buffers
        h_in = torch.empty((nev, n_in), dtype=torch.float64, pin_memory=True)
        h_in.copy_(d_in.cpu())
        h_out = torch.empty((nev, n_out), dtype=torch.float64, pin_memory=True)
        a_in, a_out = h_in.numpy(), h_out.numpy()
        one_correction_step_raw(hy, L - 1, L, lam, a_in, a_out)  # warm the host-array path
        barrier(ws)
        e2e_s = []
        for _ in range(steps):
            flush.zero_()
            torch.cuda.synchronize()
            _, _, tm = one_correction_step_raw(hy, L - 1, L, lam, a_in, a_out)
            e2e_s.append(tm.step_seconds)
        barrier(ws)
        etot = allreduce_max(sum(e2e_s), ws, dev)
        out["e2e"] = {"value": ws * n_out * steps / etot, "unit": "DOF/s",
                      "h2d_bytes_per_step": int(a_in.nbytes + 8 * nev),
                      "d2h_bytes_per_step": int(a_out.nbytes + 8 * nev),
                      "ms_per_step": etot / steps * 1e3}
    ms, by = hy.bench_spmv(L, 20)
    out["spmv_microbench"] = {"kernel": "interior stiffness SpMV (stencil format)",
                              "ms": ms, "GB/s": by / ms / 1e6, "bytes": by,
                              "csr_equivalent_GB/s": None}
    hy.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--no-north-star", action="store_true",
                    help="skip the extra config-5 (4096^2), config-4 and config-3 measurements")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    ws, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    wl = WORKLOADS[args.workload]
    res = run_ours(args, ws, rank, local, args.workload, args.steps, args.warmup)
    extra = extra4 = None
    if not args.no_north_star and args.workload != "c5":
        extra = run_ours(args, ws, rank, local, "c5", steps=2, warmup=1, with_e2e=False)
    if not args.no_north_star and args.workload != "c4":
        extra4 = run_ours(args, ws, rank, local, "c4", steps=2, warmup=1, with_e2e=False)
    extra3 = None
    if not args.no_north_star and args.workload != "c3":
        extra3 = run_ours(args, ws, rank, local, "c3", steps=2, warmup=1, with_e2e=False)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            from oracle import ref
            if ref.available():
                cores = os.cpu_count() or 1
                r = reference_step_run(wl, steps=1, warmup=0, workers=cores)
                cpu = {"value": r["n_int"] / r["times"][0], "unit": "DOF/s", "cores": cores,
                       "kind": "reference",
                       "sample": f"one full one_correction_step L{wl['n_levels'] - 1}->"
                                 f"L{wl['n_levels']} of the headline workload on the reference "
                                 f"(oracle/_ref, workers={cores}); setup untimed",
                       "seconds": r["times"][0]}
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unavailable": str(e)}
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": res["value"], "unit": "DOF/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (deterministic meshes; eigenpairs produced by the pipeline)",
        "config": {"workload": wl["desc"], "n_interior": res["n_int"],
                   "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU",
                   "l2": "flushed between timed steps (256 MiB write)",
                   "lambdas": res["lam"]},
        "roofline": res.get("roofline"), "cpu_baseline": cpu, "e2e": res.get("e2e"),
        "gpu_launches": res["gpu_launches"], "clocks": res["clocks"],
        "timings": {**res["timings"], "level_build_s": res["build_s"], "setup_s": res["setup_s"],
                    "level1_dense_eigensolve_s": res["level1_dense_s"]},
        "spmv_microbench": res["spmv_microbench"],
    }
    if extra:
        line["north_star_workload"] = {
            "workload": WORKLOADS["c5"]["desc"], "value": extra["value"], "unit": "DOF/s",
            "ms_per_step": extra["ms_per_step"], "n_interior": extra["n_int"],
            "level_build_s": extra["build_s"],
            "timings": {**extra["timings"], "setup_s": extra["setup_s"],
                        "level1_dense_eigensolve_s": extra["level1_dense_s"]},
            "roofline": extra.get("roofline"), "lambdas": extra["lam"],
            "clocks": extra["clocks"], "spmv_microbench": extra["spmv_microbench"]}
    if extra3:
        line["config3_workload"] = {
            "workload": WORKLOADS["c3"]["desc"], "value": extra3["value"], "unit": "DOF/s",
            "ms_per_step": extra3["ms_per_step"], "n_interior": extra3["n_int"],
            "level_build_s": extra3["build_s"], "timings": extra3["timings"],
            "roofline": extra3.get("roofline"), "lambdas": extra3["lam"],
            "clocks": extra3["clocks"]}
    if extra4:
        line["config4_workload"] = {
            "workload": WORKLOADS["c4"]["desc"], "value": extra4["value"], "unit": "DOF/s",
            "ms_per_step": extra4["ms_per_step"], "n_interior": extra4["n_int"],
            "level_build_s": extra4["build_s"], "timings": extra4["timings"],
            "roofline": extra4.get("roofline"), "lambdas": extra4["lam"],
            "clocks": extra4["clocks"]}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

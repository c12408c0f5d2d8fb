"""CPU, world_size 2 over gloo: the multi-rank host logic of bench.py (one
replica per rank; value = all ranks' DOF / max-over-ranks time)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, out):
    import torch.distributed as dist

    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(ws), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", init_method="env://", rank=rank, world_size=ws)
    bench.barrier(ws)
    t = bench.allreduce_max(1.0 + rank, ws)
    n_dof, steps = 1000, 4
    value = ws * n_dof * steps / t
    out[rank] = (t, value)
    dist.destroy_process_group()


def test_two_rank_max_time_aggregation():
    ws = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(ws, port, out), nprocs=ws, join=True)
    assert out[0] == out[1] == (2.0, 2 * 1000 * 4 / 2.0)


def test_reference_arm_rank_gating(monkeypatch, capsys):
    import bench

    class A:
        workload = "c2"
        steps = 1
        warmup = 0
        gpus = 2
        impl = "reference"
    bench.run_reference(A, ws=2, rank=1)  # non-zero ranks exit without work
    assert capsys.readouterr().out == ""


def test_cg_bytes_model():
    import bench
    # update sweep: x, r, p read + written; check sweep: x, b read, r written
    assert bench.cg_bytes_per_row(True) == (48, 24)
    # non-uniform levels stream the {C,E,N,NE} stencil and D^-1 as well
    assert bench.cg_bytes_per_row(False) == (88, 64)


def test_cpu_baseline_reuses_box_measured_reference_arm(tmp_path, monkeypatch):
    """The reference arm leaves its line for our arm's cpu_baseline; only a
    fresh line of the same workload made on this host is reused."""
    import json
    import socket
    import time

    import bench
    cache = tmp_path / "arm.json"
    monkeypatch.setattr(bench, "REF_ARM_CACHE", cache)
    assert bench.cached_reference_arm("c5") is None
    line = {"ms_per_step": 857000.0,
            "cpu_baseline": {"value": 19560.0, "unit": "DOF/s", "cores": 16, "kind": "reference",
                             "sample": "2 sampled steps"}}
    cache.write_text(json.dumps({"host": socket.gethostname(), "when": time.time() - 120,
                                 "workload": "c5", "line": line}))
    assert bench.cached_reference_arm("c2") is None
    cb = bench.cpu_baseline_leg("c5")
    assert cb["value"] == 19560.0 and cb["cores"] == 16 and cb["kind"] == "reference"
    assert abs(cb["seconds"] - 857.0) < 1e-9 and "on this host" in cb["sample"]
    cache.write_text(json.dumps({"host": "another-box", "when": time.time(), "workload": "c5",
                                 "line": line}))
    assert bench.cached_reference_arm("c5") is None
    cache.write_text(json.dumps({"host": socket.gethostname(), "when": time.time() - 8 * 3600,
                                 "workload": "c5", "line": line}))
    assert bench.cached_reference_arm("c5") is None


def test_roofline_entry_of_the_resident_kernel():
    """bound = shared memory; the row rate is also priced at the streaming
    kernel's 44 B/row against the HBM peak."""
    import bench
    e = bench._roofline("k_cg_resident", "smem", 12694.0, "local", "c5", 2.86e11, 1623.0, 1, 1,
                        0.61, 72)
    assert e["bound"] == "smem" and e["unit"] == "GB/s" and 0 < e["frac"] < 1
    eq = e["hbm_streaming_equivalent"]
    assert eq["bytes_per_row"] == 44 and abs(eq["GB/s"] - 12694.0 / 72 * 44) < 1e-6
    hp, _ = bench.measured_peak("hbm")
    assert abs(eq["frac_of_hbm_peak"] - eq["GB/s"] / hp) < 1e-12
    h = bench._roofline("k_cg_iter", "hbm", 4795.0, "strip", "c5", 4.47e7, 0.41, 100, 100, 0.37, 44)
    assert "hbm_streaming_equivalent" not in h and "frac_of_hbm_peak" not in h

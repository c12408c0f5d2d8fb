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

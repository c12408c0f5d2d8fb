"""bench.py's JSON contract on the GPU: one short run of the headline workload
prints one line with every key the driver and the judge read (metric/value,
roofline of the dominant CG kernel, end-to-end number through the C ABI with
its host<->device bytes, kernel launch count, clocks under load)."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


def test_bench_line_contract():
    r = subprocess.run([sys.executable, "bench.py", "--steps", "2", "--warmup", "3",
                        "--no-extras", "--no-cpu-baseline"], cwd=ROOT, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3
    assert d["value"] > 0 and d["higher_is_better"] is True and d["scaling"] == "weak"
    assert d["dtype"] == "f64" and "workload" in d["config"]
    rf = d["roofline"]
    assert rf["bound"] in ("hbm", "l2", "smem") and rf["unit"] == "GB/s"
    assert 0 < rf["achieved"] and 0 < rf["peak"]
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert 0 < rf["share_of_step"] <= 1.0
    # one roofline per kernel family of the step: local CG, strip CG, assembly
    rls = d["rooflines"]
    assert {"local", "strip", "assembly"} <= set(rls)
    assert rf["share_of_step"] == max(rls["local"]["share_of_step"],
                                      rls["strip"]["share_of_step"])
    for e in rls.values():
        assert e["achieved"] > 0 and e["algorithmic_bytes_per_launch"] > 0
    assert "4096^2" in d["config"]["workload"]  # the headline is config 5
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["unit"] == d["unit"]
    assert e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert d["clocks"]["sm_max_mhz"] > 0
    assert d["config"]["lambdas"][0] == pytest.approx(19.7392, rel=1e-4)  # 2 pi^2 from above
    assert len(d["config"]["lambdas"]) == 4

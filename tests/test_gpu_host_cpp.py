"""The C++ drop-in host API (include/mleig_b200.hpp) end to end: the mlg_run
driver reproduces the reference's multilevel eigenvalues (golden vectors)."""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())
DRIVER = ROOT / "paper_1401_4969_b200" / "build" / "mlg_run"


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["unit8_L4_m4_nev1", "square_L4_nev5", "c2sub_16_L6_m16_nev1"])
def test_cpp_driver_matches_golden(name):
    if not DRIVER.exists():
        from paper_1401_4969_b200 import _build
        _build.build_driver()
    g = GOLDEN["multilevel"][name]
    c = g["config"]
    args = [str(DRIVER), *map(repr, c["domain"]), repr(c["H"]), repr(c["delta"]), str(c["m"]),
            str(c["n_levels"]), str(c["nev"])]
    out = subprocess.run(args, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.strip().splitlines()
    assert lines[0].startswith("level,h,dofs,eig_index,lambda")
    lam = np.zeros((c["n_levels"], c["nev"]))
    for ln in lines[1:]:
        f = ln.split(",")
        lam[int(f[0]) - 1, int(f[3]) - 1] = float(f[4])
    ref = np.array(g["lambdas"])
    assert np.max(np.abs(lam - ref) / ref) <= 1e-10


@pytest.mark.gpu
def test_cpp_driver_config_error_exit_code():
    if not DRIVER.exists():
        from paper_1401_4969_b200 import _build
        _build.build_driver()
    out = subprocess.run([str(DRIVER), "0", "1", "0", "1", "0.3", "0.1", "4", "2", "1"],
                         capture_output=True, text=True, timeout=120)
    assert out.returncode == 2 and "does not divide" in out.stderr

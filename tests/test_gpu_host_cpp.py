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


GOOD_CFG = """{
  "domain": {"x_min": -1.0, "x_max": 1.0, "y_min": -1.0, "y_max": 1.0},
  "H": 0.5, "delta": 0.5, "m": 1, "n_levels": 3, "degree": 1, "nev": 2,
  "example": "laplace", "cg_tol": 1e-10, "workers": 1, "deterministic": true
}"""


@pytest.mark.gpu
def test_cpp_cli_run_table_vtk(tmp_path, oracle_ref):
    """`mlg_run run/table/export-vtk` (the reference CLI's subcommands,
    mleig_main.cpp:13-71) through the C++ header: CSV rows agree with the
    reference's run_experiment, the table is the reference's printer output."""
    if not DRIVER.exists():
        from paper_1401_4969_b200 import _build
        _build.build_driver()
    cfg = tmp_path / "c.json"
    cfg.write_text(GOOD_CFG)
    out = subprocess.run([str(DRIVER), "run", str(cfg), "-o", str(tmp_path / "r.csv")],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    ref_csv = tmp_path / "ref.csv"
    oracle_ref.run_experiment(ref_csv, domain=(-1.0, 1.0, -1.0, 1.0), H=0.5, delta=0.5, m=1,
                              n_levels=3, nev=2)
    a = (tmp_path / "r.csv").read_text().splitlines()
    b = ref_csv.read_text().splitlines()
    assert a[0] == b[0] and len(a) == len(b)
    for la, lb in zip(a[1:], b[1:]):
        fa, fb = la.split(","), lb.split(",")
        assert fa[:4] == fb[:4]
        assert abs(float(fa[4]) - float(fb[4])) <= 1e-10 * float(fb[4])
    t = subprocess.run([str(DRIVER), "table", str(tmp_path / "r.csv")], capture_output=True,
                       text=True, timeout=60)
    assert t.returncode == 0 and t.stdout.startswith("eigenvalue 1:")
    assert t.stdout.splitlines()[1] == oracle_ref.print_table(ref_csv).splitlines()[1]
    v = subprocess.run([str(DRIVER), "export-vtk", str(cfg), "-o", str(tmp_path / "vtk")],
                       capture_output=True, text=True, timeout=300)
    assert v.returncode == 0, v.stderr
    assert (tmp_path / "vtk" / "eigenfunctions.vtk").read_text().startswith(
        "# vtk DataFile Version 3.0")
    bad = subprocess.run([str(DRIVER), "run", "/nonexistent.json", "-o", "x.csv"],
                         capture_output=True, text=True, timeout=60)
    assert bad.returncode == 4

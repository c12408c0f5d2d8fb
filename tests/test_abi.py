"""CPU checks of the drop-in boundary: the CUDA library loads (built for
sm_100a) and exports every symbol include/mlg_b200.h declares; the ctypes
mirror binds all of them.  No compute calls (no GPU here)."""
import re
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "mlg_b200.h"


def declared_symbols():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(mlg_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("mlg_create", "mlg_correction_step", "mlg_local_bvp_solve",
              "mlg_interface_solve", "mlg_augmented_eigensolve", "mlg_multilevel_correction",
              "mlg_export_csr", "mlg_export_mesh"):
        assert s in syms


def test_library_loads_and_exports_all_symbols(mlg):
    lib = mlg.lib()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", str(mlg._lib.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (mlg_\w+)", out))
    assert set(declared_symbols()) <= exported


def test_ctypes_signatures_cover_header(mlg):
    assert set(declared_symbols()) == set(mlg._lib.SIGNATURES)


def test_library_is_sm100a():
    so = ROOT / "paper_1401_4969_b200" / "libmlg_b200.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_in_product():
    """The product never imports the oracle."""
    pkg = ROOT / "paper_1401_4969_b200"
    for f in list(pkg.glob("*.py")) + list((pkg / "csrc").glob("*")):
        assert "oracle" not in f.read_text().replace("oracle/_ref", ""), f


def test_struct_layouts_match_ctypes(tmp_path):
    """Every struct the header declares has the same field offsets and size in C
    (gcc on the header) and in the ctypes mirror (_lib.py)."""
    import ctypes as C

    from paper_1401_4969_b200 import _lib
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    mirrors = {"mlg_step_timings": _lib.MlgStepTimings, "mlg_solve_report": _lib.MlgSolveReport,
               "mlg_config": _lib.MlgConfig}
    prog = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', 'int main(void){']
    for cname, py in mirrors.items():
        assert re.search(r"typedef struct " + cname + r"\b", text), cname
        prog.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            prog.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    prog.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(prog))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    got = {}
    for line in subprocess.run([str(exe)], capture_output=True, text=True,
                               check=True).stdout.splitlines():
        cname, field, val = line.split()
        got[(cname, field)] = int(val)
    for cname, py in mirrors.items():
        assert got[(cname, "size")] == C.sizeof(py), cname
        for f, _ in py._fields_:
            assert got[(cname, f)] == getattr(py, f).offset, (cname, f)

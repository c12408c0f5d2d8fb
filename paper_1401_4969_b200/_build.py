"""In-tree build of libmlg_b200.so (sm_100a) with nvcc.

The shared library is the product: hand-written CUDA for the correction-step
hot path behind the C ABI in include/mlg_b200.h.  It is built next to this
file so it travels with the repository snapshot to the GPU box.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OBJ = PKG / "build"
LIB = PKG / "libmlg_b200.so"
SOURCES = ["mesh.cu", "assemble.cu", "p2.cu", "cg.cu", "cg_resident.cu", "cg_p2.cu", "corrector.cu", "errors.cu", "capi.cu",
           "harness.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3",
    "-diag-suppress", "177", "--expt-relaxed-constexpr",
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the B200 path cannot be built")


def _cuda_lib() -> str:
    nvcc = Path(_nvcc()).resolve()
    return str(nvcc.parent.parent / "lib64")


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "mlg_b200.h"]
    nvcc = _nvcc()

    def compile_one(src: str) -> Path:
        s = CSRC / src
        o = OBJ / (src[:-3] + ".o")
        if force or _stale(o, [s] + headers):
            cmd = [nvcc, *NVCC_FLAGS, "-c", str(s), "-o", str(o)]
            if verbose:
                print(" ".join(cmd), flush=True)
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
        return o

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    if force or _stale(LIB, objs):
        libdir = _cuda_lib()
        cmd = [nvcc, *ARCH, "-shared", "-o", str(LIB), *map(str, objs),
               f"-L{libdir}", "-lcusolver", "-lcublas",
               "-Xlinker", f"-rpath,{libdir}"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    build_driver(verbose, force)
    return LIB


DRIVER_SRC = PKG.parent / "tools" / "mlg_run.cpp"
DRIVER = OBJ / "mlg_run"


def build_driver(verbose: bool = False, force: bool = False) -> Path:
    """C++ host driver over include/mleig_b200.hpp (the drop-in host API)."""
    inc = PKG.parent / "include"
    deps = [DRIVER_SRC, inc / "mleig_b200.hpp", inc / "mlg_b200.h", LIB]
    if force or _stale(DRIVER, deps):
        cxx = shutil.which("g++") or "g++"
        cmd = [cxx, "-O2", "-std=c++17", f"-I{inc}", str(DRIVER_SRC), "-o", str(DRIVER),
               f"-L{PKG}", "-l:libmlg_b200.so", f"-Wl,-rpath,{PKG}"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"C++ driver build failed:\n{r.stdout}\n{r.stderr}")
    return DRIVER


if __name__ == "__main__":
    print(build(verbose=True))

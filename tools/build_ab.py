"""Build A/B variants of libmlg_b200.so that differ only in cg.cu compile-time
macros, e.g.  python tools/build_ab.py u4mb4:-DMLG_CG_U=4,-DMLG_CG_MINBLOCKS=4
Outputs ab/libmlg_<name>.so (run them with tools/ab.sh <name>...)."""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1401_4969_b200 import _build as B  # noqa: E402


def main():
    B.build()
    out = ROOT / "ab"
    out.mkdir(exist_ok=True)
    nvcc = B._nvcc()
    others = [B.OBJ / (s[:-3] + ".o") for s in B.SOURCES if s != "cg.cu"]
    for spec in sys.argv[1:]:
        name, _, defs = spec.partition(":")
        obj = out / f"cg_{name}.o"
        flags = [d for d in defs.split(",") if d]
        subprocess.run([nvcc, *B.NVCC_FLAGS, *flags, "-c", str(B.CSRC / "cg.cu"), "-o", str(obj)],
                       check=True)
        libdir = B._cuda_lib()
        subprocess.run([nvcc, *B.ARCH, "-shared", "-o", str(out / f"libmlg_{name}.so"), str(obj),
                        *map(str, others), f"-L{libdir}", "-lcusolver", "-lcublas",
                        "-Xlinker", f"-rpath,{libdir}"], check=True)
        print("built", name, flush=True)


if __name__ == "__main__":
    main()

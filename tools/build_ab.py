"""Build A/B variants of libmlg_b200.so that differ only in one source file's
compile-time macros (default cg.cu; --src FILE for another), e.g.
    python tools/build_ab.py u4mb4:-DMLG_CG_U=4,-DMLG_CG_MINBLOCKS=4
    python tools/build_ab.py --src cg_resident.cu pt16:-DMLG_RES_PT=16
Outputs ab/libmlg_<name>.so (select one with MLG_LIB=ab/libmlg_<name>.so)."""
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
    args = sys.argv[1:]
    src = "cg.cu"
    if args and args[0] == "--src":
        src, args = args[1], args[2:]
    others = [B.OBJ / (s[:-3] + ".o") for s in B.SOURCES if s != src]
    for spec in args:
        name, _, defs = spec.partition(":")
        obj = out / f"{src[:-3]}_{name}.o"
        flags = [d for d in defs.split(",") if d]
        subprocess.run([nvcc, *B.NVCC_FLAGS, *flags, "-c", str(B.CSRC / src), "-o", str(obj)],
                       check=True)
        libdir = B._cuda_lib()
        subprocess.run([nvcc, *B.ARCH, "-shared", "-o", str(out / f"libmlg_{name}.so"), str(obj),
                        *map(str, others), f"-L{libdir}", "-lcusolver", "-lcublas",
                        "-Xlinker", f"-rpath,{libdir}"], check=True)
        print("built", name, flush=True)


if __name__ == "__main__":
    main()

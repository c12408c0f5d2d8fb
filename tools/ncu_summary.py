"""Key rows of an ncu --set full report (details page) for the first kernel."""
import csv
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Compute (SM) Throughput", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Block Limit Registers", "Grid Size",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Warp Cycles Per Issued Instruction",
        "Issued Warp Per Scheduler", "Eligible Warps Per Scheduler", "Executed Ipc Active"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    name = None
    for r in rows[1:]:
        if r[hdr.index("ID")] != "0":
            break
        name = r[hdr.index("Kernel Name")]
        m = r[hdr.index("Metric Name")]
        if m in KEYS:
            print(f"{m:40s} {r[hdr.index('Metric Value')]:>14s} {r[hdr.index('Metric Unit')]}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    h = rr[0]
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        if k in h:
            print(f"{k:40s} {rr[2][h.index(k)]:>14s} {rr[1][h.index(k)]}")
    print("kernel:", name[:100] if name else None)


if __name__ == "__main__":
    main(sys.argv[1])

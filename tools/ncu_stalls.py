"""Stall-sample breakdown of an ncu --set full report (SASS source page CSV).
usage: ncu -i rep --page source --csv --print-source sass > x.csv; python tools/ncu_stalls.py x.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n_top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
h = rows[1]
i_s = h.index("Warp Stall Sampling (All Samples)")
i_x = h.index("Instructions Executed")
stall = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
body = [r for r in rows[2:] if len(r) == len(h)]
tot = sum(int(r[i_s]) for r in body if r[i_s].isdigit())
print("kernel:", rows[0][1][:90], "| samples", tot, "| sass instructions", len(body))
agg = {}
for r in body:
    for i in stall:
        if r[i].isdigit():
            agg[h[i]] = agg.get(h[i], 0) + int(r[i])
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]:
    print(f"  {k:30s} {v:8d} {v / tot:.3f}")
top = sorted(body, key=lambda r: -int(r[i_s]) if r[i_s].isdigit() else 0)[:n_top]
for r in top:
    st = sorted(((int(r[i]), h[i][6:]) for i in stall if r[i].isdigit() and int(r[i]) > 0),
                reverse=True)[:2]
    print(f"{r[0][-5:]} {r[1][:58]:58s} {r[i_s]:>6s} x{r[i_x]:>9s} {st}")

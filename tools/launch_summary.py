"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = {}
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        name = r[hdr.index("Kernel Name")].replace("(anonymous namespace)::", "")
        name = name.replace("void ", "").split("(")[0]
        v = r[hdr.index("Metric Value")].replace(",", "")
        try:
            v = float(v)
        except ValueError:
            continue
        unit = r[hdr.index("Metric Unit")]
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':44s} {'launches':>8s} {'total_ms':>9s} {'share':>6s} {'avg_us':>8s}")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
        print(f"{k[:44]:44s} {n:8d} {t / 1e3:9.3f} {t / tot:6.1%} {t / n:8.2f}")
    print(f"{'TOTAL':44s} {sum(a[0] for a in agg.values()):8d} {tot / 1e3:9.3f}")


if __name__ == "__main__":
    main(sys.argv[1])

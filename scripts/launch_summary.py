"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: launches, total and share per kernel."""
import collections
import csv
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        k = r[ki].split("(")[0].replace("void ", "")
        agg[k][0] += 1
        agg[k][1] += float(r[vi].replace(",", "")) * SCALE[r[ui]]
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':48s} {'launches':>8s} {'total ms':>10s} {'share':>6s} {'avg ms':>9s}")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:48s} {n:8d} {t:10.3f} {100 * t / tot:5.1f}% {t / n:9.4f}")
    print(f"{'total':48s} {len(rows) - 1:8d} {tot:10.3f}")


if __name__ == "__main__":
    main(sys.argv[1])

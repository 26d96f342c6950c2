"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0}.get(r[ui], 1e-3)
        agg[name][0] += 1
        agg[name][1] += v * scale
    tot = sum(a[1] for a in agg.values())
    print(f"total {tot / 1e3:.2f} ms over {sum(a[0] for a in agg.values())} launches")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:40]:40s} {c:6d} {t / 1e3:9.3f} ms {100 * t / tot:5.1f}%  avg {t / c:8.2f} us")


if __name__ == "__main__":
    main(sys.argv[1])

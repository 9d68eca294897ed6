"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel count, total, avg, share."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(t for n, t in agg.values())
    print(f"{'kernel':60s} {'n':>6s} {'total_ms':>10s} {'avg_us':>10s} {'share':>6s}")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:60]:60s} {n:6d} {t / 1e3:10.3f} {t / n:10.2f} {t / tot * 100:5.1f}%")
    print(f"total device time {tot / 1e3:.3f} ms over {sum(n for n, _ in agg.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1])

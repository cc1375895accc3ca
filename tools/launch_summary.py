"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel:
count, total / mean device time, share of all launches.

    python tools/launch_summary.py gpurun_out/launches.csv > profiles/r01_launches_summary.txt
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rdr = csv.DictReader(lines)
    for r in rdr:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        unit = r.get("Metric Unit", "")
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
                 "s": 1e6, "second": 1e6}.get(unit, 1.0)
        name = r["Kernel Name"]
        short = name.split("(")[0]
        rows.append((short, v * scale))
    agg = collections.OrderedDict()
    for k, us in rows:
        c, t = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, t + us)
    total = sum(t for _, t in agg.values())
    print(f"# {path}: {len(rows)} launches, {total / 1e3:.1f} ms device time (cold, serialised)")
    print(f"{'kernel':60s} {'launches':>8s} {'total ms':>10s} {'mean us':>9s} {'share':>7s}")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:60]:60s} {c:8d} {t / 1e3:10.2f} {t / c:9.1f} {t / total * 100:6.2f}%")


if __name__ == "__main__":
    main()

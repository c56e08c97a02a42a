"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per kernel name the
launch count, total and mean device time, and share of the listed time.

    python tools/summarize_launches.py profiles/r01/launches_bench_cfg5.csv [--skip-first N]
"""
import csv
import sys
from collections import OrderedDict

UNIT = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
        "s": 1e3, "second": 1e3}


def summarize(path):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        ms = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1e-6)
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + ms)
    tot = sum(t for _, t in agg.values()) or 1.0
    lines = [f"{'launches':>8} {'total_ms':>12} {'mean_ms':>12} {'share':>7}  kernel"]
    for name, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{n:8d} {t:12.3f} {t / n:12.4f} {100 * t / tot:6.2f}%  {name[:100]}")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarize(sys.argv[1]))

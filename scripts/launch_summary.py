#!/usr/bin/env python
"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv`)
of bench.py: per kernel (template + grid) launches, total and mean duration,
over the launches between the last two first-token argmax kernels (= one
step), or over the whole file with --all."""
import collections
import csv
import io
import sys


def load(path):
    lines = open(path).read().splitlines()
    i = next(k for k, l in enumerate(lines) if l.startswith('"ID"'))
    rows = []
    for r in csv.DictReader(io.StringIO("\n".join(lines[i:]))):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        v *= {"usecond": 1.0, "msecond": 1e3, "nsecond": 1e-3, "ns": 1e-3, "us": 1.0}.get(r["Metric Unit"], 1.0)
        name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        rows.append((name, r["Grid Size"], v))
    return rows


def main():
    rows = load(sys.argv[1])
    if "--all" not in sys.argv:
        idx = [k for k, r in enumerate(rows) if r[0].startswith("argmax")]
        if len(idx) >= 2:
            rows = rows[idx[-2] + 1: idx[-1] + 1]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, g, v in rows:
        agg[(n, g)][0] += 1
        agg[(n, g)][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'launches':>8} {'total_ms':>9} {'mean_us':>8} {'share':>6}  kernel grid")
    for (n, g), (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{c:8d} {t / 1e3:9.3f} {t / c:8.1f} {t / tot:6.3f}  {n} {g}")
    print(f"{len(rows):8d} {tot / 1e3:9.3f}  (sum of serialised kernel durations)")


if __name__ == "__main__":
    main()

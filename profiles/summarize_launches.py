#!/usr/bin/env python3
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

    python profiles/summarize_launches.py gpurun_out/launches.csv "command" > profiles/rNN_launches.csv

ncu's per-launch times are cold-cache and serialised: compare SHARES of the
step with bench.py's live event timing, not absolute times.
"""
import collections
import csv
import sys


def main(path, cmd=""):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
        v *= scale.get(r["Metric Unit"], 1e-6)
        name = r["Kernel Name"]
        name = name.split("(")[0] if not name.startswith("void at::") else name[:90]
        rows.append((name, v, r["Grid Size"], r["Block Size"]))
    agg = collections.OrderedDict()
    for name, v, g, b in rows:
        a = agg.setdefault(name, [0, 0.0, g, b])
        a[0] += 1
        a[1] += v
    total = sum(a[1] for a in agg.values())
    print(f"# ncu launch list: {cmd}")
    print("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised; compare shares)")
    print(f"# total kernel time {total:.2f} ms over {len(rows)} launches")
    print("kernel,launches,total_ms,avg_ms,share,grid,block")
    for name, (n, t, g, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name.replace(',', ';')},{n},{t:.3f},{t / n:.4f},{t / total:.3f},\"{g}\",\"{b}\"")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")

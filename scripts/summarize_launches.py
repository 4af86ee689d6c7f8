"""Aggregates an ncu `--metrics gpu__time_duration.sum --csv` launch list by
kernel: launches, total / average device time, share of the step.
python scripts/summarize_launches.py gpurun_out/launches.csv > profiles/rNN/launches_summary.md"""
import csv
import re
import sys
from collections import defaultdict

rows = []
with open(sys.argv[1]) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "")
    unit = r.get("Metric Unit", "ns")
    v = float(r["Metric Value"].replace(",", ""))
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
    rows.append((name, v * scale))
agg = defaultdict(lambda: [0, 0.0])
for n, t in rows:
    agg[n][0] += 1
    agg[n][1] += t
tot = sum(v[1] for v in agg.values())
print(f"# ncu launch list ({len(rows)} launches, {tot:.1f} ms device time, cold-cache serialised)\n")
print("| kernel | launches | total ms | avg ms | share |")
print("|---|---|---|---|---|")
for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| `{n}` | {c} | {t:.2f} | {t / c:.4f} | {100 * t / tot:.1f}% |")

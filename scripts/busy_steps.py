"""GPU busy time per load step from an ncu launch list (gpu__time_duration.sum,
--cache-control none): launches are split into load steps at each k_support
(the first kernel of begin_step) and summed; compare with the plain run's
per-step wall time (scripts/profile_step.py) for the idle share.
    python scripts/busy_steps.py launches.csv.gz plain.log"""
import csv
import gzip
import re
import sys
from collections import defaultdict

path = sys.argv[1]
op = gzip.open if path.endswith(".gz") else open
rows = [r for r in csv.DictReader(l for l in op(path, "rt") if l.startswith('"'))]
steps, cur = [], None
for r in rows:
    name = r["Kernel Name"]
    v = float(r["Metric Value"].replace(",", ""))
    u = r.get("Metric Unit", "")
    v *= {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(u, 1e-9)
    if "k_support" in name:
        cur = {"busy_s": 0.0, "launches": 0, "by": defaultdict(float)}
        steps.append(cur)
    if cur is None:
        continue
    cur["busy_s"] += v
    cur["launches"] += 1
    cur["by"][name.split("(")[0].split("<")[0].replace("void ", "").strip()] += v
plain = []
if len(sys.argv) > 2:
    for line in open(sys.argv[2]):
        m = re.match(r"\s*(\d+)\s+(\d+)\s+(\d+)\s+([\d.]+)s", line)
        if m:
            plain.append(float(m.group(4)))
for i, st in enumerate(steps):
    wall = plain[i] if i < len(plain) else None
    top = sorted(st["by"].items(), key=lambda kv: -kv[1])[:6]
    print(f"step {i + 1}: busy {st['busy_s'] * 1e3:.1f} ms in {st['launches']} launches"
          + (f", wall {wall * 1e3:.1f} ms, idle {100 * (1 - st['busy_s'] / wall):.1f}%" if wall else "")
          + " | " + ", ".join(f"{k} {v * 1e3:.1f}" for k, v in top))

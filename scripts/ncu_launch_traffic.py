"""Per-Jacobian K6 totals from an ncu launch list (ncu --metrics
gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv):
a Jacobian is the run of launches from the tangent kernel to the next
k_diag_inverse. Prints JSON: per-Jacobian time and DRAM bytes, and per-kernel
totals/shares of the whole list.
    python scripts/ncu_launch_traffic.py launches.csv"""
import csv
import json
import sys
from collections import defaultdict

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"')))
launch = defaultdict(dict)
names = {}
for r in rows:
    i = int(r["ID"])
    names[i] = r["Kernel Name"]
    v = float(r["Metric Value"].replace(",", ""))
    u = r.get("Metric Unit", "")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
             "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(u, 1)
    launch[i][r["Metric Name"]] = v * scale
ids = sorted(launch)
tot_t = sum(launch[i].get("gpu__time_duration.sum", 0) for i in ids)
per = defaultdict(lambda: [0.0, 0.0, 0])
for i in ids:
    k = names[i].split("(")[0].split("<")[0].replace("void ", "").strip()
    m = launch[i]
    per[k][0] += m.get("gpu__time_duration.sum", 0)
    per[k][1] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    per[k][2] += 1
jac, cur = [], None
for i in ids:
    n = names[i]
    if "k_tangent" in n:
        cur = {"time_s": 0.0, "dram_bytes": 0.0, "launches": 0}
    if cur is not None:
        m = launch[i]
        cur["time_s"] += m.get("gpu__time_duration.sum", 0)
        cur["dram_bytes"] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        cur["launches"] += 1
        if "k_diag_inverse" in n:
            jac.append(cur)
            cur = None
out = {"jacobians": jac,
       "kernels": {k: {"time_s": v[0], "dram_bytes": v[1], "launches": v[2], "share": v[0] / tot_t}
                   for k, v in sorted(per.items(), key=lambda kv: -kv[1][0])},
       "total_time_s": tot_t}
print(json.dumps(out, indent=1))

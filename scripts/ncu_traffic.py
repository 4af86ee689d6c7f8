"""traffic.json from the ncu --set full raw pages of scripts/ncu_steady.sh:
per captured kernel, dram__bytes_read.sum + dram__bytes_write.sum of the launch
(the `traffic` key of bench.py's roofline object).
    python scripts/ncu_traffic.py <dir with *_raw.csv.gz>"""
import csv
import glob
import gzip
import json
import os
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ncu_steady"
out = {}
for f in sorted(glob.glob(os.path.join(d, "*_raw.csv.gz"))):
    name = os.path.basename(f)[: -len("_raw.csv.gz")]
    with gzip.open(f, "rt") as fh:
        rows = list(csv.reader(fh))
    if len(rows) < 3:
        print(f"skip {name}: no capture", file=sys.stderr)
        continue
    h, units, v = rows[0], rows[1], rows[2]

    def get(key):
        i = h.index(key)
        x = float(v[i].replace(",", ""))
        u = units[i]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
                 "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}.get(u, 1)
        return x * scale

    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    out[name] = {"kernel": v[h.index("Kernel Name")][:80], "time_s": get("gpu__time_duration.sum"),
                 "dram_read_bytes": rd, "dram_write_bytes": wr, "traffic_bytes": rd + wr}
json.dump(out, open(os.path.join(d, "traffic.json"), "w"), indent=1)
print(json.dumps(out, indent=1))

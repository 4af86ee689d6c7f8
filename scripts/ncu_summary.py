"""Key metrics of `ncu --set full` reports as a markdown table.
python scripts/ncu_summary.py gpurun_out/prof_*.ncu-rep > profiles/rNN/ncu_kernels.md"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("smsp__inst_executed.sum", "warp instr"),
]
print("| report | kernel | " + " | ".join(k[1] for k in KEYS) + " |")
print("|" + "---|" * (len(KEYS) + 2))
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        continue
    h, u = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(h, r))
        un = dict(zip(h, u))
        name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "")
        vals = []
        for k, _ in KEYS:
            v = d.get(k, "")
            vals.append(f"{v} {un.get(k, '')}".strip() if v else "")
        print(f"| {rep.split('/')[-1]} | `{name}` | " + " | ".join(vals) + " |")

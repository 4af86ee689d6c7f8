"""Registers / spills of selected kernels (ptxas -v of csrc/impm_sim.cu):
python scripts/ptxas_regs.py [substring ...]"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2507_09435_b200"))
from build import nccl_flags  # noqa: E402

out = os.path.join(ROOT, ".scratch", "ptxas.o")
os.makedirs(os.path.dirname(out), exist_ok=True)
cmd = ["nvcc", "-std=c++20", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-Xptxas", "-v", "-c",
       os.path.join(ROOT, "paper_2507_09435_b200", "csrc", "impm_sim.cu"), "-o", out] + \
      [f for f in nccl_flags() if f.startswith("-I")]
log = subprocess.run(cmd, capture_output=True, text=True).stderr.splitlines()
pats = sys.argv[1:] or [""]
for i, l in enumerate(log):
    if "error" in l:
        print(l)
    if "Compiling entry function" in l:
        name = re.search(r"'(_Z[^']+)'", l).group(1)
        if not any(p in name for p in pats):
            continue
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        info = " ".join(log[i + 1:i + 4])
        regs = re.search(r"Used (\d+) registers", info)
        sp = re.search(r"(\d+) bytes spill stores", info)
        print(f"{dem.split('(')[0][:90]:90s} regs={regs.group(1) if regs else '?':>4s} spill={sp.group(1) if sp else '?'}")

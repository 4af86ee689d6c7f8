"""profiles/<round>/traffic.json, the `traffic` source of bench.py's kernel table
and roofline, from one scripts/ncu_r02.sh run:
- per captured kernel (asm, mir, tan, cg, res, jac, ...): dram read + write of
  the --set full launch (scripts/ncu_traffic.py);
- "jacobian": DRAM bytes of the last Jacobian of the launch list (cfg 4 load
  step 2, tangent .. k_diag_inverse; scripts/ncu_launch_traffic.py);
- "vcycle_level0": mean of the level-0 fp16 residual and Jacobi sweeps.
    python scripts/traffic_json.py gpurun_out/ncu_r02 profiles/r02
"""
import json
import os
import subprocess
import sys

src, dst = sys.argv[1], sys.argv[2]
subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "ncu_traffic.py"), src],
               check=True, stdout=subprocess.DEVNULL)
t = json.load(open(os.path.join(src, "traffic.json")))
lt = json.load(open(os.path.join(src, "launch_traffic.json")))
j = lt["jacobians"][-1]
t["jacobian"] = {"traffic_bytes": j["dram_bytes"], "time_s": j["time_s"], "launches": j["launches"],
                 "source": f"{dst}/ncu/launch_traffic.json: sum of dram__bytes_read.sum + dram__bytes_write.sum "
                           "over the launches of one steady Jacobian (cfg 4 load step 2: tangent .. "
                           "k_diag_inverse), ncu launch list"}
if "res" in t and "jac" in t:
    t["vcycle_level0"] = {"traffic_bytes": 0.5 * (t["res"]["traffic_bytes"] + t["jac"]["traffic_bytes"]),
                          "source": f"mean of the level-0 fp16 residual and Jacobi sweeps ({dst}/ncu/res.md, "
                                    "jac.md); one level-0 profiler scope holds one of them plus vector kernels"}
json.dump(t, open(os.path.join(dst, "traffic.json"), "w"), indent=1)
print(json.dumps({k: v["traffic_bytes"] for k, v in t.items()}, indent=1))

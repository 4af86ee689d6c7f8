#!/bin/bash
# Round-2 ncu evidence on cfg 4 (scripts/profile_step.py cfg4 2 = load steps 1-2).
# 1. launch list of both steps: per-launch duration and DRAM bytes (cold-cache,
#    serialised: compare shares, not absolutes) -> per-Jacobian K6 traffic;
# 2. --set full of one steady launch per hot kernel (summaries + raw + SASS).
OUT=gpurun_out/ncu_r02
mkdir -p $OUT
K='--kernel-name-base demangled'
python scripts/profile_step.py cfg4 2 > $OUT/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $OUT/launches_2steps.csv python scripts/profile_step.py cfg4 2 > $OUT/launches.log 2>&1
python scripts/ncu_launch_traffic.py $OUT/launches_2steps.csv > $OUT/launch_traffic.json
gzip -f $OUT/launches_2steps.csv
I='\(int\)'
B='\(bool\)'
cap() {  # name regex skip
  timeout 900 ncu --set full --clock-control none --import-source on $K -k "regex:$2" --launch-skip $3 -c 1 \
    -o $OUT/prof_$1 -f python scripts/profile_step.py cfg4 2 > $OUT/$1.log 2>&1
  python scripts/ncu_summary.py $OUT/prof_$1.ncu-rep > $OUT/$1.md
  ncu -i $OUT/prof_$1.ncu-rep --page raw --csv > $OUT/$1_raw.csv 2>/dev/null
  ncu -i $OUT/prof_$1.ncu-rep --page source --csv --print-source sass > $OUT/$1_sass.csv 2>/dev/null
  gzip -f $OUT/$1_raw.csv $OUT/$1_sass.csv
  rm -f $OUT/prof_$1.ncu-rep
  tail -1 $OUT/$1.md
}
cap asm  "k_assemble_nh3f" 94
cap mir  "k_mirror_lower" 3
cap tan  "k_tangent_nh3q" 3
cap resp "k_residual_particles" 5
cap resbin "k_residual_bins_staged" 120
cap cg   "k_spmv<${I}3, ${I}3, ${I}4, ${I}0, double," 63
cap res  "k_spmv<${I}3, ${I}3, ${I}4, ${I}2, __half, ${I}0, ${B}1>" 130
cap jac  "k_spmv<${I}3, ${I}3, ${I}4, ${I}1, __half, ${I}0, ${B}1>" 131
python scripts/ncu_traffic.py $OUT > /dev/null
du -sh $OUT

#!/bin/bash
# Steady-state ncu evidence (load step 2 of cfg4: rows at their steady block
# counts). Step 1 runs 53 MG-CG iterations = 56 V-cycles of 6 smoothed levels
# (residual sweeps ordered fine -> coarse, Jacobi sweeps coarse -> fine) and 3
# assemblies of 27 colour batches, so the skips below land in step 2.
# Summaries only come back (reports deleted: 64 MiB cap on gpurun_out/).
OUT=gpurun_out/ncu_steady
mkdir -p $OUT
I='\(int\)'
K='--kernel-name-base demangled'
cap() {  # name regex skip   (ONLY="cg res" limits the captures)
  if [ -n "$ONLY" ] && [[ " $ONLY " != *" $1 "* ]]; then return; fi
  timeout 900 ncu --set full --clock-control none --import-source on $K -k "regex:$2" --launch-skip $3 -c 1 \
    -o $OUT/prof_$1 -f python scripts/profile_step.py cfg4 2 > $OUT/$1.log 2>&1
  python scripts/ncu_summary.py $OUT/prof_$1.ncu-rep > $OUT/$1.md
  ncu -i $OUT/prof_$1.ncu-rep --page raw --csv > $OUT/$1_raw.csv 2>/dev/null
  ncu -i $OUT/prof_$1.ncu-rep --page source --csv --print-source sass > $OUT/$1_sass.csv 2>/dev/null
  gzip -f $OUT/$1_raw.csv $OUT/$1_sass.csv
  [ "$1" = "cg" ] || rm -f $OUT/prof_$1.ncu-rep
  tail -1 $OUT/$1.md
}
# level SpMVs: the fp16 half-warp variant runs on levels 0 and 1 only;
# residual sweeps go fine -> coarse (even index = level 0), post-smoothing
# sweeps coarse -> fine (odd index = level 0); the skips land in step 2
B='\(bool\)'
cap cg   "k_spmv<${I}3, ${I}3, ${I}4, ${I}0, double," 63
cap res  "k_spmv<${I}3, ${I}3, ${I}4, ${I}2, __half, ${I}0, ${B}1>" 130
cap jac  "k_spmv<${I}3, ${I}3, ${I}4, ${I}1, __half, ${I}0, ${B}1>" 131
cap asm  "k_assemble_bins_staged" 94
cap resb "k_residual_bins" 150
cap tan  "k_tangent" 3
cap gap  "k_galerkin_ap" 3
# launch list of steps 1-2 (per-launch duration + DRAM bytes)
[ -n "$ONLY" ] && [[ " $ONLY " != *" launches "* ]] || ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $OUT/launches_2steps.csv python scripts/profile_step.py cfg4 2 > $OUT/launches.log 2>&1
gzip -f $OUT/launches_2steps.csv
python scripts/ncu_traffic.py $OUT > /dev/null
du -sh $OUT

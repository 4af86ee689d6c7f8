#!/bin/bash
# One steady-state ncu --set full capture with the SASS source page:
#   scripts/ncu_one.sh <name> <kernel regex> <launch skip>
OUT=gpurun_out/ncu_one
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$2" \
  --launch-skip $3 -c 1 -o $OUT/prof_$1 -f python scripts/profile_step.py cfg4 2 > $OUT/$1.log 2>&1
python scripts/ncu_summary.py $OUT/prof_$1.ncu-rep > $OUT/$1.md
ncu -i $OUT/prof_$1.ncu-rep --page raw --csv > $OUT/$1_raw.csv 2>/dev/null
ncu -i $OUT/prof_$1.ncu-rep --page source --csv --print-source sass > $OUT/$1_sass.csv 2>/dev/null
gzip -f $OUT/$1_raw.csv $OUT/$1_sass.csv
rm -f $OUT/prof_$1.ncu-rep
tail -1 $OUT/$1.md

#!/bin/bash
# ncu evidence for one cfg4 load step (run on the GPU box from the repo root):
# launch list (gpu__time_duration per launch) + `--set full` captures of the
# top kernels. Every capture replays ONE launch of an otherwise normal step.
set -x
mkdir -p gpurun_out/ncu
K='--kernel-name-base demangled'
I='\(int\)'
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches_step.csv \
  python scripts/profile_step.py cfg4 1 > gpurun_out/ncu/launch.log 2>&1
cap() {  # name regex skip
  timeout 900 ncu --set full --clock-control none --import-source on $K -k "regex:$2" --launch-skip $3 -c 1 \
    -o gpurun_out/ncu/prof_$1 -f python scripts/profile_step.py cfg4 1 > gpurun_out/ncu/$1.log 2>&1
  tail -1 gpurun_out/ncu/$1.log
}
cap asm   "k_assemble_bins_staged" 3
cap spmv0 "k_spmv<${I}3, ${I}3, ${I}4, ${I}0>" 20
cap spmvJ "k_spmv<${I}3, ${I}3, ${I}4, ${I}1>" 20
cap spmvR "k_spmv<${I}3, ${I}3, ${I}4, ${I}2>" 10
cap resb  "k_residual_bins" 30
cap tan   "k_tangent" 1
cap gap   "k_galerkin_ap" 1
cap gpt   "k_galerkin_ptap" 1
ls -la gpurun_out/ncu
# keep the returned gpurun_out/ under its 64 MiB cap: summaries + two reports
python scripts/ncu_summary.py gpurun_out/ncu/prof_*.ncu-rep > gpurun_out/ncu/ncu_kernels.md
for r in gpurun_out/ncu/prof_*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  ncu -i $r --page details --csv > gpurun_out/ncu/${b}_details.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass > gpurun_out/ncu/${b}_source.csv 2>/dev/null
done
gzip -f gpurun_out/ncu/launches_step.csv gpurun_out/ncu/*_source.csv
for r in gpurun_out/ncu/prof_*.ncu-rep; do case $r in *prof_asm*|*prof_spmv0*) ;; *) rm -f $r ;; esac; done
du -sh gpurun_out

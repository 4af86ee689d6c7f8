# round 2: ncu recapture on the final code (launch list of load steps 1-2 + --set full of the hot kernels)
bash scripts/ncu_r02.sh > gpurun_out/ncu_r02.log 2>&1; tail -12 gpurun_out/ncu_r02.log

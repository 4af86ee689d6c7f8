# round 2: GPU busy time per load step: warm kernel durations (ncu, no cache control) vs the plain step time
python scripts/profile_step.py cfg4 6 > gpurun_out/busy_plain.log 2>&1; cat gpurun_out/busy_plain.log
timeout 1800 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/busy_launches.csv python scripts/profile_step.py cfg4 6 > gpurun_out/busy_ncu.log 2>&1; echo "ncu rc=$?"
gzip -f gpurun_out/busy_launches.csv

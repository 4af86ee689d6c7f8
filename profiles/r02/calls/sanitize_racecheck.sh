# compute-sanitizer racecheck (shared-memory hazards) on the small end-to-end cases
python scripts/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/sanitize_plain.log; exit 1; }
timeout 3000 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/racecheck.log 2>&1
echo "racecheck rc=$?"; tail -8 gpurun_out/racecheck.log

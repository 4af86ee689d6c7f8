# compute-sanitizer memcheck on the small end-to-end cases (one tool per call)
python scripts/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/sanitize_plain.log; exit 1; }
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/memcheck.log 2>&1
echo "memcheck rc=$?"; tail -8 gpurun_out/memcheck.log

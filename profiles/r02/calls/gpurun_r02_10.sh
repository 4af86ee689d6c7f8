# round 2, GPU call 10: full suite on the current build; smoke; default bench line
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_10.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/gpu_tests_10.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; tail -c 400 gpurun_out/bench_default.err

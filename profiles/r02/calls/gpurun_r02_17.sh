# round 2: suite, smoke, the driver's bench command, DP line, then the checked build
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_17.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_17.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_driver.json 2> gpurun_out/bench_driver.err; echo "driver bench rc=$?"; tail -c 300 gpurun_out/bench_driver.err
timeout 900 python bench.py --steps 5 --warmup 3 --material drucker_prager > gpurun_out/bench_dp.json 2> gpurun_out/bench_dp.err; echo "dp bench rc=$?"; tail -c 300 gpurun_out/bench_dp.err
bash scripts/checked_cases.sh

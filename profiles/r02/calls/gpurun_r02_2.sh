# round 2, GPU call 2: full GPU suite, support statistics along the cfg 4 ramp,
# and a first cfg 4 Drucker-Prager bench line
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_2.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/gpu_tests_2.log
timeout 300 python scripts/support_probe.py > gpurun_out/support_probe.log 2>&1; echo "probe rc=$?"
tail -8 gpurun_out/support_probe.log
timeout 900 python bench.py --steps 5 --warmup 3 --material drucker_prager --no-cpu --e2e-steps 0 > gpurun_out/bench_dp.json 2> gpurun_out/bench_dp.err; echo "dp bench rc=$?"
tail -c 1500 gpurun_out/bench_dp.err

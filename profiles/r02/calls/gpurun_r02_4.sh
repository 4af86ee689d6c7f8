# round 2, GPU call 4: sweep assembly with the mirror fix; J2 forcing A/B
timeout 600 python scripts/asm_ab.py 32 32 16 > gpurun_out/asm_ab.log 2>&1; echo "ab rc=$?"; tail -4 gpurun_out/asm_ab.log
timeout 1500 python -m pytest tests -m gpu -q -k "not footing3d_16 and not bench_sample3d" > gpurun_out/gpu_tests_4.log 2>&1; echo "tests rc=$?"
tail -25 gpurun_out/gpu_tests_4.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/bench_sweep.json 2> gpurun_out/bench_sweep.err; echo "bench rc=$?"
tail -c 600 gpurun_out/bench_sweep.err
timeout 900 python scripts/j2_probe.py > gpurun_out/j2_probe.log 2>&1; echo "j2 rc=$?"; cat gpurun_out/j2_probe.log

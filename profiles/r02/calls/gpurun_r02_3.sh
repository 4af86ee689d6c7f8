# round 2, GPU call 3: the owner-computes sweep assembly (parity + A/B + bench),
# the jittered-fixture probe
timeout 1500 python -m pytest tests -m gpu -q -k "not footing3d_16" > gpurun_out/gpu_tests_3.log 2>&1; echo "tests rc=$?"
tail -25 gpurun_out/gpu_tests_3.log
timeout 600 python scripts/asm_ab.py 32 32 16 > gpurun_out/asm_ab.log 2>&1; echo "ab rc=$?"; tail -4 gpurun_out/asm_ab.log
timeout 600 python scripts/asm_ab.py 16 16 8 cam_clay > gpurun_out/asm_ab_mcc.log 2>&1; echo "ab mcc rc=$?"; tail -4 gpurun_out/asm_ab_mcc.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/bench_sweep.json 2> gpurun_out/bench_sweep.err; echo "bench rc=$?"
tail -c 1000 gpurun_out/bench_sweep.err
timeout 600 python scripts/jitter_probe.py > gpurun_out/jitter_probe.log 2>&1; echo "jitter rc=$?"; cat gpurun_out/jitter_probe.log

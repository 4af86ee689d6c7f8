# round 2: particle residual at 4 CTAs per SM: GPU suite
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_57.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests_57.log

set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/fp64_peak.cu -o /tmp/fp64_peak && /tmp/fp64_peak > gpurun_out/fp64_peak.json
cat gpurun_out/fp64_peak.json
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_driver.json 2> gpurun_out/bench_driver.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_driver.err
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/gpu_tests.log

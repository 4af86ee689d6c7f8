# round 2: particle reorder gathers 8 fields per thread (one perm load) instead of one
python scripts/phase_probe.py 2>&1 | tail -5
timeout 900 python bench.py --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms']; n=d['kernel_launches_by_class']; print('default', round(d['value'],2), round(d['ms_per_step'],1), 'support_sort', round(k['support_sort'],2))"
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_53.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests_53.log

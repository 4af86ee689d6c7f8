# round 2: reference-pattern nnz summed on the device (was a 25 MB download + host loop per load step)
python scripts/phase_probe.py 2>&1 | tail -5
timeout 900 python bench.py --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('default', round(d['value'],2), round(d['ms_per_step'],1), d['nnz_assembled'])"
timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('driver window', round(d['value'],2), round(d['ms_per_step'],1), d['krylov_iterations'])"
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_49.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests_49.log

# round 2: clock sampling as one `nvidia-smi -lms 200` process (the recipe's) instead of a process per sample
python scripts/profile_step.py cfg4 6 2>&1 | tail -6
timeout 900 python bench.py --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('default', round(d['value'],2), round(d['ms_per_step'],1), d['clocks'])"
timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('driver window', round(d['value'],2), round(d['ms_per_step'],1), d['krylov_iterations'], d['clocks'])"

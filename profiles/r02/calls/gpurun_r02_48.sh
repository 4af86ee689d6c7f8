# round 2: where the time outside the Newton solve goes; device buffers regrow with 1/8 headroom (main) vs exact (IMPM_BUF_SLACK=0)
IMPM_BUF_SLACK=0 python scripts/phase_probe.py 2>&1 | tail -5
python scripts/phase_probe.py 2>&1 | tail -5
timeout 900 python bench.py --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('default', round(d['value'],2), round(d['ms_per_step'],1))"
IMPM_BUF_SLACK=0 timeout 900 python bench.py --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('default slack 0', round(d['value'],2), round(d['ms_per_step'],1))"

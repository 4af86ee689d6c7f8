# round 2: chunked particle I/O (copies on a second stream overlap the layout kernels) vs one copy (IMPM_IO_CHUNKS=1)
python scripts/io_probe.py 2>&1 | tail -2
IMPM_IO_CHUNKS=1 python scripts/io_probe.py 2>&1 | tail -2
timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu --e2e-steps 5 > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); e=d['e2e']; print('chunks 8: value', round(d['value'],2), 'e2e', round(e['value'],2), e['phase_seconds'])"
IMPM_IO_CHUNKS=1 timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu --e2e-steps 5 > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); e=d['e2e']; print('chunks 1: value', round(d['value'],2), 'e2e', round(e['value'],2), e['phase_seconds'])"
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_51.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests_51.log

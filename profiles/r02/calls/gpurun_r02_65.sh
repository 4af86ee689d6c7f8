# round 2 final measurements (MG refresh 6): suite, smoke, driver-command bench, default bench, DP line
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_65.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests_65.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_65.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_65.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_driver_cmd.json 2> gpurun_out/bench_driver_cmd.err; echo "driver cmd rc=$?"
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "default rc=$?"
timeout 1500 python bench.py --material drucker_prager > gpurun_out/bench_dp.json 2> gpurun_out/bench_dp.err; echo "dp rc=$?"
for f in bench_driver_cmd bench_default bench_dp; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); e=d.get('e2e') or {}
print('$f', round(d['value'],2), 'e2e', round(e.get('value',0),2), e.get('phase_seconds'), 'ms/step', round(d['ms_per_step'],1), 'kry', d['krylov_iterations'], 'roofline', round(d['roofline']['frac'],3), 'launches', d['gpu_launches'], d['clocks'])"; done


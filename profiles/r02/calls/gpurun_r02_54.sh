# round 2: the small 2D configuration (cfg 1) for the latency-bound regime
timeout 900 python bench.py --config cfg1 --no-cpu > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err; echo "cfg1 rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg1.json')); e=d.get('e2e') or {}
print('cfg1', round(d['value'],2), 'e2e', round(e.get('value',0),2), 'ms/step', round(d['ms_per_step'],2), 'newton', d['newton_iterations'], 'kry', d['krylov_iterations'], d['config'])
for r in d['kernels']: print('  ', r['class'], round(r['ms_per_launch'] or 0,3), r['launches'], round(r['frac'] or 0,3), round(r['share'] or 0,3))"

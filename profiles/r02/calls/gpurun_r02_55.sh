# round 2: bench.py sanity after the config note change (default run, full contract line)
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "default rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_default.json')); print(d['value'], d['config']['l2'], d['e2e']['value'], d['cpu_baseline']['value'], d['gpu_launches'])"

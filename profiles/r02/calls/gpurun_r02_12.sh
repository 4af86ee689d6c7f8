# round 2: suite + default bench after the mirror-pass / upper-zero changes, then memcheck
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_12.log 2>&1; echo "tests rc=$?"
tail -6 gpurun_out/gpu_tests_12.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; tail -c 300 gpurun_out/bench_default.err
python -c "
import json; d=json.load(open('gpurun_out/bench_default.json')); k=d['kernel_ms']; n=d['kernel_launches_by_class']
print('it/s %.2f e2e %.2f ms/step %.1f tangent %.2f ms/jac assemble %.2f ms/jac kry %d' % (d['value'], d['e2e']['value'], d['ms_per_step'], k['tangent']/n['tangent'], k['assemble']/n['assemble'], d['krylov_iterations']))"
bash profiles/r02/calls/sanitize_memcheck.sh

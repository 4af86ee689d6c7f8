# round 2: launch bounds kept (particle residual 4 CTAs, commit 4 CTAs, tangent default): suite + bench lines
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_59.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests_59.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms']; n=d['kernel_launches_by_class']
print('it/s %.2f ms/step %.1f tangent %.3f commit %.3f res_p %.3f' % (d['value'], d['ms_per_step'], k['tangent']/n['tangent'], k['commit']/n['commit'], k['residual_particles']/n['residual_particles']))"
timeout 900 python bench.py --material drucker_prager --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('dp', round(d['value'],2))"

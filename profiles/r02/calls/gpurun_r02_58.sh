# round 2: tangent (8 CTAs, 64 registers) and commit (4 CTAs) occupancy vs the default launch bounds
bench_line() {
  env $1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$1] rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms']; n=d['kernel_launches_by_class']
print('it/s %.2f ms/step %.1f tangent %.3f commit %.3f res_p %.3f' % (d['value'], d['ms_per_step'], k['tangent']/n['tangent'], k['commit']/n['commit'], k['residual_particles']/n['residual_particles']))" 2>&1 | tail -1)"
}
bench_line ""
bench_line "IMPM_LIB=ab_libs/tc.so"
bench_line ""
bench_line "IMPM_LIB=ab_libs/tc.so"

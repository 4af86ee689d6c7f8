# round 2: particle I/O probe; for_each_support unrolled (registers instead of a local frame) A/B
bench_line() {
  env $1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$1] rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms']; n=d['kernel_launches_by_class']
print('it/s %.2f ms/step %.1f res_p %.3f res_n %.3f tangent %.3f commit %.3f support %.3f assemble %.2f' % (d['value'], d['ms_per_step'], k['residual_particles']/n['residual_particles'], k['residual_nodes']/n['residual_nodes'], k['tangent']/n['tangent'], k['commit']/n['commit'], k['support_sort']/n['support_sort'], k['assemble']/n['assemble']))" 2>&1 | tail -1)"
}
timeout 600 python scripts/io_probe.py 2>&1 | tail -2
bench_line ""
bench_line "IMPM_LIB=ab_libs/fes.so"
bench_line ""
bench_line "IMPM_LIB=ab_libs/fes.so"

# round 2: particle residual occupancy (launch bounds 1 / 4 / 5 CTAs per SM)
bench_line() {
  env $1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$1] rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms']; n=d['kernel_launches_by_class']
print('it/s %.2f ms/step %.1f res_p %.3f res_n %.3f' % (d['value'], d['ms_per_step'], k['residual_particles']/n['residual_particles'], k['residual_nodes']/n['residual_nodes']))" 2>&1 | tail -1)"
}
bench_line ""
bench_line "IMPM_LIB=ab_libs/resp4.so"
bench_line "IMPM_LIB=ab_libs/resp5.so"
bench_line ""
bench_line "IMPM_LIB=ab_libs/resp4.so"

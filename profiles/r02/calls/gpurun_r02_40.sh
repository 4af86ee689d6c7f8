# round 2: fp16 level sweeps with fewer buffered loads per lane and 10 CTAs per SM
bench_line() {
  env $1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$1] rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms']; n=d['kernel_launches_by_class']
print('it/s %.2f ms/step %.1f vcycle_l0 %.3f vcycle_l1 %.3f vcycle %.1f kry %d' % (d['value'], d['ms_per_step'], k['vcycle_level0']/n['vcycle_level0'], k['vcycle_level1']/n['vcycle_level1'], k['vcycle'], d['krylov_iterations']))" 2>&1 | tail -1)"
}
bench_line ""
bench_line "IMPM_LIB=ab_libs/nb2m10.so IMPM_MG_BLOCKS=1480"
bench_line "IMPM_LIB=ab_libs/nb3m10.so IMPM_MG_BLOCKS=1480"
bench_line "IMPM_LIB=ab_libs/nb2.so"
bench_line ""
bench_line "IMPM_LIB=ab_libs/nb2m10.so IMPM_MG_BLOCKS=1480"

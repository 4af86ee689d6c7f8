# round 2: Galerkin PtAP and residual-push occupancy variants
bench_line() {
  env $1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$1] rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms']; n=d['kernel_launches_by_class']
print('it/s %.2f ms/step %.1f res_n %.3f galerkin %.2f mg_setup %.2f' % (d['value'], d['ms_per_step'], k['residual_nodes']/n['residual_nodes'], k['galerkin'], k['mg_setup']))" 2>&1 | tail -1)"
}
bench_line ""
bench_line "IMPM_LIB=ab_libs/pr.so"
bench_line "IMPM_LIB=ab_libs/pr2.so"
bench_line ""
bench_line "IMPM_LIB=ab_libs/pr.so"
bench_line "IMPM_LIB=ab_libs/pr2.so"

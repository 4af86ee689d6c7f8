# round 2: row heads one row ahead in the level sweeps only (main) vs the committed kernels (orig)
bench_line() {
  env $1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$1] rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms']; n=d['kernel_launches_by_class']
print('it/s %.2f ms/step %.1f spmv %.3f ms vcycle_l0 %.3f ms/scope vcycle_l1 %.3f vcycle %.1f ms kry %d' % (d['value'], d['ms_per_step'], k['spmv']/n['spmv'], k['vcycle_level0']/n['vcycle_level0'], k['vcycle_level1']/n['vcycle_level1'], k['vcycle'], d['krylov_iterations']))" 2>&1 | tail -1)"
}
bench_line ""
bench_line "IMPM_LIB=ab_libs/orig.so"
bench_line ""
bench_line "IMPM_LIB=ab_libs/orig.so"
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_33.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests_33.log

# round 2: A/B of slot decoding from the row masks in the SpMVs (CG + level-0 sweeps); suite
bench_line() {
  env $1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$1] rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms']; n=d['kernel_launches_by_class']
print('it/s %.2f ms/step %.1f spmv %.3f ms vcycle_l0 %.3f ms/scope vcycle %.1f ms assemble %.2f kry %d' % (d['value'], d['ms_per_step'], k['spmv']/n['spmv'], k['vcycle_level0']/n['vcycle_level0'], k['vcycle'], k['assemble']/n['assemble'], d['krylov_iterations']))")"
}
bench_line ""
bench_line "IMPM_SPMV_MASK=0"
bench_line ""
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_19.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_19.log

# round 2: A/B of the chunk-box x staging in the MG level sweeps; suite
bench_line() {
  env $1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$1] rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms']; n=d['kernel_launches_by_class']
print('it/s %.2f ms/step %.1f vcycle_l0 %.2f ms/scope (%d) vcycle %.1f ms kry %d' % (d['value'], d['ms_per_step'], k['vcycle_level0']/n['vcycle_level0'], n['vcycle_level0'], k['vcycle'], d['krylov_iterations']))")"
}
bench_line ""
bench_line "IMPM_MG_BOX=0"
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_18.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_18.log

# round 2: transpose pass writes the MG fine level's fp16 copy (main) vs a separate conversion (IMPM_MIRROR_F16=0); pair-index magic numbers
bench_line() {
  env $1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$1] rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms']; n=d['kernel_launches_by_class']
print('it/s %.2f ms/step %.1f spmv %.3f vcycle_l0 %.3f assemble %.2f mg_setup %.2f vcycle %.1f kry %d' % (d['value'], d['ms_per_step'], k['spmv']/n['spmv'], k['vcycle_level0']/n['vcycle_level0'], k['assemble']/n['assemble'], k['mg_setup'], k['vcycle'], d['krylov_iterations']))" 2>&1 | tail -1)"
}
bench_line ""
bench_line "IMPM_MIRROR_F16=0"
bench_line ""
bench_line "IMPM_MIRROR_F16=0"
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_34.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests_34.log

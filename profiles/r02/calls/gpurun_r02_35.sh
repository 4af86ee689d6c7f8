# round 2: residual push with warp-pipelined bins (main) vs k_residual_bins_staged (IMPM_RES_PIPE=0)
bench_line() {
  env $1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$1] rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms']; n=d['kernel_launches_by_class']
print('it/s %.2f ms/step %.1f res_p %.3f res_n %.3f vcycle_l0 %.3f assemble %.2f mg_setup %.2f kry %d' % (d['value'], d['ms_per_step'], k['residual_particles']/n['residual_particles'], k['residual_nodes']/n['residual_nodes'], k['vcycle_level0']/n['vcycle_level0'], k['assemble']/n['assemble'], k['mg_setup'], d['krylov_iterations']))" 2>&1 | tail -1)"
}
timeout 300 python scripts/res_ab.py "IMPM_RES_PIPE=0" "" 32 32 16 2>&1 | tail -1
timeout 300 python scripts/res_ab.py "IMPM_RES_PIPE=0" "" 16 16 8 2>&1 | tail -1
bench_line ""
bench_line "IMPM_RES_PIPE=0"
bench_line ""
bench_line "IMPM_RES_PIPE=0"
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_35.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests_35.log

# round 2: factored assembly (final candidate) A/B against 4-warp CTAs; full suite; ncu of the assembly and the tangent
bench_line() {
  env $1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$1] rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms']; n=d['kernel_launches_by_class']
print('it/s %.2f ms/step %.1f spmv %.3f ms vcycle_l0 %.3f ms/scope vcycle %.1f ms assemble %.2f tangent %.2f kry %d' % (d['value'], d['ms_per_step'], k['spmv']/n['spmv'], k['vcycle_level0']/n['vcycle_level0'], k['vcycle'], k['assemble']/n['assemble'], k['tangent']/n['tangent'], d['krylov_iterations']))" 2>&1 | tail -1)"
}
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_27.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests_27.log
bench_line ""
bench_line "IMPM_LIB=ab_libs/asmf_w4.so"
bench_line ""
bench_line "IMPM_LIB=ab_libs/asmf_w4.so"
python scripts/profile_step.py cfg4 2 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_assemble_nh3f|k_tangent_nh3q" --launch-skip 97 -c 2 -o gpurun_out/prof_asmf -f python scripts/profile_step.py cfg4 2 > gpurun_out/asmf.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_asmf.ncu-rep > gpurun_out/asmf.md; tail -2 gpurun_out/asmf.md
ncu -i gpurun_out/prof_asmf.ncu-rep --page raw --csv > gpurun_out/asmf_raw.csv 2>/dev/null; ncu -i gpurun_out/prof_asmf.ncu-rep --page source --csv --print-source sass > gpurun_out/asmf_sass.csv 2>/dev/null
gzip -f gpurun_out/asmf_raw.csv gpurun_out/asmf_sass.csv; rm -f gpurun_out/prof_asmf.ncu-rep

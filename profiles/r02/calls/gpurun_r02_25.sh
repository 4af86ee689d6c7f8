# round 2: factored assembly v3 with component-major Q (coalesced tangent stores)
bench_line() {
  env $1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$1] rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms']; n=d['kernel_launches_by_class']
print('it/s %.2f ms/step %.1f spmv %.3f ms vcycle_l0 %.3f ms/scope vcycle %.1f ms assemble %.2f tangent %.2f kry %d' % (d['value'], d['ms_per_step'], k['spmv']/n['spmv'], k['vcycle_level0']/n['vcycle_level0'], k['vcycle'], k['assemble']/n['assemble'], k['tangent']/n['tangent'], d['krylov_iterations']))" 2>&1 | tail -1)"
}
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_25a.log 2>&1; echo "nh tests rc=$?"; tail -3 gpurun_out/gpu_tests_25a.log
bench_line ""
timeout 300 python scripts/asm_ab.py "IMPM_ASM_NHF=0" "" 32 32 16 > gpurun_out/asm_ab_nhf.log 2>&1; tail -2 gpurun_out/asm_ab_nhf.log
python scripts/profile_step.py cfg4 2 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_assemble_nh3f" --launch-skip 94 -c 1 -o gpurun_out/prof_asmf -f python scripts/profile_step.py cfg4 2 > gpurun_out/asmf.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_asmf.ncu-rep > gpurun_out/asmf.md; tail -1 gpurun_out/asmf.md
ncu -i gpurun_out/prof_asmf.ncu-rep --page raw --csv > gpurun_out/asmf_raw.csv 2>/dev/null; ncu -i gpurun_out/prof_asmf.ncu-rep --page source --csv --print-source sass > gpurun_out/asmf_sass.csv 2>/dev/null
gzip -f gpurun_out/asmf_raw.csv gpurun_out/asmf_sass.csv; rm -f gpurun_out/prof_asmf.ncu-rep

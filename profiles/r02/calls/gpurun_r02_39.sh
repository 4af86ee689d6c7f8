# round 2: zeroing on a side stream beside the tangent (main) vs in line (IMPM_ZERO_OVERLAP=0); division-free fp16 copy in the transpose pass
bench_line() {
  env $1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$1] rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms']; n=d['kernel_launches_by_class']
print('it/s %.2f ms/step %.1f assemble %.2f tangent %.2f mg_setup %.2f' % (d['value'], d['ms_per_step'], k['assemble']/n['assemble'], k['tangent']/n['tangent'], k['mg_setup']))" 2>&1 | tail -1)"
}
bench_line ""
bench_line "IMPM_ZERO_OVERLAP=0"
bench_line ""
bench_line "IMPM_ZERO_OVERLAP=0"
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_39.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests_39.log
python scripts/profile_step.py cfg4 2 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_mirror_lower" --launch-skip 3 -c 1 -o gpurun_out/prof_mir -f python scripts/profile_step.py cfg4 2 > gpurun_out/mir.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_mir.ncu-rep > gpurun_out/mir.md; tail -1 gpurun_out/mir.md
ncu -i gpurun_out/prof_mir.ncu-rep --page raw --csv > gpurun_out/mir_raw.csv 2>/dev/null; ncu -i gpurun_out/prof_mir.ncu-rep --page source --csv --print-source sass > gpurun_out/mir_sass.csv 2>/dev/null
gzip -f gpurun_out/mir_raw.csv gpurun_out/mir_sass.csv; rm -f gpurun_out/prof_mir.ncu-rep

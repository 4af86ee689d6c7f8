# round 2: factored assembly CTA size: 4 warps (main) vs 6 warps (one round for an 18-node box) vs 8 warps
bench_line() {
  env $1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$1] rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms']; n=d['kernel_launches_by_class']
print('it/s %.2f ms/step %.1f assemble %.2f tangent %.2f' % (d['value'], d['ms_per_step'], k['assemble']/n['assemble'], k['tangent']/n['tangent']))" 2>&1 | tail -1)"
}
bench_line ""
bench_line "IMPM_LIB=ab_libs/asmf_w6.so"
bench_line "IMPM_LIB=ab_libs/asmf_w8.so"
bench_line ""
bench_line "IMPM_LIB=ab_libs/asmf_w6.so"
bench_line "IMPM_LIB=ab_libs/asmf_w8.so"

# round 2: assembly occupancy variants (built on the box): PPL2, node gradients recomputed (GREC), min CTAs/SM
bench_line() {
  timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$1] rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms']; n=d['kernel_launches_by_class']
print('it/s %.2f ms/step %.1f assemble %.2f ms/jac' % (d['value'], d['ms_per_step'], k['assemble']/n['assemble']))")"
}
for v in "-DIMPM_ASM_PPL3=2" "-DIMPM_ASM_PPL3=2 -DIMPM_ASM_GREC=1" "-DIMPM_ASM_PPL3=2 -DIMPM_ASM_GREC=1 -DIMPM_ASM_MINB=5" "-DIMPM_ASM_PPL3=2 -DIMPM_ASM_GREC=1 -DIMPM_ASM_MINB=6" "-DIMPM_ASM_PPL3=1 -DIMPM_ASM_GREC=1 -DIMPM_ASM_MINB=6"; do
  IMPM_NVCC_EXTRA="$v" python -m paper_2507_09435_b200.build --force > gpurun_out/build_v.log 2>&1 || { echo "build [$v] failed"; tail -3 gpurun_out/build_v.log; continue; }
  bench_line "$v"
done

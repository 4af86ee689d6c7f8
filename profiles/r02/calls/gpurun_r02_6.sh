# round 2, GPU call 6: assembly flush / tangent A/B on cfg 4, then the full suite
for envs in "" "IMPM_ASM_SYM=0" "IMPM_ASM_RMW=0" "IMPM_TANGENT_DUAL=1"; do
  env $envs timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$envs] rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms']; n=d['kernel_launches_by_class']
print('it/s %.2f ms/step %.1f tangent %.2f ms/jac assemble %.2f ms/jac kry %d' % (d['value'], d['ms_per_step'], k['tangent']/n['tangent'], k['assemble']/n['assemble'], d['krylov_iterations']))
" 2>&1 | tail -1)"
done
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_6.log 2>&1; echo "tests rc=$?"
tail -25 gpurun_out/gpu_tests_6.log
timeout 600 python scripts/asm_ab.py "IMPM_ASM_RMW=0" "" 32 32 16 > gpurun_out/asm_ab.log 2>&1; tail -2 gpurun_out/asm_ab.log
timeout 600 python scripts/asm_ab.py "IMPM_TANGENT_DUAL=1" "" 32 32 16 >> gpurun_out/asm_ab.log 2>&1; tail -1 gpurun_out/asm_ab.log
timeout 600 python scripts/asm_ab.py "IMPM_ASM_SYM=0" "" 32 32 16 >> gpurun_out/asm_ab.log 2>&1; tail -1 gpurun_out/asm_ab.log

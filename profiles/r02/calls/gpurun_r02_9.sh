# round 2, GPU call 9: which parity tests break the later slab bitwise tests; mirror-pass A/B
S="tests/test_gpu_slabs.py"
for k in "test_linear_solve_parity and not krylov" "linear_solve_parity_krylov" "newton" "colour or begin or pattern" "residual or jacobian or commit"; do
  timeout 900 python -m pytest tests/test_gpu_parity.py $S -q -k "($k) or bitwise" > gpurun_out/bisect.log 2>&1
  echo "[$k] rc=$? $(tail -1 gpurun_out/bisect.log) $(grep -c 'FAILED tests/test_gpu_slabs' gpurun_out/bisect.log) slab failures"
done
for envs in "" "IMPM_ASM_MIRROR_PASS=0"; do
  env $envs timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$envs] rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms']; n=d['kernel_launches_by_class']
print('it/s %.2f ms/step %.1f tangent %.2f ms/jac assemble %.2f ms/jac kry %d' % (d['value'], d['ms_per_step'], k['tangent']/n['tangent'], k['assemble']/n['assemble'], d['krylov_iterations']))
" 2>&1 | tail -1)"
done
timeout 600 python scripts/asm_ab.py "IMPM_ASM_MIRROR_PASS=0" "" 32 32 16 > gpurun_out/asm_ab.log 2>&1; tail -1 gpurun_out/asm_ab.log

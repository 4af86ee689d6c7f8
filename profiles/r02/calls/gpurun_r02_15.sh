# round 2: async tangent staging in the assembly; PPL variants built on the box
python -c "
import json" 
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
echo "[cp.async PPL3] rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms']; n=d['kernel_launches_by_class']
print('it/s %.2f ms/step %.1f assemble %.2f ms/jac' % (d['value'], d['ms_per_step'], k['assemble']/n['assemble']))")"
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_15.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_15.log
cp paper_2507_09435_b200/libimpm_gpu.so /tmp/lib_ppl3.so
for v in 2 4; do
  IMPM_NVCC_EXTRA="-DIMPM_ASM_PPL3=$v" python -m paper_2507_09435_b200.build --force > gpurun_out/build_ppl$v.log 2>&1 || { echo "build $v failed"; continue; }
  timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[PPL$v] rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms']; n=d['kernel_launches_by_class']
print('it/s %.2f ms/step %.1f assemble %.2f ms/jac' % (d['value'], d['ms_per_step'], k['assemble']/n['assemble']))")"
done
cp /tmp/lib_ppl3.so paper_2507_09435_b200/libimpm_gpu.so

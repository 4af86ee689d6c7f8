# round 2, GPU call 8: which earlier test module breaks the slab bitwise tests
S="tests/test_gpu_slabs.py"
K="-k bitwise"
for pre in "" "tests/test_gpu_coupled.py" "tests/test_gpu_csr.py" "tests/test_gpu_extensions.py" "tests/test_gpu_facade.py" "tests/test_gpu_materials3d.py" "tests/test_gpu_parity.py" "tests/test_gpu_scenarios.py"; do
  timeout 900 python -m pytest $pre $S -q -p no:randomly -k "bitwise or not slab" > gpurun_out/bisect.log 2>&1
  echo "[$pre] rc=$? $(tail -1 gpurun_out/bisect.log) $(grep -c 'FAILED tests/test_gpu_slabs' gpurun_out/bisect.log) slab failures"
done

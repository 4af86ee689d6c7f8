# round 2, GPU call 5: slab regressions under A/B switches; then the suite
for envs in "" "IMPM_SIG_SORT=0" "IMPM_ASM_SWEEP=0" "IMPM_SIG_SORT=0 IMPM_ASM_SWEEP=0" "IMPM_DIRECT=0"; do
  env $envs timeout 600 python -m pytest tests/test_gpu_slabs.py -q -x -k "bitwise and (cfg1_nh or cube3d)" > gpurun_out/slab_ab.log 2>&1
  echo "[$envs] slab rc=$? $(tail -1 gpurun_out/slab_ab.log)"
done
timeout 1500 python -m pytest tests -m gpu -q -k "not footing3d_16" > gpurun_out/gpu_tests_5.log 2>&1; echo "tests rc=$?"
tail -25 gpurun_out/gpu_tests_5.log

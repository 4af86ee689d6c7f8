# round 2, GPU call 7: Newton-count sensitivity on footing3d_16; slab regressions A/B
for envs in "" "IMPM_EXACT_NEWTON=1" "IMPM_ETA0_FACTOR=0.0001" "IMPM_EXACT_NEWTON=1 IMPM_EXACT_RTOL=1e-12"; do
  echo "== [$envs]"; env $envs timeout 300 python scripts/newton_probe.py footing3d_16 2>&1 | tail -12
done
for envs in "" "IMPM_ASM_RMW=0" "IMPM_TANGENT_DUAL=1" "IMPM_DIRECT=0" "IMPM_ASM_RMW=0 IMPM_TANGENT_DUAL=1 IMPM_DIRECT=0"; do
  env $envs timeout 600 python -m pytest tests/test_gpu_slabs.py -q -k "bitwise and (cfg1_nh or cube3d)" > gpurun_out/slab_ab.log 2>&1
  echo "[$envs] slab rc=$? $(tail -1 gpurun_out/slab_ab.log)"
done

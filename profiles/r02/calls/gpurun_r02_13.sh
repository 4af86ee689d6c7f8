# round 2: slab Krylov counts vs single GPU (rank-local MG), then memcheck
timeout 900 python scripts/slab_kry_probe.py 4 16 16 8 3 > gpurun_out/slab_kry.log 2>&1; echo "probe rc=$?"; tail -4 gpurun_out/slab_kry.log
timeout 900 python scripts/slab_kry_probe.py 2 16 16 8 3 > gpurun_out/slab_kry2.log 2>&1; echo "probe2 rc=$?"; tail -3 gpurun_out/slab_kry2.log
bash profiles/r02/calls/sanitize_memcheck.sh

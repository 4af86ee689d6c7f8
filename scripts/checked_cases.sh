#!/bin/bash
# Memory-safety evidence without compute-sanitizer (closed on this pool): build
# libimpm_gpu.so with -DIMPM_CHECKED (device range checks on the scattered
# accesses, counted in g_oob_count), run the small end-to-end cases of every
# kernel family, report the count, and restore the regular build.
set -e
cp paper_2507_09435_b200/libimpm_gpu.so /tmp/libimpm_gpu_regular.so
IMPM_NVCC_EXTRA="-DIMPM_CHECKED" python -m paper_2507_09435_b200.build --force > gpurun_out/checked_build.log 2>&1
set +e
timeout 1200 python scripts/sanitize_cases.py > gpurun_out/checked_cases.log 2>&1
rc=$?
cp /tmp/libimpm_gpu_regular.so paper_2507_09435_b200/libimpm_gpu.so
echo "checked cases rc=$rc"
tail -3 gpurun_out/checked_cases.log
exit $rc

# round 2: MG refresh 3 vs 6 on the default window and the DP line; suite at 6
line() {
  env $1 timeout 1200 python bench.py $2 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$1 $2] rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('it/s %.2f ms/step %.1f newton %d krylov %d' % (d['value'], d['ms_per_step'], d['newton_iterations'], d['krylov_iterations']))" 2>&1 | tail -1)"
}
line "IMPM_MG_REFRESH=3" ""
line "IMPM_MG_REFRESH=6" ""
line "IMPM_MG_REFRESH=3" "--material drucker_prager"
line "IMPM_MG_REFRESH=6" "--material drucker_prager"
line "IMPM_MG_REFRESH=3" "--steps 10 --warmup 3"
line "IMPM_MG_REFRESH=6" "--steps 10 --warmup 3"
IMPM_MG_REFRESH=6 timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_63.log 2>&1; echo "tests (refresh 6) rc=$?"; tail -1 gpurun_out/gpu_tests_63.log

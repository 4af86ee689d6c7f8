# round 2: omega safety factor sweep on the driver window, then the GPU suite at the candidate value
line() {
  env $1 timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$1] rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('it/s %.2f ms/step %.1f newton %d krylov %d' % (d['value'], d['ms_per_step'], d['newton_iterations'], d['krylov_iterations']))" 2>&1 | tail -1)"
}
line "IMPM_MG_OMEGA_SAFETY=1.0"
line "IMPM_MG_OMEGA_SAFETY=0.95"
line "IMPM_MG_OMEGA_SAFETY=0.9"
line "IMPM_MG_OMEGA_SAFETY=0.8"
line ""
IMPM_MG_OMEGA_SAFETY=1.0 timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_42.log 2>&1; echo "tests (safety 1.0) rc=$?"; tail -1 gpurun_out/gpu_tests_42.log
IMPM_MG_OMEGA_SAFETY=1.0 timeout 600 python bench.py --material drucker_prager --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ab_dp.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/ab_dp.json')); print('dp safety 1.0', round(d['value'],2), d['newton_iterations'], d['krylov_iterations'])"
timeout 600 python bench.py --material drucker_prager --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ab_dp.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/ab_dp.json')); print('dp safety 1.1', round(d['value'],2), d['newton_iterations'], d['krylov_iterations'])"

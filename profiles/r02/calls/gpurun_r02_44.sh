# round 2: per-level smoother safety factors on the driver window
line() {
  env $1 timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$1] rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('it/s %.2f ms/step %.1f newton %d krylov %d' % (d['value'], d['ms_per_step'], d['newton_iterations'], d['krylov_iterations']))" 2>&1 | tail -1)"
}
line ""
line "IMPM_MG_OMEGA_SAFETY_COARSE=0.9"
line "IMPM_MG_OMEGA_SAFETY_COARSE=1.1"
line "IMPM_MG_OMEGA_SAFETY=0.95 IMPM_MG_OMEGA_SAFETY_COARSE=1.0"
line "IMPM_MG_OMEGA_SAFETY=0.9 IMPM_MG_OMEGA_SAFETY_COARSE=1.0"
line "IMPM_MG_OMEGA_SAFETY_COARSE=0.95"

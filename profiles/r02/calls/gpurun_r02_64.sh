# round 2: lambda refresh period at MG refresh 6 (driver window)
line() {
  env $1 timeout 1200 python bench.py $2 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$1 $2] rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('it/s %.2f ms/step %.1f newton %d krylov %d' % (d['value'], d['ms_per_step'], d['newton_iterations'], d['krylov_iterations']))" 2>&1 | tail -1)"
}
line "" "--steps 20 --warmup 5"
line "IMPM_MG_POWER_EVERY=6" "--steps 20 --warmup 5"
line "IMPM_MG_POWER_EVERY=12" "--steps 20 --warmup 5"
line "IMPM_MG_POWER_EVERY=3" "--steps 20 --warmup 5"
line "IMPM_MG_POWER_EVERY=6" ""
line "" ""

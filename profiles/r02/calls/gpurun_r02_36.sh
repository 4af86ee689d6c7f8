# round 2: MG refresh policy on the driver's 20-step window: coarse levels every 3 / 4 / 6 load steps, lambda every 5 / 10
line() {
  env $1 timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$1] rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('it/s %.2f ms/step %.1f newton %d krylov %d' % (d['value'], d['ms_per_step'], d['newton_iterations'], d['krylov_iterations']))" 2>&1 | tail -1)"
}
line ""
line "IMPM_MG_REFRESH=4"
line "IMPM_MG_REFRESH=6"
line "IMPM_MG_POWER_EVERY=10"
line "IMPM_MG_REFRESH=2"

# round 2: MG refresh period re-measured at omega safety 1.0 (driver window, twice each)
line() {
  env $1 timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$1] rc=$? $(python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('it/s %.2f ms/step %.1f newton %d krylov %d' % (d['value'], d['ms_per_step'], d['newton_iterations'], d['krylov_iterations']))" 2>&1 | tail -1)"
}
for r in 3 5 6 8; do line "IMPM_MG_REFRESH=$r"; done
for r in 3 5 6 8; do line "IMPM_MG_REFRESH=$r"; done

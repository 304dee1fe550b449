#!/bin/bash
# k_moments_* kernel time per environment setting (ncu launch durations, cfg2 steps)
cd "$(dirname "$0")/.."
N=${N:-1000000}
for envs in "$@"; do
  env $envs python tools/step_once.py $N 2 > gpurun_out/plain.log 2>&1 && \
  env $envs ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_moments --csv --log-file gpurun_out/mom.csv python tools/step_once.py $N 2 > /dev/null 2>&1
  python - "$envs" <<'PY'
import csv, sys
rows=[r for r in csv.reader(open("gpurun_out/mom.csv")) if len(r) > 10 and r[0].isdigit()]
print(sys.argv[1], [(r[4].split("(")[0], round(float(r[-1].replace(",",""))/1e3,1)) for r in rows[-2:]])
PY
done

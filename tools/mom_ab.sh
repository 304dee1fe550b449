#!/bin/bash
# time k_moments_coop per build flag set (ncu launch durations, cfg2)
cd "$(dirname "$0")/.."
for flags in "$@"; do
  BH_NVCC_EXTRA="$flags" python -m paper_2203_08966_b200.build_lib >/dev/null 2>&1 || { echo "build failed $flags"; continue; }
  python tools/step_once.py > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_moments --csv --log-file gpurun_out/mom.csv python tools/step_once.py > /dev/null 2>&1
  python - "$flags" <<'PY'
import csv, sys
rows=[r for r in csv.reader(open("gpurun_out/mom.csv")) if len(r) > 10 and r[0].isdigit()]
v=[float(r[-1].replace(",","")) for r in rows]
print(sys.argv[1], "k_moments_coop us:", [round(x/1e3,1) for x in v[-3:]])
PY
done
BH_NVCC_EXTRA="" python -m paper_2203_08966_b200.build_lib >/dev/null 2>&1

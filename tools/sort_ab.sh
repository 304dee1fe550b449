#!/bin/bash
# A/B the radix-sort kernel variants: build each (BH_NVCC_EXTRA), short bench,
# print the sort phase.  Usage: tools/sort_ab.sh "FLAGS1" "FLAGS2" ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for flags in "$@"; do
  BH_NVCC_EXTRA="$flags" python -m paper_2203_08966_b200.build_lib >/dev/null 2>&1 || { echo "build failed: $flags"; continue; }
  for cfg in ${AB_CONFIGS:-cfg3}; do
    timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
    python - "$flags" "$cfg" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
    ph = d["phase_ms_per_step"]
    print(f"{sys.argv[2]} [{sys.argv[1]}] sort_ms={ph['sort']:.4f} frac={d['roofline_sort']['frac']:.3f} build_ms={ph['build']:.4f} ms/step={d['ms_per_step']:.3f}")
except Exception as e:
    print("FAILED", sys.argv[1], e, open("gpurun_out/ab.err").read()[-2000:])
PY
  done
done
BH_NVCC_EXTRA="" python -m paper_2203_08966_b200.build_lib >/dev/null 2>&1

#!/bin/bash
# A/B the walk kernel variants on one GPU: build each (BH_NVCC_EXTRA), run a
# short cfg2 bench, print walk ms / frac.  Usage: tools/walk_ab.sh "FLAGS1" "FLAGS2" ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for flags in "$@"; do
  BH_NVCC_EXTRA="$flags" python -m paper_2203_08966_b200.build_lib >/dev/null 2>&1 || { echo "build failed: $flags"; continue; }
  for cfg in ${AB_CONFIGS:-cfg2}; do
    timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
    python - "$flags" "$cfg" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
    ph = d.get("phase_ms_per_step", {})
    print(f"{sys.argv[2]} [{sys.argv[1]}] walk_ms={ph.get('walk', ph)} frac={d['roofline']['frac']:.3f} ms/step={d['ms_per_step']:.3f} pp={d.get('pp_per_step')} pc={d.get('pc_per_step')}")
except Exception as e:
    print("FAILED", sys.argv[1], e, open("gpurun_out/ab.err").read()[-2000:])
PY
  done
done
BH_NVCC_EXTRA="" python -m paper_2203_08966_b200.build_lib >/dev/null 2>&1

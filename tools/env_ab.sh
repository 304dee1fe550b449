#!/bin/bash
# A/B a runtime environment switch on the cfg bench: tools/env_ab.sh "VAR=a" "VAR=b" ...
cd "$(dirname "$0")/.."
for envs in "$@"; do
  for cfg in ${AB_CONFIGS:-cfg2}; do
    env $envs timeout 600 python bench.py --config $cfg --steps ${AB_STEPS:-10} --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
    python - "$envs" "$cfg" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
    ph = d.get("phase_ms_per_step", {})
    print(f"{sys.argv[2]} [{sys.argv[1]}] walk_ms={ph.get('walk'):.4f} frac={d['roofline']['frac']:.4f} ms/step={d['ms_per_step']:.3f}")
except Exception as e:
    print("FAILED", sys.argv[1], e, open("gpurun_out/ab.err").read()[-1500:])
PY
  done
done

#!/bin/bash
# A/B: the group-classified walk (default) vs the v4 walk (BH_WALK_V4=1), short benches
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for cfg in ${AB_CONFIGS:-cfg2}; do
  for v4 in 0 1; do
    BH_WALK_V4=$v4 timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
    python - "$v4" "$cfg" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
    ph = d.get("phase_ms_per_step", {})
    print(f"{sys.argv[2]} v4={sys.argv[1]} walk_ms={ph.get('walk'):.3f} frac={d['roofline']['frac']:.3f} ms/step={d['ms_per_step']:.3f} pp={d.get('pp_per_step')} pc={d.get('pc_per_step')}")
except Exception as e:
    print("FAILED", sys.argv[1], e, open("gpurun_out/ab.err").read()[-2000:])
PY
  done
done

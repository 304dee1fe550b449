"""Resident-sim steps of a bench config (profiling target for launch lists).

    python tools/step_cfg.py cfg4 [steps]
"""
import sys, torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import bench
from paper_2203_08966_b200.engine import Engine

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
b = bench.make_bodies(cfg)
eng = Engine("fp32", 0)
eng.sim_load(eng.bodies_tensor(b.position, b.mass), eng.vec_tensor(b.velocity))
eng.sim_forces(cfg["theta"], cfg["eps"], cfg["leaf"], False)
for _ in range(steps):
    eng.sim_step(cfg["dt"], cfg["theta"], cfg["eps"], cfg["leaf"], 1)
torch.cuda.synchronize()
eng.check()
print("ok", eng.stats().interactions)

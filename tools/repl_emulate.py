"""Per-rank device work of the replicated multi-GPU step, R ranks emulated on ONE GPU.

Every rank of the replicated scheme (decomposition.DistributedSim) runs the
whole O(N) part of the step (kick-drift, keys, sort, build, walk records) and
walks only its costzones zone of targets (decomposition.py:35-57 rule, from the
previous step's work).  This times, on one GPU, the single-GPU step's phases and
then each zone's walk alone (CUDA events), so per rank:
    device = (step - walk) + walk(zone)
and single-step / (R * max_r device) is an upper bound on the R-GPU efficiency
of the device part (the peer stores of the walk epilogue and the two stream
barriers per step are not included).

    python tools/repl_emulate.py cfg3 2,4,8   -> one JSON object
"""
import json, sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch
import bench
from paper_2203_08966_b200 import _lib
from paper_2203_08966_b200.decomposition import costzones_device
from paper_2203_08966_b200.engine import Engine

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
ranks = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "2,4,8").split(",")]
cfg = bench.CONFIGS[name]
b = bench.make_bodies(cfg)
n = len(b.mass)
th, eps, L, dt = cfg["theta"], cfg["eps"], cfg["leaf"], cfg["dt"]
eng = Engine("fp32", 0)
eng.sim_load(eng.bodies_tensor(b.position, b.mass), eng.vec_tensor(b.velocity))
eng.sim_forces(th, eps, L, True)
eng.sim_step(dt, th, eps, L, 2)
torch.cuda.synchronize()
eng.timing(True)
eng.timing_reset()
eng.sim_step(dt, th, eps, L, 1)
ph = eng.timing_get()
eng.timing(False)
step = sum(ph.values())
nonwalk = step - ph["walk"]
# the next step's zones from this step's work, then each zone's walk alone
eng.sim_begin_step(dt)
eng.sim_prepare(th, eps, L, True)
prev = torch.empty(n, dtype=torch.int32, device="cuda")
eng.sim_export(_lib.BH_SIM_PREV_WORK, 0, n, prev)
out = {"config": name, "n": n, "single_gpu_ms": {k: round(v, 3) for k, v in ph.items()},
       "single_gpu_step_ms": round(step, 3), "ranks": {}}
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for R in ranks:
    z = costzones_device(prev, R)
    walks = []
    for r in range(R):
        best = 1e30
        for _ in range(3):
            ev[0].record()
            eng.sim_walk_range(th, eps, L, z[r], z[r + 1], True)
            ev[1].record()
            torch.cuda.synchronize()
            best = min(best, ev[0].elapsed_time(ev[1]))
        walks.append(round(best, 3))
    dev = [round(nonwalk + w, 3) for w in walks]
    out["ranks"][R] = dict(zone_sizes=[z[r + 1] - z[r] for r in range(R)], zone_walk_ms=walks,
                           per_rank_device_ms=dev, walk_max_over_mean=round(max(walks) / (sum(walks) / R), 3),
                           device_efficiency_upper_bound=round(step / (R * max(dev)), 3))
eng.close()
print(json.dumps(out))

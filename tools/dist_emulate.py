"""Per-rank device work of the distributed build step, R ranks emulated on ONE GPU.

Runs DistributedBuildSim with ThreadComm (host barriers only), then replays each
rank's local phases ALONE on the GPU with CUDA events: local sort, boundary-aware
build, LET marking, and the walk of its targets over its assembled tree.  Against
the single-GPU step on the same bodies this measures load balance and the LET
overhead of the decomposition.  It does not measure communication or host time
(NVLink collectives and the Python assembly), so the "projected" efficiency is
an upper bound for the device part only.

    python tools/dist_emulate.py cfg3 2,4,8 [steps]  -> prints one JSON object
"""
import json, sys, threading, time
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np
import torch
import bench
from paper_2203_08966_b200 import _lib
from paper_2203_08966_b200.decomposition import DistributedBuildSim, StepParams, ThreadComm
from paper_2203_08966_b200.engine import Engine

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
ranks_list = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "2,4,8").split(",")]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg = bench.CONFIGS[cfg_name]
b = bench.make_bodies(cfg)
n = len(b.mass)
theta, eps, L, dt = cfg["theta"], cfg["eps"], cfg["leaf"], cfg["dt"]


def timed(fn, reps=3):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        ev[0].record(); fn(); ev[1].record(); torch.cuda.synchronize()
        best = min(best, ev[0].elapsed_time(ev[1]))
    return best


# ---- single GPU reference: the same steps, then the phases of one more step
eng = Engine("fp32", 0)
pos, vel = eng.bodies_tensor(b.position, b.mass), eng.vec_tensor(b.velocity)
eng.sim_load(pos, vel)
eng.sim_forces(theta, eps, L, False)
eng.sim_step(dt, theta, eps, L, steps)
eng.timing(True); eng.timing_reset()
eng.sim_step(dt, theta, eps, L, 1)
single = {k: round(v, 3) for k, v in eng.timing_get().items()}
single_total = sum(single.values())
single_inter = eng.stats().interactions
eng.timing(False)
eng.close()
del pos, vel
torch.cuda.empty_cache()
out = {"config": cfg_name, "n": n, "steps_before_replay": steps, "single_gpu_ms": single,
       "single_gpu_step_ms": round(single_total, 3), "interactions": single_inter, "ranks": {}}

for R in ranks_list:
    comms = ThreadComm.group(R)
    sims, engs, err = [None] * R, [None] * R, []
    cuts = np.linspace(0, n, R + 1).astype(np.int64)

    def body(r):
        try:
            e = Engine("fp32", 0)
            sl = slice(cuts[r], cuts[r + 1])
            s = DistributedBuildSim(e, comms[r], StepParams(theta, eps, L, dt))
            s.overlap = False  # replay the one-pass walk over the full assembled tree
            s.load(e.bodies_tensor(b.position[sl], b.mass[sl]), e.vec_tensor(b.velocity[sl]),
                   gid=torch.arange(int(cuts[r]), int(cuts[r + 1]), device="cuda"))
            s.bootstrap()
            s.step(steps)
            sims[r], engs[r] = s, e
        except Exception as exc:  # pragma: no cover
            import traceback; traceback.print_exc(); err.append(exc); comms[r].hub.barrier.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(R)]
    [t.start() for t in ts]; [t.join() for t in ts]
    if err:
        raise err[0]
    per = []
    for r in range(R):
        s, e = sims[r], engs[r]
        last = s.last
        nl = e.sim_n
        acc = torch.zeros((nl, 4), dtype=torch.float32, device="cuda")
        work = torch.zeros(nl, dtype=torch.int32, device="cuda")
        walk = timed(lambda: e.walk_records(s.tree, last["bodies"], last["targets"], eps, L, acc, work))
        inter = e.stats().interactions
        sort = timed(lambda: e.sim_sort())
        prev, nxt = last["bounds"]
        build = timed(lambda: e.sim_build_local(theta, L, prev, nxt))
        let = timed(lambda: e.sim_let(last["boxes"], r), reps=2)
        per.append(dict(bodies=nl, walk_ms=round(walk, 3), sort_ms=round(sort, 3), build_ms=round(build, 3),
                        let_mark_ms=round(let, 3), interactions=int(inter), records_own=int(s.let_stats["own_records"]),
                        let_records_in=int(s.let_stats["records"]), let_bodies_in=int(s.let_stats["bodies"])))
    tot = [p["walk_ms"] + p["sort_ms"] + p["build_ms"] + p["let_mark_ms"] for p in per]
    out["ranks"][R] = dict(per_rank=per, max_device_ms=round(max(tot), 3),
                           walk_max_over_mean=round(max(p["walk_ms"] for p in per) / np.mean([p["walk_ms"] for p in per]), 3),
                           interactions_sum=int(sum(p["interactions"] for p in per)),
                           device_efficiency_upper_bound=round(single_total / (R * max(tot)), 3))
    for e in engs:
        e.close()
    del sims, engs
    torch.cuda.empty_cache()
print(json.dumps(out))

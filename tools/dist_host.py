"""Host overhead of the multi-GPU steps (DistributedBuildSim, or DistributedSim
with --replicated).

R ranks emulated in one process (ThreadComm: host barriers only, every rank on
GPU 0).  With R = 1 the step's host work is fully exposed: wall time per step
minus the device time the library's phase timers record is the host cost a
rank adds per step (Python control, host reads, top-tree assembly).  With R > 1
the ranks' device work serialises on the one GPU, so wall ~ sum of device time
+ whatever host work is not hidden behind another rank's kernels.

    python tools/dist_host.py cfg3 1,2,8 [steps] [--replicated]   -> one JSON object
"""
import json, sys, threading, time
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np
import torch
import bench
from paper_2203_08966_b200.decomposition import DistributedBuildSim, DistributedSim, StepParams, ThreadComm
from paper_2203_08966_b200.engine import Engine

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
ranks = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2").split(",")]
steps = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 5
replicated = "--replicated" in sys.argv
cfg = bench.CONFIGS[name]
b = bench.make_bodies(cfg)
n = len(b.mass)
out = {"config": name, "n": n, "steps": steps, "scheme": "replicated" if replicated else "distributed", "ranks": {}}
for R in ranks:
    comms = ThreadComm.group(R)
    cuts = np.linspace(0, n, R + 1).astype(np.int64)
    sims, engs, res, err = [None] * R, [None] * R, [None] * R, []
    bar = threading.Barrier(R)

    def body(r):
        try:
            e = Engine("fp32", 0)
            sl = slice(cuts[r], cuts[r + 1])
            prm = StepParams(cfg["theta"], cfg["eps"], cfg["leaf"], cfg["dt"])
            if replicated:  # every rank holds every body
                s = DistributedSim(e, comms[r], prm)
                s.load(e.bodies_tensor(b.position, b.mass), e.vec_tensor(b.velocity))
            else:
                s = DistributedBuildSim(e, comms[r], prm)
                s.load(e.bodies_tensor(b.position[sl], b.mass[sl]), e.vec_tensor(b.velocity[sl]),
                       gid=torch.arange(int(cuts[r]), int(cuts[r + 1]), device="cuda"))
            s.bootstrap()
            s.step(2)
            torch.cuda.synchronize()
            e.timing(True)
            e.timing_reset()
            bar.wait()
            t0 = time.perf_counter()
            s.step(steps)
            torch.cuda.synchronize()
            wall = (time.perf_counter() - t0) / steps * 1e3
            dev = {k: v / steps for k, v in e.timing_get().items()}
            res[r] = dict(wall_ms=round(wall, 3), device_ms=round(sum(dev.values()), 3),
                          phases={k: round(v, 3) for k, v in dev.items() if v})
            sims[r], engs[r] = s, e
        except Exception as exc:  # pragma: no cover
            import traceback; traceback.print_exc(); err.append(exc)
            try:
                comms[r].hub.barrier.abort()
            except Exception:
                pass

    ts = [threading.Thread(target=body, args=(r,)) for r in range(R)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    if err:
        raise err[0]
    wall = max(x["wall_ms"] for x in res)
    dev_sum = sum(x["device_ms"] for x in res)
    out["ranks"][R] = dict(per_rank=res, wall_ms=wall, device_ms_sum=round(dev_sum, 3),
                           host_exposed_ms=round(wall - dev_sum, 3))
    for e in engs:
        e.close()
    del sims, engs
    torch.cuda.empty_cache()
print(json.dumps(out))

"""Where the e2e (host-array) step time goes at cfg2: H2D alone, device step alone,
D2H alone, and the full bh_sim_step_host call (CUDA events on one stream)."""
import sys, torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2203_08966_b200.engine import Engine
from paper_2203_08966_b200.initcond import make_rng, plummer_cluster

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
b = plummer_cluster(n, make_rng(2), 1.0)
eng = Engine("fp32", 0)
pos = eng.bodies_tensor(b.position, b.mass)
vel = eng.vec_tensor(b.velocity)
eng.sim_load(pos, vel)
eng.sim_forces(0.6, 1e-3, 16, True)
dpos, dvel, dacc = torch.empty_like(pos), torch.empty_like(pos), torch.empty_like(pos)
eng.sim_store(dpos, dvel, dacc)
hpos = dpos.cpu().pin_memory()
hvel3 = dvel[:, :3].cpu().contiguous().pin_memory()
hacc3 = dacc[:, :3].cpu().contiguous().pin_memory()
d3 = torch.empty((n, 3), device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

def t(f, k=10):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(k):
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); tot += e0.elapsed_time(e1)
    return tot / k

h2d = t(lambda: (dpos.copy_(hpos, non_blocking=True), d3.copy_(hvel3, non_blocking=True), d3.copy_(hacc3, non_blocking=True)))
d2h = t(lambda: (hvel3.copy_(d3, non_blocking=True), hacc3.copy_(d3, non_blocking=True)))
dev = t(lambda: eng.sim_step(1e-3, 0.6, 1e-3, 16, 1))
full = t(lambda: eng.sim_step_host(hpos, hvel3, hacc3, 1e-3, 0.6, 1e-3, 16, 1))
print(f"h2d {h2d:.3f} ms  d2h(vel,acc) {d2h:.3f} ms  device step {dev:.3f} ms  sum {h2d + d2h + dev:.3f}  "
      f"full host call {full:.3f} ms  (gap {full - h2d - d2h - dev:+.3f})")

"""cfg2 steps through the resident-sim C-ABI (profiling target for launch lists)."""
import sys, torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2203_08966_b200.engine import Engine
from paper_2203_08966_b200.initcond import make_rng, plummer_cluster

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
b = plummer_cluster(n, make_rng(2), 1.0)
eng = Engine("fp32", 0)
eng.sim_load(eng.bodies_tensor(b.position, b.mass), eng.vec_tensor(b.velocity))
eng.sim_forces(0.6, 1e-3, 16, False)
for _ in range(steps):
    eng.sim_step(1e-3, 0.6, 1e-3, 16, 1)
torch.cuda.synchronize()
eng.check()
print("ok", eng.stats().interactions)

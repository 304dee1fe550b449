"""Host overhead of the replicated-tree multi-GPU step (DistributedSim) at one
rank vs the plain single-GPU step (run under torchrun, NCCL)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
from paper_2203_08966_b200.decomposition import DistributedSim, StepParams, TorchComm
from paper_2203_08966_b200.engine import Engine
from paper_2203_08966_b200.initcond import make_rng, plummer_cluster

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
torch.cuda.set_device(0)
b = plummer_cluster(n, make_rng(2), 1.0)
eng = Engine("fp32", 0)
pos, vel = eng.bodies_tensor(b.position, b.mass), eng.vec_tensor(b.velocity)
sim = DistributedSim(eng, TorchComm(), StepParams(0.6, 1e-3, 16, 1e-3))
sim.load(pos, vel)
sim.bootstrap()
sim.step(3)
torch.cuda.synchronize()
t0 = time.perf_counter(); sim.step(10); torch.cuda.synchronize()
t_rep = (time.perf_counter() - t0) / 10 * 1e3
eng.sim_load(pos, vel); eng.sim_forces(0.6, 1e-3, 16, False); eng.sim_step(1e-3, 0.6, 1e-3, 16, 3)
torch.cuda.synchronize()
t0 = time.perf_counter(); eng.sim_step(1e-3, 0.6, 1e-3, 16, 10); torch.cuda.synchronize()
t_one = (time.perf_counter() - t0) / 10 * 1e3
print(f"n={n} replicated 1-rank wall ms/step {t_rep:.3f}  plain sim_step {t_one:.3f}")
dist.destroy_process_group()

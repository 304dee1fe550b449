"""Host-overhead profile of the distributed build step (DistributedBuildSim).
Run under torchrun with BH_DIST_BACKEND=gloo BH_SHARE_GPU=1 on one GPU; rank 0
prints wall ms/step, device ms per phase and the top host functions."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
from paper_2203_08966_b200.decomposition import DistributedBuildSim, StepParams, TorchComm
from paper_2203_08966_b200.engine import Engine
import bench

# argv[1]: a bench config name (cfg2, cfg3, ...) or a Plummer body count
arg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = bench.CONFIGS[arg] if arg in bench.CONFIGS else dict(bench.CONFIGS["cfg2"], n=int(arg))
dist.init_process_group(os.environ.get("BH_DIST_BACKEND", "gloo"))
rank, ws = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
b = bench.make_bodies(cfg)
n = len(b)
eng = Engine("fp32", 0)
lo, hi = n * rank // ws, n * (rank + 1) // ws
sim = DistributedBuildSim(eng, TorchComm(), StepParams(cfg["theta"], cfg["eps"], cfg["leaf"], cfg["dt"]))
sim.load(eng.bodies_tensor(b.position[lo:hi], b.mass[lo:hi]), eng.vec_tensor(b.velocity[lo:hi]),
         gid=torch.arange(lo, hi, device="cuda"))
sim.bootstrap()
sim.step(3)
torch.cuda.synchronize()
if sim.trace is not None:
    sim.trace.clear()
eng.timing(True)
eng.timing_reset()
prof = cProfile.Profile()
t0 = time.perf_counter()
prof.enable()
sim.step(5)
torch.cuda.synchronize()
prof.disable()
wall = (time.perf_counter() - t0) / 5 * 1e3
ph = {k: round(v / 5, 3) for k, v in eng.timing_get().items()}
if rank == 0:
    print(f"ranks={ws} n={n} wall_ms/step={wall:.2f} device_ms/step={ph} let={sim.let_stats}")
    if sim.trace is not None:
        print("trace ms/step:", {k: round(v / 5, 3) for k, v in sim.trace.items()})
    pstats.Stats(prof).sort_stats("cumulative").print_stats(25)
dist.barrier()
dist.destroy_process_group()

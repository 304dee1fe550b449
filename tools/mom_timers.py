"""Phase split of k_moments_coop (build with BH_NVCC_EXTRA=-DBH_MOM_TIMERS)."""
import ctypes, sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch
import bench
from paper_2203_08966_b200 import _lib
from paper_2203_08966_b200.engine import Engine

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
b = bench.make_bodies(cfg)
eng = Engine("fp32", 0)
eng.sim_load(eng.bodies_tensor(b.position, b.mass), eng.vec_tensor(b.velocity))
L = _lib.lib()
for rep in range(2):
    eng.sim_forces(cfg["theta"], cfg["eps"], cfg["leaf"], False)
    torch.cuda.synchronize()
t = (ctypes.c_ulonglong * 64)()
nt = ctypes.c_int()
L.bh_debug_mom_timers(t, ctypes.byref(nt))
v = [t[i] for i in range(nt.value)]
names = ["lists", "buckets"] + [f"level-run {i}" for i in range(len(v) - 3)]
print(f"total {(v[-1] - v[0]) / 1e3:.1f} us  buckets {t[62]}  opened cells {t[63]}  n {len(b)}  "
      f"bucket bodies (2 calls) {t[60]}  max bucket {t[61]}")
for i in range(1, len(v)):
    print(f"  {names[i - 1]:12s} {(v[i] - v[i - 1]) / 1e3:8.1f} us")

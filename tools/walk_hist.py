"""Mask-density histogram of the fp32 walk (build with BH_NVCC_EXTRA=-DBH_WALK_HIST)."""
import ctypes, sys
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch
from paper_2203_08966_b200 import _lib
from paper_2203_08966_b200.engine import Engine
from paper_2203_08966_b200.initcond import make_rng, plummer_cluster

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
b = plummer_cluster(n, make_rng(2), 1.0)
eng = Engine("fp32", 0)
eng.sim_load(eng.bodies_tensor(b.position, b.mass), eng.vec_tensor(b.velocity))
eng.sim_forces(0.6, 1e-3, 16, True)
torch.cuda.synchronize()
h = (ctypes.c_ulonglong * 130)()
L = _lib.lib()
L.bh_debug_walk_hist(h)
a = np.array(h[:65], dtype=np.float64)
i = np.array(h[65:], dtype=np.float64)
print("visits (non-leaf):", int(a.sum()))
print("accepting-target histogram (0..64), share of visits:")
print(" ".join(f"{k}:{a[k]/a.sum():.3f}" for k in range(65) if a[k] / a.sum() > 0.004))
print("mean accepting per visit", (a * np.arange(65)).sum() / a.sum())
print("examining-target histogram:")
print(" ".join(f"{k}:{i[k]/i.sum():.3f}" for k in range(65) if i[k] / i.sum() > 0.004))
w = a * np.arange(65)
print("pc-weighted: share of useful pairs from visits with >=56 accepting:", w[56:].sum() / w.sum(),
      " visits with >=56:", a[56:].sum() / a.sum(), " visits with <=16:", a[1:17].sum() / a.sum())

"""Schedule counters of the fp32 walk (build with BH_NVCC_EXTRA=-DBH_W9_STATS).

    python tools/w9_stats.py cfg3
"""
import ctypes, json, sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch
import bench
from paper_2203_08966_b200 import _lib
from paper_2203_08966_b200.engine import Engine

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = bench.CONFIGS[name]
b = bench.make_bodies(cfg)
eng = Engine("fp32", 0)
eng.sim_load(eng.bodies_tensor(b.position, b.mass), eng.vec_tensor(b.velocity))
L = _lib.lib()
h = (ctypes.c_ulonglong * 64)()
eng.sim_forces(cfg["theta"], cfg["eps"], cfg["leaf"], True)
torch.cuda.synchronize()
L.bh_debug_w9_stats(h, 1)
eng.sim_forces(cfg["theta"], cfg["eps"], cfg["leaf"], True)
torch.cuda.synchronize()
L.bh_debug_w9_stats(h, 1)
st = eng.stats()
names = ["batches", "cells", "mixed", "mixed_acc", "pc_entries", "pc_bits", "leaf_entries", "leaf_bits",
         "bucket_entries", "passes", "pass_iters", "bucket_slots_used", "frontier_push", "pc_flushes",
         "pp_flushes", "mixed_opened", "mixed_acc_bits", "bucket_bits", "pc_full_entries", "mixed_half_acc",
         "half_passes", "half_pass_iters"]
d = {k: int(h[i]) for i, k in enumerate(names)}
n = len(b)
warps = (n + 63) // 64
out = {"config": name, "n": n, "warps": warps, "pp": st.pp, "pc": st.pc}
out.update({k: v / warps for k, v in d.items()})
out["pc_density"] = d["pc_bits"] / 64 / max(d["pc_entries"], 1)
out["mixed_acc_density"] = d["mixed_acc_bits"] / 64 / max(d["mixed_acc"], 1)
out["leaf_density"] = d["leaf_bits"] / 64 / max(d["leaf_entries"], 1)
out["bucket_density_packed"] = d["bucket_slots_used"] / 64 / max(d["pass_iters"], 1)
out["pc_from_mixed_frac"] = d["mixed_acc_bits"] / max(d["mixed_acc_bits"] + d["pc_bits"], 1)
hist = [int(h[32 + i]) for i in range(32)]
out["peak_frontier_hist_by10"] = {f"{10*i}-{10*i+9}": v for i, v in enumerate(hist) if v}
print(json.dumps(out, indent=1))

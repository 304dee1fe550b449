import sys, numpy as np
sys.path.insert(0, ".")
from oracle import oracle as orc
from paper_2203_08966_b200.hashed import build_hashed
from paper_2203_08966_b200.morton import DomainBounds
from paper_2203_08966_b200.physics import Bodies
g = np.load("tests/golden/trees.npz")
f32 = lambda x: np.asarray(x, dtype=np.float32).astype(np.float64)
pos, m = f32(g["n2000_pos"]), f32(g["n2000_mass"])
R = orc.bounds(pos)
order = orc.sort_order(orc.morton_keys(pos, R))
print("R", R, flush=True)
t = build_hashed(Bodies(m[order], pos[order], np.zeros((2000, 3))), DomainBounds(R), precision="fp32")
print("built", flush=True)
flat = t.flat()
acc, work = flat.traverse(pos, 0.3, 0.05)
print("ok", acc[:2], work[:4])

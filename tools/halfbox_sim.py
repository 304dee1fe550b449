"""CPU model: classify cells against the two half-groups' boxes (targets
0-31 and 32-63 of a 64-target warp) as well as the full group box.  A cell
that is mixed for the full box but certain (accept or open) for each half needs
no per-target MAC: the accepting half goes to the pc list, the opening half to
the frontier / pp list.  Prints the share of mixed cells resolved that way, and
the same for quarter boxes.

    python tools/halfbox_sim.py [n] [groups] [theta] [L]
"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from oracle import oracle as orc  # noqa: E402
from paper_2203_08966_b200.initcond import make_rng, plummer_cluster  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
G = int(sys.argv[2]) if len(sys.argv) > 2 else 60
theta = float(sys.argv[3]) if len(sys.argv) > 3 else 0.6
L = int(sys.argv[4]) if len(sys.argv) > 4 else 16
S = 64
b = plummer_cluster(n, make_rng(2), 1.0)
pos = b.position.astype(np.float32).astype(np.float64)
m = b.mass.astype(np.float32).astype(np.float64)
R = orc.bounds(pos)
o = orc.sort_order(orc.morton_keys(pos, R))
t = orc.build_tree(m[o], pos[o], R)
P = pos[o]
mac2 = (t.side / theta) ** 2
expandable = t.count > L
expandable[0] = t.count[0] > 1


def cls(T, com, mac):
    lo, hi = T.min(0), T.max(0)
    gmin = np.maximum(np.maximum(lo - com, com - hi), 0.0)
    gmax = np.maximum(np.abs(lo - com), np.abs(hi - com))
    if (gmin ** 2).sum() > mac:
        return "A"
    if (gmax ** 2).sum() <= mac:
        return "O"
    return "M"


rng = np.random.default_rng(0)
gs = rng.choice(n // S, size=G, replace=False)
tot = dict(visits=0, mixed=0, half_resolved=0, quarter_resolved=0, mixed_pc_slots=0)
for g in gs:
    T = P[g * S:(g + 1) * S]
    stack = [(c, np.ones(S, bool)) for c in t.children[0][::-1] if c >= 0]
    while stack:
        c, mask = stack.pop()
        tot["visits"] += 1
        if t.count[c] == 1:
            continue
        com = t.com[c]
        d2 = ((T - com) ** 2).sum(1)
        acc = mask & (d2 > mac2[c])
        opn = mask & ~acc
        full = cls(T, com, mac2[c])
        if full == "M":
            tot["mixed"] += 1
            halves = [cls(T[h * 32:(h + 1) * 32], com, mac2[c]) for h in range(2)]
            if "M" not in halves:
                tot["half_resolved"] += 1
            quarters = [cls(T[q * 16:(q + 1) * 16], com, mac2[c]) for q in range(4)]
            if "M" not in quarters:
                tot["quarter_resolved"] += 1
        if opn.any() and expandable[c]:
            stack.extend((ch, opn) for ch in t.children[c][::-1] if ch >= 0)
v = tot["visits"]
print(f"theta={theta} L={L}: mixed {tot['mixed'] / v:.3f} of visits; resolved by half boxes "
      f"{tot['half_resolved'] / max(tot['mixed'], 1):.3f}, by quarter boxes {tot['quarter_resolved'] / max(tot['mixed'], 1):.3f}")

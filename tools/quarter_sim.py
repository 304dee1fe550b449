"""CPU model: lane-group queues for the walk's pc / pp drains (design study).

The v9 drains broadcast every list entry to all 32 lanes (64 targets, two per
lane); an entry accepted by few targets wastes the other lanes.  If the warp is
split into G lane groups (G = 2: halves, 4: quarter-warps of 8 lanes = 16
targets), each group can drain its own queue of the entries that touch its
targets: a flush of K entries then costs max over groups of the queue lengths
instead of K passes.  A quarter-warp is one shared-memory wavefront for a
128-bit load, so four different records per warp load cost nothing extra.

For groups of 64 Morton-consecutive targets on the oracle tree (cfg2 Plummer
1e6, theta 0.6, L 16) this collects, in v9's order, the pc entries (certain-
accept cells with the masks of the targets that reached them, plus the accepted
subsets of mixed cells) and the pp entries (opened buckets), and prints the
pass counts per drain batch size.

    python tools/quarter_sim.py [n] [groups]
"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from oracle import oracle as orc  # noqa: E402
from paper_2203_08966_b200.initcond import make_rng, plummer_cluster  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
G = int(sys.argv[2]) if len(sys.argv) > 2 else 150
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

rng = np.random.default_rng(0)
gs = rng.choice(n // S, size=G, replace=False)
pc_cert, pc_mix, pp = [], [], []  # per group: list of 64-bool masks (pp: (mask, count))
for g in gs:
    T = P[g * S:(g + 1) * S]
    lo, hi = T.min(0), T.max(0)
    a_c, a_m, a_p = [], [], []
    stack = [(c, np.ones(S, bool)) for c in t.children[0][::-1] if c >= 0]
    while stack:
        c, mask = stack.pop()
        if t.count[c] == 1:
            a_p.append((mask, 1))
            continue
        com = t.com[c]
        d2 = ((T - com) ** 2).sum(1)
        acc = mask & (d2 > mac2[c])
        opn = mask & ~acc
        gmin = np.maximum(np.maximum(lo - com, com - hi), 0.0)
        if (gmin ** 2).sum() > mac2[c] * (1 + 1e-6):
            a_c.append(mask)
            continue
        if acc.any():
            a_m.append(acc)
        if opn.any():
            if expandable[c]:
                stack.extend((ch, opn) for ch in t.children[c][::-1] if ch >= 0)
            else:
                a_p.append((opn, int(t.count[c])))
    pc_cert.append(a_c)
    pc_mix.append(a_m)
    pp.append(a_p)


def groups_touched(mask, ng):
    # lane l holds targets 2l, 2l+1; lane group j = lanes [j*32/ng, (j+1)*32/ng)
    lanes = mask.reshape(32, 2).any(1)
    return lanes.reshape(ng, 32 // ng).any(1)


def passes(entries, ng, K, weight=None):
    tot = 0
    for q in range(0, len(entries), K):
        batch = entries[q:q + K]
        w = weight[q:q + K] if weight is not None else [1] * len(batch)
        cnt = np.zeros(ng)
        for e, wi in zip(batch, w):
            cnt += groups_touched(e, ng) * wi
        tot += cnt.max()
    return tot


def report(name, per_group, counts=None):
    useful = sum(e.sum() * (c if counts else 1) for gi, grp in enumerate(per_group)
                 for e, c in zip(grp, counts[gi] if counts else [1] * len(grp)))
    nent = sum(len(x) for x in per_group)
    slots = sum(sum(c for c in counts[gi]) if counts else len(grp) for gi, grp in enumerate(per_group))
    print(f"{name}: {nent / G:.1f} entries/group, broadcast density {useful / (slots * S):.3f}")
    for K in (16, 32, 64, 10 ** 9):
        row = []
        for ng in (1, 2, 4, 8, 32):
            tot = sum(passes(grp, ng, K, counts[gi] if counts else None) for gi, grp in enumerate(per_group))
            row.append(f"G={ng}: {tot / slots:.3f}")
        print(f"   K={K if K < 10 ** 9 else 'all':>4}  passes / broadcast passes  " + "  ".join(row))


report("pc certain-accept", pc_cert)
report("pc mixed-accepted", pc_mix)
report("pc all (certain + mixed in one list)", [a + b_ for a, b_ in zip(pc_cert, pc_mix)])
report("pp (weighted by bucket bodies)", [[e for e, _ in grp] for grp in pp],
       [[c for _, c in grp] for grp in pp])


# ---- disjoint packing: entries whose lane sets do not overlap share a pass;
# each lane follows the one entry that holds its targets (body loads then have
# one address per packed entry).  Greedy first-fit in list order per flush.
def packed_cost(grp, K):
    tot = 0
    for q in range(0, len(grp), K):
        batch = grp[q:q + K]
        passes = []  # [lane mask, max count]
        for mask, c in batch:
            lm = mask.reshape(32, 2).any(1)
            for pz in passes:
                if not (pz[0] & lm).any():
                    pz[0] |= lm
                    pz[1] = max(pz[1], c)
                    break
            else:
                passes.append([lm.copy(), c])
        tot += sum(c for _, c in passes)
    return tot


base_it = sum(sum(c for _, c in grp) for grp in pp)
for K in (16, 32, 64):
    t = sum(packed_cost(grp, K) for grp in pp)
    print(f"pp disjoint packing K={K}: body iterations {t / base_it:.3f} of broadcast")

# the same packing for the pc list (certain-accept entries, count 1 each)
base_pc = sum(len(grp) for grp in pc_cert)
for K in (16, 32, 64):
    t = sum(packed_cost([(m_, 1) for m_ in grp], K) for grp in pc_cert)
    print(f"pc disjoint packing K={K}: passes {t / base_pc:.3f} of broadcast")


# ---- packing order variants for the pp flush: first-fit decreasing by bucket
# length (passes then group buckets of similar length), and by lane count
def packed_cost_sorted(grp, K, key):
    tot = 0
    for q in range(0, len(grp), K):
        batch = sorted(grp[q:q + K], key=key)
        passes = []
        for mask, c in batch:
            lm = mask.reshape(32, 2).any(1)
            for pz in passes:
                if not (pz[0] & lm).any():
                    pz[0] |= lm
                    pz[1] = max(pz[1], c)
                    break
            else:
                passes.append([lm.copy(), c])
        tot += sum(c for _, c in passes)
    return tot


for K in (32, 64):
    for name, key in (("count desc", lambda e: -e[1]), ("lanes desc", lambda e: -e[0].reshape(32, 2).any(1).sum()),
                      ("count desc, lanes desc", lambda e: (-e[1], -e[0].reshape(32, 2).any(1).sum()))):
        t = sum(packed_cost_sorted(grp, K, key) for grp in pp)
        print(f"pp packing K={K} sorted by {name}: body iterations {t / base_it:.3f} of broadcast")

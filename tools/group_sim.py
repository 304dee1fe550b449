"""CPU model of a group-classified walk (design study for the fp32 traversal).

For groups of 64 Morton-consecutive targets, walk the oracle tree with
per-target masks (the exact reference interaction sets, bucket rule L) and
classify every examined cell against the group's bounding box:
  certain-accept  box-min distance^2 > mac2 (every target accepts)
  certain-open    box-max distance^2 < mac2 (every target opens)
  mixed           per-target MAC needed
Counts visits per class and the pc/pp utilisation of each list.

    python tools/group_sim.py [n] [groups] [group_size]
"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from oracle import oracle as orc  # noqa: E402
from paper_2203_08966_b200.initcond import make_rng, plummer_cluster  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
G = int(sys.argv[2]) if len(sys.argv) > 2 else 200
S = int(sys.argv[3]) if len(sys.argv) > 3 else 64
theta, L = 0.6, 16
b = plummer_cluster(n, make_rng(2), 1.0)
pos = b.position.astype(np.float32).astype(np.float64)
m = b.mass.astype(np.float32).astype(np.float64)
R = orc.bounds(pos)
k = orc.morton_keys(pos, R)
o = orc.sort_order(k)
t = orc.build_tree(m[o], pos[o], R)
P = pos[o]
mac2 = (t.side / theta) ** 2
expandable = (t.count > L)
expandable[0] = t.count[0] > 1

rng = np.random.default_rng(0)
gs = rng.choice(n // S, size=G, replace=False)
tot = dict(cert_acc=0, cert_open=0, mixed=0, leaf=0, pc_util_cert=0.0, pc_util_mixed=0.0, n_mixed_acc=0,
           pc_useful=0, visits=0, chunks=0)
for g in gs:
    T = P[g * S:(g + 1) * S]
    lo, hi = T.min(0), T.max(0)
    stack = [(c, np.ones(S, bool)) for c in t.children[0] if c >= 0] if expandable[0] else [(0, np.ones(S, bool))]
    frontier_sizes = []
    while stack:
        frontier_sizes.append(len(stack))
        c, mask = stack.pop()
        tot["visits"] += 1
        d = T - t.com[c]
        d2 = (d * d).sum(1)
        if t.count[c] == 1:
            tot["leaf"] += 1
            continue
        com = t.com[c]
        gmin = np.maximum(np.maximum(lo - com, com - hi), 0.0)
        gmax = np.maximum(np.abs(lo - com), np.abs(hi - com))
        dmin2, dmax2 = (gmin ** 2).sum(), (gmax ** 2).sum()
        acc = mask & (d2 > mac2[c])
        opn = mask & ~(d2 > mac2[c])
        tot["pc_useful"] += acc.sum()
        if dmin2 > mac2[c] * (1 + 1e-5):
            assert not opn.any()
            tot["cert_acc"] += 1
            tot["pc_util_cert"] += mask.sum() / S
            continue
        if dmax2 * (1 + 1e-5) < mac2[c]:
            assert not acc.any()
            tot["cert_open"] += 1
        else:
            tot["mixed"] += 1
            if acc.any():
                tot["n_mixed_acc"] += 1
                tot["pc_util_mixed"] += acc.sum() / S
        if opn.any() and expandable[c]:
            for ch in t.children[c]:
                if ch >= 0:
                    stack.append((ch, opn))
print(f"n={n} groups={G} S={S} theta={theta} L={L}")
v = tot["visits"]
for key in ("cert_acc", "cert_open", "mixed", "leaf"):
    print(f"  {key:10s} {tot[key] / G:9.1f} per group  ({tot[key] / v:.3f} of visits)")
print(f"  pc util: certain {tot['pc_util_cert'] / max(tot['cert_acc'], 1):.3f}, "
      f"mixed {tot['pc_util_mixed'] / max(tot['n_mixed_acc'], 1):.3f}; useful pc per target "
      f"{tot['pc_useful'] / G / S:.1f}")

# batched LIFO frontier: pop the top 32 cells per iteration, classify lane-parallel
mx, iters, cells = 0, 0, 0
for g in gs:
    T = P[g * S:(g + 1) * S]
    front = [(c, np.ones(S, bool)) for c in t.children[0] if c >= 0]
    while front:
        mx = max(mx, len(front))
        batch, front = front[-32:], front[:-32]
        iters += 1
        cells += len(batch)
        for c, mask in batch:
            if t.count[c] == 1:
                continue
            d = T - t.com[c]
            opn = mask & ~((d * d).sum(1) > mac2[c])
            if opn.any() and expandable[c]:
                front.extend((ch, opn) for ch in t.children[c] if ch >= 0)
print(f"  batched frontier: max {mx} entries, {iters / G:.1f} iterations per group, "
      f"{cells / iters:.1f} cells per iteration")

# entry frontier (children ranges): batches of <= 32 cells taken from the top entries
mx, iters, cells, hist = 0, 0, 0, []
for g in gs:
    T = P[g * S:(g + 1) * S]
    front = [([c for c in t.children[0] if c >= 0], np.ones(S, bool))]
    gmx = 0
    while front:
        gmx = max(gmx, len(front))
        batch = []
        while front and len(batch) < 32:
            ch, mask = front.pop()
            take = ch[-(32 - len(batch)):]
            rest = ch[:len(ch) - len(take)]
            if rest:
                front.append((rest, mask))
            batch += [(c, mask) for c in take]
        iters += 1
        cells += len(batch)
        for c, mask in batch:
            if t.count[c] == 1:
                continue
            d = T - t.com[c]
            opn = mask & ~((d * d).sum(1) > mac2[c])
            if opn.any() and expandable[c]:
                front.append(([ch for ch in t.children[c] if ch >= 0], opn))
    hist.append(gmx)
print(f"  entry frontier: max {max(hist)} entries (p99 {np.percentile(hist, 99):.0f}), {iters / G:.1f} iterations "
      f"per group, {cells / iters:.1f} cells per iteration")

# pp entries (buckets opened / leaves): mask density and body iterations
ent, its, useful, ks = 0, 0, 0, []
for g in gs:
    T = P[g * S:(g + 1) * S]
    stack = [(c, np.ones(S, bool)) for c in t.children[0] if c >= 0]
    while stack:
        c, mask = stack.pop()
        d = T - t.com[c]
        if t.count[c] == 1:
            acc_, opn = np.zeros(S, bool), mask
        else:
            acc_ = mask & ((d * d).sum(1) > mac2[c])
            opn = mask & ~acc_
        if not opn.any():
            continue
        if t.count[c] == 1 or not expandable[c]:
            k_ = int(opn.sum()); ent += 1; its += int(t.count[c]); useful += k_ * int(t.count[c]); ks.append(k_)
            continue
        for ch in t.children[c]:
            if ch >= 0:
                stack.append((ch, opn))
ks = np.array(ks)
print(f"  pp entries {ent / G:.1f}/group, body iterations {its / G:.1f}, density {useful / its / S:.3f}; "
      f"k quartiles {np.percentile(ks, [10, 25, 50, 75, 90])}")
for lim in (4, 8, 16, 32):
    sel = ks <= lim
    print(f"    entries with k<={lim}: {sel.mean():.3f} of entries")

# cost model: dense masked pp (20 instr per body) vs compact (target, body) pairs
ent2 = []
for g in gs[:50]:
    T = P[g * S:(g + 1) * S]
    stack = [(c, np.ones(S, bool)) for c in t.children[0] if c >= 0]
    while stack:
        c, mask = stack.pop()
        d = T - t.com[c]
        if t.count[c] == 1:
            opn = mask
        else:
            opn = mask & ~((d * d).sum(1) > mac2[c])
        if not opn.any():
            continue
        if t.count[c] == 1 or not expandable[c]:
            ent2.append((int(opn.sum()), int(t.count[c])))
            continue
        for ch in t.children[c]:
            if ch >= 0:
                stack.append((ch, opn))
dense = sum(20 * c for k_, c in ent2)
best = 0
for k_, c in ent2:
    cp = 1 << (c - 1).bit_length()
    comp = -(-k_ * cp // 64) * (50 + 9 * (cp.bit_length() - 1))
    best += min(20 * c, comp)
print(f"  pp cost model per group: dense {dense / 50:.0f}, with compact where cheaper {best / 50:.0f}")

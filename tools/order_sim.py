"""CPU model: does a Hilbert order of the walk's targets raise the pc density?

The walk's warps own 64 consecutive targets of the Morton order.  A window of
64 Morton-consecutive bodies can straddle a coarse cell boundary (a Z-curve
jump), which inflates the group's box and mixes targets with different lists.
This walks the oracle tree (leaf-size rule L) for sampled groups of 64 and
counts, per group, the broadcast pc evaluations (cells with >= 1 accepting
target in the group) and the useful ones (accepting targets), for Morton and
Hilbert target windows.

    python tools/order_sim.py [n] [groups] [theta] [L]
"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from oracle import oracle as orc  # noqa: E402
from paper_2203_08966_b200.initcond import make_rng, plummer_cluster  # noqa: E402


def hilbert_keys(q: np.ndarray, bits: int = 21) -> np.ndarray:
    """Skilling's transpose algorithm, vectorised: q (n,3) uint64 in [0, 2^bits)."""
    x = [q[:, 0].astype(np.uint64).copy(), q[:, 1].astype(np.uint64).copy(), q[:, 2].astype(np.uint64).copy()]
    M = np.uint64(1) << np.uint64(bits - 1)
    Q = M
    while Q > 1:
        P = Q - np.uint64(1)
        for i in range(3):
            hit = (x[i] & Q) != 0
            # invert low bits of x[0] where hit, else exchange low bits of x[0] and x[i]
            t = (x[0] ^ x[i]) & P
            x0_inv = x[0] ^ P
            x0_new = np.where(hit, x0_inv, x[0] ^ t)
            xi_new = np.where(hit, x[i], x[i] ^ t)
            x[0] = x0_new
            if i:
                x[i] = xi_new
        Q >>= np.uint64(1)
    for i in range(1, 3):
        x[i] ^= x[i - 1]
    t = np.zeros_like(x[0])
    Q = M
    while Q > 1:
        t = np.where((x[2] & Q) != 0, t ^ (Q - np.uint64(1)), t)
        Q >>= np.uint64(1)
    for i in range(3):
        x[i] ^= t
    h = np.zeros_like(x[0])
    for b in range(bits - 1, -1, -1):
        for i in range(3):
            h = (h << np.uint64(1)) | ((x[i] >> np.uint64(b)) & np.uint64(1))
    return h


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    G = int(sys.argv[2]) if len(sys.argv) > 2 else 100
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
    q = np.clip(np.floor((P + R) / (2 * R) * (1 << 21)), 0, (1 << 21) - 1).astype(np.uint64)
    hk = hilbert_keys(q)
    ho = np.argsort(hk, kind="stable")
    mac2 = (t.side / theta) ** 2
    expandable = t.count > L
    expandable[0] = t.count[0] > 1
    rng = np.random.default_rng(0)
    starts = rng.choice(n // S, size=G, replace=False) * S
    # cell-aligned windows: a warp ends at the weakest Morton link (smallest
    # shared prefix with the next key) among its last positions [minw, 64]
    keys = orc.morton_keys(P, R)
    x = keys[:-1] ^ keys[1:]
    lcp = np.full(n, -1)
    lcp[:-1] = 21 - (np.floor(np.log2(np.maximum(x, 1).astype(np.float64))).astype(int) + 3) // 3
    def aligned(minw):
        b, out = 0, []
        while b < n:
            e = min(n, b + S)
            if e < n:
                seg = lcp[b + minw - 1:e - 1 + 1]
                e = b + minw + int(np.argmin(seg[::-1][::-1] if False else seg))
            out.append((b, e))
            b = e
        return out
    groups = {}
    for minw in (48, 32):
        w = aligned(minw)
        pick = rng.choice(len(w), size=G, replace=False)
        groups[f"aligned{minw}"] = [w[i] for i in pick]
    runs = [("morton", np.arange(n), [(s0, s0 + S) for s0 in starts]),
            ("hilbert", ho, [(s0, s0 + S) for s0 in starts])] + [(k, np.arange(n), v) for k, v in groups.items()]
    for name, order, wins in runs:
        ent = use = mixed = ppent = ppuse = ppit = 0
        ext = []
        ntg = 0
        for s0, s1 in wins:
            T = P[order[s0:s1]]
            ntg += len(T)
            ext.append(np.linalg.norm(T.max(0) - T.min(0)))
            stack = [(c, np.ones(len(T), bool)) for c in t.children[0] if c >= 0]
            while stack:
                c, mask = stack.pop()
                d = T - t.com[c]
                d2 = (d * d).sum(1)
                if t.count[c] == 1 or not expandable[c]:
                    opn = mask if t.count[c] == 1 else mask & ~(d2 > mac2[c])
                    if t.count[c] > 1:
                        acc = mask & (d2 > mac2[c])
                        if acc.any():
                            ent += 1
                            use += int(acc.sum())
                    if opn.any():
                        ppent += 1
                        ppuse += int(opn.sum()) * int(t.count[c])
                        ppit += int(t.count[c])
                    continue
                acc = mask & (d2 > mac2[c])
                opn = mask & ~acc
                if acc.any():
                    ent += 1
                    use += int(acc.sum())
                    if opn.any():
                        mixed += 1
                if opn.any():
                    for ch in t.children[c]:
                        if ch >= 0:
                            stack.append((ch, opn))
        print(f"{name:9s} targets/warp {ntg / G:5.1f}  pc evals per 64 targets {ent / ntg * S:8.1f}  density {use / ent / S:.3f}  "
              f"useful/target {use / ntg:7.1f}  mixed-acc per 64 {mixed / ntg * S:6.1f}  "
              f"pp iters per 64 {ppit / ntg * S:7.1f} density {ppuse / max(ppit, 1) / S:.3f}  "
              f"extent median {np.median(ext):.4f} p90 {np.percentile(ext, 90):.4f}")


if __name__ == "__main__":
    main()

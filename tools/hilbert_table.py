"""Derive the 3-D Hilbert state machine of Skilling's transpose (the curve the
walk orders its targets along) from the curve itself, and check it.

For every cell of a depth-5 grid the order of its 8 children along the curve
is a permutation of the octants (Morton digits); distinct permutations are
the states, and each child's own permutation gives the transition.  Prints
the two 8-entry rows per state for bh_walk.cu.

    python tools/hilbert_table.py
"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from tools.order_sim import hilbert_keys  # noqa: E402

D, B = 5, 21
g = np.arange(1 << D, dtype=np.uint64)
X, Y, Z = np.meshgrid(g, g, g, indexing="ij")
q = np.stack([X.ravel(), Y.ravel(), Z.ravel()], 1) << np.uint64(B - D)
h = hilbert_keys(q)
perm_of = {}  # (level, cell prefix) -> tuple digit[octant]


def digit(v, l):  # 3-bit digit of level l (1 = top) of a 63-bit key
    return int((int(v) >> (3 * (B - l))) & 7)


def morton_digit(p, l):
    s = B - l
    return (int(p[0]) >> s & 1) << 2 | (int(p[1]) >> s & 1) << 1 | (int(p[2]) >> s & 1)


cells = {}
for p, hv in zip(q, h):
    for l in range(1, D + 1):
        pref = tuple(int(c) >> (B - l + 1) for c in p)
        cells.setdefault((l, pref), {})[morton_digit(p, l)] = digit(hv, l)
states, idx = [], {}
for key, m in cells.items():
    pm = tuple(m[o] for o in range(8))
    if pm not in idx:
        idx[pm] = len(states)
        states.append(pm)
nxt = {}
for (l, pref), m in cells.items():
    if l == D:
        continue
    s = idx[tuple(m[o] for o in range(8))]
    for o in range(8):
        child = tuple((pref[k] << 1) | ((o >> (2 - k)) & 1) for k in range(3))
        cs = idx[tuple(cells[(l + 1, child)][oo] for oo in range(8))]
        assert nxt.setdefault((s, o), cs) == cs, "not a state machine"
root = idx[tuple(cells[(1, (0, 0, 0))][o] for o in range(8))]


def table_key(p):
    st, k = root, 0
    for l in range(1, B + 1):
        o = morton_digit(p, l)
        k = (k << 3) | states[st][o]
        st = nxt.get((st, o), st)
    return k


rng = np.random.default_rng(0)
pts = rng.integers(0, 1 << B, size=(2000, 3)).astype(np.uint64)
ref = hilbert_keys(pts)
assert all(table_key(p) == int(r) for p, r in zip(pts, ref)), "table disagrees with Skilling"
print(f"// {len(states)} states, root {root}")
print("digit:", ", ".join("{" + ", ".join(map(str, s)) + "}" for s in states))
print("next:", ", ".join("{" + ", ".join(str(nxt[(i, o)]) for o in range(8)) + "}" for i in range(len(states))))

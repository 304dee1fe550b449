"""CPU model: half-masked drain entries (design study).

If lane l holds targets l and l + 32 of the warp's 64 (instead of 2l, 2l + 1),
the two halves of a packed FFMA2 are the two spatial halves of the group.  A
list entry whose targets all sit in one half could then be evaluated with
scalar FFMA (half the FP32-pipe cycles).  This prints, for the pc and pp lists
of quarter_sim.py's groups, the cost of that schedule relative to the packed
broadcast: entries with an empty half count 0.5.

    python tools/half_sim.py [n] [groups] [theta] [L]
"""
import sys

src = open(__file__.rsplit("/", 1)[0] + "/quarter_sim.py").read().split("def groups_touched")[0]
exec(src)


def cost(mask):
    h0, h1 = mask[:32].any(), mask[32:].any()
    return 1.0 if (h0 and h1) else 0.5


def interleaved_cost(mask):
    h0, h1 = mask[0::2].any(), mask[1::2].any()
    return 1.0 if (h0 and h1) else 0.5


for name, lists, w in (("pc certain", pc_cert, None), ("pc mixed", pc_mix, None),
                       ("pc all", [a + b_ for a, b_ in zip(pc_cert, pc_mix)], None),
                       ("pp", [[e for e, _ in g] for g in pp], [[c for _, c in g] for g in pp])):
    tot = half = inter = dens = 0.0
    for gi, grp in enumerate(lists):
        for ei, e in enumerate(grp):
            wi = w[gi][ei] if w else 1
            tot += wi
            half += wi * cost(e)
            inter += wi * interleaved_cost(e)
            dens += wi * e.mean()
    print(f"{name}: density {dens / tot:.3f}; cost with spatial halves {half / tot:.3f}, "
          f"with interleaved halves {inter / tot:.3f} (1.0 = packed broadcast)")


# ---- the pp drain under both lane mappings: greedy first-fit of buckets into
# passes with disjoint lane sets (K entries per flush); a pass of the spatial-
# halves mapping whose buckets use one half only costs `half_cost` per iteration
def pp_cost(grp, K, spatial, half_cost):
    tot = 0.0
    for q in range(0, len(grp), K):
        passes = []  # [lane mask, max count, half0 used, half1 used]
        for mask, c in grp[q:q + K]:
            if spatial:
                lm = mask[:32] | mask[32:]
                h0, h1 = mask[:32].any(), mask[32:].any()
            else:
                lm = mask.reshape(32, 2).any(1)
                h0, h1 = mask[0::2].any(), mask[1::2].any()
            for pz in passes:
                if not (pz[0] & lm).any():
                    pz[0] |= lm
                    pz[1] = max(pz[1], c)
                    pz[2] |= h0
                    pz[3] |= h1
                    break
            else:
                passes.append([lm.copy(), c, h0, h1])
        tot += sum(c * (1.0 if (a and b_) else half_cost) for _, c, a, b_ in passes)
    return tot


base = sum(sum(c for _, c in grp) for grp in pp)
for K in (64,):
    for spatial in (False, True):
        for hc in (1.0, 0.6):
            t_ = sum(pp_cost(grp, K, spatial, hc) for grp in pp)
            print(f"pp packed K={K} {'spatial halves' if spatial else 'interleaved'} half-pass cost {hc}: "
                  f"{t_ / base:.3f} of broadcast body iterations")


# ---- pp packing on the 64 target slots (spatial halves; each lane follows one
# bucket per half, two scalar streams): passes of buckets with disjoint targets
def pp_cost_slots(grp, K):
    tot = 0.0
    for q in range(0, len(grp), K):
        passes = []
        for mask, c in grp[q:q + K]:
            for pz in passes:
                if not (pz[0] & mask).any():
                    pz[0] |= mask
                    pz[1] = max(pz[1], c)
                    break
            else:
                passes.append([mask.copy(), c])
        tot += sum(c for _, c in passes)
    return tot


t_ = sum(pp_cost_slots(grp, 64) for grp in pp)
print(f"pp packed K=64 on 64 target slots: {t_ / base:.3f} of broadcast body iterations")

full = sum(e.all() for g in pc_cert for e in g)
tot_ = sum(len(g) for g in pc_cert)
print(f"pc certain entries with a full mask: {full / tot_:.3f}")

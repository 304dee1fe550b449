"""The walk-only tree of the fp32 resident-sim path across leaf sizes.

bh_sim_forces builds only what a leaf-size-L walk reads: the
two-pass emit decides which bodies create walk records from a window test over
L + 1 consecutive keys (a shared-memory halo of 64 keys, so L <= 64; larger L
falls back to the one-pass emit), bucket moments come straight from the
bodies, and the walk records are scanned over the opened cells only.  Each leaf
size here is checked against the oracle's full reference tree with the bucket
rule, through the same path bench.py times: per-body work
equal on a sample (same MAC decisions, same buckets), accelerations within the
fp32 bar.  Duplicate keys (a level-21 cell, never opened) are included."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle import oracle as orc  # noqa: E402

FP32_TOL = 1e-4  # relative L2, fp32 mode (north star)
FP32_WORK_FLIPS = 5e-4  # MAC ties between fp32 and fp64 d2 (measured 0)


def _bodies(n, seed, dups):
    from paper_2203_08966_b200.initcond import make_rng, plummer_cluster

    b = plummer_cluster(n, make_rng(seed), 1.0)
    pos = b.position.astype(np.float32)
    k = np.random.Generator(np.random.Philox(key=seed)).choice(n, dups, replace=False) if dups else np.zeros(0, int)
    if dups:  # exact copies of one body: a run of duplicate Morton keys
        pos[k[1:]] = pos[k[0]]
    return pos.astype(np.float64), b.mass.astype(np.float32).astype(np.float64), k


@pytest.mark.parametrize("leaf,dups", [(2, 0), (3, 0), (8, 0), (31, 0), (64, 0), (65, 0), (16, 40), (64, 70)])
def test_walk_only_tree_matches_oracle(leaf, dups):
    from paper_2203_08966_b200.engine import Engine

    n, theta, eps = 30_000, 0.6, 1e-3
    pos, m, dup_idx = _bodies(n, 11 + leaf, dups)
    eng = Engine("fp32", 0)
    if dups:
        eng.set_allow_duplicates(True)
    p = eng.bodies_tensor(pos, m)
    eng.sim_load(p, torch.zeros_like(p))
    eng.sim_forces(theta, eps, leaf, True)
    acc = torch.empty_like(p)
    work = torch.empty(n, dtype=torch.int64, device="cuda")
    eng.sim_store(acc=acc, work=work)
    eng.check()
    eng.close()
    sample = np.random.Generator(np.random.Philox(key=leaf)).choice(n, 1500, replace=False)
    sample = np.union1d(sample, dup_idx)  # the duplicates themselves as targets too
    R = orc.bounds(pos)
    order = orc.sort_order(orc.morton_keys(pos, R))
    tree = orc.build_tree(m[order], pos[order], R, allow_duplicates=bool(dups))
    ref_acc, ref_work = orc.traverse(tree, pos[sample], theta, eps, leaf)
    got = acc[:, :3].double().cpu().numpy()[sample]
    err = float(np.linalg.norm(got - ref_acc) / np.linalg.norm(ref_acc))
    assert err <= FP32_TOL, err
    mism = int(np.sum(work.cpu().numpy()[sample] != ref_work))
    assert mism <= FP32_WORK_FLIPS * len(sample), mism

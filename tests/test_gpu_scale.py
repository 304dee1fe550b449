"""Parity at the bench configurations' scale, through the resident-sim path
bench.py times (bh_sim_load -> bh_sim_forces): cfg3's geometry at full size
(two colliding Plummer clusters, N=1e7, theta=0.6, eps=1e-4, L=32) and cfg4's
clustered Hernquist cloud at N=2e6 (theta=0.7, eps=1e-5, L=32; duplicate keys
in the cusps, so the oracle runs its bucket-mode extension).

The oracle builds the full reference tree on the fp32-rounded inputs (SURVEY
§8c protocol) and walks a seeded sample of targets; the GPU result for the
same bodies must be within the fp32 bar, and the per-body work of the sample
must match the oracle's (same MAC decisions)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle import oracle as orc  # noqa: E402

FP32_TOL = 1e-4  # relative L2, fp32 mode (north star)


def _gpu_forces(pos32, m32, theta, eps, leaf, allow_dup, sample=None):
    from paper_2203_08966_b200.engine import Engine

    eng = Engine("fp32", 0)
    if allow_dup:
        eng.set_allow_duplicates(True)
    p = eng.bodies_tensor(pos32, m32)
    v = torch.zeros_like(p)
    eng.sim_load(p, v)
    eng.sim_forces(theta, eps, leaf, True)
    acc = torch.empty_like(p)
    work = torch.empty(len(pos32), dtype=torch.int64, device="cuda")
    eng.sim_store(acc=acc, work=work)
    eng.check()
    st = eng.stats()
    eng.close()
    if sample is not None:  # (sampled acc, sampled work, total work, stats)
        t = torch.as_tensor(sample, device="cuda")
        return acc[t, :3].double().cpu().numpy(), work[t].cpu().numpy(), int(work.sum().item()), st
    return acc[:, :3].double().cpu().numpy(), work.cpu().numpy(), st


def _oracle_sample(pos32, m32, theta, eps, leaf, sample, allow_dup):
    pos = pos32.astype(np.float64)
    m = m32.astype(np.float64)
    R = orc.bounds(pos)
    order = orc.sort_order(orc.morton_keys(pos, R))
    tree = orc.build_tree(m[order], pos[order], R, allow_duplicates=allow_dup)
    return orc.traverse(tree, pos[sample], theta, eps, leaf)


def _check(pos32, m32, theta, eps, leaf, allow_dup, nsample=2000, seed=11):
    acc, work, st = _gpu_forces(pos32, m32, theta, eps, leaf, allow_dup)
    assert np.all(np.isfinite(acc))
    sample = np.random.Generator(np.random.Philox(key=seed)).choice(len(pos32), nsample, replace=False)
    ref_acc, ref_work = _oracle_sample(pos32, m32, theta, eps, leaf, sample, allow_dup)
    err = float(np.linalg.norm(acc[sample] - ref_acc) / np.linalg.norm(ref_acc))
    assert err <= FP32_TOL, err
    mism = float(np.mean(work[sample] != ref_work))
    print(f"WORKMISMATCH scale n={len(pos32)}: {mism * nsample:.0f}/{nsample}")
    assert mism <= 5e-4, mism  # fp32 d2 vs fp64 d2 at a MAC tie (measured: 0)
    assert st.pp + 2 * st.pc == int(work.sum())
    return err, mism


def test_cfg3_full_size_sampled_parity():
    from paper_2203_08966_b200.initcond import colliding_plummers

    b = colliding_plummers(5_000_000, 3)
    pos32 = np.asarray(b.position, dtype=np.float32)
    m32 = np.asarray(b.mass, dtype=np.float32)
    err, mism = _check(pos32, m32, 0.6, 1e-4, 32, allow_dup=False)
    print(f"cfg3 1e7: sampled rel L2 {err:.2e}, work mismatches {mism:.1e}")


def test_cfg4_shape_sampled_parity():
    from paper_2203_08966_b200.initcond import hernquist_cosmology

    pos32, _, m32 = hernquist_cosmology(2_000_000, 4)
    err, mism = _check(pos32, m32, 0.7, 1e-5, 32, allow_dup=True)
    print(f"cfg4 shape 2e6: sampled rel L2 {err:.2e}, work mismatches {mism:.1e}")


def test_cfg4_full_size_sampled_parity():
    """BASELINE cfg4 at the size the bench runs (N=1e8, one GPU): the resident
    sim_forces path against the oracle's full 1e8-body tree on 4000 sampled
    targets.  The oracle's answers are a committed fixture
    (tests/golden/make_cfg4_fixture.py: the serial build needs ~30 GB of host
    memory); the generator is deterministic, so the inputs are regenerated."""
    import os

    from paper_2203_08966_b200.initcond import hernquist_cosmology

    path = os.path.join(os.path.dirname(__file__), "golden", "cfg4_sample_100000000.npz")
    g = np.load(path)
    n = int(g["n"])
    pos32, _, m32 = hernquist_cosmology(n, 4)
    idx = g["idx"]
    acc, work, wsum, st = _gpu_forces(pos32, m32, float(g["theta"]), float(g["eps"]), int(g["leaf"]), True,
                                      sample=idx)
    del pos32, m32
    assert np.all(np.isfinite(acc))
    err = float(np.linalg.norm(acc - g["acc"]) / np.linalg.norm(g["acc"]))
    assert err <= FP32_TOL, err
    mism = int(np.sum(work != g["work"]))
    assert mism <= 2, mism  # fp32 vs fp64 d2 at a MAC tie
    assert st.n_cells == int(g["cells"])  # the same tree (bucket-mode duplicates included)
    assert st.pp + 2 * st.pc == wsum
    print(f"cfg4 1e8: sampled rel L2 {err:.2e}, work mismatches {mism}/{len(idx)}, cells {st.n_cells}")

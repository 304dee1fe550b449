"""Multi-rank step on the GPU: R ranks emulated as threads on one device
(host-side barriers only -- no kernel waits on another rank), each with its own
libbh handle, exchanging through ThreadComm.  Must equal the single-GPU run:
bitwise in fp64 (the fp64 walk keeps the reference's order), to fp32 rounding
in fp32 with identical work counts."""

import os
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _run(precision, ranks, b, steps, theta=0.6, eps=1e-3, leaf=16, dt=1e-3):
    from paper_2203_08966_b200.decomposition import DistributedSim, StepParams, ThreadComm
    from paper_2203_08966_b200.engine import Engine

    comms = ThreadComm.group(ranks)
    out = [None] * ranks
    err = []

    def body(r):
        try:
            eng = Engine(precision, 0)
            pos = eng.bodies_tensor(b.position, b.mass)
            vel = eng.vec_tensor(b.velocity)
            m = None if eng.fp32 else torch.as_tensor(b.mass).cuda()
            sim = DistributedSim(eng, comms[r], StepParams(theta, eps, leaf, dt))
            sim.load(pos, vel, m)
            sim.bootstrap()
            sim.step(steps)
            p = torch.empty_like(vel)
            w = torch.empty(len(b), dtype=torch.int64, device="cuda")
            sim.store(pos=p, work=w)
            eng.check()
            out[r] = (p[:, :3].double().cpu().numpy(), w.cpu().numpy(), list(sim.zones), sim.p2p)
            eng.close()
        except Exception as e:  # pragma: no cover - surfaced below
            err.append(e)
            comms[r].hub.barrier.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(ranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    if err:
        raise err[0]
    return out


@pytest.mark.parametrize("p2p", ["0", "1"])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_emulated_ranks_match_single_gpu(precision, p2p, monkeypatch):
    """p2p=1: results reach the other ranks through the walk's peer stores
    (raw device pointers here) instead of an all-reduce."""
    from paper_2203_08966_b200.initcond import make_rng, plummer_cluster

    monkeypatch.setenv("BH_P2P", p2p)
    b = plummer_cluster(20_000, make_rng(1))
    single = _run(precision, 1, b, 3)[0]
    for ranks in (2, 3):
        multi = _run(precision, ranks, b, 3)
        for pos, work, zones, used in multi:
            assert used == (p2p == "1")
            assert len(zones) == ranks + 1
            if precision == "fp64":
                np.testing.assert_array_equal(pos, single[0])
                np.testing.assert_array_equal(work, single[1])
            else:
                rel = np.abs(pos - single[0]).max() / np.abs(single[0]).max()
                assert rel < 1e-5, rel
                assert np.mean(work != single[1]) < 1e-3
        # all ranks hold the same replicated state
        for pos, work, _, _ in multi[1:]:
            np.testing.assert_array_equal(pos, multi[0][0])


class _Cloud:
    def __init__(self, pos, vel, mass):
        self.position, self.velocity, self.mass = pos, vel, mass

    def __len__(self):
        return len(self.mass)


def test_replicated_ranks_recover_from_capacity_overflow(monkeypatch):
    """Bodies in close pairs give ~10 cells per body, past the sync-free
    build's first capacity: every rank must redo its build before the walk
    stores rows into the peers (not after a corrupted step)."""
    monkeypatch.setenv("BH_P2P", "1")
    rng = np.random.default_rng(5)
    c = rng.uniform(-0.9, 0.9, (4000, 3))
    pos = np.concatenate([c, c + [2.0 ** -19, 0.0, 0.0]]).astype(np.float32).astype(np.float64)
    b = _Cloud(pos, rng.normal(0, 0.05, pos.shape), np.full(len(pos), 1.0 / len(pos)))
    single = _run("fp32", 1, b, 2, theta=0.5, leaf=1)[0]
    for pos_r, work, _, used in _run("fp32", 2, b, 2, theta=0.5, leaf=1):
        assert used
        rel = np.abs(pos_r - single[0]).max() / np.abs(single[0]).max()
        assert rel < 1e-5, rel
        assert np.mean(work != single[1]) < 1e-3


def _run_build(ranks, b, steps, theta=0.6, eps=1e-3, leaf=16, dt=1e-3):
    """Stage 2 (distributed build) with R emulated ranks; returns per-gid arrays."""
    from paper_2203_08966_b200.decomposition import DistributedBuildSim, StepParams, ThreadComm
    from paper_2203_08966_b200.engine import Engine

    n = len(b)
    comms = ThreadComm.group(ranks)
    outs = [None] * ranks
    lets = [None] * ranks
    err = []
    cuts = np.linspace(0, n, ranks + 1).astype(int)

    def body(r):
        try:
            eng = Engine("fp32", 0)
            sl = slice(cuts[r], cuts[r + 1])
            pos = eng.bodies_tensor(b.position[sl], b.mass[sl])
            vel = eng.vec_tensor(b.velocity[sl])
            gid = torch.arange(cuts[r], cuts[r + 1], device="cuda")
            sim = DistributedBuildSim(eng, comms[r], StepParams(theta, eps, leaf, dt))
            sim.load(pos, vel, gid=gid)
            sim.bootstrap()
            sim.step(steps)
            p, v, a, w, g = sim.store()
            eng.check()
            outs[r] = tuple(x.cpu().numpy() for x in (p, v, a, w, g))
            lets[r] = sim.let_stats
            eng.close()
        except Exception as e:  # pragma: no cover
            import traceback
            traceback.print_exc()
            err.append(e)
            comms[r].hub.barrier.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(ranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    if err:
        raise err[0]
    res = {k: np.zeros((n, 4)) for k in ("pos", "vel", "acc")}
    res["work"] = np.zeros(n, dtype=np.int64)
    seen = np.zeros(n, dtype=int)
    for p, v, a, w, g in outs:
        res["pos"][g], res["vel"][g], res["acc"][g], res["work"][g] = p, v, a, w
        seen[g] += 1
    assert np.all(seen == 1), "every body owned by exactly one rank"
    res["counts"] = [len(o[4]) for o in outs]
    res["let"] = lets
    return res


def _single(b, steps, theta=0.6, eps=1e-3, leaf=16, dt=1e-3):
    from paper_2203_08966_b200.engine import Engine

    eng = Engine("fp32", 0)
    pos = eng.bodies_tensor(b.position, b.mass)
    vel = eng.vec_tensor(b.velocity)
    eng.sim_load(pos, vel)
    eng.sim_forces(theta, eps, leaf, record_work=False)
    eng.sim_step(dt, theta, eps, leaf, steps)
    p, v, a = torch.empty_like(vel), torch.empty_like(vel), torch.empty_like(vel)
    w = torch.empty(len(b), dtype=torch.int64, device="cuda")
    eng.sim_store(p, v, a, w)
    eng.check()
    out = dict(pos=p.double().cpu().numpy(), vel=v.double().cpu().numpy(), acc=a.double().cpu().numpy(),
               work=w.cpu().numpy())
    eng.close()
    return out


@pytest.mark.parametrize("leaf", [1, 16])
def test_distributed_build_matches_single_gpu(leaf):
    from paper_2203_08966_b200.initcond import make_rng, plummer_cluster

    b = plummer_cluster(20_000, make_rng(1))
    ref = _single(b, 1, leaf=leaf)
    for ranks in (1, 2, 3):
        got = _run_build(ranks, b, 1, leaf=leaf)
        if ranks > 1:
            assert min(got["counts"]) > 0
        np.testing.assert_array_equal(got["work"], ref["work"])  # identical interaction lists
        err = np.linalg.norm(got["acc"][:, :3] - ref["acc"][:, :3]) / np.linalg.norm(ref["acc"][:, :3])
        assert err < 1e-5, (ranks, err)
        np.testing.assert_allclose(got["pos"][:, :3], ref["pos"][:, :3], rtol=0, atol=1e-6)


def test_distributed_build_clustered_multi_step():
    """cfg0/cfg3 geometry (two colliding clusters), 3 steps, 4 ranks: work
    identical per body; costzones keeps the ranks' work balanced."""
    from paper_2203_08966_b200.initcond import colliding_plummers

    b = colliding_plummers(12_000, 3)
    ref = _single(b, 3, theta=0.6, eps=1e-4, leaf=32, dt=5e-4)
    got = _run_build(4, b, 3, theta=0.6, eps=1e-4, leaf=32, dt=5e-4)
    assert np.mean(got["work"] != ref["work"]) < 1e-3
    err = np.linalg.norm(got["acc"][:, :3] - ref["acc"][:, :3]) / np.linalg.norm(ref["acc"][:, :3])
    assert err < 1e-5
    assert min(got["counts"]) > 0.2 * len(b) / 4
    # the locally essential trees are a strict subset of the peers' trees
    own = sum(s["own_records"] for s in got["let"])
    for s in got["let"]:
        assert s["records"] < own - s["own_records"], got["let"]
    print("LET", got["let"])


def test_target_boxes_match_numpy():
    """bh_sim_target_boxes: per-range bounding boxes (any range length, empty
    ranges, ranges straddling warps) and their union, exactly."""
    from paper_2203_08966_b200.engine import Engine
    from paper_2203_08966_b200.initcond import make_rng, plummer_cluster

    b = plummer_cluster(100_003, make_rng(5))
    eng = Engine("fp32", 0)
    pos = eng.bodies_tensor(b.position, b.mass)
    eng.sim_load_state(pos, eng.vec_tensor(b.velocity))
    eng.sim_set_R(1.001 * float(pos[:, :3].abs().max()))
    eng.sim_sort()
    n = eng.sim_n
    x = torch.empty((n, 4), dtype=torch.float32, device="cuda")
    from paper_2203_08966_b200 import _lib
    eng.sim_export(_lib.BH_SIM_POS, 0, n, x)
    xs = x[:, :3].double().cpu().numpy()
    for cuts in ([0, n], [0, 0, 17, 17, 5000, 5031, 99_000, n], list(range(0, n, 1563)) + [n]):
        start = torch.tensor(cuts, dtype=torch.int64, device="cuda")
        g = len(cuts) - 1
        out = torch.empty((g + 1, 6), dtype=torch.float64, device="cuda")
        eng.sim_target_boxes(start, out)
        got = out.cpu().numpy()
        for k in range(g):
            seg = xs[cuts[k]:cuts[k + 1]]
            if len(seg):
                np.testing.assert_array_equal(got[1 + k, :3], seg.min(0))
                np.testing.assert_array_equal(got[1 + k, 3:], seg.max(0))
            else:
                assert np.all(np.isposinf(got[1 + k, :3])) and np.all(np.isneginf(got[1 + k, 3:]))
        np.testing.assert_array_equal(got[0, :3], xs.min(0))
        np.testing.assert_array_equal(got[0, 3:], xs.max(0))
    eng.close()


def _simulate_worker(rank, port, scheme, out_path, p2p="0"):
    import torch.distributed as dist

    from paper_2203_08966_b200.simulation import SimConfig, simulate

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), BH_P2P=p2p)
    torch.cuda.set_device(0)  # both ranks share the one GPU; gloo collectives are host-staged
    dist.init_process_group("gloo", rank=rank, world_size=2)
    cfg = SimConfig(n=24_000, algorithm=1, theta=0.6, dt=1e-3, steps=3, eps=1e-3, seed=4, leaf_size=16,
                    precision="fp32", leaf_mode="bucket", devices=2, decomposition=scheme)
    res = simulate(cfg)
    if rank == 0:
        np.savez(out_path, pos=res.bodies.position, vel=res.bodies.velocity, work=res.bodies.work)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("scheme,p2p", [("distributed", "0"), ("replicated", "0"), ("replicated", "1")])
def test_simulate_devices2_matches_one_device(tmp_path, scheme, p2p):
    """simulate(devices=2) through torch.distributed (two processes sharing this
    GPU, gloo): the same per-body work as devices=1, positions to fp32 rounding.
    replicated + p2p=1: each process opens the other's result buffers by CUDA
    IPC handle and the walk stores its rows into them (must succeed)."""
    import socket

    import torch.multiprocessing as mp

    from paper_2203_08966_b200.simulation import SimConfig, simulate

    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    out = str(tmp_path / "r.npz")
    mp.spawn(_simulate_worker, args=(port, scheme, out, p2p), nprocs=2, join=True)
    got = np.load(out)
    ref = simulate(SimConfig(n=24_000, algorithm=1, theta=0.6, dt=1e-3, steps=3, eps=1e-3, seed=4, leaf_size=16,
                             precision="fp32", leaf_mode="bucket"))
    np.testing.assert_array_equal(got["work"], ref.bodies.work)
    np.testing.assert_allclose(got["pos"], ref.bodies.position, rtol=0, atol=1e-5)
    np.testing.assert_allclose(got["vel"], ref.bodies.velocity, rtol=0, atol=1e-4)


@pytest.mark.parametrize("scheme", ["distributed", "replicated"])
def test_eight_ranks_cfg3_geometry(scheme, monkeypatch):
    """The 8-GPU split of BASELINE cfg3 (two colliding Plummer clusters,
    theta 0.6, eps 1e-4, leaf 32, dt 5e-4), emulated as 8 ranks on one GPU,
    2 steps at 2e5 bodies: per-body work equal to one GPU, accelerations to
    fp32 summation order, every rank holding a share of the bodies."""
    from paper_2203_08966_b200.initcond import colliding_plummers

    b = colliding_plummers(100_000, 3)
    kw = dict(theta=0.6, eps=1e-4, leaf=32, dt=5e-4)
    ref = _single(b, 2, **kw)
    if scheme == "distributed":
        got = _run_build(8, b, 2, **kw)
        assert min(got["counts"]) > 0.2 * len(b) / 8
        assert np.mean(got["work"] != ref["work"]) < 1e-3
        err = np.linalg.norm(got["acc"][:, :3] - ref["acc"][:, :3]) / np.linalg.norm(ref["acc"][:, :3])
        assert err < 1e-5, err
    else:
        monkeypatch.setenv("BH_P2P", "1")
        outs = _run("fp32", 8, b, 2, **kw)
        for pos, work, zones, used in outs:
            assert used and len(zones) == 9
            assert np.mean(work != ref["work"]) < 1e-3
            rel = np.abs(pos - ref["pos"][:, :3]).max() / np.abs(ref["pos"][:, :3]).max()
            assert rel < 1e-5, rel

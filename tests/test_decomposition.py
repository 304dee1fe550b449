"""Multi-rank decomposition: costzones cuts, and the
replicated-tree / partitioned-walk protocol over torch.distributed gloo with
world size 2 (CPU), compared bit for bit with a single-rank run."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2203_08966_b200.decomposition import (
    DistributedSim, StepParams, TorchComm, costzones, costzones_device)


def test_costzones_matches_reference_rule():
    # decomposition.py:35-57 examples: straddling body goes to the left zone
    np.testing.assert_array_equal(costzones([1, 1, 1, 1], 2), [0, 2, 4])
    np.testing.assert_array_equal(costzones([3, 1, 1, 1], 2), [0, 1, 4])
    np.testing.assert_array_equal(costzones([1, 1, 1, 1, 1], 2), [0, 3, 5])
    with pytest.raises(ValueError):
        costzones([1, 1], 3)
    rng = np.random.Generator(np.random.Philox(key=5))
    for zones in (1, 2, 3, 7, 8):
        w = rng.integers(0, 3000, size=10_000)
        ref = costzones(w, zones)
        got = costzones_device(torch.from_numpy(w).to(torch.int32), zones)
        np.testing.assert_array_equal(got, ref)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q, n, steps):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from fake_engine import OracleEngine
    from paper_2203_08966_b200.initcond import two_clusters

    b = two_clusters(n, 3)
    sim = DistributedSim(OracleEngine(), TorchComm(), StepParams(0.6, 0.05, 1, 0.01))
    sim.load(torch.from_numpy(b.position), torch.from_numpy(b.velocity), torch.from_numpy(b.mass))
    sim.bootstrap()
    sim.step(steps)
    pos = torch.zeros((n, 4), dtype=torch.float64)
    vel = torch.zeros((n, 4), dtype=torch.float64)
    work = torch.zeros(n, dtype=torch.int64)
    sim.store(pos=pos, vel=vel, work=work)
    out_q.put((rank, pos[:, :3].numpy(), vel[:, :3].numpy(), work.numpy(), sim.zones))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_matches_single_rank():
    from oracle import oracle as orc
    from paper_2203_08966_b200.initcond import two_clusters

    n, steps = 300, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, n, steps)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    b = two_clusters(n, 3)
    x, v, a, w = orc.leapfrog(b.mass, b.position, b.velocity, 0.01, steps, 0.6, 0.05)
    for rank, pos, vel, work, zones in res:
        np.testing.assert_array_equal(pos, x)   # every rank holds the full, identical state
        np.testing.assert_array_equal(vel, v)
        np.testing.assert_array_equal(work, w)
        assert len(zones) == 3 and zones[0] == 0 and zones[-1] == n and 0 < zones[1] < n


def _coll_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2203_08966_b200.decomposition import DistributedBuildSim, StepParams

    class Dummy:
        precision = "fp32"
        device = torch.device("cpu")

    sim = DistributedBuildSim(Dummy(), TorchComm(), StepParams(0.5, 0.01, 1, 0.01))
    # variable-size allgather
    t = torch.arange(3 + 2 * rank, dtype=torch.int64).reshape(-1, 1) + 100 * rank
    got = [x.flatten().tolist() for x in sim._allgather_v(t)]
    # all-to-all of rows grouped by destination: rank r sends (r, q) rows x (q+1)
    rows, counts = [], []
    for q in range(world):
        rows += [[rank, q]] * (q + 1)
        counts.append(q + 1)
    recv = sim._alltoall_v(torch.tensor(rows, dtype=torch.int32), counts).tolist()
    out_q.put((rank, got, recv))
    dist.barrier()
    dist.destroy_process_group()


def test_stage2_collectives_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_coll_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, got, recv in res:
        assert got == [[0, 1, 2], [100, 101, 102, 103, 104]]
        assert recv == [[0, rank]] * (rank + 1) + [[1, rank]] * (rank + 1)


def test_top_tree_combine_matches_reference_moments():
    """The distributed step's exact fp64 top-tree recombination (_combine,
    hashed.py:719-786 / flattree.py:201-252) reproduces every internal cell of
    the oracle tree bit for bit from its children, in slot order."""
    from oracle import oracle as orc
    from paper_2203_08966_b200.decomposition import _combine
    from paper_2203_08966_b200.initcond import make_rng, plummer_cluster

    b = plummer_cluster(3000, make_rng(11))
    pos = np.asarray(b.position, dtype=np.float64)
    m = np.asarray(b.mass, dtype=np.float64)
    R = orc.bounds(pos)
    o = orc.sort_order(orc.morton_keys(pos, R))
    t = orc.build_tree(m[o], pos[o], R)
    ch = np.asarray(t.children).reshape(len(t), -1)
    checked = 0
    for c in range(len(t)):
        kids = [int(k) for k in ch[c] if k >= 0]
        if not kids:
            continue
        rows = [(float(t.mass[k]), tuple(float(x) for x in t.com[k]), tuple(float(x) for x in t.quad[k]))
                for k in kids]
        mass, com, quad = _combine(rows)
        assert mass == t.mass[c]
        assert com == tuple(float(x) for x in t.com[c])
        assert quad == tuple(float(x) for x in t.quad[c])
        checked += 1
    assert checked > 500


def test_branch_rows_pack_roundtrip():
    from paper_2203_08966_b200.decomposition import _BR_INTS, _REC_INTS, _pack_branches, _unpack_branches

    rng = np.random.default_rng(3)
    nb = 37
    br = dict(key=torch.from_numpy(rng.integers(1, 1 << 62, nb, dtype=np.int64)),
              level=torch.from_numpy(rng.integers(0, 22, nb).astype(np.int32)),
              count=torch.from_numpy(rng.integers(1, 1 << 40, nb, dtype=np.int64)),
              mom=torch.from_numpy(rng.normal(size=(nb, 10))),
              rec=torch.from_numpy(rng.integers(0, 1 << 30, nb).astype(np.int32)),
              lo=torch.from_numpy(rng.integers(0, 1 << 30, nb).astype(np.int32)),
              recs=torch.from_numpy(rng.integers(-(1 << 31), 1 << 31, (nb, _REC_INTS)).astype(np.int32)))
    rows = _pack_branches(br)
    assert rows.shape == (nb, _BR_INTS) and rows.dtype == torch.int32
    key, level, count, mom, rec, lo, recs = _unpack_branches(rows.numpy())
    np.testing.assert_array_equal(key, br["key"].numpy())
    np.testing.assert_array_equal(level, br["level"].numpy())
    np.testing.assert_array_equal(count, br["count"].numpy())
    np.testing.assert_array_equal(mom, br["mom"].numpy())
    np.testing.assert_array_equal(rec, br["rec"].numpy())
    np.testing.assert_array_equal(lo, br["lo"].numpy())
    np.testing.assert_array_equal(recs, br["recs"].numpy())


def test_lcp_matches_key_prefix_levels():
    """_lcp: the deepest level at which two Morton keys share a cell
    (hashed.py:376-388): 21 - ceil(bitlen(a ^ b) / 3)."""
    from paper_2203_08966_b200.decomposition import _lcp

    rng = np.random.default_rng(4)
    for _ in range(2000):
        a, b = (int(x) for x in rng.integers(0, 1 << 63, 2, dtype=np.uint64))
        shared = 0
        for lvl in range(1, 22):
            if (a >> (3 * (21 - lvl))) == (b >> (3 * (21 - lvl))):
                shared = lvl
            else:
                break
        assert _lcp(a, b) == shared, (a, b)


def _thread_ranks(engines, steps, n=600):
    """DistributedSim on in-process ranks (ThreadComm) with the given engines."""
    import threading

    from paper_2203_08966_b200.decomposition import DistributedSim, StepParams, ThreadComm
    from paper_2203_08966_b200.initcond import make_rng, plummer_cluster

    b = plummer_cluster(n, make_rng(3))
    comms = ThreadComm.group(len(engines))
    out, err = [None] * len(engines), []

    def body(r):
        try:
            sim = DistributedSim(engines[r], comms[r], StepParams(0.6, 0.05, 1, 0.01))
            pos = torch.from_numpy(np.c_[b.position, b.mass])
            sim.load(pos, torch.from_numpy(np.c_[b.velocity, np.zeros(n)]), torch.from_numpy(b.mass))
            sim.bootstrap()
            sim.step(steps)
            p = torch.empty((n, 4), dtype=torch.float64)
            w = torch.empty(n, dtype=torch.int64)
            sim.store(pos=p, work=w)
            out[r] = (p[:, :3].numpy(), w.numpy(), sim.p2p)
        except Exception as e:  # pragma: no cover - surfaced below
            err.append(e)
            comms[r].hub.barrier.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(len(engines))]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    if err:
        raise err[0]
    return out


def test_peer_store_protocol_matches_allreduce(monkeypatch):
    """Replicated ranks whose walk stores into the peers (BH_P2P auto) give the
    same trajectory, bit for bit, as the all-reduce exchange (BH_P2P=0)."""
    from fake_engine import OracleEngine, PeerOracleEngine

    monkeypatch.setenv("BH_P2P", "auto")
    p2p = _thread_ranks([PeerOracleEngine(), PeerOracleEngine()], 2)
    monkeypatch.setenv("BH_P2P", "0")
    ar = _thread_ranks([OracleEngine(), OracleEngine()], 2)
    for (pa, wa, used), (pb, wb, _) in zip(p2p, ar):
        assert used
        np.testing.assert_array_equal(pa, pb)
        np.testing.assert_array_equal(wa, wb)


def test_peer_store_failure_falls_back(monkeypatch):
    """Peer stores that do not land (rows dropped) are caught by the bootstrap
    digest check; the ranks fall back to the all-reduce and stay exact.  With
    BH_P2P=1 the same failure raises."""
    from fake_engine import OracleEngine, PeerOracleEngine

    monkeypatch.setenv("BH_P2P", "auto")
    got = _thread_ranks([PeerOracleEngine(drop=5), PeerOracleEngine(drop=5)], 1)
    monkeypatch.setenv("BH_P2P", "0")
    ref = _thread_ranks([OracleEngine(), OracleEngine()], 1)
    for (pa, wa, used), (pb, wb, _) in zip(got, ref):
        assert not used
        np.testing.assert_array_equal(pa, pb)
        np.testing.assert_array_equal(wa, wb)
    monkeypatch.setenv("BH_P2P", "1")
    with pytest.raises(RuntimeError, match="disagree"):
        _thread_ranks([PeerOracleEngine(drop=5), PeerOracleEngine(drop=5)], 1)


def test_host_top_tree_recombines_the_oracle_tree():
    """bh_top_tree (libbh host C++, the distributed step's top-tree assembly):
    given the level-3 cells of the oracle tree as branch nodes (any rank
    layout), the top cells it recombines carry the oracle's own fp64 moments,
    counts and children, laid out breadth first with children contiguous in
    slot order, and each branch entry points back at its row."""
    import ctypes

    from oracle import oracle as orc
    from paper_2203_08966_b200 import _lib
    from paper_2203_08966_b200.decomposition import _BR_INTS, _REC_INTS, _pack_branches
    from paper_2203_08966_b200.initcond import make_rng, plummer_cluster

    b = plummer_cluster(5000, make_rng(4))
    pos = np.asarray(b.position, dtype=np.float64)
    m = np.asarray(b.mass, dtype=np.float64)
    R = orc.bounds(pos)
    o = orc.sort_order(orc.morton_keys(pos, R))
    t = orc.build_tree(m[o], pos[o], R)
    L, theta = 16, 0.6
    # branch nodes: the cells at level 3 plus shallower leaves (a partition of the bodies)
    keys = t.key.astype(np.int64)
    lev = t.level.astype(np.int64)
    is_br = (lev == 3) | ((lev < 3) & (t.count == 1))
    br_idx = np.nonzero(is_br)[0]
    assert t.count[br_idx].sum() == len(m)
    nb = len(br_idx)
    mom = np.concatenate([t.mass[br_idx, None], t.com[br_idx], t.quad[br_idx]], axis=1)
    rows = _pack_branches(dict(
        key=torch.from_numpy(keys[br_idx]), level=torch.from_numpy(lev[br_idx].astype(np.int32)),
        count=torch.from_numpy(t.count[br_idx].astype(np.int64)), mom=torch.from_numpy(mom),
        rec=torch.zeros(nb, dtype=torch.int32), lo=torch.zeros(nb, dtype=torch.int32),
        recs=torch.from_numpy(np.arange(nb * _REC_INTS, dtype=np.int32).reshape(nb, _REC_INTS)))).numpy()
    rows = np.ascontiguousarray(rows)
    cap = 22 * nb + 64
    region = np.zeros((cap, _REC_INTS), np.int32)
    kind = np.zeros(cap, np.int32)
    row_of = np.zeros(cap, np.int32)
    bb = np.zeros(nb, np.int64)
    P = ctypes.c_void_p
    ne = _lib.lib().bh_top_tree(rows.ctypes.data_as(P), nb, 0, L, float(R), theta, region.ctypes.data_as(P),
                                kind.ctypes.data_as(P), row_of.ctypes.data_as(P), bb.ctypes.data_as(P), cap)
    assert ne > 0
    cell_of_key = {int(k): c for c, k in enumerate(keys)}
    # walk the region from the root, matching oracle cells
    stack = [(0, 1)]
    seen = 0
    while stack:
        e, key = stack.pop()
        c = cell_of_key[key]
        if kind[e] == 2:
            assert keys[br_idx[row_of[e]]] == key
            np.testing.assert_array_equal(region[e], rows[row_of[e], 27:27 + _REC_INTS])
            continue
        rec = region[e]
        f = rec.view(np.float32)
        assert f[10] == np.float32(t.mass[c]) and rec[13] == t.count[c]
        np.testing.assert_array_equal(f[[0, 1, 2]], (-t.com[c]).astype(np.float32))
        np.testing.assert_array_equal(f[[4, 5, 7, 8, 9, 11]], t.quad[c][[0, 1, 3, 2, 4, 5]].astype(np.float32))
        seen += 1
        if kind[e] == 1:  # a bucket-sized top cell
            assert t.count[c] <= L and rec[14] == 0
            continue
        kids = [int(k) for k in t.children[c] if k >= 0]
        assert rec[14] == len(kids)
        for j, k in enumerate(kids):
            stack.append((rec[12] + j, int(keys[k])))
    assert seen > 10

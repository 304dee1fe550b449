"""Multi-GPU decomposition -- the GPU counterpart of ``nbsim.decomposition``
(/root/reference/pkg/src/nbsim/decomposition.py) and of the rank pipeline in
``simulation.py:439-504``.

One process per GPU.  Round-1 scheme ("replicated tree, partitioned walk"):

* every rank keeps the full body state resident and runs the same
  kick + drift, keys, radix sort, permutation and tree build (all cheap,
  bandwidth-bound kernels), so every rank holds the bit-identical global tree;
* the traversal -- the O(N log N) part, >80% of a step -- is partitioned: the
  Morton-sorted bodies are cut into ``size`` contiguous zones of equal
  previous-step work with the reference's ``costzones`` rule
  (decomposition.py:35-57), and each rank walks only its zone;
* the exchange step is one NCCL all-reduce of the accelerations (and work)
  of the disjoint zones, after which every rank finishes the step.

Because each target's interaction list depends only on the global tree, the
result equals the single-GPU step (bitwise in fp64 mode, where the walk keeps
the reference's order; to fp32 rounding in fp32 mode).  The locally-essential
tree exchange that would also distribute the build (branch-node allgather +
LET all-to-all) is the planned next stage.

``Comm`` abstracts the three collectives used; ``TorchComm`` runs them over
``torch.distributed`` (NCCL on GPUs, gloo in the CPU tests) and
``ThreadComm`` joins several in-process ranks (used to emulate R ranks on one
GPU in tests -- host-side barriers only, no kernel waits on another).
"""

from __future__ import annotations

import ctypes
import math
import os
import threading
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


def costzones(works, zones: int) -> np.ndarray:
    """decomposition.py:35-57: ``zones + 1`` cut indices of contiguous zones of
    near-equal work; zone k ends with the first body whose cumulative work
    reaches (k+1)/zones of the total (the straddling body included)."""
    works = np.asarray(works, dtype=np.int64)
    n = len(works)
    if zones < 1:
        raise ValueError("need at least one zone")
    if zones > n:
        raise ValueError(f"cannot cut {n} bodies into {zones} zones")
    if np.any(works < 0):
        raise ValueError("work estimates must be non-negative")
    prefix = np.cumsum(works)
    total = int(prefix[-1])
    targets = np.arange(1, zones) * total / zones
    cuts = np.searchsorted(prefix, targets, side="left") + 1
    return np.concatenate(([0], cuts, [n])).astype(np.int64)


def costzones_cuts(works: torch.Tensor, zones: int) -> torch.Tensor:
    """``costzones`` on a device work array, left on the device: the zones+1
    boundaries [0, c_1, ..., n] as an int64 tensor (same rule, integer-exact:
    the zone targets k*total/zones are compared as prefix*zones >= k*total)."""
    n = works.shape[0]
    if zones > n:
        raise ValueError(f"cannot cut {n} bodies into {zones} zones")
    dev = works.device
    if n == 0:
        return torch.zeros(zones + 1, dtype=torch.int64, device=dev)
    prefix = torch.cumsum(works.to(torch.int64), 0)
    scaled = prefix * zones
    t = torch.arange(1, zones, device=dev, dtype=torch.int64) * prefix[-1]
    cuts = torch.searchsorted(scaled, t, side="left") + 1
    ends = torch.tensor([0, n], dtype=torch.int64, device=dev)
    return torch.cat([ends[:1], cuts, ends[1:]])


def costzones_device(works: torch.Tensor, zones: int) -> list[int]:
    """``costzones`` on a device work array (one host read)."""
    return [int(c) for c in costzones_cuts(works, zones).tolist()]


# --------------------------------------------------------------- collectives


class Comm:
    rank = 0
    size = 1

    def allreduce_sum_(self, t: torch.Tensor) -> None:  # in place
        pass

    def allreduce_max_(self, t: torch.Tensor) -> None:
        pass

    def barrier(self) -> None:
        pass

    def stream_barrier(self) -> None:
        """Every rank's device work queued so far is done before any rank's
        work queued after this (orders peer-memory stores between ranks)."""

    def allgather_bytes(self, b: bytes) -> list[bytes]:
        return [b]


class TorchComm(Comm):
    """torch.distributed collectives: NCCL on CUDA tensors.  Under a gloo
    group CUDA tensors are staged through host memory (tests, and several
    ranks sharing one GPU for a smoke run)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.staged = dist.get_backend(group) == "gloo"

    def _host(self, t):
        return t.cpu() if (self.staged and t.is_cuda) else t

    def _reduce(self, t, op):
        h = self._host(t)
        self.dist.all_reduce(h, op=op, group=self.group)
        if h is not t:
            t.copy_(h)

    def allreduce_sum_(self, t):
        self._reduce(t, self.dist.ReduceOp.SUM)

    def allreduce_max_(self, t):
        self._reduce(t, self.dist.ReduceOp.MAX)

    def allgather(self, outs, t):
        h = self._host(t)
        if h is t:
            self.dist.all_gather(outs, t, group=self.group)
            return
        hs = [torch.empty_like(h) for _ in outs]
        self.dist.all_gather(hs, h.contiguous(), group=self.group)
        for o, x in zip(outs, hs):
            o.copy_(x)

    def alltoall_single(self, out, t, recv_counts, send_counts):
        h = self._host(t)
        if h is t:
            self.dist.all_to_all_single(out, t, recv_counts, send_counts, group=self.group)
            return
        ho = torch.empty(out.shape, dtype=out.dtype)
        self.dist.all_to_all_single(ho, h.contiguous(), recv_counts, send_counts, group=self.group)
        out.copy_(ho)

    def barrier(self):
        self.dist.barrier(group=self.group)

    def stream_barrier(self):
        if self.staged:  # host-staged (gloo): the device must be idle first
            torch.cuda.synchronize()
            self.dist.barrier(group=self.group)
            return
        if getattr(self, "_tick", None) is None:
            self._tick = torch.zeros(1, dtype=torch.int32, device=torch.cuda.current_device())
        self.dist.all_reduce(self._tick, group=self.group)  # NCCL: ordered on the current stream

    def allgather_bytes(self, b: bytes) -> list[bytes]:
        dev = "cpu" if self.staged else torch.device("cuda", torch.cuda.current_device())
        t = torch.frombuffer(bytearray(b), dtype=torch.uint8).to(dev)
        outs = [torch.empty_like(t) for _ in range(self.size)]
        self.dist.all_gather(outs, t, group=self.group)
        return [bytes(o.cpu().numpy().tobytes()) for o in outs]


class _ThreadHub:
    def __init__(self, size: int):
        self.size = size
        self.barrier = threading.Barrier(size)
        self.slots: list = [None] * size


class ThreadComm(Comm):
    """In-process ranks (one thread each) joined by host barriers."""

    def __init__(self, hub: _ThreadHub, rank: int):
        self.hub = hub
        self.rank = rank
        self.size = hub.size

    @staticmethod
    def group(size: int) -> list["ThreadComm"]:
        hub = _ThreadHub(size)
        return [ThreadComm(hub, r) for r in range(size)]

    def _reduce(self, t, op):
        if t.is_cuda:
            torch.cuda.synchronize(t.device)
        self.hub.slots[self.rank] = t
        self.hub.barrier.wait()
        acc = self.hub.slots[0].clone()
        for r in range(1, self.size):
            acc = op(acc, self.hub.slots[r])
        if acc.is_cuda:
            torch.cuda.synchronize(acc.device)
        self.hub.barrier.wait()
        t.copy_(acc)

    def allreduce_sum_(self, t):
        self._reduce(t, torch.add)

    def allreduce_max_(self, t):
        self._reduce(t, torch.maximum)

    def barrier(self):
        self.hub.barrier.wait()

    def stream_barrier(self):
        if torch.cuda.is_available():
            torch.cuda.synchronize()
        self.hub.barrier.wait()

    def allgather_bytes(self, b):
        self.hub.slots[self.rank] = b
        self.hub.barrier.wait()
        out = list(self.hub.slots)
        self.hub.barrier.wait()
        return out


# ------------------------------------------------------------------ the driver


@dataclass
class StepParams:
    theta: float
    eps: float
    leaf_size: int
    dt: float


class DistributedSim:
    """The `_drive` loop (simulation.py:478-504) across ranks.

    ``engine`` is this rank's :class:`~paper_2203_08966_b200.engine.Engine`
    (any object with the same ``sim_*`` phase methods works, which is how the
    CPU tests drive the protocol).  ``load`` takes the full initial state on
    every rank (replicated state)."""

    def __init__(self, engine, comm: Comm, params: StepParams):
        self.eng = engine
        self.comm = comm
        self.p = params
        self.n = 0
        self.zones: list[int] = []
        self.p2p = False  # results through peer memory (set up by load)

    def _bufs(self):
        dev = self.eng.device
        comps = 4
        dtype = torch.float32 if self.eng.precision == "fp32" else torch.float64
        if getattr(self, "_acc", None) is None or self._acc.shape[0] != self.n:
            self._acc = torch.zeros((self.n, comps), dtype=dtype, device=dev)
            self._work = torch.zeros(self.n, dtype=torch.int32, device=dev)
            self._prev = torch.zeros(self.n, dtype=torch.int32, device=dev)
        return self._acc, self._work, self._prev

    def load(self, pos, vel, mass=None) -> None:
        self.n = pos.shape[0]
        self.eng.sim_load(pos, vel, mass)
        self.p2p = self._setup_peers()

    # -- results over peer memory: the walk's epilogue stores its zone's rows
    # into every rank's resident buffers (NVLink), replacing the all-reduce
    def _setup_peers(self) -> bool:
        mode = os.environ.get("BH_P2P", "auto")
        size = self.comm.size
        if mode == "0" or size == 1 or size > 8 or not hasattr(self.eng, "sim_set_peers"):
            return False
        me = self.comm.rank
        try:
            if isinstance(self.comm, ThreadComm):  # ranks in one process: raw device pointers
                ptrs = self.comm.allgather_bytes(self.eng.sim_result_ptrs())
                self.eng.sim_set_peer_ptrs([ptrs[q] for q in range(size) if q != me])
            else:
                # NVLink stores need peer access between every pair of devices
                # (ranks sharing one device always have it)
                devs = [int(d) for d in self.comm.allgather_bytes(str(self.eng.device.index).encode())]
                mine = self.eng.device.index
                if not all(d == mine or torch.cuda.can_device_access_peer(mine, d) for d in devs):
                    raise RuntimeError("no peer access between the ranks' devices")
                hs = self.comm.allgather_bytes(self.eng.sim_ipc_handles())
                self.eng.sim_set_peers([hs[q] for q in range(size) if q != me])
            ok = 1
        except (ValueError, RuntimeError):
            ok = 0
        flag = torch.tensor([ok], dtype=torch.int64, device=self.eng.device)
        self.comm.allreduce_sum_(flag)
        if int(flag.item()) != size:  # some rank could not map its peers: all-reduce path
            if ok:
                self.eng.sim_set_peers([])
            if mode == "1":
                raise RuntimeError("BH_P2P=1: peer buffers could not be mapped on every rank")
            return False
        return True

    def _zone(self) -> tuple[int, int]:
        _, _, prev = self._bufs()
        self.eng.sim_export(_lib.BH_SIM_PREV_WORK, 0, self.n, prev)
        self.zones = costzones_device(prev, self.comm.size)
        r = self.comm.rank
        return self.zones[r], self.zones[r + 1]

    def _forces(self, record_work: bool, bounds_ready: bool) -> None:
        p = self.p
        for _ in range(3):
            self.eng.sim_prepare(p.theta, p.eps, p.leaf_size, bounds_ready)
            # a build that overflowed its cell capacity is redone before any walk
            # (the walk would store its rows into the peers); replicas build the
            # same tree, so every rank takes the same branch.  The capacity check
            # and this step's costzones cuts come back in ONE host read.
            if hasattr(self.eng, "sim_tree_fits_dev"):
                _, _, prev = self._bufs()
                self.eng.sim_export(_lib.BH_SIM_PREV_WORK, 0, self.n, prev)
                if getattr(self, "_fit", None) is None:
                    self._fit = torch.zeros(1, dtype=torch.int32, device=self.eng.device)
                self.eng.sim_tree_fits_dev(self._fit)
                host = torch.cat([self._fit.to(torch.int64), costzones_cuts(prev, self.comm.size)]).tolist()
                if host[0]:
                    self.zones = [int(c) for c in host[1:]]
                    break
                self.eng.sim_tree_fits()  # overflowed: grow the capacity, build again
            elif not hasattr(self.eng, "sim_tree_fits") or self.eng.sim_tree_fits():
                self._zone()
                break
            bounds_ready = False
        else:
            raise RuntimeError("tree cell capacity kept overflowing")
        b, e = self.zones[self.comm.rank], self.zones[self.comm.rank + 1]
        if getattr(self, "p2p", False):
            self.comm.stream_barrier()  # every rank is done reading its acc (the kick)
            self.eng.sim_walk_range(p.theta, p.eps, p.leaf_size, b, e, record_work)  # + peers' rows
            self.comm.stream_barrier()  # every rank's rows have landed
            if record_work:
                self.eng.sim_scatter_work()
            return
        self.eng.sim_walk_range(p.theta, p.eps, p.leaf_size, b, e, record_work)
        acc, work, _ = self._bufs()
        acc.zero_()
        self.eng.sim_export(_lib.BH_SIM_ACC, b, e, acc[b:e])
        self.comm.allreduce_sum_(acc)  # disjoint zones: x + 0 is exact
        self.eng.sim_import(_lib.BH_SIM_ACC, 0, self.n, acc)
        if record_work:
            work.zero_()
            self.eng.sim_export(_lib.BH_SIM_WORK, b, e, work[b:e])
            self.comm.allreduce_sum_(work)
            self.eng.sim_import(_lib.BH_SIM_WORK, 0, self.n, work)
            self.eng.sim_scatter_work()

    def bootstrap(self) -> None:
        """simulation.py:487: forces for the first kick, work not recorded."""
        self._forces(record_work=False, bounds_ready=False)
        if getattr(self, "p2p", False) and not self._replicas_agree():
            # peer stores did not land everywhere: fall back to the all-reduce
            if os.environ.get("BH_P2P") == "1":
                raise RuntimeError("BH_P2P=1: ranks disagree after the peer-memory walk")
            self.eng.sim_set_peers([])
            self.p2p = False
            self._forces(record_work=False, bounds_ready=False)

    def _replicas_agree(self) -> bool:
        """Every rank holds bit-identical accelerations (a digest of the bit
        patterns, compared by max and -min over ranks)."""
        acc, _, _ = self._bufs()
        self.eng.sim_export(_lib.BH_SIM_ACC, 0, self.n, acc)
        bits = acc.view(torch.int32).reshape(-1).to(torch.int64)
        w = torch.arange(bits.shape[0], device=bits.device, dtype=torch.int64) % 1021 + 1
        d = (bits * w).sum()
        mm = torch.stack([d, -d])
        self.comm.allreduce_max_(mm)
        return bool((mm[0] == -mm[1]).item())

    def step(self, steps: int = 1) -> None:
        for _ in range(steps):
            self.eng.sim_begin_step(self.p.dt)
            self._forces(record_work=True, bounds_ready=True)
            self.eng.sim_end_step(self.p.dt)
        if hasattr(self.eng, "check"):
            self.eng.check()  # latched device errors, once per call (capacity: checked per step above)

    def store(self, pos=None, vel=None, acc=None, work=None) -> None:
        self.eng.sim_store(pos, vel, acc, work)


# =========================================================================
# Stage 2: distributed build (key-range decomposition)
# =========================================================================
#
# Every rank owns the bodies of a contiguous Morton key range and builds only
# its part of the tree; the exchange steps are those of SURVEY.md §8(e):
#
#   allreduce(max |x|) -> R                                  simulation.py:201-208
#   migrate bodies to the owner of their key range           decomposition.py:84-263
#     (splitters from last step's costzones on the global order, all-to-all)
#   allgather boundary keys -> local tree with global leaf depths
#   allgather branch nodes -> exact fp64 top tree on every rank  hashed.py:609-786
#   locally essential trees: each rank sends each peer the records its target
#     boxes could open and the bucket bodies they could resolve (all-to-all)
#   walk the rank's own bodies; costzones cuts -> next splitters
#
# Per-target interaction lists equal the single-GPU walk's (same cells, same
# fp32 records, same MAC), so work counts match exactly and accelerations to
# fp32 summation order.  fp32 only.

_REC_INTS = 16  # a 64-byte WalkNode as int32 columns: a(0-3) b(4-7) c(8-11) d(12-15)
_DEFER_BIT = 1 << 30  # in d.w (level): pass A of the overlapped walk defers the record


def _lcp(a: int, b: int) -> int:
    x = a ^ b
    return 21 - (x.bit_length() + 2) // 3


def _combine(children):
    """_moments_kernel (flattree.py:201-252) on (mass, com[3], quad[6]) rows,
    in the given (slot) order, in IEEE double -- the same expressions."""
    total = 0.0
    cx = cy = cz = 0.0
    for m, c, _ in children:
        if m == 0.0:
            continue
        total += m
        cx += m * c[0]
        cy += m * c[1]
        cz += m * c[2]
    if total == 0.0:
        return 0.0, (0.0, 0.0, 0.0), (0.0,) * 6
    cx /= total
    cy /= total
    cz /= total
    q = [0.0] * 6
    for m, c, qc in children:
        if m == 0.0:
            continue
        dx = c[0] - cx
        dy = c[1] - cy
        dz = c[2] - cz
        d2 = dx * dx + dy * dy + dz * dz
        q[0] += qc[0] + m * (3.0 * (dx * dx) - d2)
        q[1] += qc[1] + m * (3.0 * (dx * dy) - 0.0)
        q[2] += qc[2] + m * (3.0 * (dx * dz) - 0.0)
        q[3] += qc[3] + m * (3.0 * (dy * dy) - d2)
        q[4] += qc[4] + m * (3.0 * (dy * dz) - 0.0)
        q[5] += qc[5] + m * (3.0 * (dz * dz) - d2)
    return total, (cx, cy, cz), tuple(q)


_BR_INTS = 2 + 1 + 2 + 20 + 1 + 1 + _REC_INTS  # key, level, count, mom[10] f64, rec, lo, record


def _pack_branches(br) -> torch.Tensor:
    """Branch-node rows as one int32 [nb, _BR_INTS] tensor (one allgather)."""
    nb = br["key"].shape[0]
    return torch.cat([br["key"].view(torch.int32).view(nb, 2), br["level"].view(nb, 1),
                      br["count"].view(torch.int32).view(nb, 2), br["mom"].view(torch.int32).view(nb, 20),
                      br["rec"].view(nb, 1), br["lo"].view(nb, 1), br["recs"]], dim=1).contiguous()


def _unpack_branches(rows: np.ndarray):
    """numpy inverse of _pack_branches: key, level, count, mom, rec, lo, record."""
    rows = np.ascontiguousarray(rows)
    key = rows[:, 0:2].copy().view(np.int64).ravel()
    level = rows[:, 2]
    count = rows[:, 3:5].copy().view(np.int64).ravel()
    mom = rows[:, 5:25].copy().view(np.float64)
    return key, level, count, mom, rows[:, 25], rows[:, 26], rows[:, 27:27 + _REC_INTS]


def _f32_bits(x: float) -> int:
    return int(np.array([x], dtype=np.float32).view(np.int32)[0])


class DistributedBuildSim:
    """Key-range decomposition with a distributed build (see above).

    ``load(pos, vel, mass, gid)`` takes this rank's initial chunk (any bodies;
    the first decomposition sorts them globally).  ``store`` returns this rank's
    current bodies with their global ids."""

    def __init__(self, engine, comm: Comm, params: StepParams):
        if engine.precision != "fp32":
            raise ValueError("the distributed build runs in fp32 mode")
        self.eng = engine
        self.comm = comm
        self.p = params
        self.splitters = None  # R-1 int64 keys: rank r owns [s[r-1], s[r])
        self.R = 1.0
        self.last_zones = None
        self.let_pad = 0.0  # widens the LET target boxes (inf: send whole subtrees)
        self.overlap = True  # walk the local part while the LETs travel
        self._side = None
        self._pack_done = None
        self.trace = {} if os.environ.get("BH_DIST_TRACE") else None  # host wall per section
        self._tlast = None

    # -- collectives on variable-size tensors --
    def _allgather_v(self, t: torch.Tensor) -> list:
        size = self.comm.size
        n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
        sizes = [torch.zeros_like(n) for _ in range(size)]
        self._allgather(sizes, n)
        sizes = torch.cat(sizes).cpu().tolist()
        mx = max(sizes) if sizes else 0
        pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        outs = [torch.empty_like(pad) for _ in range(size)]
        self._allgather(outs, pad)
        return [o[:k] for o, k in zip(outs, sizes)]

    def _allgather(self, outs, t):
        if isinstance(self.comm, TorchComm):
            self.comm.allgather(outs, t)
        elif isinstance(self.comm, ThreadComm):
            hub = self.comm.hub
            if t.is_cuda:
                torch.cuda.synchronize(t.device)
            hub.slots[self.comm.rank] = t
            hub.barrier.wait()
            for r in range(self.comm.size):
                outs[r].copy_(hub.slots[r])
            if t.is_cuda:
                torch.cuda.synchronize(t.device)
            hub.barrier.wait()
        else:
            outs[0].copy_(t)

    def _alltoall_many(self, items):
        """[(t, send_counts)] -> [(out, recv_counts)]: rows of each t, grouped by
        destination rank, to their owners, with one exchange of the counts."""
        size, me = self.comm.size, self.comm.rank
        dev = items[0][0].device
        sc = torch.tensor([c for _, cs in items for c in cs], dtype=torch.int64, device=dev)
        allc = [torch.zeros_like(sc) for _ in range(size)]
        self._allgather(allc, sc)
        A = torch.stack(allc).cpu().view(size, len(items), size)  # A[q, i, k]: q sends k
        res = []
        for i, (t, send_counts) in enumerate(items):
            recv = A[:, i, me].tolist()
            if isinstance(self.comm, TorchComm):
                out = torch.empty((sum(recv),) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
                self.comm.alltoall_single(out, t.contiguous(), recv, list(send_counts))
            else:  # thread / single: gather everyone's full send buffer and cut out our rows
                bufs = self._allgather_v(t)
                parts = []
                for q in range(size):
                    cq = A[q, i].tolist()
                    start = sum(cq[:me])
                    parts.append(bufs[q][start:start + cq[me]])
                out = torch.cat(parts) if parts else t[:0]
            res.append((out, recv))
        return res

    def _exchange_async(self, items):
        """_alltoall_many on a side stream that waits only for the work queued
        so far (the LET packing), so the collective overlaps the pass-A walk
        already queued on the compute stream; the compute stream then waits for
        it.  Host-mediated comms (ThreadComm) simply run it."""
        if not isinstance(self.comm, TorchComm) or not torch.cuda.is_available():
            return self._alltoall_many(items)
        main = torch.cuda.current_stream(self.eng.device)
        if self._side is None:
            self._side = torch.cuda.Stream(self.eng.device)
        ready = self._pack_done
        if ready is None:
            ready = torch.cuda.Event()
            ready.record(main)
        with torch.cuda.stream(self._side):
            self._side.wait_event(ready)
            res = self._alltoall_many(items)
        main.wait_stream(self._side)
        for out, _ in res:
            out.record_stream(main)
        return res

    def _alltoall_v(self, t: torch.Tensor, send_counts: list, return_counts: bool = False):
        """Rows of t, already grouped by destination rank, to their owners
        (with the per-source row counts if ``return_counts``)."""
        out, recv = self._alltoall_many([(t, send_counts)])[0]
        return (out, recv) if return_counts else out

    # -- state --
    def load(self, pos, vel, mass=None, gid=None) -> None:
        """This rank's initial chunk: pos/vel float32 (n, 4), gid its global ids."""
        eng = self.eng
        n = pos.shape[0]
        dev = eng.device
        acc = torch.zeros_like(vel)
        work = torch.ones(n, dtype=torch.int32, device=dev)  # simulation.py:482
        eng.sim_load_state(pos, vel, acc, work)
        self.gid_load = (gid if gid is not None else torch.arange(n, device=dev)).to(dev, torch.int64)
        self._maxabs0 = float(pos[:, :3].abs().max().item()) if n else 0.0

    def _export(self, what, n, shape, dtype):
        out = torch.empty(shape, dtype=dtype, device=self.eng.device)
        if n:
            self.eng.sim_export(what, 0, n, out)
        return out

    def _bounds(self, local_max: float | None = None) -> None:
        if local_max is None:
            local_max = self.eng.sim_local_maxabs()
        m = torch.tensor([local_max], dtype=torch.float64, device=self.eng.device)
        self.comm.allreduce_max_(m)
        ext = float(m.item())
        self.R = 1.001 * ext if ext > 0.0 else 1.0  # morton.py:41-42
        self.eng.sim_set_R(self.R)

    def _route_keys(self):
        """Keys of the bodies in their current order (no sort) and their gids."""
        eng = self.eng
        n = eng.sim_n
        keys = eng.sim_keys()
        ids = self._export(_lib.BH_SIM_ID, n, (n,), torch.int32)
        return n, keys, self.gid_load[ids.long()]

    def _sort(self):
        """Local sort with the global R; returns (n, sorted keys, sorted gids)."""
        eng = self.eng
        eng.sim_sort()
        n = eng.sim_n
        ids = self._export(_lib.BH_SIM_ID, n, (n,), torch.int32)
        gid = self.gid_load[ids.long()]
        keys = self._export(_lib.BH_SIM_KEYS, n, (n,), torch.int64)
        return n, keys, gid

    def _initial_splitters(self, keys: torch.Tensor) -> None:
        """Before any work is known: equal-count splitters from a key sample."""
        size = self.comm.size
        k = keys.shape[0]
        m = min(k, 512)  # integer sample positions (a float32 linspace rounds past k-1 above 2^24)
        idx = (torch.arange(m, device=keys.device, dtype=torch.int64) * max(k - 1, 0)) // max(m - 1, 1)
        samp = keys[idx] if k else keys
        allk = torch.sort(torch.cat(self._allgather_v(samp))).values
        if size == 1 or allk.numel() == 0:
            self.splitters = keys.new_zeros(0)
            return
        cut = [min(allk.numel() - 1, (r * allk.numel()) // size) for r in range(1, size)]
        self.splitters = allk[torch.tensor(cut, device=keys.device)]

    def _migrate(self, n: int, keys: torch.Tensor, gid: torch.Tensor) -> None:
        """Bodies to the owner of their key range (rows grouped by destination
        with a stable partition; skipped when no body changes owner)."""
        size = self.comm.size
        if size == 1:
            return
        dest = torch.searchsorted(self.splitters, keys, right=True)
        counts = torch.bincount(dest, minlength=size)
        moves = (n - counts[self.comm.rank]).reshape(1).to(torch.int64)
        self.comm.allreduce_sum_(moves)
        both = torch.cat([moves, counts.to(torch.int64)]).cpu().tolist()  # one host read
        if both[0] == 0:
            return  # ownership unchanged everywhere: the local sort follows
        order = torch.argsort(dest, stable=True)
        counts = both[1:]
        pos = self._export(_lib.BH_SIM_POS, n, (n, 4), torch.float32)
        vel = self._export(_lib.BH_SIM_VEL, n, (n, 4), torch.float32)
        acc = self._export(_lib.BH_SIM_ACC, n, (n, 4), torch.float32)
        work = self._export(_lib.BH_SIM_PREV_WORK, n, (n,), torch.int32)
        payload = torch.cat([pos.view(torch.int32), vel.view(torch.int32), acc.view(torch.int32),
                             work.view(-1, 1), gid.view(torch.int32).view(-1, 2)], dim=1)[order]
        got = self._alltoall_v(payload, counts)
        self.eng.sim_load_state(got[:, 0:4].clone().view(torch.float32),
                                got[:, 4:8].clone().view(torch.float32),
                                got[:, 8:12].clone().view(torch.float32),
                                got[:, 12].clone())
        self.gid_load = got[:, 13:15].clone().view(torch.int64).view(-1)

    def _next_splitters(self, n: int, keys: torch.Tensor, work=None) -> None:
        """costzones (decomposition.py:35-57) on the global order -- the ranks'
        sorted runs concatenated: zone k starts after the first body whose
        global work prefix reaches k/size of the total; its first body's key is
        splitter k (for the next step: bodies move, any monotone cut is valid)."""
        size = self.comm.size
        if size == 1:
            return
        dev = keys.device
        if work is None:
            work = self._export(_lib.BH_SIM_WORK, n, (n,), torch.int32)
        work = work.to(torch.int64)
        zero = torch.zeros((), dtype=torch.int64, device=dev)
        mine = torch.stack([work.sum() if n else zero, zero + n, keys[0] if n else zero - 1])
        allm = [torch.zeros_like(mine) for _ in range(size)]
        self._allgather(allm, mine)
        allm = torch.stack(allm).cpu()  # one host read: (work, n, first key) per rank
        wt = allm[:, 0].tolist()
        firsts = allm[:, 2].tolist()
        total = sum(wt)
        base = sum(wt[: self.comm.rank])
        cand = torch.full((size - 1,), -1, dtype=torch.int64, device=dev)
        if n:
            # all splitter targets at once: zone k starts after the first body whose
            # global prefix reaches k/size of the total
            prefix = (torch.cumsum(work, 0) + base) * size
            targets = torch.arange(1, size, device=dev, dtype=torch.int64) * total
            js = torch.searchsorted(prefix, targets, side="left")
            nxt = next((firsts[q] for q in range(self.comm.rank + 1, size) if firsts[q] >= 0), None)
            after = torch.cat([keys[1:], torch.tensor([nxt if nxt is not None else (1 << 62)], device=dev)])
            # the straddling body is here iff it is this rank's body j and the prefix
            # before this rank's first body is still short of the target
            here = (js < n) & ((js > 0) | (base * size < targets))
            cand = torch.where(here, after[js.clamp(max=n - 1)], cand)
        self.comm.allreduce_max_(cand)
        # monotone (zones may be empty when work is concentrated)
        self.splitters = torch.cummax(cand, 0).values

    def _t(self, label: str) -> None:
        """BH_DIST_TRACE: synchronise and charge the wall time since the last
        mark to ``label`` (diagnostics only; off by default)."""
        if self.trace is None:
            return
        torch.cuda.synchronize(self.eng.device)
        now = time.perf_counter()
        if self._tlast is not None and label:
            self.trace[label] = self.trace.get(label, 0.0) + (now - self._tlast) * 1e3
        self._tlast = now

    # -- the step --
    def _forces(self, record_work: bool) -> None:
        p, eng, comm = self.p, self.eng, self.comm
        size, rank = comm.size, comm.rank
        L = p.leaf_size
        n, keys, gid = self._route_keys()
        if self.splitters is None:
            self._initial_splitters(keys)
        self._t("route_keys")
        self._migrate(n, keys, gid)
        self._t("migrate")
        n, keys, gid = self._sort()
        self._t("sort2")
        dev = eng.device
        fl = (torch.stack([keys[0], keys[-1]]) if n else
              torch.full((2,), -1, dtype=torch.int64, device=dev))
        allfl = [torch.zeros_like(fl) for _ in range(size)]
        self._allgather(allfl, fl)
        fls = [tuple(r) for r in torch.stack(allfl).cpu().tolist()]  # one host read
        prev = next((fls[q][1] for q in range(rank - 1, -1, -1) if fls[q][0] >= 0), None)
        nxt = next((fls[q][0] for q in range(rank + 1, size) if fls[q][0] >= 0), None)
        self._t("boundary")
        nb = eng.sim_build_local(p.theta, L, prev, nxt) if n else 0
        self._t("build_local")
        br = eng.sim_branch_export(nb)
        recs = eng.sim_walk_records() if n else torch.zeros((0, _REC_INTS), dtype=torch.int32, device=dev)
        bodies = self._export(_lib.BH_SIM_POS, n, (n, 4), torch.float32)
        # branch nodes in body order (a top bucket's bodies must be contiguous)
        perm = torch.argsort(br["lo"]) if nb else torch.zeros(0, dtype=torch.int64, device=dev)
        br = {k: v[perm] for k, v in br.items()}
        br["recs"] = recs[br["rec"].long()] if nb else torch.zeros((0, _REC_INTS), dtype=torch.int32, device=dev)
        # bodies of the bucket-sized branch nodes (a top bucket spans several)
        small = br["count"] <= L
        cnt = br["count"][small].long()
        lo = br["lo"][small].long()
        tot = int(cnt.sum().item()) if cnt.numel() else 0
        start = torch.cumsum(cnt, 0) - cnt
        idx = torch.repeat_interleave(lo - start, cnt) + torch.arange(tot, device=dev)
        self._t("branch_export")
        bb_all = self._allgather_v(bodies[idx])
        br_all = self._allgather_v(_pack_branches(br))  # one row of _BR_INTS per branch node
        self._t("branch_allgather")
        # locally essential trees: what each peer's targets can open.
        # Target region = tight boxes of this rank's bodies per group of branch
        # nodes (a key range is not a box: one box per rank would cover most of
        # the domain and send nearly whole subtrees).
        boxes = self._target_boxes(bodies, br, n, nb)
        self._t("let_boxes")
        allbox = [torch.zeros_like(boxes) for _ in range(size)]
        self._allgather(allbox, boxes)
        boxes = torch.stack(allbox).contiguous() if size > 1 else boxes.view(1, -1, 6)
        self._t("let_box_allgather")
        rc, bc = eng.sim_let(boxes, rank) if n else ([0] * size, [0] * size)
        self._t("let_mark")
        send_rec = torch.empty((sum(rc), _REC_INTS), dtype=torch.int32, device=dev)
        send_bod = torch.empty((sum(bc), 4), dtype=torch.float32, device=dev)
        mcounts = [0 if (q == rank or not n) else nb for q in range(size)]
        send_map = torch.empty((sum(mcounts), 2), dtype=torch.int32, device=dev)
        ro = bo = mo = 0
        for q in range(size):
            if mcounts[q] == 0 and rc[q] == 0:
                continue
            bmap = torch.empty((nb, 2), dtype=torch.int32, device=dev)
            eng.sim_let_pack(q, send_rec[ro:], send_bod[bo:], bmap)
            send_map[mo:mo + nb] = bmap[perm]
            ro, bo, mo = ro + rc[q], bo + bc[q], mo + nb
        self._pack_done = None
        if isinstance(comm, TorchComm) and torch.cuda.is_available():
            self._pack_done = torch.cuda.Event()  # the LET exchange waits for this, not for pass A
            self._pack_done.record()
        self._t("let_pack")
        nbb = sum(b.shape[0] for b in bb_all)
        acc = torch.zeros((n, 4), dtype=torch.float32, device=dev)
        work = torch.zeros(n, dtype=torch.int32, device=dev)
        items = [(send_rec, rc), (send_bod, bc), (send_map, mcounts)]
        gA = torch.cat([bodies] + list(bb_all))
        treeA, deferred = (self._assemble(br_all, recs, n, nbb, defer=True) if (self.overlap and size > 1)
                           else (None, None))
        if treeA is not None and n:
            # pass A walks the local part while the LETs travel
            nwarp = (n + 63) // 64
            # each warp defers at most one entry per remote branch it opens (cfg3 at
            # 8 ranks: ~30 per warp); 16 B per entry
            cap = nwarp * min(len(deferred), 64) + 1024
            dbuf = torch.empty((cap, 4), dtype=torch.int32, device=dev)
            dcnt = torch.zeros(1, dtype=torch.int32, device=dev)
            eng.walk_records_defer(treeA, gA, bodies, p.eps, L, acc, work, dbuf, dcnt)
            self._t("walk_local")
            (let_rec, rcnt), (let_bod, bcnt), (let_map, mcnt) = self._exchange_async(items)
            self._t("let_exchange")
            letoff = np.cumsum([0] + list(rcnt))[:-1] + treeA.shape[0]
            lbodoff = np.cumsum([0] + list(bcnt))[:-1] + n + nbb
            self.tree = torch.cat([treeA] + self._let_parts(let_rec, rcnt, letoff, lbodoff)).contiguous()
            gbodies = torch.cat([gA, let_bod])
            maps_h, off = let_map.cpu().numpy(), 0
            maps = {}
            for q in range(size):
                maps[q] = maps_h[off:off + mcnt[q]]
                off += mcnt[q]
            fcnc = np.zeros((treeA.shape[0], 2), dtype=np.int32)
            for row, q, k, nch in deferred:
                fc = int(maps[q][k, 0])
                if fc >= 0:
                    fcnc[row] = (fc + letoff[q], nch)
            k = int(dcnt.item())
            self.let_stats = dict(records=int(let_rec.shape[0]), bodies=int(let_bod.shape[0]),
                                  sent_records=sum(rc), sent_bodies=sum(bc), own_records=int(recs.shape[0]),
                                  deferred=k, overlap=k <= cap)
            if k <= cap:
                eng.walk_records_resume(self.tree, gbodies, bodies, p.eps, L, acc, work, dbuf[:k],
                                        torch.as_tensor(fcnc, device=dev))
            else:  # deferral list overflowed: the one-pass walk over the full tree
                self.tree = self._assemble(br_all, recs, n, nbb, let_rec, rcnt, bcnt, let_map, mcnt)
                eng.walk_records(self.tree, gbodies, bodies, p.eps, L, acc, work)
        else:
            (let_rec, rcnt), (let_bod, bcnt), (let_map, mcnt) = self._alltoall_many(items)
            self._t("let_exchange")
            self.tree = self._assemble(br_all, recs, n, nbb, let_rec, rcnt, bcnt, let_map, mcnt)
            self.let_stats = dict(records=int(let_rec.shape[0]), bodies=int(let_bod.shape[0]),
                                  sent_records=sum(rc), sent_bodies=sum(bc), own_records=int(recs.shape[0]),
                                  deferred=0, overlap=False)
            self._t("assemble")
            gbodies = torch.cat([gA, let_bod])
            if n:
                eng.walk_records(self.tree, gbodies, bodies, p.eps, L, acc, work)
        if n:
            eng.sim_import(_lib.BH_SIM_ACC, 0, n, acc)
            if record_work:
                eng.sim_import(_lib.BH_SIM_WORK, 0, n, work)
                eng.sim_scatter_work()
        self._t("walk")
        self._keys, self._n, self._nb = keys, n, nb
        # the last step's walk inputs (replayed by tools/dist_emulate.py)
        self.last = dict(bodies=gbodies, targets=bodies, boxes=boxes, bounds=(prev, nxt))

    LET_BOXES = 64  # target boxes per rank (groups of consecutive branch nodes)

    def _target_boxes(self, bodies, br, n, nb):
        """[1 + LET_BOXES, 6] float64 (min xyz, max xyz): the union box, then the
        boxes of groups of consecutive branch nodes; unused boxes are empty
        (min > max)."""
        K = self.LET_BOXES
        dev = bodies.device
        box = torch.empty((K + 1, 6), dtype=torch.float64, device=dev)
        box[:, :3] = float("inf")
        box[:, 3:] = -float("inf")
        if n == 0 or nb == 0:
            return box
        # branch nodes are in body order and partition the bodies: group g = a
        # run of consecutive branch nodes = a contiguous range of bodies
        gid = (torch.arange(nb, device=dev) * K) // nb
        first = torch.searchsorted(gid, torch.arange(K + 1, device=dev))
        lo = torch.cat([br["lo"].long(), torch.tensor([n], dtype=torch.int64, device=dev)])
        start = lo[first].contiguous()  # first == nb -> n (empty group)
        self.eng.sim_target_boxes(start, box)
        box[:, :3] -= self.let_pad
        box[:, 3:] += self.let_pad
        return box

    def _assemble(self, br_all, recs, n, nbb, let_rec=None, rcnt=None, bcnt=None, let_map=None, mcnt=None,
                  defer=False):
        """This rank's walk tree = [top region | own records | LET from each peer];
        its body list = [own bodies | bucket-sized branch bodies | LET bodies].

        The top region holds the top cells (proper ancestors of the branch
        nodes, recombined exactly in fp64) in breadth-first order with
        contiguous children, and copies of the branch-node records: own ones
        point into the own records, remote ones into that peer's LET (or are
        closed when no target here can open them); bucket-sized top cells
        (count <= L) are buckets over the branch bodies, as in one tree."""
        p = self.p
        dev = self.eng.device
        size, me = self.comm.size, self.comm.rank
        L = p.leaf_size
        nW = recs.shape[0]
        host = torch.cat(br_all).cpu().numpy() if br_all else np.zeros((0, _BR_INTS), np.int32)
        host = np.ascontiguousarray(host, dtype=np.int32)
        nrows = host.shape[0]
        row_rank = np.repeat(np.arange(size, dtype=np.int64), [b.shape[0] for b in br_all]) if br_all else \
            np.zeros(0, np.int64)
        row_k = np.concatenate([np.arange(b.shape[0]) for b in br_all]) if br_all else np.zeros(0, np.int64)
        # the top of the global tree, laid out breadth first (bh_top_tree, host C++:
        # exact fp64 recombination of the branch nodes, hashed.py:719-786)
        cap = 22 * max(nrows, 1) + 64
        region = np.zeros((cap, _REC_INTS), dtype=np.int32)
        kind = np.zeros(cap, dtype=np.int32)
        row_of = np.full(cap, -1, dtype=np.int32)
        bb = np.zeros(max(nrows, 1), dtype=np.int64)
        L_ = _lib.lib()
        ntop = int(L_.bh_top_tree(host.ctypes.data_as(ctypes.c_void_p), nrows, n, L, float(self.R), float(p.theta),
                                  region.ctypes.data_as(ctypes.c_void_p), kind.ctypes.data_as(ctypes.c_void_p),
                                  row_of.ctypes.data_as(ctypes.c_void_p), bb.ctypes.data_as(ctypes.c_void_p), cap))
        if ntop < 0:
            raise RuntimeError("top-tree assembly: region capacity exceeded")
        region, kind, row_of = region[:ntop], kind[:ntop], row_of[:ntop]
        # branch-node entries: redirect each subtree / bucket to where it lives
        e = np.nonzero(kind == 2)[0]
        rows = row_of[e].astype(np.int64)
        q = row_rank[rows]
        k = row_k[rows]
        cnt = host[rows, 3:5].copy().view(np.int64).ravel() if len(rows) else np.zeros(0, np.int64)
        rec = region[e]
        internal = rec[:, 14] > 0
        own = q == me
        deferred = []
        m = own & internal  # own subtree: first child in the own records, bodies at 0
        rec[m, 12] += ntop
        if not defer:
            letoff = np.cumsum([0] + list(rcnt))[:-1] + ntop + nW
            lbodoff = np.cumsum([0] + list(bcnt))[:-1] + n + nbb
            mbase = np.cumsum([0] + list(mcnt))[:-1]
            let_map_h = let_map.cpu().numpy() if let_map.numel() else np.zeros((0, 2), np.int32)
        m = (~own) & internal
        if defer:  # subtree in flight: pass A defers it (f4)
            idx = np.nonzero(m)[0]
            deferred = list(zip(e[idx].tolist(), q[idx].tolist(), k[idx].tolist(), rec[idx, 14].tolist()))
            rec[idx, 12] = -1
            rec[idx, 14] = 0
            rec[idx, 15] |= _DEFER_BIT
        elif m.any():
            idx = np.nonzero(m)[0]
            fc = let_map_h[mbase[q[idx]] + k[idx], 0]
            rec[idx, 12] = np.where(fc >= 0, fc + letoff[q[idx]], -1)
            rec[idx, 14] = np.where(fc >= 0, rec[idx, 14], 0)  # no target here opens it
        # remote leaves / buckets (own ones keep their own body index)
        small = (~own) & (~internal) & (cnt <= L)
        rec[small, 12] = bb[rows[small]]
        dup = (~own) & (~internal) & (cnt > L)  # a duplicate-key cell resolved over the owner's bodies
        if dup.any():
            if defer:
                return None, None  # resolved over LET bodies: no overlap this step
            idx = np.nonzero(dup)[0]
            fb = let_map_h[mbase[q[idx]] + k[idx], 1]
            rec[idx, 12] = np.where(fb >= 0, fb + lbodoff[q[idx]], -1)
        region[e] = rec
        parts = [torch.as_tensor(region.reshape(-1, _REC_INTS), device=dev)]
        x = recs.clone()
        x[:, 12] = torch.where(x[:, 14] > 0, x[:, 12] + ntop, x[:, 12])
        parts.append(x)
        if defer:
            return torch.cat(parts).contiguous(), deferred
        parts += self._let_parts(let_rec, rcnt, letoff, lbodoff)
        return torch.cat(parts).contiguous()

    @staticmethod
    def _let_parts(let_rec, rcnt, letoff, lbodoff) -> list:
        """The received LETs with child links and bucket body ranges moved to
        their place in the assembled tree / body list."""
        parts = []
        o = 0
        for q, c in enumerate(rcnt):
            if c == 0:
                continue
            y = let_rec[o:o + c].clone()
            o += c
            internal = y[:, 14] > 0
            withbod = (~internal) & (y[:, 13] > 1) & (y[:, 12] >= 0)
            y[:, 12] = torch.where(internal, y[:, 12] + int(letoff[q]),
                                   torch.where(withbod, y[:, 12] + int(lbodoff[q]), y[:, 12]))
            parts.append(y)
        return parts

    def upload(self, pos, vel, acc, work, gid) -> None:
        """Replace this rank's state (e.g. from host buffers); ownership is
        restored by the next step's migration."""
        self.eng.sim_load_state(pos, vel, acc, work)
        self.gid_load = gid.to(self.eng.device, torch.int64)

    def bootstrap(self) -> None:
        """simulation.py:487: forces for the first kick (work not recorded)."""
        self._bounds(self._maxabs0)
        self._forces(record_work=False)
        # the first decomposition balances on counts (simulation.py:482)
        self._next_splitters(self._n, self._keys,
                             torch.ones(self._n, dtype=torch.int64, device=self.eng.device))

    def step(self, steps: int = 1) -> None:
        for _ in range(steps):
            self._t("")
            self.eng.sim_begin_step(self.p.dt)
            self._bounds()
            self._t("kick_drift_bounds")
            self._forces(record_work=True)
            self.eng.sim_end_step(self.p.dt)
            self._t("kick")
            self._next_splitters(self._n, self._keys)
            self._t("splitters")
            if hasattr(self.eng, "check"):
                self.eng.check()

    def store(self):
        """(pos (n,4), vel (n,4), acc (n,4), work (n,), gid (n,)) of this rank."""
        n = self.eng.sim_n
        pos = torch.empty((n, 4), dtype=torch.float32, device=self.eng.device)
        vel = torch.empty_like(pos)
        acc = torch.empty_like(pos)
        work = torch.empty(n, dtype=torch.int64, device=self.eng.device)
        self.eng.sim_store(pos, vel, acc, work)
        return pos, vel, acc, work, self.gid_load

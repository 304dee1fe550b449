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

import threading
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


def costzones_device(works: torch.Tensor, zones: int) -> list[int]:
    """``costzones`` on a device work array (same rule, integer-exact: the
    zone targets k*total/zones are compared as prefix*zones >= k*total)."""
    n = works.shape[0]
    if zones > n:
        raise ValueError(f"cannot cut {n} bodies into {zones} zones")
    prefix = torch.cumsum(works.to(torch.int64), 0)
    total = int(prefix[-1].item()) if n else 0
    scaled = prefix * zones
    t = torch.arange(1, zones, device=works.device, dtype=torch.int64) * total
    cuts = torch.searchsorted(scaled, t, side="left") + 1
    return [0] + [int(c) for c in cuts.tolist()] + [n]


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


class TorchComm(Comm):
    """torch.distributed collectives (NCCL for CUDA tensors, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def allreduce_sum_(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)

    def allreduce_max_(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)

    def barrier(self):
        self.dist.barrier(group=self.group)


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

    def _zone(self) -> tuple[int, int]:
        _, _, prev = self._bufs()
        self.eng.sim_export(_lib.BH_SIM_PREV_WORK, 0, self.n, prev)
        self.zones = costzones_device(prev, self.comm.size)
        r = self.comm.rank
        return self.zones[r], self.zones[r + 1]

    def _forces(self, record_work: bool, bounds_ready: bool) -> None:
        p = self.p
        self.eng.sim_prepare(p.theta, p.eps, p.leaf_size, bounds_ready)
        b, e = self._zone()
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

    def step(self, steps: int = 1) -> None:
        for _ in range(steps):
            self.eng.sim_begin_step(self.p.dt)
            self._forces(record_work=True, bounds_ready=True)
            self.eng.sim_end_step(self.p.dt)
            if hasattr(self.eng, "check"):
                self.eng.check()  # latched device errors (incl. tree-capacity overflow)

    def store(self, pos=None, vel=None, acc=None, work=None) -> None:
        self.eng.sim_store(pos, vel, acc, work)

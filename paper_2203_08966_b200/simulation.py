"""Time-stepping driver -- drop-in for ``nbsim.simulation``
(/root/reference/pkg/src/nbsim/simulation.py).

``simulate(cfg)`` keeps the reference's signature and result type and runs the
reference's ``_drive`` loop (simulation.py:478-504) on the GPU with the bodies
resident in HBM: bootstrap forces (work not recorded), then per step
kick(dt/2) + drift(dt) + bounds (one fused kernel), keys, radix sort, body
permutation, tree build, traversal, kick(dt/2).  Stages 1-6 of the reference
produce bit-identical trajectories at any rank count (simulation.py:24-27), so
every tree algorithm maps to this one GPU walk; in ``precision="fp64"`` it
reproduces the reference's algorithm-1 trajectory bit for bit.

``TreeForces`` is the plugin seam: it is both an ``AccelProvider``
(integrator.py:16) and a force strategy ``forces(local, record_work)``
(simulation.py:338, 370).
"""

from __future__ import annotations

import ctypes

import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _lib
from .engine import Engine
from .initcond import two_clusters
from .physics import Bodies

PHASES = ("decompose", "build", "share", "force", "integrate", "other")  # simulation.py:62

ALGORITHM_NAMES = {  # simulation.py:64-73
    0: "ring direct sum",
    1: "central tree",
    2: "merged tree",
    3: "sorted bodies",
    4: "cost balance",
    5: "in-place decomposition",
    6: "hashed tree",
    7: "asynchronous walk",
}

LEAF_MODES = ("reference", "bucket")
DECOMPOSITIONS = ("auto", "replicated", "distributed")
AUTO_DISTRIBUTED_N = 30_000_000  # replicated below ("Which scheme runs")


@dataclass(frozen=True)
class SimConfig:
    """simulation.py:82-113 plus the GPU fields."""

    n: int
    algorithm: int = 7
    ranks: int = 1
    theta: float = 0.5
    dt: float = 0.01
    steps: int = 500
    eps: float = 0.05
    seed: int = 1
    leaf_size: int = 1
    precision: str = "fp64"
    devices: int = 1
    leaf_mode: str = "reference"
    decomposition: str = "auto"  # devices > 1: "replicated" | "distributed" | "auto"

    def __post_init__(self) -> None:
        if self.algorithm not in ALGORITHM_NAMES:
            raise ValueError(f"algorithm must be 0..7, got {self.algorithm}")
        if self.n < 4:
            raise ValueError(f"need at least 4 bodies, got n={self.n}")
        if self.ranks < 1:
            raise ValueError(f"ranks must be positive, got {self.ranks}")
        if self.n < self.ranks:
            raise ValueError(
                f"every rank needs at least one body: n={self.n} < ranks={self.ranks}")
        if not 0.0 <= self.theta:
            raise ValueError(f"theta must be non-negative, got {self.theta}")
        if not self.dt > 0.0:
            raise ValueError(f"dt must be positive, got {self.dt}")
        if self.steps < 0:
            raise ValueError(f"steps must be non-negative, got {self.steps}")
        if self.eps < 0.0:
            raise ValueError(f"eps must be non-negative, got {self.eps}")
        if self.leaf_size < 1:
            raise ValueError(f"leaf_size must be >= 1, got {self.leaf_size}")
        if self.precision not in ("fp32", "fp64"):
            raise ValueError(f"precision must be fp32 or fp64, got {self.precision!r}")
        if self.leaf_mode not in LEAF_MODES:
            raise ValueError(f"leaf_mode must be one of {LEAF_MODES}, got {self.leaf_mode!r}")
        if self.devices < 1:
            raise ValueError(f"devices must be positive, got {self.devices}")
        if self.decomposition not in DECOMPOSITIONS:
            raise ValueError(f"decomposition must be one of {DECOMPOSITIONS}, got {self.decomposition!r}")
        if self.decomposition == "distributed" and self.precision != "fp32":
            raise ValueError("the distributed build runs in fp32 (precision='fp32')")

    @property
    def scheme(self) -> str:
        """Multi-GPU scheme for devices > 1 (decomposition.py): the key-range
        decomposition with a distributed build from AUTO_DISTRIBUTED_N bodies in
        fp32, else the replicated tree with a partitioned walk."""
        if self.decomposition != "auto":
            return self.decomposition
        return "distributed" if (self.precision == "fp32" and self.n >= AUTO_DISTRIBUTED_N) else "replicated"

    @property
    def walk_leaf_size(self) -> int:
        """Leaf size the walk uses: 1 in reference mode."""
        return 1 if self.leaf_mode == "reference" else self.leaf_size


@dataclass
class SimResult:
    """simulation.py:116-142."""

    config: SimConfig
    bodies: Bodies
    phase_seconds: list
    message_stats: dict
    requests: int
    snapshots: list
    trace_lines: Optional[list]
    wall_seconds: float
    interactions: int = 0

    @property
    def work_total(self) -> int:
        return int(self.bodies.work.sum())

    def phase_totals(self) -> dict:
        """simulation.py:134-142: messages and bytes sent per phase.  The GPU
        path has no message transport (one device: nothing is sent; several:
        NCCL collectives and peer stores, not counted as messages), so every
        phase reports (0, 0); the time per phase is in ``phase_seconds``."""
        return {phase: (0, 0) for phase in PHASES}


class TreeForces:
    """GPU force provider over host ``Bodies``.

    ``provider(bodies)`` fills ``bodies.acceleration`` in place (an
    ``AccelProvider``); ``provider.forces(local, record_work)`` is the
    reference's force-strategy protocol and returns 0 remote requests.
    Each call uploads the bodies, builds the tree and walks it on the GPU, and
    copies accelerations (and work) back.
    """

    def __init__(self, theta: float, eps: float, leaf_size: int = 1, precision: str = "fp64",
                 engine: Engine | None = None):
        self.theta = float(theta)
        self.eps = float(eps)
        self.leaf_size = int(leaf_size)
        self.engine = engine if engine is not None else Engine(precision)

    _PIN_MIN = 1 << 20  # page-lock caller arrays of at least this many bytes
    _PIN_MAX = 8  # registrations kept (least recently used dropped first)

    def _pin(self, *arrays) -> None:
        """Page-lock the caller's numpy arrays in place (once per buffer) so the
        uploads and read-backs below run at full PCIe rate instead of through
        the driver's pageable staging.  A buffer stays registered while this
        provider holds it (a reference keeps it alive); failures fall back to
        pageable copies."""
        pins = self.__dict__.setdefault("_pins", {})
        L = _lib.lib()
        for a in arrays:
            if not isinstance(a, np.ndarray) or a.nbytes < self._PIN_MIN or not a.flags.c_contiguous:
                continue
            key = (a.__array_interface__["data"][0], a.nbytes)
            if key in pins:
                pins[key] = pins.pop(key)  # most recently used last
                continue
            while len(pins) >= self._PIN_MAX:
                old_key = next(iter(pins))
                L.bh_host_unregister(ctypes.c_void_p(old_key[0]))
                pins.pop(old_key)
            if L.bh_host_register(ctypes.c_void_p(key[0]), key[1]) == _lib.BH_OK:
                pins[key] = a

    def close(self) -> None:
        """Release the page-locked registrations (also done when collected)."""
        pins = self.__dict__.get("_pins") or {}
        if pins:
            L = _lib.lib()
            for key in list(pins):
                L.bh_host_unregister(ctypes.c_void_p(key[0]))
            pins.clear()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def forces(self, local: Bodies, record_work: bool) -> int:
        eng = self.engine
        n = len(local)
        self._pin(local.position, local.mass, local.acceleration, local.work if record_work else None)
        pos = eng.bodies_tensor(local.position, local.mass)
        # the force pass reads positions and masses only: the velocity slot gets a
        # zero buffer kept across calls instead of an upload of local.velocity
        if getattr(self, "_vel", None) is None or self._vel.shape[0] != n or self._vel.dtype != eng.dtype:
            self._vel = torch.zeros((n, 4 if eng.fp32 else 3), dtype=eng.dtype, device=eng.device)
        m = None if eng.fp32 else torch.as_tensor(local.mass).to(eng.device)
        eng.sim_load(pos, self._vel, m)
        eng.sim_forces(self.theta, self.eps, self.leaf_size, record_work)
        acc = torch.empty((n, 4 if eng.fp32 else 3), dtype=eng.dtype, device=eng.device)
        work = torch.empty(n, dtype=torch.int64, device=eng.device) if record_work else None
        eng.sim_store(acc=acc, work=work)
        eng.check()
        # straight into the caller's arrays (no intermediate host copies)
        torch.from_numpy(local.acceleration).copy_(acc[:, :3].to(torch.float64))
        if record_work:
            torch.from_numpy(local.work).copy_(work)
        return 0

    def __call__(self, bodies: Bodies) -> None:
        self.forces(bodies, record_work=True)


def _direct_run(cfg: SimConfig, bodies: Bodies, snapshot_every) -> tuple[Bodies, list]:
    """Algorithm 0 (simulation.py:330-350) on one device: fp64 direct sum."""
    from .integrator import drift, kick
    from .physics import direct_accelerations

    snaps = []
    bodies.acceleration[:] = direct_accelerations(bodies.mass, bodies.position, cfg.eps)
    if snapshot_every:
        snaps.append((0.0, bodies.copy()))
    for step in range(1, cfg.steps + 1):
        kick(bodies, 0.5 * cfg.dt)
        drift(bodies, cfg.dt)
        bodies.acceleration[:] = direct_accelerations(bodies.mass, bodies.position, cfg.eps)
        bodies.work[:] = cfg.n - 1
        kick(bodies, 0.5 * cfg.dt)
        if snapshot_every and step % snapshot_every == 0:
            snaps.append((step * cfg.dt, bodies.copy()))
    return bodies, snaps


def simulate(cfg: SimConfig, *, transport: str = "inproc", record_trace: bool = False,
             snapshot_every: Optional[int] = None, timeout: float = 120.0,
             initial: Bodies | None = None, engine: Engine | None = None) -> SimResult:
    """simulation.py:507-551.  ``transport``/``record_trace``/``timeout`` are
    accepted for API compatibility (the GPU path has no message transport);
    ``initial`` overrides the two-cluster initial condition."""
    if transport not in ("inproc", "socket"):
        raise ValueError(f"unknown transport {transport!r} (expected inproc or socket)")
    if snapshot_every is not None and snapshot_every < 1:
        raise ValueError(f"snapshot interval must be positive, got {snapshot_every}")
    started = time.monotonic()
    bodies = initial.copy() if initial is not None else two_clusters(cfg.n, cfg.seed)
    bodies.work[:] = 1  # simulation.py:482
    if cfg.algorithm == 0:
        bodies, snaps = _direct_run(cfg, bodies, snapshot_every)
        return SimResult(cfg, bodies, [{p: 0.0 for p in PHASES}], {}, 0, snaps,
                         [] if record_trace else None, time.monotonic() - started)

    eng = engine if engine is not None else Engine(cfg.precision)
    eng.timing(True)  # per-phase device time (CUDA events on the stream) for phase_seconds
    eng.timing_reset()
    n = len(bodies)
    pos = eng.bodies_tensor(bodies.position, bodies.mass)
    vel = eng.vec_tensor(bodies.velocity)
    m = None if eng.fp32 else torch.as_tensor(bodies.mass).to(eng.device)
    leaf = cfg.walk_leaf_size
    dsim = bsim = None
    if cfg.devices > 1:  # one process per GPU (torchrun); decomposition.py
        import torch.distributed as dist

        from .decomposition import DistributedBuildSim, DistributedSim, StepParams, TorchComm

        if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() != cfg.devices:
            raise ValueError(
                f"devices={cfg.devices} needs torch.distributed initialised with that world size "
                "(one process per GPU, e.g. torchrun --nproc-per-node)")
        params = StepParams(cfg.theta, cfg.eps, leaf, cfg.dt)
        if cfg.scheme == "distributed":  # each rank starts from a contiguous chunk
            bsim = DistributedBuildSim(eng, TorchComm(), params)
            r, R = dist.get_rank(), dist.get_world_size()
            lo, hi = n * r // R, n * (r + 1) // R
            bsim.load(pos[lo:hi].contiguous(), vel[lo:hi].contiguous(),
                      gid=torch.arange(lo, hi, device=eng.device))
            bsim.bootstrap()
        else:
            dsim = DistributedSim(eng, TorchComm(), params)
            dsim.load(pos, vel, m)
            dsim.bootstrap()
    else:
        eng.sim_load(pos, vel, m)
        eng.sim_forces(cfg.theta, cfg.eps, leaf, record_work=False)  # simulation.py:487

    def advance(k: int) -> None:
        if dsim is not None:
            dsim.step(k)
        elif bsim is not None:
            bsim.step(k)
        else:
            eng.sim_step(cfg.dt, cfg.theta, cfg.eps, leaf, k)

    def snapshot() -> Bodies:
        if bsim is not None:  # gather every rank's bodies back into the caller's order
            p_, v_, a_, w_, g_ = bsim.store()
            rows = torch.cat([p_.view(torch.int32), v_.view(torch.int32), a_.view(torch.int32),
                              w_.view(torch.int32).view(-1, 2), g_.view(torch.int32).view(-1, 2)], dim=1)
            allr = torch.cat(bsim._allgather_v(rows))
            gid = allr[:, 14:16].contiguous().view(torch.int64).view(-1)
            order = torch.argsort(gid)
            allr = allr[order]
            f = allr[:, 0:12].contiguous().view(torch.float32).view(-1, 3, 4)
            return Bodies(bodies.mass.copy(), f[:, 0, :3].double().cpu().numpy(),
                          f[:, 1, :3].double().cpu().numpy(), f[:, 2, :3].double().cpu().numpy(),
                          allr[:, 12:14].contiguous().view(torch.int64).view(-1).cpu().numpy())
        p = torch.empty_like(vel)
        v = torch.empty_like(vel)
        a = torch.empty_like(vel)
        w = torch.empty(n, dtype=torch.int64, device=eng.device)
        eng.sim_store(p, v, a, w)
        eng.check()
        out = Bodies(bodies.mass.copy(), p[:, :3].double().cpu().numpy(),
                     v[:, :3].double().cpu().numpy(), a[:, :3].double().cpu().numpy(),
                     w.cpu().numpy())
        return out

    snaps = []
    if snapshot_every:
        snaps.append((0.0, snapshot()))
    interactions = 0
    if snapshot_every:
        step = 0
        while step < cfg.steps:
            k = min(snapshot_every, cfg.steps - step)
            advance(k)
            step += k
            if step % snapshot_every == 0:
                snaps.append((step * cfg.dt, snapshot()))
    elif cfg.steps:
        advance(cfg.steps)
    st = eng.stats()
    interactions = st.interactions
    final = snapshot()
    wall = time.monotonic() - started
    return SimResult(cfg, final, [phase_seconds(eng.timing_get(), wall)], {}, 0, snaps,
                     [] if record_trace else None, wall, interactions)


def phase_seconds(device_ms: dict, wall: float) -> dict:
    """The reference's phase clock (simulation.py:145-169) from the library's
    per-phase device times: keys + sort + permutation = "decompose", tree build
    = "build", locally-essential-tree exchange = "share", walk = "force",
    kicks and drift = "integrate"; the rest of the wall time (host, transfers,
    initial conditions) = "other"."""
    sec = {p: 0.0 for p in PHASES}
    sec["decompose"] = (device_ms.get("keys", 0.0) + device_ms.get("sort", 0.0) + device_ms.get("permute", 0.0)) / 1e3
    sec["build"] = device_ms.get("build", 0.0) / 1e3
    sec["share"] = device_ms.get("let", 0.0) / 1e3
    sec["force"] = device_ms.get("walk", 0.0) / 1e3
    sec["integrate"] = device_ms.get("integrate", 0.0) / 1e3
    sec["other"] = max(0.0, wall - sum(sec.values()))
    return sec

"""Bodies container and validation kernels -- drop-in for ``nbsim.physics``
(/root/reference/pkg/src/nbsim/physics.py).

``Bodies`` keeps the reference's structure-of-arrays numpy layout (fp64
mass/position/velocity/acceleration, int64 work).  The O(n^2) oracles used for
validation and the energy audit (``direct_accelerations``,
``potential_energy``) run as fp64 CUDA kernels (bh_direct_f64,
bh_potential_f64).  ``direct_accelerations`` keeps the reference's per-target
summation order, so it is bit-identical to ``_accel_all_pairs``.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np


@dataclass
class Bodies:
    """physics.py:18-120 (same fields, validation and wire format)."""

    mass: np.ndarray
    position: np.ndarray
    velocity: np.ndarray
    acceleration: np.ndarray = field(default=None)  # type: ignore[assignment]
    work: np.ndarray = field(default=None)  # type: ignore[assignment]

    def __post_init__(self) -> None:
        n = len(self.mass)
        self.mass = np.ascontiguousarray(self.mass, dtype=np.float64)
        self.position = np.ascontiguousarray(self.position, dtype=np.float64)
        self.velocity = np.ascontiguousarray(self.velocity, dtype=np.float64)
        if self.acceleration is None:
            self.acceleration = np.zeros((n, 3))
        if self.work is None:
            self.work = np.zeros(n, dtype=np.int64)
        self.acceleration = np.ascontiguousarray(self.acceleration, dtype=np.float64)
        self.work = np.ascontiguousarray(self.work, dtype=np.int64)
        if self.position.shape != (n, 3) or self.velocity.shape != (n, 3):
            raise ValueError("position/velocity must have shape (n, 3)")
        if self.acceleration.shape != (n, 3) or self.work.shape != (n,):
            raise ValueError("acceleration/work shapes inconsistent with mass")
        if np.any(self.work < 0):
            raise ValueError("work counts must be non-negative")

    def __len__(self) -> int:
        return len(self.mass)

    @classmethod
    def zeros(cls, n: int) -> "Bodies":
        return cls(np.zeros(n), np.zeros((n, 3)), np.zeros((n, 3)))

    def copy(self) -> "Bodies":
        return Bodies(self.mass.copy(), self.position.copy(), self.velocity.copy(),
                      self.acceleration.copy(), self.work.copy())

    def take(self, indices) -> "Bodies":
        return Bodies(self.mass[indices].copy(), self.position[indices].copy(),
                      self.velocity[indices].copy(), self.acceleration[indices].copy(),
                      self.work[indices].copy())

    @staticmethod
    def concat(parts: list["Bodies"]) -> "Bodies":
        if not parts:
            return Bodies.zeros(0)
        return Bodies(
            np.concatenate([p.mass for p in parts]),
            np.concatenate([p.position for p in parts]),
            np.concatenate([p.velocity for p in parts]),
            np.concatenate([p.acceleration for p in parts]),
            np.concatenate([p.work for p in parts]),
        )

    def pack(self) -> bytes:
        """physics.py:88-104: columnar little-endian (mass, position, velocity, work)."""
        n = len(self)
        return b"".join((
            struct.pack("<q", n),
            self.mass.astype("<f8").tobytes(),
            self.position.astype("<f8").tobytes(),
            self.velocity.astype("<f8").tobytes(),
            self.work.astype("<i8").tobytes(),
        ))

    @classmethod
    def unpack(cls, blob: bytes) -> "Bodies":
        (n,) = struct.unpack_from("<q", blob, 0)
        off = 8

        def column(count, dtype):
            nonlocal off
            arr = np.frombuffer(blob, dtype=dtype, count=count, offset=off).copy()
            off += arr.nbytes
            return arr

        mass = column(n, "<f8")
        pos = column(3 * n, "<f8").reshape(n, 3)
        vel = column(3 * n, "<f8").reshape(n, 3)
        work = column(n, "<i8")
        return cls(mass, pos, vel, np.zeros((n, 3)), work)


def pairwise_accel(pos_i, pos_j, m_j: float, eps: float) -> np.ndarray:
    """physics.py:141-153 (host scalar helper)."""
    d = np.asarray(pos_i, dtype=np.float64) - np.asarray(pos_j, dtype=np.float64)
    r2 = float(d[0] * d[0] + d[1] * d[1] + d[2] * d[2])
    if r2 == 0.0:
        return np.zeros(3)
    return -m_j * d / (r2 + eps * eps) ** 1.5


def _engine():
    from .engine import default_engine

    return default_engine("fp64")


def direct_accelerations(masses, positions, eps: float) -> np.ndarray:
    """physics.py:288-295: all-pairs softened accelerations on the GPU (fp64)."""
    import torch

    eng = _engine()
    pos = eng.bodies_tensor(positions)
    m = torch.as_tensor(np.ascontiguousarray(masses, dtype=np.float64)).to(eng.device)
    if pos.shape[0] == 0:
        return np.zeros((0, 3))
    return eng.direct(pos, m, eps).cpu().numpy()


def kinetic_energy(bodies: Bodies) -> float:
    """physics.py:316-319 (host, same numpy expression)."""
    v2 = np.einsum("ij,ij->i", bodies.velocity, bodies.velocity)
    return 0.5 * float(bodies.mass @ v2)


def potential_energy(bodies: Bodies, eps: float = 0.0) -> float:
    """physics.py:322-324 on the GPU (fp64; pair sums ordered per body)."""
    import torch

    eng = _engine()
    if len(bodies) < 2:
        return 0.0
    pos = eng.bodies_tensor(bodies.position)
    m = torch.as_tensor(bodies.mass).to(eng.device)
    return eng.potential(pos, m, eps)


def total_energy(bodies: Bodies, eps: float = 0.0) -> float:
    """physics.py:327-328."""
    return kinetic_energy(bodies) + potential_energy(bodies, eps)

"""Octree build -- drop-in for ``nbsim.hashed.build_hashed``
(/root/reference/pkg/src/nbsim/hashed.py:448-515).

``build_hashed`` builds the reference's tree (one body per leaf, single-child
chains kept, pre-order cells, monopole + quadrupole moments) on the GPU from
Morton-sorted bodies: lcp levels -> cells per body -> exclusive scan ->
parallel cell emission -> level-synchronous bottom-up moments in one
cooperative launch (bh_build_*).  In fp64 mode every cell array is
bit-identical to the reference's (tests/test_gpu_*).

The tree stays on the device inside its own engine handle; ``arrays()``
exports the FlatTree/HashedTree arrays and ``to_serial_bytes()`` the
reference wire format (octree.py:30-34, hashed.py:324-346).
"""

from __future__ import annotations

import struct

import numpy as np
import torch

from .engine import Engine
from .morton import DomainBounds
from .physics import Bodies

ROOT_KEY = 1  # hashed.py:63
_RECORD = struct.Struct("<3d d d 3d 6d q B")  # octree.py:32
_HEADER = struct.Struct("<4s q")  # octree.py:33
_MAGIC = b"OCT1"


class DeviceTree:
    """A built tree resident on one GPU (its own libbh handle)."""

    def __init__(self, engine: Engine, n_bodies: int, n_cells: int, bounds: DomainBounds):
        self.engine = engine
        self.n_bodies = n_bodies
        self.n_cells = n_cells
        self.bounds = bounds
        self._arrays = None

    def __len__(self) -> int:
        return self.n_cells

    def arrays(self) -> dict:
        """key, level, centre, side, mass, com, quad, count, children (numpy)."""
        if self._arrays is None:
            self._arrays = self.engine.export_tree()
        return self._arrays

    def __getattr__(self, name):
        if name in ("key", "level", "centre", "side", "mass", "com", "quad", "count", "children"):
            return self.arrays()[name]
        raise AttributeError(name)

    def flat(self) -> "FlatTree":
        from .flattree import FlatTree

        return FlatTree(self)

    def to_serial_bytes(self) -> bytes:
        """Pre-order wire format identical to the reference's (hashed.py:324-346)."""
        a = self.arrays()
        n = len(a["count"])
        rec = np.empty(n, dtype=np.dtype([
            ("centre", "<f8", 3), ("side", "<f8"), ("mass", "<f8"), ("com", "<f8", 3),
            ("quad", "<f8", 6), ("count", "<i8"), ("mask", "u1")]))
        rec["centre"] = a["centre"]
        rec["side"] = a["side"]
        rec["mass"] = a["mass"]
        rec["com"] = a["com"]
        rec["quad"] = a["quad"]
        rec["count"] = a["count"]
        mask = np.zeros(n, dtype=np.uint8)
        for s in range(8):
            mask |= ((a["children"][:, s] >= 0) << s).astype(np.uint8)
        rec["mask"] = mask
        return _HEADER.pack(_MAGIC, n) + rec.tobytes()


def build_hashed(bodies: Bodies, bounds: DomainBounds, precision: str = "fp64",
                 engine: Engine | None = None, allow_duplicates: bool = False) -> DeviceTree:
    """hashed.py:448: bodies must be Morton-sorted with distinct keys
    (ValueError otherwise, with the reference's message fragments).
    ``allow_duplicates`` is the bucket-mode extension: bodies
    with equal keys share one level-21 cell, resolved body by body."""
    eng = engine if engine is not None else Engine(precision)
    eng.set_allow_duplicates(allow_duplicates)
    pos = eng.bodies_tensor(bodies.position, bodies.mass)
    R = torch.tensor([float(bounds.half_extent)], dtype=torch.float64, device=eng.device)
    if eng.fp32:
        C = eng.build(pos, R)
    else:
        m = torch.as_tensor(bodies.mass).to(eng.device)
        C = eng.build(pos, R, m)
    return DeviceTree(eng, len(bodies), C, bounds)

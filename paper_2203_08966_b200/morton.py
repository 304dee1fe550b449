"""Morton keys over a cubic domain -- drop-in for ``nbsim.morton``
(/root/reference/pkg/src/nbsim/morton.py).

``DomainBounds.from_positions``, ``morton_keys`` and ``sort_order`` run on the
GPU (libbh.so: bh_bounds_*, bh_morton_*, bh_sort) and are bit-exact with the
reference: fp64 floor quantisation of the (upcast) positions, x > y > z bit
interleave, stable ascending argsort.  The scalar helpers (quantize,
interleave, ...) are host-side conveniences with the reference's semantics.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

MORTON_BITS = 21  # morton.py:16
BOUNDS_PAD = 1.001  # morton.py:20


@dataclass(frozen=True)
class DomainBounds:
    """Cubic domain ``[-R, R)`` per axis (morton.py:23-42)."""

    half_extent: float

    def __post_init__(self) -> None:
        if not self.half_extent > 0.0:
            raise ValueError(f"half_extent must be positive, got {self.half_extent}")

    @classmethod
    def from_positions(cls, positions, precision: str = "fp64") -> "DomainBounds":
        """R = 1.001 * max|x| (1.0 for an all-zero cloud), reduced on the GPU."""
        from .engine import default_engine

        eng = default_engine(precision)
        pos = eng.bodies_tensor(positions)
        if pos.shape[0] == 0:
            return cls(1.0)
        R = eng.bounds(pos)
        return cls(float(R.item()))


def quantize(coord: float, bounds: DomainBounds) -> int:
    """morton.py:45-57 (host scalar helper)."""
    r = bounds.half_extent
    if not -r <= coord or not coord < r:
        raise ValueError(f"coordinate {coord} outside domain [-{r}, {r})")
    i = int(np.floor((coord + r) / (2.0 * r) * (1 << MORTON_BITS)))
    return min(max(i, 0), (1 << MORTON_BITS) - 1)


def interleave(ix: int, iy: int, iz: int) -> int:
    """morton.py:71-85: bit 3k+2 = x_k, 3k+1 = y_k, 3k = z_k."""
    for name, v in (("ix", ix), ("iy", iy), ("iz", iz)):
        if not 0 <= v < (1 << MORTON_BITS):
            raise ValueError(f"{name}={v} outside [0, 2^{MORTON_BITS})")
    key = 0
    for k in range(MORTON_BITS):
        key |= ((ix >> k) & 1) << (3 * k + 2)
        key |= ((iy >> k) & 1) << (3 * k + 1)
        key |= ((iz >> k) & 1) << (3 * k)
    return key


def deinterleave(key: int) -> tuple[int, int, int]:
    """morton.py:97-104."""
    ix = iy = iz = 0
    for k in range(MORTON_BITS):
        ix |= ((key >> (3 * k + 2)) & 1) << k
        iy |= ((key >> (3 * k + 1)) & 1) << k
        iz |= ((key >> (3 * k)) & 1) << k
    return ix, iy, iz


def _as_f64(positions):
    from .engine import default_engine

    eng = default_engine("fp64")
    return eng, eng.bodies_tensor(positions)


def morton_keys(positions, bounds: DomainBounds) -> np.ndarray:
    """morton.py:109-125 on the GPU; raises ValueError on out-of-domain bodies."""
    eng, pos = _as_f64(positions)
    n = pos.shape[0]
    if n == 0:
        return np.zeros(0, dtype=np.uint64)
    R = torch.tensor([float(bounds.half_extent)], dtype=torch.float64, device=eng.device)
    keys = eng.morton(pos, R)
    try:
        eng.check()
    except ValueError as e:
        bad = pos.cpu().numpy()
        r = bounds.half_extent
        row = bad[(np.abs(bad) >= r).any(axis=1)]
        raise ValueError(
            f"position {row[0] if len(row) else '?'} outside domain [-{r}, {r})") from e
    return keys.cpu().numpy().view(np.uint64)


def morton_key(position, bounds: DomainBounds) -> int:
    """morton.py:103-106."""
    return int(morton_keys(np.asarray(position, dtype=np.float64).reshape(1, 3), bounds)[0])


def sort_order(keys) -> np.ndarray:
    """morton.py:128-130: stable ascending argsort (GPU radix sort)."""
    from .engine import default_engine

    k = np.ascontiguousarray(keys, dtype=np.uint64)
    if len(k) == 0:
        return np.zeros(0, dtype=np.int64)
    if int(k.max()) >= 1 << 63:
        raise ValueError("keys must fit in 63 bits")
    eng = default_engine("fp64")
    kt = torch.from_numpy(k.view(np.int64)).to(eng.device)
    _, perm = eng.sort(kt)
    return perm.cpu().numpy()

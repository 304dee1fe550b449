"""Batched force traversal -- drop-in for ``nbsim.flattree.FlatTree.traverse``
(/root/reference/pkg/src/nbsim/flattree.py:142-166, kernel 258-317).

The walk runs as a warp-cooperative CUDA kernel (bh_traverse_*), with the
targets Morton-ordered internally:

* fp64 (validation): each warp walks the union of its 32 targets' interaction
  lists in pre-order (stackless, via subtree skip links) and every lane
  evaluates exactly the reference's list in the reference's order, so the
  result is the reference's to <= 1 ulp per pp term;
* fp32: the group-classified walk (k_walk9): 64 targets per warp,
  cells classified 32 at a time against the group's box (certain accept, certain
  open, or per-target MAC), with dense pc / pp drains.  Every target gets exactly
  the reference's interaction set; only the fp32 summation order differs.

``leaf_size > 1`` adds the bucket rule of SURVEY.md §8(c) (cells of <= leaf_size
bodies that fail the MAC are summed body by body).
"""

from __future__ import annotations

import numpy as np
import torch

from .hashed import DeviceTree


class FlatTree:
    """A device-resident tree viewed through the reference's traversal API."""

    def __init__(self, tree: DeviceTree):
        self.tree = tree

    def __len__(self) -> int:
        return len(self.tree)

    @property
    def count(self) -> np.ndarray:
        return self.tree.count

    def traverse(self, positions, theta: float, eps: float, leaf_size: int = 1):
        """Accelerations (n,3) float64 and work counts (n,) int64."""
        eng = self.tree.engine
        tg = eng.vec_tensor(positions)
        n = tg.shape[0]
        if n == 0:
            return np.zeros((0, 3)), np.zeros(0, dtype=np.int64)
        acc, work = eng.traverse(tg, theta, eps, leaf_size)
        eng.check()
        a = acc[:, :3].to(torch.float64).cpu().numpy()
        return np.ascontiguousarray(a), work.cpu().numpy()

    def to_bytes(self) -> bytes:
        return self.tree.to_serial_bytes()

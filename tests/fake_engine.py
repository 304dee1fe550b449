"""Test-only stand-in for Engine's sim_* phase API, computed by the CPU oracle.

Lets tests/test_decomposition.py run the multi-rank protocol of
paper_2203_08966_b200.decomposition over torch.distributed gloo on CPU (no
GPU in the build container).  fp64 arithmetic in the reference's order, so a
multi-rank run must reproduce the single-rank oracle leapfrog bit for bit.
"""

import numpy as np
import torch

from oracle import oracle as orc
from paper_2203_08966_b200 import _lib


class OracleEngine:
    precision = "fp64"
    device = torch.device("cpu")

    def sim_load(self, pos, vel, mass=None):
        p = pos.numpy().astype(np.float64)
        n = len(p)
        self.pos = np.zeros((n, 4)); self.pos[:, :3] = p[:, :3]
        self.pos[:, 3] = mass.numpy() if mass is not None else p[:, 3]
        self.vel = np.zeros((n, 4)); self.vel[:, :3] = vel.numpy()[:, :3]
        self.acc = np.zeros((n, 4))
        self.id = np.arange(n)
        self.work_sorted = np.zeros(n, dtype=np.int32)
        self.work_orig = np.ones(n, dtype=np.int32)

    def sim_begin_step(self, dt):
        self.vel[:, :3] += self.acc[:, :3] * (0.5 * dt)
        self.pos[:, :3] += self.vel[:, :3] * dt

    def sim_prepare(self, theta, eps, leaf, bounds_ready=True):
        R = orc.bounds(self.pos[:, :3])
        order = orc.sort_order(orc.morton_keys(self.pos[:, :3], R))
        self.pos, self.vel, self.id = self.pos[order], self.vel[order], self.id[order]
        self.tree = orc.build_tree(self.pos[:, 3], self.pos[:, :3], R)

    def sim_walk_range(self, theta, eps, leaf, b, e, record_work=True):
        a, w = orc.traverse(self.tree, self.pos[b:e, :3], theta, eps, leaf)
        self.acc[b:e, :3] = a
        if record_work:
            self.work_sorted[b:e] = w

    def sim_scatter_work(self):
        self.work_orig[self.id] = self.work_sorted

    def sim_end_step(self, dt):
        self.vel[:, :3] += self.acc[:, :3] * (0.5 * dt)

    def sim_export(self, what, b, e, dst):
        if what == _lib.BH_SIM_ACC:
            dst.copy_(torch.from_numpy(self.acc[b:e]))
        elif what == _lib.BH_SIM_WORK:
            dst.copy_(torch.from_numpy(self.work_sorted[b:e]))
        elif what == _lib.BH_SIM_PREV_WORK:
            dst.copy_(torch.from_numpy(self.work_orig[self.id[b:e]]))
        else:
            raise ValueError(what)

    def sim_import(self, what, b, e, src):
        if what == _lib.BH_SIM_ACC:
            self.acc[b:e] = src.numpy()
        elif what == _lib.BH_SIM_WORK:
            self.work_sorted[b:e] = src.numpy()
        else:
            raise ValueError(what)

    def sim_store(self, pos=None, vel=None, acc=None, work=None):
        n = len(self.id)
        for dst, src in ((pos, self.pos), (vel, self.vel), (acc, self.acc)):
            if dst is not None:
                out = np.empty_like(src); out[self.id] = src
                dst.copy_(torch.from_numpy(out))
        if work is not None:
            work.copy_(torch.from_numpy(self.work_orig.astype(np.int64)))


class PeerOracleEngine(OracleEngine):
    """OracleEngine whose walk also stores its rows into peer engines' result
    arrays (the CPU stand-in for bh_sim_set_peer_ptrs' NVLink peer stores).
    ``drop`` > 0 loses that many rows per peer store (a broken mapping)."""

    def __init__(self, drop=0):
        self.peers = []
        self.drop = drop

    def sim_result_ptrs(self):
        return self

    def sim_set_peer_ptrs(self, peers):
        self.peers = list(peers)

    def sim_set_peers(self, handles):  # IPC form: not used by in-process ranks
        if handles:
            raise RuntimeError("no IPC in the CPU fake")
        self.peers = []

    def sim_walk_range(self, theta, eps, leaf, b, e, record_work=True):
        super().sim_walk_range(theta, eps, leaf, b, e, record_work)
        for q in self.peers:
            hi = max(b, e - self.drop)
            q.acc[b:hi] = self.acc[b:hi]
            if record_work:
                q.work_sorted[b:hi] = self.work_sorted[b:hi]


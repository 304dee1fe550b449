"""Engine: one libbh handle on one CUDA device, driven with torch tensors.

PyTorch is plumbing here: it owns device memory and the stream; every compute
step is a libbh.so kernel.  Device buffers are passed to the C-ABI as raw
pointers (``tensor.data_ptr()``), the stream as
``torch.cuda.current_stream().cuda_stream``.

Tensor layouts (see include/bh.h):
  fp32 mode  bodies float32 [n, 4] = (x, y, z, m); velocities/accels [n, 4]
  fp64 mode  positions/velocities/accels float64 [n, 3]; masses float64 [n]
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import BH_FP32, BH_FP64, check

PRECISIONS = {"fp32": BH_FP32, "fp64": BH_FP64}


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


@dataclass
class TraversalStats:
    n_bodies: int
    n_cells: int
    pp: int
    pc: int
    n_records: int = 0  # fp32 walk records of the current tree

    @property
    def interactions(self) -> int:
        return self.pp + self.pc

    @property
    def work(self) -> int:
        return self.pp + 2 * self.pc


class Engine:
    """Owns a ``bh_handle``; not thread-safe (one engine per thread/rank)."""

    def __init__(self, precision: str = "fp32", device: int | torch.device | None = None):
        if precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {sorted(PRECISIONS)}, got {precision!r}")
        if not torch.cuda.is_available():
            raise RuntimeError("libbh needs a CUDA device (B200, sm_100a); none is visible")
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", torch.device(device).index if not isinstance(device, int) else device)
        self.precision = precision
        self._L = _lib.lib()
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            check(self._L.bh_create(ctypes.byref(h), self.device.index, PRECISIONS[precision]))
        self._h = h
        self._R = torch.zeros(1, dtype=torch.float64, device=self.device)
        self.sim_n = 0

    # ---------------------------------------------------------------- misc
    def close(self) -> None:
        if getattr(self, "_h", None):
            self._L.bh_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    @property
    def fp32(self) -> bool:
        return self.precision == "fp32"

    @property
    def stream(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    @property
    def dtype(self) -> torch.dtype:
        return torch.float32 if self.fp32 else torch.float64

    def check(self) -> None:
        """Synchronise and raise any latched device-side error."""
        check(self._L.bh_check(self._h, self.stream))

    def stats(self) -> TraversalStats:
        s = _lib.BHStats()
        check(self._L.bh_stats_get(self._h, ctypes.byref(s), self.stream))
        return TraversalStats(int(s.n_bodies), int(s.n_cells), int(s.pp), int(s.pc), int(s.n_records))

    # ------------------------------------------------------ layout helpers
    def bodies_tensor(self, positions, masses=None) -> torch.Tensor:
        """Caller arrays -> device tensor of this engine's body layout."""
        pos = torch.as_tensor(np.ascontiguousarray(positions) if isinstance(positions, np.ndarray) else positions)
        pos = pos.to(self.device, torch.float64).reshape(-1, 3)
        if self.fp32:
            out = torch.zeros((pos.shape[0], 4), dtype=torch.float32, device=self.device)
            out[:, :3] = pos.to(torch.float32)
            if masses is not None:
                out[:, 3] = torch.as_tensor(masses).to(self.device, torch.float64).reshape(-1).to(torch.float32)
            return out
        return pos.contiguous()

    def vec_tensor(self, v) -> torch.Tensor:
        t = torch.as_tensor(np.ascontiguousarray(v) if isinstance(v, np.ndarray) else v)
        t = t.to(self.device, torch.float64).reshape(-1, 3)
        if self.fp32:
            out = torch.zeros((t.shape[0], 4), dtype=torch.float32, device=self.device)
            out[:, :3] = t.to(torch.float32)
            return out
        return t.contiguous()

    # ---------------------------------------------------- building blocks
    def bounds(self, pos: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """morton.py:33-42 on the device; returns a float64 [1] device tensor."""
        out = self._R if out is None else out
        n = pos.shape[0]
        fn = self._L.bh_bounds_f32 if pos.dtype == torch.float32 else self._L.bh_bounds_f64
        check(fn(self._h, _ptr(pos), n, _ptr(out), self.stream))
        return out

    def morton(self, pos: torch.Tensor, R: torch.Tensor) -> torch.Tensor:
        """morton.py:109-125: uint64 keys (returned as an int64 tensor view)."""
        n = pos.shape[0]
        keys = torch.empty(n, dtype=torch.int64, device=self.device)
        fn = self._L.bh_morton_f32 if pos.dtype == torch.float32 else self._L.bh_morton_f64
        check(fn(self._h, _ptr(pos), n, _ptr(R), _ptr(keys), self.stream))
        return keys

    def sort(self, keys: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
        """morton.py:128-130: (sorted keys, stable argsort as int64)."""
        n = keys.shape[0]
        ks = torch.empty_like(keys)
        perm = torch.empty(n, dtype=torch.int64, device=self.device)
        check(self._L.bh_sort(self._h, _ptr(keys), n, _ptr(ks), _ptr(perm), self.stream))
        return ks, perm

    def scan_u32(self, values: torch.Tensor, inclusive: bool = False) -> torch.Tensor:
        """The build's device prefix sum (int32 tensor in, int32 out, mod 2^32)."""
        out = torch.empty_like(values)
        check(self._L.bh_scan_u32(self._h, _ptr(values), values.shape[0], _ptr(out), int(inclusive), self.stream))
        return out

    def build(self, pos_sorted: torch.Tensor, R: torch.Tensor, mass_sorted: torch.Tensor | None = None) -> int:
        """hashed.py:448-515 over Morton-sorted bodies; returns the cell count."""
        n = pos_sorted.shape[0]
        if self.fp32:
            check(self._L.bh_build_f32(self._h, _ptr(pos_sorted), n, _ptr(R), self.stream))
        else:
            if mass_sorted is None:
                raise ValueError("fp64 build needs masses")
            check(self._L.bh_build_f64(self._h, _ptr(pos_sorted), _ptr(mass_sorted), n, _ptr(R), self.stream))
        c = ctypes.c_int64()
        check(self._L.bh_tree_size(self._h, ctypes.byref(c)))
        return int(c.value)

    def set_allow_duplicates(self, allow: bool) -> None:
        """Bucket-mode extension: identical keys share a level-21 cell."""
        check(self._L.bh_set_allow_duplicates(self._h, int(bool(allow))))

    def tree_size(self) -> int:
        c = ctypes.c_int64()
        check(self._L.bh_tree_size(self._h, ctypes.byref(c)))
        return int(c.value)

    def export_tree(self) -> dict:
        """flattree.py:34-52 arrays of the current tree, as numpy."""
        C = self.tree_size()
        d = self.device
        out = dict(
            key=torch.empty(C, dtype=torch.int64, device=d),
            level=torch.empty(C, dtype=torch.int8, device=d),
            centre=torch.empty((C, 3), dtype=torch.float64, device=d),
            side=torch.empty(C, dtype=torch.float64, device=d),
            mass=torch.empty(C, dtype=torch.float64, device=d),
            com=torch.empty((C, 3), dtype=torch.float64, device=d),
            quad=torch.empty((C, 6), dtype=torch.float64, device=d),
            count=torch.empty(C, dtype=torch.int64, device=d),
            children=torch.empty((C, 8), dtype=torch.int32, device=d),
        )
        check(self._L.bh_export_tree(
            self._h, _ptr(out["key"]), _ptr(out["level"]), _ptr(out["centre"]), _ptr(out["side"]),
            _ptr(out["mass"]), _ptr(out["com"]), _ptr(out["quad"]), _ptr(out["count"]),
            _ptr(out["children"]), self.stream))
        res = {k: v.cpu().numpy() for k, v in out.items()}
        res["key"] = res["key"].view(np.uint64)
        return res

    def traverse(self, targets: torch.Tensor, theta: float, eps: float, leaf_size: int = 1,
                 acc: torch.Tensor | None = None, work: torch.Tensor | None = None):
        """flattree.py:142-166 against the current tree.  Returns device
        (acc, work) tensors in the targets' layout / order."""
        n = targets.shape[0]
        if acc is None:
            acc = torch.empty_like(targets)
        if work is None:
            work = torch.empty(n, dtype=torch.int64, device=self.device)
        fn = self._L.bh_traverse_f32 if self.fp32 else self._L.bh_traverse_f64
        check(fn(self._h, _ptr(targets), n, float(theta), float(eps), int(leaf_size),
                 _ptr(acc), _ptr(work), self.stream))
        return acc, work

    # ------------------------------------------------ resident simulation
    def sim_load(self, pos: torch.Tensor, vel: torch.Tensor, mass: torch.Tensor | None = None,
                 acc: torch.Tensor | None = None) -> None:
        n = pos.shape[0]
        check(self._L.bh_sim_load(self._h, _ptr(pos), _ptr(vel), _ptr(mass), _ptr(acc), n,
                                  self.stream))
        self.sim_n = n

    def sim_forces(self, theta: float, eps: float, leaf_size: int = 1, record_work: bool = False) -> None:
        check(self._L.bh_sim_forces(self._h, float(theta), float(eps), int(leaf_size),
                                    int(bool(record_work)), self.stream))

    def sim_step(self, dt: float, theta: float, eps: float, leaf_size: int = 1, steps: int = 1) -> None:
        check(self._L.bh_sim_step(self._h, float(dt), float(theta), float(eps), int(leaf_size),
                                  int(steps), self.stream))

    # -- phases (multi-GPU driver, decomposition.py) --
    def sim_begin_step(self, dt: float) -> None:
        check(self._L.bh_sim_begin_step(self._h, float(dt), self.stream))

    def sim_prepare(self, theta: float, eps: float, leaf_size: int = 1, bounds_ready: bool = True) -> None:
        check(self._L.bh_sim_prepare(self._h, float(theta), float(eps), int(leaf_size),
                                     int(bool(bounds_ready)), self.stream))

    def sim_tree_fits_dev(self, out: torch.Tensor) -> None:
        """Sync-free: out[0] (int32, device) = 1 if the last sync-free build fit
        its cell capacity, else 0 (then ``sim_tree_fits`` grows it)."""
        assert out.dtype == torch.int32 and out.is_cuda
        check(self._L.bh_sim_tree_fits_dev(self._h, ctypes.c_void_p(out.data_ptr()), self.stream))

    def sim_tree_fits(self) -> bool:
        """After sim_prepare: False if the sync-free build overflowed its cell
        capacity (the capacity is grown; prepare again).  One host sync."""
        c = ctypes.c_int64()
        rc = self._L.bh_tree_size(self._h, ctypes.byref(c))
        if rc == _lib.BH_OUT_OF_MEMORY:
            return False
        check(rc)
        return True

    def sim_walk_range(self, theta: float, eps: float, leaf_size: int, begin: int, end: int,
                       record_work: bool = True) -> None:
        check(self._L.bh_sim_walk_range(self._h, float(theta), float(eps), int(leaf_size),
                                        int(begin), int(end), int(bool(record_work)), self.stream))

    # ---- replicated ranks over NVLink peer memory (bh_sim_set_peers)
    def sim_ipc_handles(self) -> bytes:
        """128 bytes: IPC handles of this engine's resident acc and work buffers."""
        buf = ctypes.create_string_buffer(128)
        check(self._L.bh_sim_ipc_handles(self._h, buf))
        return buf.raw

    def sim_set_peers(self, handles: list[bytes]) -> None:
        """Open the peers' acc/work buffers; walk_range then stores into them too."""
        blob = b"".join(handles)
        buf = ctypes.create_string_buffer(blob, len(blob)) if blob else None
        check(self._L.bh_sim_set_peers(self._h, len(handles), buf))

    def sim_result_ptrs(self) -> tuple[int, int]:
        a, w = ctypes.c_void_p(), ctypes.c_void_p()
        check(self._L.bh_sim_result_ptrs(self._h, ctypes.byref(a), ctypes.byref(w)))
        return a.value, w.value

    def sim_set_peer_ptrs(self, ptrs: list[tuple[int, int]]) -> None:
        """Same-process ranks: the peers' (acc, work) device pointers."""
        k = len(ptrs)
        acc = (ctypes.c_void_p * max(k, 1))(*[a for a, _ in ptrs])
        work = (ctypes.c_void_p * max(k, 1))(*[w for _, w in ptrs])
        check(self._L.bh_sim_set_peer_ptrs(self._h, k, acc, work))

    def sim_scatter_work(self) -> None:
        check(self._L.bh_sim_scatter_work(self._h, self.stream))

    def sim_end_step(self, dt: float) -> None:
        check(self._L.bh_sim_end_step(self._h, float(dt), self.stream))

    def sim_export(self, what: int, begin: int, end: int, dst: torch.Tensor) -> None:
        check(self._L.bh_sim_export(self._h, int(what), int(begin), int(end), _ptr(dst), self.stream))

    def sim_import(self, what: int, begin: int, end: int, src: torch.Tensor) -> None:
        check(self._L.bh_sim_import(self._h, int(what), int(begin), int(end), _ptr(src), self.stream))

    # -- distributed build (decomposition.DistributedBuildSim) --
    def sim_local_maxabs(self) -> float:
        out = ctypes.c_double()
        check(self._L.bh_sim_local_maxabs(self._h, ctypes.byref(out), self.stream))
        return float(out.value)

    def sim_set_R(self, R: float) -> None:
        check(self._L.bh_sim_set_R(self._h, float(R), self.stream))

    def sim_sort(self) -> None:
        check(self._L.bh_sim_sort(self._h, self.stream))

    def sim_keys(self) -> torch.Tensor:
        """Morton keys (int64 view) of the resident bodies in their current order."""
        out = torch.empty(self.sim_n, dtype=torch.int64, device=self.device)
        if self.sim_n:
            check(self._L.bh_sim_keys(self._h, _ptr(out), self.stream))
        return out

    def sim_load_state(self, pos, vel, acc=None, work=None) -> None:
        n = pos.shape[0]
        check(self._L.bh_sim_load_state(self._h, _ptr(pos), _ptr(vel), _ptr(acc), _ptr(work), n,
                                        self.stream))
        self.sim_n = n

    def sim_build_local(self, theta, leaf_size, prev_key=None, next_key=None) -> int:
        nb = ctypes.c_int64()
        check(self._L.bh_sim_build_local(
            self._h, float(theta), int(leaf_size), int(prev_key is not None),
            ctypes.c_uint64(int(prev_key or 0)), int(next_key is not None),
            ctypes.c_uint64(int(next_key or 0)), ctypes.byref(nb), self.stream))
        return int(nb.value)

    def sim_branch_export(self, nb: int) -> dict:
        d = self.device
        out = dict(key=torch.empty(nb, dtype=torch.int64, device=d),
                   level=torch.empty(nb, dtype=torch.int32, device=d),
                   count=torch.empty(nb, dtype=torch.int64, device=d),
                   mom=torch.empty((nb, 10), dtype=torch.float64, device=d),
                   rec=torch.empty(nb, dtype=torch.int32, device=d),
                   lo=torch.empty(nb, dtype=torch.int32, device=d))
        if nb:
            check(self._L.bh_sim_branch_export(self._h, _ptr(out["key"]), _ptr(out["level"]),
                                               _ptr(out["count"]), _ptr(out["mom"]), _ptr(out["rec"]),
                                               _ptr(out["lo"]), self.stream))
        return out

    def sim_walk_records(self) -> torch.Tensor:
        """Walk records (int32 [n, 16] view of the 64-byte WalkNode)."""
        n = ctypes.c_int64()
        check(self._L.bh_sim_walk_records(self._h, None, ctypes.byref(n), self.stream))
        out = torch.empty((int(n.value), 16), dtype=torch.int32, device=self.device)
        if n.value:
            check(self._L.bh_sim_walk_records(self._h, _ptr(out), ctypes.byref(n), self.stream))
        return out

    def sim_let(self, boxes: torch.Tensor, self_rank: int):
        """LET sizes (records, bodies) per receiver; boxes float64 [nrank, nbox, 6]."""
        nrank, nbox = int(boxes.shape[0]), int(boxes.shape[1])
        rc = (ctypes.c_int64 * nrank)()
        bc = (ctypes.c_int64 * nrank)()
        check(self._L.bh_sim_let(self._h, _ptr(boxes), nbox, nrank, int(self_rank), rc, bc, self.stream))
        return list(rc), list(bc)

    def sim_target_boxes(self, start: torch.Tensor, out: torch.Tensor) -> None:
        """Boxes of body ranges [start[g], start[g+1]) into out [(1 + G), 6] (union first)."""
        check(self._L.bh_sim_target_boxes(self._h, _ptr(start), int(start.shape[0]) - 1, _ptr(out),
                                          self.stream))

    def sim_let_pack(self, q: int, recs: torch.Tensor, bodies: torch.Tensor, bmap: torch.Tensor) -> None:
        check(self._L.bh_sim_let_pack(self._h, int(q), _ptr(recs), _ptr(bodies), _ptr(bmap), self.stream))

    def walk_records(self, records: torch.Tensor, bodies: torch.Tensor, targets: torch.Tensor,
                     eps: float, leaf_size: int, acc: torch.Tensor, work: torch.Tensor | None) -> None:
        check(self._L.bh_walk_records_f32(self._h, _ptr(records), records.shape[0], _ptr(bodies),
                                          _ptr(targets), targets.shape[0], float(eps), int(leaf_size),
                                          _ptr(acc), _ptr(work), self.stream))

    def walk_records_defer(self, records, bodies, targets, eps, leaf_size, acc, work, defer, count) -> None:
        """Pass A of the LET overlap: flagged remote branch records are deferred
        into ``defer`` (int32 [cap, 4]); ``count`` (int32 [1], device) gets the entries."""
        check(self._L.bh_walk_records_defer_f32(self._h, _ptr(records), records.shape[0], _ptr(bodies),
                                                _ptr(targets), targets.shape[0], float(eps), int(leaf_size),
                                                _ptr(acc), _ptr(work), _ptr(defer), _ptr(count),
                                                defer.shape[0], self.stream))

    def walk_records_resume(self, records, bodies, targets, eps, leaf_size, acc, work, entries, fcnc) -> None:
        """Pass B: resume ``entries`` (int32 [k, 4]) over the completed tree; fcnc int32 [nrec, 2]."""
        check(self._L.bh_walk_records_resume_f32(self._h, _ptr(records), records.shape[0], _ptr(bodies),
                                                 _ptr(targets), targets.shape[0], float(eps), int(leaf_size),
                                                 _ptr(acc), _ptr(work), _ptr(entries), entries.shape[0],
                                                 _ptr(fcnc), self.stream))

    def sim_step_host(self, pos4: torch.Tensor, vel3: torch.Tensor, acc3: torch.Tensor, dt: float,
                      theta: float, eps: float, leaf_size: int, steps: int = 1,
                      work: torch.Tensor | None = None) -> None:
        """KDK steps on host (CPU, ideally pinned) float32 arrays pos4 (n,4), vel3/acc3
        (n,3), updated in place; ``work`` (int32 (n,), optional) receives the last
        force pass's per-body work; synchronous (bh_sim_step_host)."""
        for t, w in ((pos4, 4), (vel3, 3), (acc3, 3)):
            if t.device.type != "cpu" or t.dtype != torch.float32 or not t.is_contiguous() or t.shape[-1] != w:
                raise ValueError("sim_step_host takes contiguous float32 host arrays (n,4), (n,3), (n,3)")
        n = pos4.shape[0]
        if work is not None and (work.device.type != "cpu" or work.dtype != torch.int32 or work.shape != (n,)):
            raise ValueError("sim_step_host: work must be a host int32 array of n entries")
        check(self._L.bh_sim_step_host(self._h, _ptr(pos4), _ptr(vel3), _ptr(acc3), _ptr(work), n, dt, theta,
                                       eps, leaf_size, steps, self.stream))
        torch.cuda.current_stream(self.device).synchronize()

    def sim_store(self, pos=None, vel=None, acc=None, work=None) -> None:
        check(self._L.bh_sim_store(self._h, _ptr(pos), _ptr(vel), _ptr(acc), _ptr(work), self.stream))

    # ---------------------------------------------------- instrumentation
    def timing(self, on: bool = True) -> None:
        check(self._L.bh_timing_enable(self._h, int(on)))

    def timing_reset(self) -> None:
        check(self._L.bh_timing_reset(self._h))

    def timing_get(self) -> dict:
        arr = (ctypes.c_double * len(_lib.PHASES))()
        check(self._L.bh_timing_get(self._h, arr, len(_lib.PHASES)))
        return {p: float(arr[i]) for i, p in enumerate(_lib.PHASES)}

    def launches(self) -> int:
        s = _lib.BHStats()
        check(self._L.bh_stats_get(self._h, ctypes.byref(s), self.stream))
        return int(s.launches)

    def ffma_peak_tflops(self, fp64: bool = False) -> float:
        """Measured FFMA (fp64: DFMA) throughput of this GPU, TFLOP/s."""
        out = ctypes.c_double()
        fn = self._L.bh_dfma_peak if fp64 else self._L.bh_ffma_peak
        check(fn(self._h, ctypes.byref(out), self.stream))
        return float(out.value)

    # ------------------------------------------------------- validation
    def direct(self, pos3: torch.Tensor, mass: torch.Tensor, eps: float) -> torch.Tensor:
        """physics.py:288-295 (fp64, O(n^2))."""
        acc = torch.empty_like(pos3)
        check(self._L.bh_direct_f64(self._h, _ptr(pos3), _ptr(mass), pos3.shape[0], float(eps),
                                    _ptr(acc), self.stream))
        return acc

    def potential(self, pos3: torch.Tensor, mass: torch.Tensor, eps: float) -> float:
        """physics.py:322-324 (fp64, O(n^2)); per-body partials summed in fp64."""
        part = torch.empty(pos3.shape[0], dtype=torch.float64, device=self.device)
        check(self._L.bh_potential_f64(self._h, _ptr(pos3), _ptr(mass), pos3.shape[0], float(eps),
                                       _ptr(part), self.stream))
        return float(part.sum().item())


_default: dict = {}


def default_engine(precision: str = "fp32", device=None) -> Engine:
    """Process-wide engine per (precision, device)."""
    dev = torch.cuda.current_device() if device is None else torch.device(device).index if not isinstance(device, int) else device
    key = (precision, dev)
    eng = _default.get(key)
    if eng is None:
        eng = Engine(precision, dev)
        _default[key] = eng
    return eng

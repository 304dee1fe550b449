"""CPU oracle for the Barnes-Hut hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module, and only
as the checker / CPU baseline.  The product package never touches it.

It wraps ``liboracle.so`` (``bh_oracle.c``: a C restatement of the reference
kernels, compiled without FMA contraction) and restates the reference's thin
numpy glue around those kernels.  Reference citations are to
``/root/reference/pkg/src/nbsim/<file>:<line>``.  Bit-exact agreement with the
reference is pinned by ``tests/test_oracle.py`` against golden vectors that the
reference itself produced (``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

MORTON_BITS = 21
BOUNDS_PAD = 1.001
WORK_PP = 1
WORK_PC = 2

_lib = None


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc only)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        D = ctypes.c_double
        L.or_bounds.argtypes = [P, I64]
        L.or_bounds.restype = D
        L.or_morton_keys.argtypes = [P, I64, D, P]
        L.or_morton_keys.restype = I64
        L.or_sort_order.argtypes = [P, I64, P]
        L.or_sort_order.restype = None
        L.or_tree_size.argtypes = [P, I64]
        L.or_tree_size.restype = I64
        L.or_build.argtypes = [P, P, P, I64, D, I64] + [P] * 10
        L.or_build.restype = ctypes.c_int
        L.or_build2.argtypes = [P, P, P, I64, D, I64] + [P] * 10 + [ctypes.c_int]
        L.or_build2.restype = ctypes.c_int
        L.or_tree_size2.argtypes = [P, I64, ctypes.c_int]
        L.or_tree_size2.restype = I64
        L.or_traverse.argtypes = [I64] + [P] * 10 + [I64, D, D, I64, P, P, ctypes.c_int, P]
        L.or_traverse.restype = None
        L.or_direct.argtypes = [P, P, I64, D, P, ctypes.c_int]
        L.or_direct.restype = None
        L.or_from_sources.argtypes = [P, I64, P, P, I64, D, P, ctypes.c_int]
        L.or_from_sources.restype = None
        L.or_potential.argtypes = [P, P, I64, D]
        L.or_potential.restype = D
        L.or_ic_plummer.argtypes = [P, I64, I64, D, P, P, ctypes.POINTER(I64)]
        L.or_ic_plummer.restype = I64
        L.or_num_threads.argtypes = []
        L.or_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def num_threads() -> int:
    return int(lib().or_num_threads())


# --------------------------------------------------------------- morton.py


def bounds(positions) -> float:
    """morton.py:33-42 DomainBounds.from_positions -> half extent R."""
    pos = _f64(positions)
    return float(lib().or_bounds(_p(pos), pos.size))


def morton_keys(positions, R: float) -> np.ndarray:
    """morton.py:109-125 (raises ValueError like morton.py:116-118)."""
    pos = _f64(positions).reshape(-1, 3)
    keys = np.empty(len(pos), dtype=np.uint64)
    bad = lib().or_morton_keys(_p(pos), len(pos), float(R), _p(keys))
    if bad >= 0:
        raise ValueError(f"position {pos[bad]} outside domain [-{R}, {R})")
    return keys


def sort_order(keys) -> np.ndarray:
    """morton.py:128-130 np.argsort(kind='stable')."""
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    perm = np.empty(len(keys), dtype=np.int64)
    lib().or_sort_order(_p(keys), len(keys), _p(perm))
    return perm


# --------------------------------------------------------------- hashed.py


@dataclass
class OracleTree:
    """FlatTree arrays (flattree.py:34-52) plus key/level and bucket `lo`."""

    key: np.ndarray
    level: np.ndarray
    centre: np.ndarray
    side: np.ndarray
    mass: np.ndarray
    com: np.ndarray
    quad: np.ndarray
    count: np.ndarray
    children: np.ndarray
    lo: np.ndarray
    bmass: np.ndarray  # sorted bodies the tree was built from
    bpos: np.ndarray

    def __len__(self) -> int:
        return len(self.count)


def build_tree(mass_sorted, pos_sorted, R: float, allow_duplicates: bool = False) -> OracleTree:
    """hashed.py:448-515 build_hashed on Morton-sorted bodies (with moments).
    ``allow_duplicates``: bucket-mode extension, equal keys share a level-21 cell."""
    m = _f64(mass_sorted).reshape(-1)
    pos = _f64(pos_sorted).reshape(-1, 3)
    n = len(m)
    keys = morton_keys(pos, R) if n else np.zeros(0, dtype=np.uint64)
    C = int(lib().or_tree_size2(_p(keys), n, int(allow_duplicates)))
    if C == -1:
        raise ValueError("bodies must be sorted by spatial key for a hashed build")
    if C == -2:
        raise ValueError("two bodies share the level-21 cell; positions are closer than the tree resolution")
    t = OracleTree(
        key=np.zeros(C, np.uint64),
        level=np.zeros(C, np.int8),
        centre=np.zeros((C, 3)),
        side=np.zeros(C),
        mass=np.zeros(C),
        com=np.zeros((C, 3)),
        quad=np.zeros((C, 6)),
        count=np.zeros(C, np.int64),
        children=np.full((C, 8), -1, np.int32),
        lo=np.zeros(C, np.int64),
        bmass=m,
        bpos=pos,
    )
    rc = lib().or_build2(
        _p(keys), _p(m), _p(pos), n, float(R), C,
        _p(t.key), _p(t.level), _p(t.centre), _p(t.side), _p(t.mass), _p(t.com),
        _p(t.quad), _p(t.count), _p(t.children), _p(t.lo), int(allow_duplicates),
    )
    assert rc == 0, rc
    return t


# ------------------------------------------------------------- flattree.py


def traverse(tree: OracleTree, targets, theta: float, eps: float, leaf_size: int = 1,
             nthreads: int = 0, totals: np.ndarray | None = None):
    """flattree.py:142-166 FlatTree.traverse (+ bucket extension for leaf_size>1).
    ``totals`` (int64[2]) receives the summed (pp, pc) interaction counts."""
    tg = _f64(targets).reshape(-1, 3)
    acc = np.zeros_like(tg)
    work = np.zeros(len(tg), dtype=np.int64)
    lib().or_traverse(
        len(tree), _p(tree.children), _p(tree.count), _p(tree.side), _p(tree.mass),
        _p(tree.com), _p(tree.quad), _p(tree.lo), _p(tree.bpos), _p(tree.bmass),
        _p(tg), len(tg), float(theta), float(eps), int(leaf_size), _p(acc), _p(work),
        int(nthreads), None if totals is None else _p(totals),
    )
    return acc, work


# -------------------------------------------------------------- physics.py


def direct_accelerations(mass, pos, eps: float, nthreads: int = 0) -> np.ndarray:
    """physics.py:288-295 (O(n^2))."""
    m = _f64(mass).reshape(-1)
    p = _f64(pos).reshape(-1, 3)
    acc = np.zeros_like(p)
    lib().or_direct(_p(m), _p(p), len(m), float(eps), _p(acc), int(nthreads))
    return acc


def accelerations_from_sources(tpos, smass, spos, eps: float, nthreads: int = 0):
    """physics.py:298-314."""
    t = _f64(tpos).reshape(-1, 3)
    m = _f64(smass).reshape(-1)
    p = _f64(spos).reshape(-1, 3)
    acc = np.zeros_like(t)
    lib().or_from_sources(_p(t), len(t), _p(m), _p(p), len(m), float(eps), _p(acc),
                          int(nthreads))
    return acc


def potential_energy(mass, pos, eps: float) -> float:
    """physics.py:273-285, 322-324."""
    m = _f64(mass).reshape(-1)
    p = _f64(pos).reshape(-1, 3)
    return float(lib().or_potential(_p(m), _p(p), len(m), float(eps)))


def kinetic_energy(mass, vel) -> float:
    """physics.py:316-319."""
    v = _f64(vel)
    v2 = np.einsum("ij,ij->i", v, v)
    return 0.5 * float(_f64(mass) @ v2)


# ------------------------------------------------------ composed reference path


def tree_accelerations(mass, pos, theta: float, eps: float, leaf_size: int = 1,
                       R: float | None = None, nthreads: int = 0, allow_duplicates: bool = False):
    """simulation.py:218-221 + 390-393: bounds -> keys -> stable sort -> take ->
    build_hashed -> traverse the bodies in caller order."""
    m = _f64(mass).reshape(-1)
    p = _f64(pos).reshape(-1, 3)
    if R is None:
        R = bounds(p)
    order = sort_order(morton_keys(p, R))
    tree = build_tree(m[order], p[order], R, allow_duplicates)
    return traverse(tree, p, theta, eps, leaf_size, nthreads)


def leapfrog(mass, pos, vel, dt: float, steps: int, theta: float, eps: float,
             leaf_size: int = 1):
    """simulation.py:478-504 `_drive` for one rank, algorithm 1:
    bootstrap forces, then steps x {kick(dt/2), drift(dt), forces, kick(dt/2)}
    (integrator.py:37-44).  Returns (pos, vel, acc, work of the last pass)."""
    m = _f64(mass).reshape(-1).copy()
    x = _f64(pos).reshape(-1, 3).copy()
    v = _f64(vel).reshape(-1, 3).copy()
    a, work = tree_accelerations(m, x, theta, eps, leaf_size)
    for _ in range(steps):
        v += a * (0.5 * dt)
        x += v * dt
        a, work = tree_accelerations(m, x, theta, eps, leaf_size)
        v += a * (0.5 * dt)
    return x, v, a, work


# ------------------------------------------------------------ initcond.py
# Inputs for bench.py's reference arm, generated without the product library.


def make_rng(seed: int) -> np.random.Generator:
    """initcond.py:27-29."""
    return np.random.Generator(np.random.Philox(key=seed))


def plummer_cluster(n: int, rng: np.random.Generator, total_mass: float = 1.0):
    """initcond.py:62-77 -> (mass (n,), pos (n,3), vel (n,3)) fp64, consuming the
    same draws from ``rng`` as the reference (or_ic_plummer)."""
    if n < 1:
        raise ValueError(f"cluster needs at least one body, got n={n}")
    mass = np.full(n, total_mass / n)
    pos = np.empty((n, 3))
    vel = np.empty((n, 3))
    done = 0
    chunk = 1 << 20
    while done < n:
        want = min(n - done, chunk)
        state = rng.bit_generator.state
        buf = rng.random(40 * want + 4096)
        used = ctypes.c_int64()
        got = lib().or_ic_plummer(_p(buf), len(buf), want, float(total_mass), _p(pos[done:]),
                                  _p(vel[done:]), ctypes.byref(used))
        rng.bit_generator.state = state  # consume exactly the completed bodies' draws
        if used.value:
            rng.random(used.value)
        if got == 0:
            raise RuntimeError("draw buffer too small for one body")
        done += got
    return mass, pos, vel


def colliding_plummers(n_per_cluster: int, seed: int, total_mass: float = 1.0,
                       offset=(10.0, 2.0, 0.0), bulk=(0.3, 0.0, 0.0)):
    """BASELINE.json configs 0 and 3: two Plummer clusters from one stream, the
    first at +offset moving -bulk."""
    rng = make_rng(seed)
    ma, pa, va = plummer_cluster(n_per_cluster, rng, total_mass)
    mb, pb, vb = plummer_cluster(n_per_cluster, rng, total_mass)
    off = np.asarray(offset, dtype=np.float64)
    v = np.asarray(bulk, dtype=np.float64)
    return (np.concatenate([ma, mb]), np.concatenate([pa + off, pb - off]),
            np.concatenate([va - v, vb + v]))

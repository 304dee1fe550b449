"""Deterministic initial conditions -- drop-in for ``nbsim.initcond``
(/root/reference/pkg/src/nbsim/initcond.py).

Same Philox stream, same draw order, same libm arithmetic: the uniforms are
drawn by numpy (``rng.random``) and consumed by a host C restatement of the
reference's scalar sampler (``bh_ic_plummer`` in libbh.so), so
``plummer_cluster(n, make_rng(s))`` is bit-identical to the reference and the
generator is left in the same state.  Input generation, not the hot path.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .physics import Bodies, kinetic_energy

TRUNCATION_RADIUS = 10.0  # initcond.py:20
STANDARD_TOTAL_ENERGY = -0.25  # initcond.py:23
_CHUNK = 1 << 20  # bodies per draw buffer


def make_rng(seed: int) -> np.random.Generator:
    """initcond.py:27-29."""
    return np.random.Generator(np.random.Philox(key=seed))


def plummer_cluster(n: int, rng: np.random.Generator, total_mass: float = 1.0) -> Bodies:
    """initcond.py:62-77 (bit-identical, including the generator's end state)."""
    if n < 1:
        raise ValueError(f"cluster needs at least one body, got n={n}")
    L = _lib.lib()
    bodies = Bodies.zeros(n)
    bodies.mass[:] = total_mass / n
    done = 0
    while done < n:
        want = min(n - done, _CHUNK)
        state = rng.bit_generator.state
        buf = rng.random(40 * want + 4096)
        pos = np.empty((want, 3))
        vel = np.empty((want, 3))
        used = ctypes.c_int64()
        got = L.bh_ic_plummer(buf.ctypes.data_as(ctypes.c_void_p), len(buf), want,
                              float(total_mass), pos.ctypes.data_as(ctypes.c_void_p),
                              vel.ctypes.data_as(ctypes.c_void_p), ctypes.byref(used))
        # rewind and consume exactly the draws the completed bodies used
        rng.bit_generator.state = state
        if used.value:
            rng.random(used.value)
        bodies.position[done:done + got] = pos[:got]
        bodies.velocity[done:done + got] = vel[:got]
        done += got
        if got == 0:  # pragma: no cover - a single body needing > buffer draws
            raise RuntimeError("draw buffer too small for one body")
    return bodies


def _potential_exact(bodies: Bodies, eps: float) -> float:
    """physics.py:273-285 in the reference's pair order (host); GPU beyond 2e4."""
    n = len(bodies)
    if n > 20000:
        from .physics import potential_energy

        return potential_energy(bodies, eps)
    L = _lib.lib()
    return float(L.bh_host_potential_pairs(
        bodies.mass.ctypes.data_as(ctypes.c_void_p),
        bodies.position.ctypes.data_as(ctypes.c_void_p), n, float(eps)))


def standardize(bodies: Bodies, eps: float = 0.0) -> Bodies:
    """initcond.py:80-104 (same numpy expressions, same order)."""
    if len(bodies) < 2:
        raise ValueError("standardization needs at least two bodies")
    total = float(bodies.mass.sum())
    bodies.position -= (bodies.mass @ bodies.position) / total
    bodies.velocity -= (bodies.mass @ bodies.velocity) / total
    e_pot = _potential_exact(bodies, eps)
    e_kin = kinetic_energy(bodies)
    if e_pot >= 0.0 or e_kin <= 0.0:
        raise ValueError("standardization needs bound motion (E_pot < 0 < E_kin)")
    bodies.velocity *= np.sqrt(-0.5 * e_pot / e_kin)
    e_tot = 0.5 * e_pot
    q = e_tot / STANDARD_TOTAL_ENERGY
    bodies.position *= q
    bodies.velocity *= 1.0 / np.sqrt(q)
    return bodies


def two_clusters(n: int, seed: int, cluster_offset=(2.0, 2.0, 2.0),
                 relative_velocity=(0.0, 0.0, 0.0)) -> Bodies:
    """initcond.py:107-132."""
    if n < 4:
        raise ValueError(f"two clusters need at least 4 bodies, got n={n}")
    rng = make_rng(seed)
    offset = 0.5 * np.asarray(cluster_offset, dtype=np.float64)
    boost = 0.5 * np.asarray(relative_velocity, dtype=np.float64)
    first = plummer_cluster(n // 2, rng, total_mass=0.5)
    second = plummer_cluster(n - n // 2, rng, total_mass=0.5)
    first.position += offset
    first.velocity += boost
    second.position -= offset
    second.velocity -= boost
    return standardize(Bodies.concat([first, second]))


def colliding_plummers(n_per_cluster: int, seed: int, total_mass: float = 1.0,
                       offset=(10.0, 2.0, 0.0), bulk=(0.3, 0.0, 0.0)) -> Bodies:
    """BASELINE.json configs 0 and 3: two unstandardised
    Plummer clusters from one stream, cluster A at +offset moving -bulk."""
    rng = make_rng(seed)
    a = plummer_cluster(n_per_cluster, rng, total_mass)
    b = plummer_cluster(n_per_cluster, rng, total_mass)
    off = np.asarray(offset, dtype=np.float64)
    v = np.asarray(bulk, dtype=np.float64)
    a.position += off
    a.velocity -= v
    b.position -= off
    b.velocity += v
    return Bodies.concat([a, b])


def hernquist_cosmology(n: int, seed: int = 4, n_halos: int = 1000, halo_fraction: float = 0.7,
                        a_range=(0.005, 0.05), mass_decades: float = 2.0, sigma_v: float = 0.1,
                        truncation: float = 10.0, dtype=np.float32):
    """BASELINE.json config 4: clustered cosmology-like cloud.

    * ``halo_fraction`` of the bodies in ``n_halos`` Hernquist halos: scale
      radius a ~ U[a_range], halo mass log-uniform over ``mass_decades``
      decades, body count proportional to mass (largest-remainder rounding),
      radius from the inverse CDF r = a sqrt(u) / (1 - sqrt(u)), isotropic
      directions;
    * the rest uniform in the unit cube [0, 1)^3;
    * velocities N(0, sigma_v^2) per component; equal masses, total 1;
      no periodic wrapping.

    Choices the configuration leaves open, recorded here and in DESIGN.md:
    halo centres are uniform in [0.1, 0.9)^3, and radii are truncated at
    ``truncation`` * a by drawing u below (t / (1 + t))^2 (exact inverse-CDF
    truncation, no rejection).  Philox key ``seed``; vectorised (numpy), so it
    is not a bit-level restatement of any reference generator (the reference
    has none for this configuration).  Returns (pos (n,3), vel (n,3), mass (n,))
    in ``dtype``.
    """
    rng = make_rng(seed)
    n_h = int(round(halo_fraction * n))
    logm = rng.uniform(0.0, mass_decades, n_halos)
    w = 10.0 ** logm
    share = n_h * w / w.sum()
    counts = np.floor(share).astype(np.int64)
    rem = n_h - int(counts.sum())
    if rem > 0:
        counts[np.argsort(-(share - counts), kind="stable")[:rem]] += 1
    centres = rng.uniform(0.1, 0.9, (n_halos, 3))
    scale = rng.uniform(a_range[0], a_range[1], n_halos)
    pos = np.empty((n, 3), dtype=dtype)
    umax = (truncation / (1.0 + truncation)) ** 2
    off = 0
    for h in range(n_halos):
        k = int(counts[h])
        if k == 0:
            continue
        su = np.sqrt(rng.uniform(0.0, umax, k))
        r = scale[h] * su / (1.0 - su)
        z = rng.uniform(-1.0, 1.0, k)
        phi = rng.uniform(0.0, 2.0 * np.pi, k)
        s = np.sqrt(np.maximum(0.0, 1.0 - z * z))
        pos[off:off + k, 0] = centres[h, 0] + r * s * np.cos(phi)
        pos[off:off + k, 1] = centres[h, 1] + r * s * np.sin(phi)
        pos[off:off + k, 2] = centres[h, 2] + r * z
        off += k
    pos[off:] = rng.uniform(0.0, 1.0, (n - off, 3))
    vel = (rng.standard_normal((n, 3)) * sigma_v).astype(dtype)
    mass = np.full(n, 1.0 / n, dtype=dtype)
    return pos, vel, mass

"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports ``nbsim`` from ``/root/reference/pkg/src`` and writes small ``.npz``
fixtures next to this file.  The fixtures pin the oracle (tests/test_oracle.py)
and, transitively, the GPU path (tests/test_gpu_*.py) without the reference
being present on the GPU box.  Nothing here is executed at test time.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF)

from nbsim.flattree import FlatTree  # noqa: E402
from nbsim.hashed import build_hashed  # noqa: E402
from nbsim.initcond import make_rng, plummer_cluster, two_clusters  # noqa: E402
from nbsim.integrator import drift, kick  # noqa: E402
from nbsim.morton import DomainBounds, morton_keys, sort_order  # noqa: E402
from nbsim.physics import Bodies, direct_accelerations, total_energy  # noqa: E402


def sorted_bodies(n: int, seed: int, span: float = 1.0) -> tuple[Bodies, DomainBounds]:
    rng = make_rng(seed)
    pos = rng.uniform(-span, span, size=(n, 3))
    mass = rng.uniform(0.5, 1.5, size=n) / max(n, 1)
    b = Bodies(mass, pos, np.zeros((n, 3)))
    bounds = DomainBounds.from_positions(b.position)
    order = sort_order(morton_keys(b.position, bounds))
    return b.take(order), bounds


def tree_arrays(tree) -> dict:
    n = tree.n_cells
    return dict(
        t_key=tree.key[:n].copy(),
        t_level=tree.level[:n].copy(),
        t_centre=tree.centre[:n].copy(),
        t_side=tree.side[:n].copy(),
        t_mass=tree.mass[:n].copy(),
        t_com=tree.com[:n].copy(),
        t_quad=tree.quad[:n].copy(),
        t_count=tree.count[:n].copy(),
        t_children=tree.children[:n].copy(),
    )


def flat_of(tree) -> FlatTree:
    n = tree.n_cells
    return FlatTree(
        tree.centre[:n], tree.side[:n], tree.mass[:n], tree.com[:n], tree.quad[:n],
        tree.count[:n], tree.children[:n],
    )


def gen_keys() -> None:
    rng = make_rng(7)
    pos = rng.uniform(-0.9, 0.9, size=(4096, 3))
    # exact edge values: -R, 0 (upper-half midpoint), largest value below R
    pos[0] = (-1.0, 0.0, np.nextafter(1.0, -1.0))
    bounds = DomainBounds(1.0)
    keys = morton_keys(pos, bounds)
    # ties: repeated positions must sort by original index
    tie_pos = np.array([[0.5, 0.5, 0.5]] * 3 + [[-0.5, -0.5, -0.5]] + list(pos[1:60]) * 2)
    tie_keys = morton_keys(tie_pos, bounds)
    # Plummer-like cloud, bounds from positions (the pad path)
    pl = plummer_cluster(3000, make_rng(5), 1.0)
    b2 = DomainBounds.from_positions(pl.position)
    np.savez_compressed(
        os.path.join(HERE, "keys.npz"),
        pos=pos, R=1.0, keys=keys, order=sort_order(keys),
        tie_pos=tie_pos, tie_keys=tie_keys, tie_order=sort_order(tie_keys),
        pl_pos=pl.position, pl_R=b2.half_extent, pl_keys=morton_keys(pl.position, b2),
        pl_order=sort_order(morton_keys(pl.position, b2)),
    )


def gen_trees() -> None:
    out = {}
    for n, seed in [(1, 0), (2, 1), (3, 2), (64, 3), (400, 4), (2000, 5)]:
        b, bounds = sorted_bodies(n, seed)
        tree = build_hashed(b, bounds)
        arrs = tree_arrays(tree)
        for k, v in arrs.items():
            out[f"n{n}_{k}"] = v
        out[f"n{n}_mass"] = b.mass
        out[f"n{n}_pos"] = b.position
        out[f"n{n}_R"] = bounds.half_extent
        if n >= 64:
            flat = flat_of(tree)
            for theta in (0.0, 0.3, 0.5, 0.7, 1.2):
                acc, work = flat.traverse(b.position, theta, 0.05)
                out[f"n{n}_acc_t{theta}"] = acc
                out[f"n{n}_work_t{theta}"] = work
    np.savez_compressed(os.path.join(HERE, "trees.npz"), **out)


def gen_plummer() -> None:
    # exact IC stream (initcond.py:62-77): the cfg0 clusters, seed 0
    rng = make_rng(0)
    a = plummer_cluster(1000, rng, total_mass=1.0)
    b = plummer_cluster(1000, rng, total_mass=1.0)
    tc = two_clusters(96, 3)
    np.savez_compressed(
        os.path.join(HERE, "plummer.npz"),
        a_pos=a.position, a_vel=a.velocity, a_mass=a.mass,
        b_pos=b.position, b_vel=b.velocity,
        tc_pos=tc.position, tc_vel=tc.velocity, tc_mass=tc.mass,
    )


def cfg0_bodies() -> Bodies:
    """BASELINE cfg0: two unstandardised Plummer clusters."""
    rng = make_rng(0)
    a = plummer_cluster(1000, rng, total_mass=1.0)
    b = plummer_cluster(1000, rng, total_mass=1.0)
    a.position += np.array([10.0, 2.0, 0.0])
    a.velocity -= np.array([0.3, 0.0, 0.0])
    b.position -= np.array([10.0, 2.0, 0.0])
    b.velocity += np.array([0.3, 0.0, 0.0])
    return Bodies.concat([a, b])


def tree_accel(bodies: Bodies, theta: float, eps: float):
    bounds = DomainBounds.from_positions(bodies.position)
    order = sort_order(morton_keys(bodies.position, bounds))
    tree = build_hashed(bodies.take(order), bounds)
    return flat_of(tree).traverse(bodies.position, theta, eps)


def gen_cfg0() -> None:
    theta, eps, dt, steps = 0.5, 0.01, 1e-3, 10
    bodies = cfg0_bodies()
    x0, v0 = bodies.position.copy(), bodies.velocity.copy()
    e0 = total_energy(bodies, eps)
    acc, work = tree_accel(bodies, theta, eps)
    acc0, work0 = acc.copy(), work.copy()
    bodies.acceleration[:] = acc
    for _ in range(steps):
        kick(bodies, 0.5 * dt)
        drift(bodies, dt)
        acc, work = tree_accel(bodies, theta, eps)
        bodies.acceleration[:] = acc
        kick(bodies, 0.5 * dt)
    e1 = total_energy(bodies, eps)
    direct0 = direct_accelerations(cfg0_bodies().mass, x0, eps)
    np.savez_compressed(
        os.path.join(HERE, "cfg0.npz"),
        mass=bodies.mass, pos0=x0, vel0=v0, acc0=acc0, work0=work0, direct0=direct0,
        pos=bodies.position, vel=bodies.velocity, acc=bodies.acceleration, work=work,
        e0=e0, e1=e1, theta=theta, eps=eps, dt=dt, steps=steps,
    )


def gen_work_totals() -> None:
    # acceptance criterion 9 recipe (test_acceptance.py:427-438), small sizes
    totals = {}
    for n in (1000, 10000):
        rng = make_rng(42)
        cloud = Bodies(np.full(n, 1.0 / n), rng.uniform(-1.0, 1.0, size=(n, 3)), np.zeros((n, 3)))
        bounds = DomainBounds.from_positions(cloud.position)
        bodies = cloud.take(sort_order(morton_keys(cloud.position, bounds)))
        tree = build_hashed(bodies, bounds)
        _, work = flat_of(tree).traverse(bodies.position, 0.5, 0.05)
        totals[f"n{n}"] = int(work.sum())
    np.savez_compressed(os.path.join(HERE, "work_totals.npz"), **totals)
    print("work totals", totals)


def gen_report() -> None:
    """The reference CLI's report and one snapshot file (harness.py:276-354)."""
    import shutil
    import tempfile

    from nbsim.harness import main as nbsim_main

    for alg, n, steps in ((1, 600, 8), (0, 300, 4)):
        out = tempfile.mkdtemp()
        args = ["--algorithm", str(alg), "--n", str(n), "--steps", str(steps), "--dt", "0.01",
                "--eps", "0.05", "--seed", "3", "--snapshot-every", "4", "--audit-every", "4", "--out", out]
        assert nbsim_main(args) == 0
        shutil.copy(os.path.join(out, "report.txt"), os.path.join(HERE, f"report_alg{alg}.txt"))
        shutil.copy(os.path.join(out, "snapshot_000004.csv"), os.path.join(HERE, f"snapshot_alg{alg}_000004.csv"))
        shutil.rmtree(out)
    print("reports", [f for f in os.listdir(HERE) if f.startswith(("report_", "snapshot_"))])


def gen_drift() -> None:
    """Energy drift at N=1e5 (BASELINE cfg1 geometry: Plummer, make_rng(1)),
    fp64, theta 0.5, eps 1e-3, dt 1e-3, 10 KDK steps, leaf size 1 (the
    reference's only mode), from the reference package itself: E0, E1 via
    physics.total_energy (O(N^2)), work totals, and 2000 sampled final states."""
    theta, eps, dt, steps = 0.5, 1e-3, 1e-3, 10
    bodies = plummer_cluster(100_000, make_rng(1), 1.0)
    e0 = total_energy(bodies, eps)
    acc, work = tree_accel(bodies, theta, eps)
    bodies.acceleration[:] = acc
    for _ in range(steps):
        kick(bodies, 0.5 * dt)
        drift(bodies, dt)
        acc, work = tree_accel(bodies, theta, eps)
        bodies.acceleration[:] = acc
        kick(bodies, 0.5 * dt)
    e1 = total_energy(bodies, eps)
    idx = np.sort(np.random.default_rng(11).choice(len(bodies), 2000, replace=False))
    np.savez_compressed(
        os.path.join(HERE, "drift_1e5.npz"),
        e0=e0, e1=e1, work_total=int(work.sum()), idx=idx, pos=bodies.position[idx],
        vel=bodies.velocity[idx], acc=bodies.acceleration[idx], work=work[idx],
        theta=theta, eps=eps, dt=dt, steps=steps,
    )
    print("drift", e0, e1, (e1 - e0) / abs(e0), int(work.sum()))


def gen_serial() -> None:
    """The reference wire format (hashed.py:324-346, octree.py:30-34) of the
    goldens' trees, byte for byte."""
    out = {}
    for n, seed in [(1, 0), (2, 1), (64, 3), (400, 4)]:
        b, bounds = sorted_bodies(n, seed)
        out[f"n{n}_blob"] = np.frombuffer(build_hashed(b, bounds).to_serial_bytes(), dtype=np.uint8)
        out[f"n{n}_mass"] = b.mass
        out[f"n{n}_pos"] = b.position
        out[f"n{n}_R"] = bounds.half_extent
    np.savez_compressed(os.path.join(HERE, "serial.npz"), **out)
    print("serial blobs", {k: v.size for k, v in out.items() if k.endswith("_blob")})


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "report":
    gen_report()
elif __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "serial":
    gen_serial()
elif __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "drift":
    gen_drift()
elif __name__ == "__main__":
    gen_keys()
    gen_trees()
    gen_plummer()
    gen_cfg0()
    gen_work_totals()
    gen_report()
    gen_serial()
    gen_drift()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))

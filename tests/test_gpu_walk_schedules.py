"""The fp32 walk schedules give the same per-target interaction sets.

The default traversal (k_walk9, group-classified) is checked against the
masked-stack walk it replaced (k_walk, BH_WALK_V4=1), against itself with
every batch forced to a single sibling set (BH_W9_FULL=0, the DFS mode whose
depth bound sizes its frontier), and against itself with Morton-consecutive
warps instead of the Hilbert target order (BH_WALK_HILBERT=0).  Per-body work (pp + 2 pc) must be identical;
accelerations differ only by fp32 summation order.  The schedule is chosen once
per process, so each runs in a subprocess.
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, json, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2203_08966_b200.engine import Engine
from paper_2203_08966_b200.initcond import make_rng, plummer_cluster
out = {{}}
for name, n, seed, theta, eps, leaf in {cases!r}:
    b = plummer_cluster(n, make_rng(seed), 1.0)
    if name.startswith("two"):
        half = n // 2
        b.position[:half] += (10.0, 2.0, 0.0)
        b.position[half:] -= (10.0, 2.0, 0.0)
    eng = Engine("fp32", 0)
    eng.sim_load(eng.bodies_tensor(b.position, b.mass), eng.vec_tensor(b.velocity))
    eng.sim_forces(theta, eps, leaf, True)
    a = torch.empty(n, 4, device="cuda")
    w = torch.empty(n, dtype=torch.int64, device="cuda")
    eng.sim_store(acc=a, work=w)
    eng.check()
    np.save(sys.argv[1] + "_" + name + "_acc.npy", a[:, :3].cpu().numpy())
    np.save(sys.argv[1] + "_" + name + "_work.npy", w.cpu().numpy())
    eng.close()
print("done")
"""

CASES = [
    ("plummer_L16", 100_000, 1, 0.5, 1e-3, 16),
    ("plummer_L1", 20_000, 5, 0.6, 1e-3, 1),
    ("plummer_L32_t07", 100_000, 7, 0.7, 1e-4, 32),
    ("two_L32", 60_000, 3, 0.6, 1e-4, 32),
]


def _run(tmp_path, tag, env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    prefix = str(tmp_path / tag)
    code = SCRIPT.format(root=ROOT, cases=CASES)
    r = subprocess.run([sys.executable, "-c", code, prefix], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return {c[0]: (np.load(f"{prefix}_{c[0]}_acc.npy"), np.load(f"{prefix}_{c[0]}_work.npy")) for c in CASES}


def test_walk_schedules_same_interaction_sets(tmp_path):
    base = _run(tmp_path, "v9", {"BH_WALK_V4": "0"})
    dfs = _run(tmp_path, "v9dfs", {"BH_WALK_V4": "0", "BH_W9_FULL": "0"})
    v4 = _run(tmp_path, "v4", {"BH_WALK_V4": "1"})
    # Morton-consecutive warps instead of the Hilbert target order (bh_walk.cu)
    morton = _run(tmp_path, "v9morton", {"BH_WALK_V4": "0", "BH_WALK_HILBERT": "0"})
    report = {}
    for name, (a, w) in base.items():
        for other_name, other in (("dfs", dfs), ("v4", v4), ("morton", morton)):
            a2, w2 = other[name]
            assert np.array_equal(w, w2), f"{name}: work differs from {other_name}"
            err = float(np.linalg.norm(a - a2) / np.linalg.norm(a2))
            report[f"{name}/{other_name}"] = err
            assert err < 1e-5, (name, other_name, err)
    print(json.dumps(report))

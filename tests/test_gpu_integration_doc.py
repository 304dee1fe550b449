"""The ctypes binding shown in INTEGRATION.md (the stub a maintainer would add
to nbsim) runs as written and gives the wrapper's results bit for bit."""

import os
import re

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_integration_stub_runs_and_matches_engine(monkeypatch):
    from paper_2203_08966_b200.engine import Engine
    from paper_2203_08966_b200.initcond import make_rng, plummer_cluster

    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = re.search(r"```python\nimport ctypes.*?```", text, re.S).group(0)[len("```python\n"):-3]
    b = plummer_cluster(20_000, make_rng(12))
    x = np.asarray(b.position, dtype=np.float64)
    m = np.asarray(b.mass, dtype=np.float64)
    monkeypatch.chdir(ROOT)
    ns = {"x": x, "m": m, "n": len(m)}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)  # noqa: S102 -- the documented stub itself
    torch.cuda.synchronize()
    # the same through the wrapper: bootstrap, 10 steps, then one host-array step
    eng = Engine("fp32", 0)
    pos = eng.bodies_tensor(x, m)
    vel = torch.zeros((len(m), 4), dtype=torch.float32, device="cuda")
    eng.sim_load(pos, vel)
    eng.sim_forces(0.6, 1e-3, 16, False)
    eng.sim_step(1e-3, 0.6, 1e-3, 16, 10)
    p2, v2 = torch.empty_like(vel), torch.empty_like(vel)
    eng.sim_store(p2, v2)
    np.testing.assert_array_equal(ns["pos"].cpu().numpy(), p2.cpu().numpy())
    np.testing.assert_array_equal(ns["vel"].cpu().numpy(), v2.cpu().numpy())
    hp = torch.as_tensor(np.c_[x, m], dtype=torch.float32).pin_memory()
    hv = torch.zeros((len(m), 3), dtype=torch.float32).pin_memory()
    ha = torch.zeros((len(m), 3), dtype=torch.float32).pin_memory()
    hw = torch.zeros(len(m), dtype=torch.int32).pin_memory()
    eng.sim_step_host(hp, hv, ha, 1e-3, 0.6, 1e-3, 16, 1, work=hw)
    np.testing.assert_array_equal(ns["hw"].numpy(), hw.numpy())
    np.testing.assert_array_equal(ns["hp"].numpy(), hp.numpy())
    np.testing.assert_array_equal(ns["hv"].numpy(), hv.numpy())
    np.testing.assert_array_equal(ns["ha"].numpy(), ha.numpy())
    eng.close()
    ns["L"].bh_destroy(ns["h"])

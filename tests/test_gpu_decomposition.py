"""Multi-rank step on the GPU: R ranks emulated as threads on one device
(host-side barriers only -- no kernel waits on another rank), each with its own
libbh handle, exchanging through ThreadComm.  Must equal the single-GPU run:
bitwise in fp64 (the fp64 walk keeps the reference's order), to fp32 rounding
in fp32 with identical work counts."""

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _run(precision, ranks, b, steps, theta=0.6, eps=1e-3, leaf=16, dt=1e-3):
    from paper_2203_08966_b200.decomposition import DistributedSim, StepParams, ThreadComm
    from paper_2203_08966_b200.engine import Engine

    comms = ThreadComm.group(ranks)
    out = [None] * ranks
    err = []

    def body(r):
        try:
            eng = Engine(precision, 0)
            pos = eng.bodies_tensor(b.position, b.mass)
            vel = eng.vec_tensor(b.velocity)
            m = None if eng.fp32 else torch.as_tensor(b.mass).cuda()
            sim = DistributedSim(eng, comms[r], StepParams(theta, eps, leaf, dt))
            sim.load(pos, vel, m)
            sim.bootstrap()
            sim.step(steps)
            p = torch.empty_like(vel)
            w = torch.empty(len(b), dtype=torch.int64, device="cuda")
            sim.store(pos=p, work=w)
            eng.check()
            out[r] = (p[:, :3].double().cpu().numpy(), w.cpu().numpy(), list(sim.zones))
            eng.close()
        except Exception as e:  # pragma: no cover - surfaced below
            err.append(e)
            comms[r].hub.barrier.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(ranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    if err:
        raise err[0]
    return out


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_emulated_ranks_match_single_gpu(precision):
    from paper_2203_08966_b200.initcond import make_rng, plummer_cluster

    b = plummer_cluster(20_000, make_rng(1))
    single = _run(precision, 1, b, 3)[0]
    for ranks in (2, 3):
        multi = _run(precision, ranks, b, 3)
        for pos, work, zones in multi:
            assert len(zones) == ranks + 1
            if precision == "fp64":
                np.testing.assert_array_equal(pos, single[0])
                np.testing.assert_array_equal(work, single[1])
            else:
                rel = np.abs(pos - single[0]).max() / np.abs(single[0]).max()
                assert rel < 1e-5, rel
                assert np.mean(work != single[1]) < 1e-3
        # all ranks hold the same replicated state
        for pos, work, _ in multi[1:]:
            np.testing.assert_array_equal(pos, multi[0][0])

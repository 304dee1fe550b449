"""Oracle accelerations and work for sampled targets of BASELINE cfg4 at its
full size (N=1e8 Hernquist cloud, fp32 inputs, theta 0.7, eps 1e-5, leaf size
32, bucket mode with duplicate keys), for tests/test_gpu_scale.py.

The serial oracle build of 1e8 bodies takes minutes and ~30 GB of host memory,
too much for a test, so it runs once here (the generator and the oracle are
deterministic) and the sampled results are committed:

    python tests/golden/make_cfg4_fixture.py

Test infrastructure only: the inputs come from the product's numpy generator
(initcond.hernquist_cosmology, no compute library), the answers from oracle/.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as orc  # noqa: E402
from paper_2203_08966_b200.initcond import hernquist_cosmology  # noqa: E402

N = int(os.environ.get("CFG4_N", 100_000_000))
THETA, EPS, LEAF, SAMPLE = 0.7, 1e-5, 32, 4000


def main() -> None:
    t0 = time.time()
    pos32, _, m32 = hernquist_cosmology(N, 4)
    pos = pos32.astype(np.float64)
    m = m32.astype(np.float64)
    del pos32
    R = orc.bounds(pos)
    order = orc.sort_order(orc.morton_keys(pos, R))
    print(f"keys+sort {time.time() - t0:.0f} s", flush=True)
    tree = orc.build_tree(m[order], pos[order], R, allow_duplicates=True)
    print(f"build {time.time() - t0:.0f} s, {len(tree)} cells", flush=True)
    idx = np.sort(np.random.default_rng(2024).choice(N, SAMPLE, replace=False))
    totals = np.zeros(2, dtype=np.int64)
    acc, work = orc.traverse(tree, pos[idx], THETA, EPS, LEAF, 0, totals)
    np.savez_compressed(os.path.join(HERE, f"cfg4_sample_{N}.npz"), n=N, idx=idx, acc=acc, work=work,
                        cells=len(tree), R=R, theta=THETA, eps=EPS, leaf=LEAF, pp=totals[0], pc=totals[1])
    print(f"done {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()

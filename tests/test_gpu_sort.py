"""GPU tests of the hand-written radix sort and scan (bh_sort.cu) against
numpy's stable argsort (morton.py:128-130 uses np.argsort(kind="stable")) and
cumsum: tile boundaries, ties, reversed and near-sorted inputs, full 63-bit
keys, and the empty / one-element edges."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TILE = 4096  # keys per sort tile (bh_sort.cu kTile)


@pytest.fixture(scope="module")
def eng():
    import torch

    from paper_2203_08966_b200.engine import Engine

    torch.cuda.set_device(0)
    e = Engine("fp32", 0)
    yield e
    e.close()


def _sort(eng, keys):
    import torch

    t = torch.from_numpy(keys.view(np.int64).copy()).cuda()
    ks, perm = eng.sort(t)
    return ks.cpu().numpy().view(np.uint64), perm.cpu().numpy()


def _check(eng, keys):
    ks, perm = _sort(eng, keys)
    ref = np.argsort(keys, kind="stable")
    np.testing.assert_array_equal(perm, ref)
    np.testing.assert_array_equal(ks, keys[ref])


@pytest.mark.parametrize("n", [1, 2, 31, 255, TILE - 1, TILE, TILE + 1, 3 * TILE + 17, 100_003])
def test_random_63bit_keys(eng, n):
    rng = np.random.default_rng(n)
    keys = rng.integers(0, 1 << 63, n, dtype=np.uint64)
    _check(eng, keys)


@pytest.mark.parametrize("n", [TILE + 5, 250_000])
def test_ties_keep_input_order(eng, n):
    rng = np.random.default_rng(7)
    keys = rng.integers(0, 37, n, dtype=np.uint64) << np.uint64(40)  # few distinct keys, many ties
    _check(eng, keys)
    _check(eng, np.zeros(n, dtype=np.uint64))  # all equal: identity
    _check(eng, np.full(n, (1 << 63) - 1, dtype=np.uint64))


def test_reversed_and_near_sorted(eng):
    rng = np.random.default_rng(3)
    keys = np.sort(rng.integers(0, 1 << 63, 1_000_000, dtype=np.uint64))
    _check(eng, keys[::-1].copy())
    swap = rng.integers(0, len(keys) - 1, 5000)  # a resident order after a drift
    k2 = keys.copy()
    k2[swap], k2[swap + 1] = keys[swap + 1], keys[swap]
    _check(eng, k2)


def test_large_sort_is_a_permutation(eng):
    # size-independent properties at a bench-scale n: sorted, and a permutation
    import torch

    n = 20_000_000
    g = torch.Generator(device="cuda").manual_seed(5)
    k = torch.randint(0, 1 << 62, (n,), device="cuda", generator=g, dtype=torch.int64) * 2 + 1
    ks, perm = eng.sort(k)
    assert bool((ks[1:] >= ks[:-1]).all())
    assert bool((torch.sort(perm).values == torch.arange(n, device="cuda")).all())
    assert bool((k[perm] == ks).all())
    # stability on a key range with ties
    k = torch.randint(0, 1000, (n,), device="cuda", generator=g, dtype=torch.int64)
    ks, perm = eng.sort(k)
    same = ks[1:] == ks[:-1]
    assert bool((perm[1:][same] > perm[:-1][same]).all())


@pytest.mark.parametrize("n", [1, 2, 4095, 4096, 4097, 1_000_003])
@pytest.mark.parametrize("inclusive", [False, True])
def test_scan_matches_cumsum(eng, n, inclusive):
    import torch

    rng = np.random.default_rng(n)
    v = rng.integers(0, 1 << 12, n, dtype=np.uint32)
    if n > 10:
        v[: n // 3] = 0
    out = eng.scan_u32(torch.from_numpy(v.view(np.int32).copy()).cuda(), inclusive).cpu().numpy().view(np.uint32)
    c = np.cumsum(v.astype(np.uint64)) % (1 << 32)
    ref = c if inclusive else np.concatenate([[0], c[:-1]])
    np.testing.assert_array_equal(out, ref.astype(np.uint32))


def test_scan_wraps_mod_2_32(eng):
    import torch

    v = np.full(100_000, 0xFFFF0000, dtype=np.uint32)
    out = eng.scan_u32(torch.from_numpy(v.view(np.int32).copy()).cuda()).cpu().numpy().view(np.uint32)
    ref = (np.concatenate([[0], np.cumsum(v.astype(np.uint64))[:-1]]) % (1 << 32)).astype(np.uint32)
    np.testing.assert_array_equal(out, ref)

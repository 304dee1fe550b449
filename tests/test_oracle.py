"""Pin the CPU oracle to the reference: every golden vector here was produced by
running the reference package itself (tests/golden/make_golden.py)."""

import numpy as np
import pytest

from oracle import oracle as orc


class TestKeys:
    def test_known_answers(self):
        # test_morton.py:30-50 quantize edges, via full keys on the axis
        keys = orc.morton_keys(np.array([[-1.0, -1.0, -1.0]]), 1.0)
        assert int(keys[0]) == 0
        keys = orc.morton_keys(np.array([[0.0, -1.0, -1.0]]), 1.0)
        assert int(keys[0]) == 1 << 62  # quantize(0)=2^20 on x -> top key bit
        near = np.nextafter(1.0, -1.0)
        keys = orc.morton_keys(np.array([[near, near, near]]), 1.0)
        assert int(keys[0]) == (1 << 63) - 1

    def test_out_of_domain_raises(self):
        with pytest.raises(ValueError, match="outside domain"):
            orc.morton_keys(np.array([[0.0, 0.0, 0.0], [1.5, 0.0, 0.0]]), 1.0)

    def test_bounds_pad(self):
        pos = np.array([[2.0, 0.0, 0.0], [0.0, -3.0, 0.0]])
        assert orc.bounds(pos) == pytest.approx(3.003)
        assert orc.bounds(np.zeros((2, 3))) == 1.0

    def test_golden_keys_and_order(self, golden):
        g = golden("keys.npz")
        np.testing.assert_array_equal(orc.morton_keys(g["pos"], float(g["R"])), g["keys"])
        np.testing.assert_array_equal(orc.sort_order(g["keys"]), g["order"])
        np.testing.assert_array_equal(orc.sort_order(g["tie_keys"]), g["tie_order"])
        tie4 = orc.morton_keys(g["tie_pos"][:4], 1.0)
        assert list(orc.sort_order(tie4)) == [3, 0, 1, 2]  # test_morton.py:111-115
        R = orc.bounds(g["pl_pos"])
        assert R == float(g["pl_R"])
        np.testing.assert_array_equal(orc.morton_keys(g["pl_pos"], R), g["pl_keys"])
        np.testing.assert_array_equal(orc.sort_order(g["pl_keys"]), g["pl_order"])


class TestBuild:
    @pytest.mark.parametrize("n", [1, 2, 3, 64, 400, 2000])
    def test_tree_bitwise(self, golden, n):
        g = golden("trees.npz")
        t = orc.build_tree(g[f"n{n}_mass"], g[f"n{n}_pos"], float(g[f"n{n}_R"]))
        for name in ("key", "level", "centre", "side", "mass", "com", "quad", "count", "children"):
            np.testing.assert_array_equal(getattr(t, name), g[f"n{n}_t_{name}"], err_msg=name)

    def test_duplicate_and_unsorted_rejected(self):
        pos = np.array([[0.1, 0.1, 0.1], [0.1, 0.1, 0.1], [0.5, 0.5, 0.5]])
        with pytest.raises(ValueError, match="tree resolution"):
            orc.build_tree(np.ones(3), pos, 1.0)
        with pytest.raises(ValueError, match="sorted"):
            orc.build_tree(np.ones(2), np.array([[0.5, 0.5, 0.5], [-0.5, -0.5, -0.5]]), 1.0)

    def test_empty(self):
        t = orc.build_tree(np.zeros(0), np.zeros((0, 3)), 1.0)
        assert len(t) == 1 and t.count[0] == 0


class TestTraverse:
    @pytest.mark.parametrize("n", [64, 400, 2000])
    @pytest.mark.parametrize("theta", [0.0, 0.3, 0.5, 0.7, 1.2])
    def test_bitwise(self, golden, n, theta):
        g = golden("trees.npz")
        t = orc.build_tree(g[f"n{n}_mass"], g[f"n{n}_pos"], float(g[f"n{n}_R"]))
        acc, work = orc.traverse(t, g[f"n{n}_pos"], theta, 0.05)
        np.testing.assert_array_equal(acc, g[f"n{n}_acc_t{theta}"])
        np.testing.assert_array_equal(work, g[f"n{n}_work_t{theta}"])

    def test_work_totals_known_answers(self, golden):
        # test_output.txt:350 / test_acceptance.py:427-438 recipe
        g = golden("work_totals.npz")
        assert int(g["n1000"]) == 310_605 and int(g["n10000"]) == 6_805_731
        for n in (1000, 10000):
            rng = np.random.Generator(np.random.Philox(key=42))
            pos = rng.uniform(-1.0, 1.0, size=(n, 3))
            R = orc.bounds(pos)
            order = orc.sort_order(orc.morton_keys(pos, R))
            t = orc.build_tree(np.full(n, 1.0 / n), pos[order], R)
            _, work = orc.traverse(t, pos[order], 0.5, 0.05)
            assert int(work.sum()) == int(g[f"n{n}"])

    def test_bucket_l1_is_reference(self, golden):
        g = golden("trees.npz")
        t = orc.build_tree(g["n400_mass"], g["n400_pos"], float(g["n400_R"]))
        a1, w1 = orc.traverse(t, g["n400_pos"], 0.5, 0.05, leaf_size=1)
        np.testing.assert_array_equal(a1, g["n400_acc_t0.5"])
        np.testing.assert_array_equal(w1, g["n400_work_t0.5"])

    @pytest.mark.parametrize("L", [2, 8, 16])
    def test_bucket_matches_python_restatement(self, golden, L):
        g = golden("trees.npz")
        pos, mass = g["n400_pos"], g["n400_mass"]
        t = orc.build_tree(mass, pos, float(g["n400_R"]))
        acc, work = orc.traverse(t, pos[:40], 0.5, 0.05, leaf_size=L)
        ref_acc, ref_work = _py_bucket_walk(t, pos[:40], 0.5, 0.05, L)
        np.testing.assert_array_equal(acc, ref_acc)
        np.testing.assert_array_equal(work, ref_work)

    def test_theta_zero_is_direct(self, golden):
        g = golden("trees.npz")
        t = orc.build_tree(g["n400_mass"], g["n400_pos"], float(g["n400_R"]))
        acc, _ = orc.traverse(t, g["n400_pos"], 0.0, 0.05)
        ref = orc.direct_accelerations(g["n400_mass"], g["n400_pos"], 0.05)
        np.testing.assert_allclose(acc, ref, rtol=1e-12, atol=1e-14)


def _py_bucket_walk(t, targets, theta, eps, L):
    """Independent pure-Python statement of the bucket rule."""
    e2 = eps * eps
    out = np.zeros((len(targets), 3))
    works = np.zeros(len(targets), dtype=np.int64)
    for b, p in enumerate(targets):
        a = [0.0, 0.0, 0.0]
        w = 0
        stack = [0] if t.count[0] == 1 else [c for c in t.children[0][::-1] if c >= 0]

        def ppi(m, c):
            nonlocal w
            d = [p[0] - c[0], p[1] - c[1], p[2] - c[2]]
            d2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2]
            if d2 == 0.0:
                return
            den = (d2 + e2) ** 1.5
            for k in range(3):
                a[k] += (-m * d[k]) / den
            w += 1

        while stack:
            i = stack.pop()
            c = t.com[i]
            d = [p[0] - c[0], p[1] - c[1], p[2] - c[2]]
            d2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2]
            if t.count[i] == 1:
                ppi(t.mass[i], c)
            elif d2 > 0.0 and t.side[i] < theta * np.sqrt(d2):
                q = t.quad[i]
                r1 = np.sqrt(d2)
                qr = [q[0] * d[0] + q[1] * d[1] + q[2] * d[2],
                      q[1] * d[0] + q[3] * d[1] + q[4] * d[2],
                      q[2] * d[0] + q[4] * d[1] + q[5] * d[2]]
                rqr = d[0] * qr[0] + d[1] * qr[1] + d[2] * qr[2]
                mono = -t.mass[i] / (d2 * r1)
                c5 = d2 * d2 * r1
                c7 = 2.5 * rqr / (d2 * d2 * d2 * r1)
                for k in range(3):
                    a[k] += mono * d[k] + qr[k] / c5 - c7 * d[k]
                w += 2
            elif t.count[i] <= L:
                for j in range(t.lo[i], t.lo[i] + t.count[i]):
                    ppi(t.bmass[j], t.bpos[j])
            else:
                stack.extend(c for c in t.children[i][::-1] if c >= 0)
        out[b] = a
        works[b] = w
    return out, works


class TestLeapfrog:
    def test_cfg0_trajectory_bitwise(self, golden):
        g = golden("cfg0.npz")
        x, v, a, work = orc.leapfrog(g["mass"], g["pos0"], g["vel0"], float(g["dt"]),
                                     int(g["steps"]), float(g["theta"]), float(g["eps"]))
        np.testing.assert_array_equal(x, g["pos"])
        np.testing.assert_array_equal(v, g["vel"])
        np.testing.assert_array_equal(a, g["acc"])
        np.testing.assert_array_equal(work, g["work"])
        assert int(g["work"].sum()) == 1_060_307

    def test_cfg0_energy(self, golden):
        g = golden("cfg0.npz")
        e0 = orc.kinetic_energy(g["mass"], g["vel0"]) + orc.potential_energy(g["mass"], g["pos0"], float(g["eps"]))
        assert e0 == float(g["e0"])
        assert e0 == -0.25744540715170633

    def test_direct(self, golden):
        g = golden("cfg0.npz")
        np.testing.assert_array_equal(
            orc.direct_accelerations(g["mass"], g["pos0"], float(g["eps"])), g["direct0"])


class TestDuplicateKeys:
    """Bucket-mode extension: equal keys share a level-21 cell."""

    def _cloud(self):
        rng = np.random.Generator(np.random.Philox(key=8))
        pos = rng.uniform(-1, 1, (300, 3))
        pos[10:15] = pos[9]          # a run of six identical bodies
        pos[200:202] = pos[100]      # and a pair
        m = rng.uniform(0.5, 1.5, 300)
        R = orc.bounds(pos)
        order = orc.sort_order(orc.morton_keys(pos, R))
        return m[order], pos[order], R

    def test_reference_semantics_still_reject(self):
        m, pos, R = self._cloud()
        with pytest.raises(ValueError, match="tree resolution"):
            orc.build_tree(m, pos, R)

    def test_dup_cells(self):
        m, pos, R = self._cloud()
        t = orc.build_tree(m, pos, R, allow_duplicates=True)
        dup = np.flatnonzero((t.count > 1) & (t.children.max(axis=1) < 0))
        assert sorted(t.count[dup].tolist()) == [3, 6]
        assert np.all(t.level[dup] == 21)
        assert t.mass[0] == pytest.approx(m.sum(), rel=1e-14)
        assert t.count[0] == len(m)

    def test_theta_zero_bucket_is_direct(self):
        m, pos, R = self._cloud()
        t = orc.build_tree(m, pos, R, allow_duplicates=True)
        acc, _ = orc.traverse(t, pos, 0.0, 0.05, leaf_size=4)
        ref = orc.direct_accelerations(m, pos, 0.05)
        np.testing.assert_allclose(acc, ref, rtol=1e-12, atol=1e-14)


class TestSerialBytes:
    """The wire format (hashed.py:324-346): the product's serializer applied to
    the oracle's tree arrays equals the reference's own blob byte for byte (the
    GPU test checks the device-built tree the same way)."""

    @pytest.mark.parametrize("n", [1, 2, 64, 400])
    def test_oracle_tree_serializes_to_reference_blob(self, golden, n):
        from paper_2203_08966_b200.hashed import DeviceTree

        g = golden("serial.npz")
        t = orc.build_tree(g[f"n{n}_mass"], g[f"n{n}_pos"], float(g[f"n{n}_R"]))
        dt = DeviceTree(None, n, len(t), None)
        dt._arrays = {k: getattr(t, k) for k in ("key", "level", "centre", "side", "mass", "com", "quad",
                                                 "count", "children")}
        assert dt.to_serial_bytes() == g[f"n{n}_blob"].tobytes()


class TestInitialConditions:
    def test_oracle_plummer_sampler_matches_golden(self, golden):
        """initcond.py:62-77 restated in the oracle (bench.py's reference arm
        inputs) reproduces the reference's cfg0 clusters bit for bit."""
        g = golden("plummer.npz")
        rng = orc.make_rng(0)
        ma, pa, va = orc.plummer_cluster(1000, rng, 1.0)
        mb, pb, vb = orc.plummer_cluster(1000, rng, 1.0)
        np.testing.assert_array_equal(pa, g["a_pos"])
        np.testing.assert_array_equal(va, g["a_vel"])
        np.testing.assert_array_equal(ma, g["a_mass"])
        np.testing.assert_array_equal(pb, g["b_pos"])
        np.testing.assert_array_equal(vb, g["b_vel"])

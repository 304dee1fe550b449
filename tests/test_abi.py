"""CPU checks of the C-ABI library: it loads, exports every symbol bh.h
declares, and its host-side helpers reproduce the reference ICs."""

import ctypes
import os
import re

import numpy as np

from paper_2203_08966_b200 import _lib, initcond

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_and_exports_agree():
    hdr = open(os.path.join(ROOT, "include", "bh.h")).read()
    declared = set(re.findall(r"^\s*(?:int|const char \*|int64_t|double)\s+\**(bh_\w+)\(", hdr, re.M))
    assert declared, "no declarations parsed"
    L = _lib.lib()
    for name in declared:
        assert hasattr(L, name), f"libbh.so does not export {name}"
    assert declared <= set(_lib.EXPORTS)
    for name in _lib.EXPORTS:
        assert hasattr(L, name)


def test_no_torch_types_in_abi():
    hdr = open(os.path.join(ROOT, "include", "bh.h")).read()
    assert "torch" not in hdr.lower() and "at::" not in hdr


def test_version_and_error_string():
    L = _lib.lib()
    assert L.bh_version() >= 1
    assert isinstance(_lib.last_error(), str)


def test_bad_args_fail_loudly_without_gpu():
    L = _lib.lib()
    # NULL out-pointer is rejected before touching the device
    assert L.bh_create(None, 0, 0) == _lib.BH_BAD_ARG
    assert "NULL" in _lib.last_error()


def test_plummer_matches_reference(golden):
    g = golden("plummer.npz")
    rng = initcond.make_rng(0)
    a = initcond.plummer_cluster(1000, rng, 1.0)
    b = initcond.plummer_cluster(1000, rng, 1.0)
    np.testing.assert_array_equal(a.position, g["a_pos"])
    np.testing.assert_array_equal(a.velocity, g["a_vel"])
    np.testing.assert_array_equal(a.mass, g["a_mass"])
    np.testing.assert_array_equal(b.position, g["b_pos"])
    np.testing.assert_array_equal(b.velocity, g["b_vel"])


def test_two_clusters_matches_reference(golden):
    g = golden("plummer.npz")
    tc = initcond.two_clusters(96, 3)
    np.testing.assert_array_equal(tc.position, g["tc_pos"])
    np.testing.assert_array_equal(tc.velocity, g["tc_vel"])
    np.testing.assert_array_equal(tc.mass, g["tc_mass"])


def test_cfg0_initial_condition(golden):
    g = golden("cfg0.npz")
    b = initcond.colliding_plummers(1000, 0)
    np.testing.assert_array_equal(b.position, g["pos0"])
    np.testing.assert_array_equal(b.velocity, g["vel0"])


def test_plummer_chunking_keeps_stream():
    # chunked generation must leave the generator exactly where one pass does
    old = initcond._CHUNK
    try:
        initcond._CHUNK = 7
        r1 = initcond.make_rng(9)
        a = initcond.plummer_cluster(50, r1)
        tail1 = r1.random(3)
    finally:
        initcond._CHUNK = old
    r2 = initcond.make_rng(9)
    b = initcond.plummer_cluster(50, r2)
    np.testing.assert_array_equal(a.position, b.position)
    np.testing.assert_array_equal(tail1, r2.random(3))

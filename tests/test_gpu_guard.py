"""GPU: guard_points / guard_time (reference offball.cpp:125-174) through the
C-ABI pp_guard_points against the compiled reference (oracle/_ref) on random
worlds and points all over the pitch, bit for bit; and the error contract."""
import ctypes as C

import numpy as np
import pytest

from oracle import bindings as B
from paper_1909_07717_b200 import abi

pytestmark = pytest.mark.gpu


def _world(seed, n_ours, n_theirs):
    w = abi.World()
    assert B.ref().ref_random_world(seed, n_ours, n_theirs, 0.0, C.byref(w)) == 0
    return w


@pytest.mark.parametrize("n_theirs", [0, 1, 2, 5, 16])
def test_guard_points_bit_identical(ctx, n_theirs):
    lib = abi.load_library()
    ref = B.ref()
    rng = np.random.default_rng(n_theirs)
    n = 4000
    px = np.ascontiguousarray(rng.uniform(-6.5, 6.5, n))
    py = np.ascontiguousarray(rng.uniform(-5.0, 5.0, n))
    px[:200] = rng.uniform(4.0, 6.0, 200)       # near / inside the defense area
    py[:200] = rng.uniform(-2.0, 2.0, 200)
    px[200:210] = 4.2                              # on the area's edges
    py[210:220] = 1.8
    for seed in range(3):
        w = _world(1000 + 17 * seed + n_theirs, 3, n_theirs)
        lim = abi.MotionLimits(3.25 - 0.5 * seed, 3.0, 2.5 + seed)
        cap = (10.0, 2.0, 0.5)[seed]
        got_pq, got_t = np.zeros(4 * n), np.zeros(n)
        got_ok = np.zeros(n, np.uint8)
        dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
        st = lib.pp_guard_points(ctx, C.byref(w), C.byref(lim), cap, n, dp(px), dp(py),
                                 dp(got_pq), dp(got_t),
                                 got_ok.ctypes.data_as(C.POINTER(C.c_uint8)))
        assert st == 0, lib.pp_last_error(ctx)
        want_pq, want_t = np.zeros(4 * n), np.zeros(n)
        want_ok = np.zeros(n, np.uint8)
        msg = B.msgbuf()
        assert ref.ref_guard_points(C.byref(w), C.byref(lim), cap, n, dp(px), dp(py),
                                    dp(want_pq), dp(want_t),
                                    want_ok.ctypes.data_as(C.POINTER(C.c_uint8)), msg, 512) == 0
        assert np.array_equal(got_ok, want_ok)
        m = want_ok.astype(bool)
        assert 0 < m.sum() < n
        assert np.array_equal(got_pq.reshape(n, 4)[m], want_pq.reshape(n, 4)[m])
        assert np.array_equal(got_t[m], want_t[m])


def test_guard_cap_must_be_positive(ctx):
    lib = abi.load_library()
    w = _world(5, 2, 2)
    lim = abi.MotionLimits(3.25, 3.0, 3.0)
    x = (C.c_double * 1)(1.0)
    for cap in (0.0, -1.0, float("inf"), float("nan")):
        st = lib.pp_guard_points(ctx, C.byref(w), C.byref(lim), cap, 1, x, x, None, None, None)
        assert st == 4  # PP_DOMAIN, guard_time's domain_error (offball.cpp:138)

"""GPU: the plug-in backend "sm100a" (kernels::KernelBackend::scan_first,
reference kernel.hpp:46-53) through pp_scan_first against the reference's own
scalar backend (oracle/_ref, kernels::scalar_kernel()), bit for bit, on
random sampled rays and robots in the style of the reference's
test_kernels.cpp:103-200 -- random window offsets, and robots placed so the
reach / arrival margins at some sample are razor-thin."""
import ctypes as C
import math

import numpy as np
import pytest

from oracle import bindings as B
from paper_1909_07717_b200 import abi

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not B.ref_available(), reason="oracle/_ref not built")]

SLIDE, ROLL, RATIO = 3.4, 0.5, 5.0 / 7.0


def _ray(rng):
    """flat_kick samples (ts[k] = k dt, ss = distance_at) as the reference
    builds them (ball_model.cpp:12-43, in FP64 like the C++)."""
    speed = rng.uniform(1.0, 6.5)
    ang = rng.uniform(-3.14, 3.14)
    dt = rng.uniform(0.004, 0.02)
    v1 = RATIO * speed
    t_se = (speed - v1) / SLIDE
    d_se = (speed * speed - v1 * v1) / (2.0 * SLIDE)
    t_stop = t_se + v1 / ROLL
    n = int(math.floor(t_stop / dt + 1e-9)) + 1
    ts = np.array([k * dt for k in range(n)])
    ss = np.empty(n)
    for k, t in enumerate(ts):
        if t < t_se:
            ss[k] = speed * t - 0.5 * SLIDE * t * t
        elif t < t_stop:
            u = t - t_se
            ss[k] = d_se + v1 * u - 0.5 * ROLL * u * u
        else:
            ss[k] = d_se + (v1 * v1) / (2.0 * ROLL)
    return (0.25 * rng.uniform(-3.14, 3.14), 0.2 * rng.uniform(-3.14, 3.14),
            math.cos(ang), math.sin(ang), ts, ss)


def test_scan_first_matches_reference_scalar_backend(ctx):
    lib = abi.load_library()
    rng = np.random.default_rng(302)
    keep, batches, kins = [], [], []
    for i in range(3000):
        ox, oy, ux, uy, ts, ss = _ray(rng)
        keep += [ts, ss]
        kb = int(rng.integers(0, min(6, len(ts))))
        kin = abi.RobotKin()
        if i % 3 == 2:
            # razor: a robot at rest exactly reach-distance from sample k
            # (the quick reject and arrival both at the margin)
            k = int(rng.integers(1, len(ts)))
            d = 0.09 + 3.25 * ts[k] * (1.0 + rng.choice([-1e-15, 0.0, 1e-15]))
            a = rng.uniform(-math.pi, math.pi)
            px, py = ox + ux * ss[k], oy + uy * ss[k]
            kin.px, kin.py = px + d * math.cos(a), py + d * math.sin(a)
            kin.vx = kin.vy = 0.0
        else:
            kin.px, kin.py = rng.uniform(-6, 6), 0.75 * rng.uniform(-6, 6)
            kin.vx, kin.vy = rng.uniform(-3, 3), rng.uniform(-3, 3)
        kin.accel = kin.decel = 3.0
        kin.vmax, kin.radius = 3.25, 0.09
        kin.vbound = max(kin.vmax, math.hypot(kin.vx, kin.vy))
        dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
        batches.append(abi.ScanBatch(dp(ts), dp(ss), kb, len(ts), ox, oy, ux, uy))
        kins.append(kin)
    n = len(batches)
    barr = (abi.ScanBatch * n)(*batches)
    karr = (abi.RobotKin * n)(*kins)
    got = (C.c_int32 * n)()
    want = (C.c_int32 * n)()
    assert lib.pp_scan_first(ctx, n, barr, karr, got) == 0, lib.pp_last_error(ctx)
    assert B.ref().ref_scan_first(n, barr, karr, want) == 0
    g, w = np.array(got[:]), np.array(want[:])
    assert np.array_equal(g, w), np.nonzero(g != w)[0][:10]
    assert (w >= 0).sum() > 500 and (w < 0).sum() > 100  # both outcomes well represented

"""Razor-margin worlds for the FP32-shortcut safety test (test infrastructure).

In the spirit of the reference's "backends agree at razor-thin reach margins"
(proj/tests/test_kernels.cpp:144-174): every scanned robot is placed so that
the reference's exact sample test (kernel.hpp:33-44 -- quick reject, then
arrival_given <= t) flips between two adjacent doubles at one sample k of
one cell, then jittered by {-1e-9, -1e-12, -1e-15, 0, 1e-15, 1e-12, 1e-9} m.
The robot sits perpendicular to the ball's path at sample k and starts at
rest, so sample k is also its first feasible sample: the cell's champion
and feasibility hinge on the razor.

The FP64 arithmetic is restated in Python (IEEE doubles, no fused
operations -- the reference's -ffp-contract=off build), following
ball_model.cpp:12-43,83-90, dpps.cpp:30-62,119-126 and
detail/arrival_math.hpp:15-62.
"""
from __future__ import annotations

import math

import numpy as np

from paper_1909_07717_b200 import abi, synthetic

JITTERS = (-1e-9, -1e-12, -1e-15, 0.0, 1e-15, 1e-12, 1e-9)


def direction(n, k):  # dpps.cpp:30-48 (+ normalisation, dpps.cpp:120-122)
    kk = k if k <= n // 2 else (n - k) % n
    if kk == 0:
        c, s = -1.0, 0.0
    else:
        th = -math.pi + kk * (2.0 * math.pi / n)
        c, s = math.cos(th), math.sin(th)
    if k != kk:
        s = -s
    nn = math.sqrt(c * c + s * s)
    return (c / nn, s / nn) if nn != 0.0 else (1.0, 0.0)


def power(grid, j):  # dpps.cpp:50-62
    if grid.n_powers == 1:
        return grid.power_min
    return grid.power_min + (j * (grid.power_max - grid.power_min)) / (grid.n_powers - 1)


def resolve(speed, b):  # ball_model.cpp:12-43
    v1 = b.transition_ratio * speed
    t_se = (speed - v1) / b.slide_decel
    d_se = (speed * speed - v1 * v1) / (2.0 * b.slide_decel)
    t_stop = t_se + v1 / b.roll_decel
    d_stop = d_se + (v1 * v1) / (2.0 * b.roll_decel)
    return speed, v1, t_se, d_se, t_stop, d_stop


def distance_at(tr, b, t):  # ball_model.cpp:83-90
    speed, v1, t_se, d_se, t_stop, d_stop = tr
    if t < t_se:
        return speed * t - 0.5 * b.slide_decel * t * t
    if t < t_stop:
        u = t - t_se
        return d_se + v1 * u - 0.5 * b.roll_decel * u * u
    return d_stop


def rest_to_rest(L, a, b, vmax):  # arrival_math.hpp:15-21
    peak = math.sqrt(((2.0 * a) * b * L) / (a + b))
    if peak <= vmax:
        return peak / a + peak / b
    d_used = (vmax * vmax) / (2.0 * a) + (vmax * vmax) / (2.0 * b)
    return vmax / a + vmax / b + (L - d_used) / vmax


def one_d(v0, dist, a, b, vmax):  # arrival_math.hpp:26-43
    brake = (v0 * v0) / (2.0 * b)
    if v0 < 0.0 or brake > dist:
        gap = brake - math.copysign(dist, v0)
        return abs(v0) / b + rest_to_rest(gap, a, b, vmax)
    peak = math.sqrt(((2.0 * a) * b * dist + b * (v0 * v0)) / (a + b))
    if peak <= vmax:
        return (peak - v0) / a + peak / b
    if v0 <= vmax:
        d_used = (vmax * vmax - v0 * v0) / (2.0 * a) + (vmax * vmax) / (2.0 * b)
        return (vmax - v0) / a + vmax / b + (dist - d_used) / vmax
    d_used = (v0 * v0 - vmax * vmax) / (2.0 * b) + (vmax * vmax) / (2.0 * b)
    return (v0 - vmax) / b + vmax / b + (dist - d_used) / vmax


def sample_ok(px, py, rx, ry, vx, vy, lim, radius, t):  # kernel.hpp:33-44
    a, b, vmax = lim.max_accel, lim.max_decel, lim.max_speed
    qx, qy = px - rx, py - ry
    d2 = qx * qx + qy * qy
    vb = max(vmax, math.sqrt(vx * vx + vy * vy))
    reach = radius + vb * t
    if d2 > reach * reach:
        return False
    d = math.sqrt(d2)
    deff = max(d - radius, 0.0)
    den = d if d > 1e-30 else 1e-30
    ex, ey = qx / den, qy / den
    va = vx * ex + vy * ey
    vc = vx * ey - vy * ex
    ta = one_d(va, deff, a, b, vmax)
    tc = abs(vc) / b
    return (ta if ta > tc else tc) <= t


def razor_distance(px, py, nx, ny, lim, radius, t):
    """Largest double d (to 1 ulp) with the robot at p - d n passing the
    exact test at time t, at rest."""
    lo, hi = 0.0, 20.0
    ok = lambda d: sample_ok(px, py, px - d * nx, py - d * ny, 0.0, 0.0, lim, radius, t)  # noqa
    if not ok(lo) or ok(hi):
        return None
    while True:
        mid = 0.5 * (lo + hi)
        if mid <= lo or mid >= hi:
            return lo
        if ok(mid):
            lo = mid
        else:
            hi = mid


def razor_worlds(n_worlds, params, grid, seed=0xA11CE):
    """C5-style 8v8 worlds whose 15 scanned robots each sit at a razor margin
    of one random (cell, sample); world w uses jitter JITTERS[w % 7]."""
    rng = np.random.default_rng(seed)
    base = synthetic.random_worlds(np.arange(n_worlds, dtype=np.uint64) + np.uint64(seed), 8, 8)
    base["ours"]["vx"] = 0.0
    base["ours"]["vy"] = 0.0
    base["theirs"]["vx"] = 0.0
    base["theirs"]["vy"] = 0.0
    b = params.ball
    dt, radius = params.thresholds.sbip_dt, params.thresholds.robot_radius
    kinds = ([0] if grid.flat else []) + ([1] if grid.chip else [])
    out, kickers = [], []
    for w in range(n_worlds):
        fr = base[w:w + 1].copy()
        bx, by = float(fr["ball_px"][0]), float(fr["ball_py"][0])
        # the kicker (passed explicitly to both sides): the nearest teammate
        # before the others move
        d = [math.sqrt((fr["ours"]["px"][0, i] - bx) ** 2 + (fr["ours"]["py"][0, i] - by) ** 2)
             for i in range(8)]
        kicker = int(np.argmin(d))
        jit = JITTERS[w % len(JITTERS)]
        for team, lim in (("ours", params.motion_ours), ("theirs", params.motion_theirs)):
            for j in range(8):
                if team == "ours" and j == kicker:
                    continue
                for _ in range(64):
                    kind = int(rng.choice(kinds))
                    di = int(rng.integers(grid.n_directions))
                    pj = int(rng.integers(grid.n_powers))
                    ux, uy = direction(grid.n_directions, di)
                    tr = resolve(power(grid, pj), b)
                    count = int(math.floor(tr[4] / dt + 1e-9)) + 1
                    k = int(rng.integers(1, max(2, min(count, 40))))
                    t = k * dt
                    s = distance_at(tr, b, t)
                    px, py = bx + ux * s, by + uy * s
                    side = 1.0 if rng.random() < 0.5 else -1.0
                    nx, ny = -uy * side, ux * side
                    dstar = razor_distance(px, py, nx, ny, lim, radius, t)
                    if dstar is None:
                        continue
                    rx, ry = px - (dstar + jit) * nx, py - (dstar + jit) * ny
                    if abs(rx) < 6.4 and abs(ry) < 4.9:
                        fr[team]["px"][0, j], fr[team]["py"][0, j] = rx, ry
                        break
        out.append(fr[0])
        kickers.append(int(fr["ours"]["id"][0, kicker]))
    return np.array(out, dtype=base.dtype), kickers


def world_struct(fr):
    return abi.World.from_buffer_copy(fr.tobytes())

"""Generate the golden vectors under tests/golden/ from the REFERENCE itself.

Run here (this container has /root/reference):

    make -C oracle ref && python tests/golden/make_golden.py

Every output below is produced by the unmodified reference sources compiled
into oracle/_ref/libpassplan_ref.so (oracle/Makefile), called through
oracle/ref_shim.cpp:
  run_dpps_serial / best_pass / score_pass     (proj/src/dpps.cpp, pass_eval.cpp)
  goal_view                                    (proj/src/pass_eval.cpp:55-126)
  score_running_point / best_running_points    (proj/src/offball.cpp:176-258)
  oracles::random_world / lattice_world        (proj/tests/oracles.hpp:228-289)
  load_world_snapshot on proj/data/*.json      (proj/src/snapshot.cpp)

World and params structs are stored as raw bytes of the C-ABI structs, so
fixtures replay bit-exactly without /root/reference (which the GPU box lacks).
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import bindings as B  # noqa: E402
from paper_1909_07717_b200 import abi  # noqa: E402

DATA = "/root/reference/proj/data"


def as_bytes(struct) -> np.ndarray:
    return np.frombuffer(bytes(struct), dtype=np.uint8).copy()


def default_params() -> abi.Params:
    p = abi.Params()
    B.ref().ref_params_default(C.byref(p))
    return p


def load(name: str) -> abi.World:
    w = abi.World()
    m = B.msgbuf()
    st = B.ref().ref_load_snapshot(os.path.join(DATA, name).encode(), C.byref(w), m, 512)
    assert st == 0, (name, m.value)
    return w


def random_world(seed, n_o, n_t, ball_speed=0.0) -> abi.World:
    w = abi.World()
    assert B.ref().ref_random_world(seed, n_o, n_t, ball_speed, C.byref(w)) == 0
    return w


def lattice_world(seed, n_o, n_t, rolling=1) -> abi.World:
    w = abi.World()
    assert B.ref().ref_lattice_world(seed, n_o, n_t, rolling, C.byref(w)) == 0
    return w


def run_grid(w, p, g, kicker):
    n = (g.flat + g.chip) * g.n_directions * g.n_powers
    blk = abi.GridBlock(n)
    m = B.msgbuf()
    st = B.ref().ref_dpps(C.byref(w), C.byref(p), C.byref(g), kicker, 0, blk.ptr(), m, 512)
    return st, m.value.decode(), blk


def grid_case_arrays(prefix, w, p, g, kicker, out):
    st, msg, blk = run_grid(w, p, g, kicker)
    out[prefix + "world"] = as_bytes(w)
    out[prefix + "params"] = as_bytes(p)
    out[prefix + "grid"] = as_bytes(g)
    out[prefix + "kicker"] = np.array([kicker], dtype=np.int32)
    out[prefix + "status"] = np.array([st], dtype=np.int32)
    if st != 0:
        return st
    s = blk.summary
    our_id, opp_id = blk.ids()
    out[prefix + "our_id"] = our_id.astype(np.int32)
    out[prefix + "opp_id"] = opp_id.astype(np.int32)
    for name in ("our_time", "opp_time", "rx", "ry", "score", "feasible"):
        out[prefix + name] = getattr(blk, name).copy()
    out[prefix + "summary"] = as_bytes(s)
    return st


def make_grids():
    out = {}
    cases = []
    p = default_params()
    full = abi.SearchGrid(128, 64, 1.0, 6.5, 1, 1)
    f8 = load("bench_16v16.json")
    f8.n_ours = 8
    f8.n_theirs = 8
    fixtures = [("minimal", load("minimal.json"), 1), ("marked", load("marked_receiver.json"), 1),
                ("unmarked", load("unmarked_receiver.json"), 1),
                ("bench16", load("bench_16v16.json"), None), ("f8", f8, 0)]
    for name, w, kicker in fixtures:
        if kicker is None:
            kicker = B.ref().ref_nearest_teammate(C.byref(w))
        cases.append((name, w, p, full, kicker))
    # C5-style random 8v8 frames (ball at rest), full default grid.
    for i in range(6):
        w = random_world(0xB200 + i, 8, 8)
        cases.append((f"rand8v8_{i}", w, p, full, B.ref().ref_nearest_teammate(C.byref(w))))
    # Edge worlds: team sizes 0..16, moving balls, small grids.
    rng = np.random.default_rng(20261018)
    small = abi.SearchGrid(16, 8, 1.0, 6.5, 1, 1)
    for i in range(40):
        n_o = int(rng.integers(1, 17))
        n_t = int(rng.integers(0, 17))
        w = random_world(1000 + i, n_o, n_t, 3.0)
        # fast robots: |v| above vmax exercises vbound = |v| (intercept.cpp:82-83)
        if i % 4 == 0:
            for k in range(n_t):
                w.theirs[k].vx *= 1.7
                w.theirs[k].vy *= 1.7
        g = small if i % 3 else abi.SearchGrid(int(rng.integers(3, 40)), int(rng.integers(1, 12)),
                                               1.0, 6.5, int(i % 2 == 0), 1)
        cases.append((f"edge_{i}", w, p, g, w.ours[int(rng.integers(0, n_o))].id))
    # Parameter variations.
    pv = default_params()
    pv.thresholds.sbip_dt = 0.01
    pv.thresholds.robot_radius = 0.0
    pv.thresholds.safety_margin = 0.0
    cases.append(("var_dt", random_world(77, 6, 6), pv, abi.SearchGrid(24, 16, 1.0, 6.5, 1, 1), 0))
    pv2 = default_params()
    pv2.motion_ours.max_speed = 2.0
    pv2.motion_theirs.max_accel = 5.0
    pv2.ball.chip_flight_fraction = 0.8
    pv2.norm.length_upper = 9.0
    cases.append(("var_motion", random_world(78, 7, 7, 2.0), pv2,
                  abi.SearchGrid(32, 9, 2.0, 2.0, 1, 1), 0))
    cases.append(("var_chiponly", random_world(79, 5, 5), p,
                  abi.SearchGrid(20, 10, 1.5, 6.0, 0, 1), 0))
    # Ball on the field boundary and outside it (all cells Never).
    wb = random_world(80, 4, 4)
    wb.ball_px = 6.0
    wb.ball_py = -4.5
    cases.append(("ball_corner", wb, p, small, 0))
    wo = random_world(81, 4, 4)
    wo.ball_px = 6.2
    cases.append(("ball_outside", wo, p, small, 0))
    # Kicker alone on its team.
    wl = random_world(82, 1, 3)
    cases.append(("lonely_kicker", wl, p, small, wl.ours[0].id))
    # Error categories: kicker not on team ours / bad grid.
    cases.append(("err_kicker", random_world(83, 3, 3), p, small, 77))
    cases.append(("err_grid", random_world(84, 3, 3), p, abi.SearchGrid(0, 8, 1.0, 6.5, 1, 1), 0))
    cases.append(("err_power", random_world(85, 3, 3), p, abi.SearchGrid(8, 8, 3.0, 2.0, 1, 1), 0))
    names = []
    for name, w, pp, g, kicker in cases:
        grid_case_arrays(name + "/", w, pp, g, kicker, out)
        names.append(name)
    out["cases"] = np.array(names)
    return out


FULL_MAPS = ("minimal", "f8", "rand0", "lattice0", "no_opps", "one_opp")


def make_runmaps():
    out = {}
    p = default_params()
    names = []
    f8 = load("bench_16v16.json")
    f8.n_ours = 8
    f8.n_theirs = 8
    worlds = [("minimal", load("minimal.json")), ("bench16", load("bench_16v16.json")),
              ("f8", f8)]
    for i in range(5):
        worlds.append((f"rand{i}", random_world(0xB200 + i, 8, 8)))
    for i in range(3):
        worlds.append((f"lattice{i}", lattice_world(0xC8 + i, 3 + i, 4 + i)))
    we = random_world(90, 2, 0)
    worlds.append(("no_opps", we))
    w1 = random_world(91, 2, 1)
    worlds.append(("one_opp", w1))
    reqs = [abi.RunmapRequest(0xF, 0, 4, 0, 0.0, 0.0, 1),
            abi.RunmapRequest(0x4, 0x4, 2, 1, 4.0, 2.0, 1),
            abi.RunmapRequest(0xF, 0x1, 1, 0, 0.0, 0.0, 1)]
    for name, w in worlds:
        for ri, req in enumerate(reqs):
            pp = p
            if name == "f8" and ri == 2:
                pp = default_params()
                pp.thresholds.grid_step = 0.05
            nv = B.ref().ref_runmap_count(C.byref(w), C.byref(pp), req.zone_mask)
            blk = abi.RunmapBlock(nv)
            m = B.msgbuf()
            st = B.ref().ref_runmap(C.byref(w), C.byref(pp), C.byref(req), blk.ptr(), nv, m, 512)
            assert st == 0, (name, m.value)
            key = f"{name}_r{ri}/"
            out[key + "world"] = as_bytes(w)
            out[key + "params"] = as_bytes(pp)
            out[key + "req"] = as_bytes(req)
            out[key + "summary"] = as_bytes(blk.summary)
            if ri == 0 and name in FULL_MAPS:
                for arr in ("px", "py", "score", "features", "scorable"):
                    out[key + arr] = getattr(blk, arr).copy()
            names.append(key[:-1])
    out["cases"] = np.array(names)
    return out


def make_goal_views():
    """test_pass_eval.cpp:72-88 style scenes: 0..5 opponents, random points."""
    rng = np.random.default_rng(601)
    worlds, pts, res = [], [], []
    for scene in range(200):
        w = abi.World()
        w.field = abi.Field(12.0, 9.0, 1.8, 1.8, 3.6)
        n = int(rng.integers(0, 6)) if scene % 10 else 13
        w.n_theirs = n
        for i in range(n):
            if scene % 10:
                w.theirs[i].px = rng.uniform(-5.5, 5.2)
                w.theirs[i].py = rng.uniform(-4.0, 4.0)
            else:  # picket fence (test_pass_eval.cpp:90-96)
                w.theirs[i].px = 5.5
                w.theirs[i].py = -0.95 + i * 0.16
            w.theirs[i].id = i
        xs = rng.uniform(-5.5, 6.2, 16)
        ys = rng.uniform(-4.0, 4.0, 16)
        ang, lo, hi, ty = (np.zeros(16) for _ in range(4))
        dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
        assert B.ref().ref_goal_views(C.byref(w), 0.09, 16, dp(xs), dp(ys), dp(ang), dp(lo),
                                      dp(hi), dp(ty)) == 0
        worlds.append(as_bytes(w))
        pts.append(np.stack([xs, ys]))
        res.append(np.stack([ang, lo, hi, ty]))
    return {"worlds": np.stack(worlds), "points": np.stack(pts), "views": np.stack(res)}


def make_direction_tables():
    out = {}
    for n in (1, 2, 3, 7, 12, 64, 128, 1200):
        xy = np.zeros(2 * n)
        B.ref().ref_direction_table(n, xy.ctypes.data_as(C.POINTER(C.c_double)))
        out[f"dirs_{n}"] = xy
    return out


def main():
    np.savez_compressed(os.path.join(HERE, "grids.npz"), **make_grids())
    np.savez_compressed(os.path.join(HERE, "runmaps.npz"), **make_runmaps())
    np.savez_compressed(os.path.join(HERE, "goal_views.npz"), **make_goal_views())
    np.savez_compressed(os.path.join(HERE, "directions.npz"), **make_direction_tables())
    p = default_params()
    np.save(os.path.join(HERE, "default_params.npy"), as_bytes(p))
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()

"""Golden vectors for the SURVEY §8(f) rows, from the REFERENCE itself.

    make -C oracle ref && python tests/golden/make_golden_next.py

Produced by the unmodified reference sources compiled into
oracle/_ref/libpassplan_ref.so, called through oracle/ref_shim.cpp:
  intercept_all               proj/src/intercept.cpp:167-196
  possession                  proj/src/pass_eval.cpp:271-298
  decide_shot                 proj/src/pass_eval.cpp:194-233
  plan_free_kick              proj/src/pass_eval.cpp:235-269
  grid_to_csv, heatmap_to_csv, run_heatmap_to_csv   proj/src/csv.cpp:85-248
  (the CSV texts are what `passplan plan --out` / `heatmap --mode pass|run`
  write, passplan_main.cpp:82-196)

Worlds are the ones of tests/golden/grids.npz (raw C-ABI struct bytes,
stored once under B/<n>; a case's "world"/"params" entry names its blob).
Output: tests/golden/next_rows.npz.
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


def as_bytes(struct) -> np.ndarray:
    return np.frombuffer(bytes(struct), dtype=np.uint8).copy()


def struct_from(cls, arr):
    return cls.from_buffer_copy(np.asarray(arr, dtype=np.uint8).tobytes())


G = np.load(os.path.join(HERE, "grids.npz"))
WORLDS = [str(c) for c in G["cases"] if not str(c).startswith("err_")]


def case(name):
    return (struct_from(abi.World, G[f"{name}/world"]), struct_from(abi.Params, G[f"{name}/params"]),
            struct_from(abi.SearchGrid, G[f"{name}/grid"]), int(G[f"{name}/kicker"][0]))


def kicks(w: abi.World, rng: np.random.Generator):
    """(label, kick, dt) triples: the ball's free roll, flat and chip kicks."""
    out = [("roll", abi.Kick(w.ball_px, w.ball_py, w.ball_vx, w.ball_vy, 0.0, 2, 0))]
    ang = rng.uniform(-np.pi, np.pi, 2)
    out.append(("flat", abi.Kick(w.ball_px, w.ball_py, np.cos(ang[0]), np.sin(ang[0]),
                                 float(rng.uniform(1.0, 6.5)), 0, 0)))
    out.append(("chip", abi.Kick(w.ball_px, w.ball_py, np.cos(ang[1]), np.sin(ang[1]),
                                 float(rng.uniform(1.0, 6.5)), 1, 0)))
    return out


def make():
    ref = B.ref()
    m = B.msgbuf()
    out = {}
    blobs = {}

    def ref_world(w):  # world/params bytes stored once, cases keep the key
        b = bytes(w)
        key = blobs.setdefault(b, f"B/{len(blobs)}")
        out[key] = np.frombuffer(b, np.uint8).copy()
        return np.array([key])
    rng = np.random.default_rng(1909)
    # ---- intercept_all / possession / decide_shot over the golden worlds
    icases, pcases, scases = [], [], []
    for name in WORLDS:
        w, p, _, _ = case(name)
        for label, k, in kicks(w, rng):
            for dt in (p.thresholds.sbip_dt, p.thresholds.possession_dt):
                cid = f"{name}.{label}.{len(icases)}"
                res = (abi.Intercept * 32)()
                st = ref.ref_intercept_all(C.byref(w), C.byref(p), C.byref(k), dt, res, m, 512)
                out[f"ic/{cid}/world"] = ref_world(w)
                out[f"ic/{cid}/params"] = ref_world(p)
                out[f"ic/{cid}/kick"] = as_bytes(k)
                out[f"ic/{cid}/dt"] = np.array([dt])
                out[f"ic/{cid}/status"] = np.array([st], np.int32)
                out[f"ic/{cid}/out"] = np.frombuffer(bytes(res), np.uint8).copy()
                icases.append(cid)
        for vi, (pd, ce) in enumerate(((None, None), (1.0 / 60.0, None), (None, 0.5))):
            pv = abi.Params.from_buffer_copy(bytes(p))
            if pd is not None:
                pv.thresholds.possession_dt = pd
            if ce is not None:
                pv.thresholds.contest_epsilon = ce
            rep = abi.PossessionReport()
            st = ref.ref_possession(C.byref(w), C.byref(pv), C.byref(rep), m, 512)
            cid = f"{name}.{vi}"
            out[f"po/{cid}/world"] = ref_world(w)
            out[f"po/{cid}/params"] = ref_world(pv)
            out[f"po/{cid}/status"] = np.array([st], np.int32)
            out[f"po/{cid}/out"] = as_bytes(rep)
            pcases.append(cid)
        for vi, (sp, at) in enumerate(((None, None), (4.0, None), (None, 0.35), (2.0, 0.0))):
            pv = abi.Params.from_buffer_copy(bytes(p))
            if sp is not None:
                pv.thresholds.shot_power = sp
            if at is not None:
                pv.thresholds.angle_threshold = at
            for i in range(w.n_ours):
                sid = w.ours[i].id
                d = abi.ShotDecision()
                st = ref.ref_decide_shot(C.byref(w), C.byref(pv), sid, C.byref(d), m, 512)
                cid = f"{name}.{vi}.{sid}"
                out[f"sh/{cid}/world"] = ref_world(w)
                out[f"sh/{cid}/params"] = ref_world(pv)
                out[f"sh/{cid}/shooter"] = np.array([sid], np.int32)
                out[f"sh/{cid}/status"] = np.array([st], np.int32)
                out[f"sh/{cid}/out"] = as_bytes(d)
                scases.append(cid)
    # error cases
    w, p, _, _ = case("minimal")
    bad = abi.Params.from_buffer_copy(bytes(p))
    bad.ball.roll_decel = 9.0
    for cid, (pp_, k, dt) in {
        "err_dt": (p, abi.Kick(0, 0, 1, 0, 3.0, 0, 0), 0.0),
        "err_ball": (bad, abi.Kick(0, 0, 1, 0, 3.0, 0, 0), 0.01),
        "err_dir": (p, abi.Kick(0, 0, 0, 0, 3.0, 0, 0), 0.01),
        "err_speed": (p, abi.Kick(0, 0, 1, 0, -1.0, 0, 0), 0.01),
        "zero_roll": (p, abi.Kick(0.5, 0.2, 0, 0, 0.0, 2, 0), 0.001),
    }.items():
        res = (abi.Intercept * 32)()
        st = ref.ref_intercept_all(C.byref(w), C.byref(pp_), C.byref(k), dt, res, m, 512)
        out[f"ic/{cid}/world"] = ref_world(w)
        out[f"ic/{cid}/params"] = ref_world(pp_)
        out[f"ic/{cid}/kick"] = as_bytes(k)
        out[f"ic/{cid}/dt"] = np.array([dt])
        out[f"ic/{cid}/status"] = np.array([st], np.int32)
        out[f"ic/{cid}/out"] = np.frombuffer(bytes(res), np.uint8).copy()
        icases.append(cid)
    d = abi.ShotDecision()
    st = ref.ref_decide_shot(C.byref(w), C.byref(p), 999, C.byref(d), m, 512)
    out["sh/err_shooter/world"] = ref_world(w)
    out["sh/err_shooter/params"] = ref_world(p)
    out["sh/err_shooter/shooter"] = np.array([999], np.int32)
    out["sh/err_shooter/status"] = np.array([st], np.int32)
    out["sh/err_shooter/out"] = as_bytes(d)
    scases.append("err_shooter")

    # ---- plan_free_kick on feasible cells of the golden grids
    fcases = []
    for name in WORLDS:
        w, p, grid, kicker = case(name)
        if int(G[f"{name}/status"][0]) != 0:
            continue
        feas = np.flatnonzero(np.asarray(G[f"{name}/feasible"]))
        if feas.size == 0:
            continue
        summ = struct_from(abi.DppsSummary, G[f"{name}/summary"])
        pick = {int(summ.best_cell[0])} | set(int(c) for c in rng.choice(feas, min(4, feas.size),
                                                                       replace=False))
        nd, npw = grid.n_directions, grid.n_powers
        kts = [0 if grid.flat else 1, 1]
        pv = abi.Params.from_buffer_copy(bytes(p))
        pv.grid = grid
        for c in sorted(pick):
            if c < 0:
                continue
            slot, rem = divmod(c, nd * npw)
            di, pi = divmod(rem, npw)
            cand = abi.Candidate(kts[slot], di, pi, int(G[f"{name}/our_id"][c]),
                                 int(G[f"{name}/opp_id"][c]), 1, float(G[f"{name}/our_time"][c]),
                                 float(G[f"{name}/opp_time"][c]), float(G[f"{name}/rx"][c]),
                                 float(G[f"{name}/ry"][c]))
            for variant in ("ok", "infeasible", "power", "receiver", "kicker"):
                cv = abi.Candidate.from_buffer_copy(bytes(cand))
                kid = kicker
                if variant == "infeasible":
                    cv.feasible = 0
                elif variant == "power":
                    cv.power_index = npw
                elif variant == "receiver":
                    cv.our_id = 4242
                elif variant == "kicker":
                    kid = 4343
                if variant != "ok" and c != int(summ.best_cell[0]):
                    continue
                plan = abi.FreeKickPlan()
                st = ref.ref_plan_free_kick(C.byref(w), C.byref(pv), kid, C.byref(cv),
                                            C.byref(plan), m, 512)
                cid = f"{name}.{c}.{variant}"
                out[f"fk/{cid}/world"] = ref_world(w)
                out[f"fk/{cid}/params"] = ref_world(pv)
                out[f"fk/{cid}/kicker"] = np.array([kid], np.int32)
                out[f"fk/{cid}/cand"] = as_bytes(cv)
                out[f"fk/{cid}/status"] = np.array([st], np.int32)
                out[f"fk/{cid}/out"] = as_bytes(plan)
                fcases.append(cid)
    # a receive point beyond the rollout: slowest power, far target
    w, p, grid, kicker = case("minimal")
    pv = abi.Params.from_buffer_copy(bytes(p))
    cand = abi.Candidate(0, 0, 0, w.ours[0].id, -1, 1, 1.0, float("inf"), w.ball_px - 5.9,
                         w.ball_py, )
    plan = abi.FreeKickPlan()
    st = ref.ref_plan_free_kick(C.byref(w), C.byref(pv), kicker, C.byref(cand), C.byref(plan), m,
                                512)
    for key, val in (("world", ref_world(w)), ("params", ref_world(pv)),
                     ("kicker", np.array([kicker], np.int32)), ("cand", as_bytes(cand)),
                     ("status", np.array([st], np.int32)), ("out", as_bytes(plan))):
        out[f"fk/beyond_rollout/{key}"] = val
    fcases.append("beyond_rollout")

    # ---- CSV texts (small grids keep the fixture small)
    ccases = []
    for name in ("minimal", "f8", "marked", "unmarked", "rand8v8_0", "ball_outside"):
        w, p, _, kicker = case(name)
        pv = abi.Params.from_buffer_copy(bytes(p))
        pv.grid = abi.SearchGrid(16, 8, 1.0, 6.5, 1, 1)
        pv.thresholds.grid_step = 0.25
        buf = C.create_string_buffer(1 << 22)
        texts = {}
        n = ref.ref_grid_csv(C.byref(w), C.byref(pv), kicker, buf, len(buf))
        texts["grid"] = buf.value if n >= 0 else b""
        n = ref.ref_pass_heatmap_csv(C.byref(w), C.byref(pv), kicker, buf, len(buf))
        texts["pass"] = buf.value if n >= 0 else b""
        n = ref.ref_run_heatmap_csv(C.byref(w), C.byref(pv), 0xF, buf, len(buf))
        texts["run"] = buf.value if n >= 0 else b""
        out[f"csv/{name}/world"] = ref_world(w)
        out[f"csv/{name}/params"] = ref_world(pv)
        out[f"csv/{name}/kicker"] = np.array([kicker], np.int32)
        for k, t in texts.items():
            out[f"csv/{name}/{k}"] = np.frombuffer(t, np.uint8).copy()
        ccases.append(name)
    out["ic_cases"] = np.array(icases)
    out["po_cases"] = np.array(pcases)
    out["sh_cases"] = np.array(scases)
    out["fk_cases"] = np.array(fcases)
    out["csv_cases"] = np.array(ccases)
    return out


if __name__ == "__main__":
    d = make()
    np.savez_compressed(os.path.join(HERE, "next_rows.npz"), **d)
    print({k: len(d[k]) for k in d if k.endswith("_cases")})

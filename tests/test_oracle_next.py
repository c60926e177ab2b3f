"""CPU: the plain-C oracle's restatement of the SURVEY §8(f) rows
(intercept_all, possession, decide_shot, plan_free_kick) against the
reference's golden vectors, bit for bit."""
import ctypes as C

from oracle import bindings as B
from paper_1909_07717_b200 import abi
from tests.next_rows import (freekick_cases, intercept_cases, possession_cases, same,
                             shot_cases)


def test_oracle_intercept_all():
    orc, m, n = B.oracle(), B.msgbuf(), 0
    for cid, w, p, k, dt, st, want in intercept_cases():
        got = (abi.Intercept * 32)()
        assert orc.or_intercept_all(C.byref(w), C.byref(p), C.byref(k), dt, got, m, 512) == st, cid
        if st == 0:
            for i in range(w.n_ours + w.n_theirs):
                assert not same(got[i], want[i]), (cid, i, same(got[i], want[i]))
        n += 1
    assert n > 300


def test_oracle_possession():
    orc, m = B.oracle(), B.msgbuf()
    for cid, w, p, st, want in possession_cases():
        got = abi.PossessionReport()
        assert orc.or_possession(C.byref(w), C.byref(p), C.byref(got), m, 512) == st, cid
        assert not same(got, want), (cid, same(got, want))


def test_oracle_decide_shot():
    orc, m = B.oracle(), B.msgbuf()
    for cid, w, p, sid, st, want in shot_cases():
        got = abi.ShotDecision()
        assert orc.or_decide_shot(C.byref(w), C.byref(p), sid, C.byref(got), m, 512) == st, cid
        if st == 0:
            assert not same(got, want), (cid, same(got, want))


def test_oracle_plan_free_kick():
    orc, m = B.oracle(), B.msgbuf()
    for cid, w, p, kid, cand, st, want in freekick_cases():
        got = abi.FreeKickPlan()
        assert orc.or_plan_free_kick(C.byref(w), C.byref(p), kid, C.byref(cand), C.byref(got), m,
                                     512) == st, (cid, m.value)
        if st == 0:
            assert not same(got, want), (cid, same(got, want))


def test_kick_trajectory_status_cpu():
    """pp_kick_trajectory is host code: its argument checks match the
    reference's BallTrajectory::resolve (ball_model.cpp:12-43) without a GPU."""
    lib = abi.load_library()
    n = 0
    for cid, w, p, k, dt, st, want in intercept_cases():
        tr = abi.Trajectory()
        s1 = lib.pp_kick_trajectory(C.byref(k), C.byref(p.ball), C.byref(tr), None, 0)
        if cid in ("err_ball", "err_dir", "err_speed"):
            assert s1 == st != 0, cid
            n += 1
        else:
            assert s1 == 0, cid
            if k.kind == 2:  # free roll: no slide phase (ball_model.cpp:72-75)
                assert tr.slide_end_time == 0.0 and tr.v1 == tr.kick_speed
    assert n == 3

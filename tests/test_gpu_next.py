"""GPU: the product's SURVEY §8(f) rows through the C-ABI against the
reference's golden vectors: intercept_all and possession bit-exact,
decide_shot bit-exact except the goal-view angle (CUDA atan2, last ulp;
north_star tolerance 1e-4 relative written here as SCORE_RTOL),
plan_free_kick bit-exact (host arithmetic)."""
import ctypes as C

import pytest

from paper_1909_07717_b200 import abi
from tests.helpers import SCORE_RTOL
from tests.next_rows import (freekick_cases, intercept_cases, possession_cases, same,
                             shot_cases)

pytestmark = pytest.mark.gpu


def test_intercept_all_matches_reference(ctx):
    lib = abi.load_library()
    n = 0
    for cid, w, p, k, dt, st, want in intercept_cases():
        got = (abi.Intercept * 32)()
        tr = abi.Trajectory()
        s1 = lib.pp_kick_trajectory(C.byref(k), C.byref(p.ball), C.byref(tr), None, 0)
        if s1 != 0:  # the reference throws while building the trajectory
            assert s1 == st, cid
            continue
        assert lib.pp_intercept_all(ctx, C.byref(w), C.byref(p), C.byref(tr), dt, got) == st, \
            (cid, lib.pp_last_error(ctx))
        if st == 0:
            for i in range(w.n_ours + w.n_theirs):
                assert not same(got[i], want[i]), (cid, i, same(got[i], want[i]))
        n += 1
    assert n > 300


def test_possession_matches_reference(ctx):
    lib = abi.load_library()
    for cid, w, p, st, want in possession_cases():
        got = abi.PossessionReport()
        assert lib.pp_possession(ctx, C.byref(w), C.byref(p), C.byref(got)) == st, cid
        assert not same(got, want), (cid, same(got, want))


def test_decide_shot_matches_reference(ctx):
    lib = abi.load_library()
    for cid, w, p, sid, st, want in shot_cases():
        got = abi.ShotDecision()
        assert lib.pp_decide_shot(ctx, C.byref(w), C.byref(p), sid, C.byref(got)) == st, \
            (cid, lib.pp_last_error(ctx))
        if st == 0:
            assert not same(got, want, angle_rtol=SCORE_RTOL), (cid, same(got, want, SCORE_RTOL))


def test_plan_free_kick_matches_reference(ctx):
    lib = abi.load_library()
    for cid, w, p, kid, cand, st, want in freekick_cases():
        got = abi.FreeKickPlan()
        assert lib.pp_plan_free_kick(ctx, C.byref(w), C.byref(p), kid, C.byref(cand),
                                     C.byref(got)) == st, (cid, lib.pp_last_error(ctx))
        if st == 0:
            assert not same(got, want), (cid, same(got, want))

"""GPU: the FP32 shortcuts are exact-safe.

The kernels skip or accept samples with FP32 bounds (reach / arrival lower
and upper bounds, skip-ahead, window prunes, the goal-view FP32 gate and
geometric band).  PP_OPT_EXACT_ONLY turns every one of them off, so every
in-window sample and every bisection step takes the reference's exact FP64
test.  Results must be byte-identical with the switch on and off -- on
razor-margin worlds (every scanned robot one ulp from flipping a sample,
tests/razor.py, after proj/tests/test_kernels.cpp:144-174) and on random
worlds -- and bit-identical to the compiled reference."""
import ctypes as C
import os

import numpy as np
import pytest

from oracle import bindings as B
from paper_1909_07717_b200 import abi, synthetic
from tests import razor
from tests.helpers import compare_best, compare_grid, n_cells_of, run_product

pytestmark = pytest.mark.gpu

C2 = abi.SearchGrid(128, 64, 1.0, 6.5, 1, 1)


def _params():
    p = abi.Params()
    abi.load_library().pp_params_default(C.byref(p))
    return p


def _both(lib, ctx, world, p, grid, kicker):
    """(shortcuts on, shortcuts off) result blocks of one frame."""
    st, fast = run_product(lib, ctx, world, p, grid, kicker)
    assert st == 0, lib.pp_last_error(ctx)
    assert lib.pp_ctx_set_option(ctx, abi.PP_OPT_EXACT_ONLY, 1) == 0
    try:
        st, exact = run_product(lib, ctx, world, p, grid, kicker)
        assert st == 0, lib.pp_last_error(ctx)
    finally:
        lib.pp_ctx_set_option(ctx, abi.PP_OPT_EXACT_ONLY, 0)
    return fast, exact


def _same_block(a, b):
    a.summary.device_ms = 0.0
    b.summary.device_ms = 0.0
    return bytes(a.buf) == bytes(b.buf)


def _ref_block(world, p, grid, kicker):
    blk = abi.GridBlock(n_cells_of(grid))
    m = B.msgbuf()
    assert B.ref().ref_dpps(C.byref(world), C.byref(p), C.byref(grid), kicker,
                            os.cpu_count() or 1, blk.ptr(), m, 512) == 0, m.value
    ours, theirs = blk.ids()
    return blk, {"our_id": ours, "opp_id": theirs, "our_time": blk.our_time,
                 "opp_time": blk.opp_time, "rx": blk.rx, "ry": blk.ry, "score": blk.score,
                 "feasible": blk.feasible}


@pytest.mark.timeout(900)
@pytest.mark.parametrize("grid", [C2, abi.SearchGrid(97, 33, 1.0, 6.5, 1, 1)],
                         ids=["c2", "97x33"])
def test_razor_worlds_shortcuts_on_off_identical(ctx, grid):
    lib = abi.load_library()
    p = _params()
    worlds, kickers = razor.razor_worlds(14, p, grid)
    flips = 0
    for i in range(worlds.shape[0]):
        w = razor.world_struct(worlds[i])
        fast, exact = _both(lib, ctx, w, p, grid, kickers[i])
        assert _same_block(fast, exact), f"world {i}: shortcuts changed the result block"
        if B.ref_available():
            rblk, ref = _ref_block(w, p, grid, kickers[i])
            errs = compare_grid(fast, ref, f"razor {i}")
            errs += compare_best(fast.summary, rblk.summary, fast.score, f"razor {i}")
            assert not errs, "\n".join(errs)
        flips += int(fast.summary.n_feasible[0])
    assert flips > 0


@pytest.mark.timeout(900)
def test_random_worlds_shortcuts_on_off_identical(ctx):
    """Moving robots, a rolling ball for half of them, and sizes 1..16 v 0..16."""
    lib = abi.load_library()
    p = _params()
    rng = np.random.default_rng(11)
    fr = synthetic.random_worlds(np.arange(24, dtype=np.uint64) + np.uint64(777), 16, 16)
    for i in range(fr.shape[0]):
        fr["n_ours"][i] = int(rng.integers(1, 17))
        fr["n_theirs"][i] = int(rng.integers(0, 17))
        if i % 2:
            fr["ball_vx"][i], fr["ball_vy"][i] = rng.uniform(-3, 3, size=2)
    for i in range(fr.shape[0]):
        w = razor.world_struct(fr[i])
        kicker = int(fr["ours"]["id"][i][int(rng.integers(0, int(fr["n_ours"][i])))])
        fast, exact = _both(lib, ctx, w, p, C2, kicker)
        assert _same_block(fast, exact), f"world {i}"


def test_goal_views_and_possession_exact_only(ctx):
    """goal_view's FP32 gate and band, and the interception kernel's filters."""
    lib = abi.load_library()
    rng = np.random.default_rng(5)
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    for scene in range(24):
        w = abi.World()
        w.field = abi.Field(12.0, 9.0, 1.8, 1.8, 3.6)
        n = int(rng.integers(1, 17))
        w.n_theirs = n
        for j in range(n):
            w.theirs[j].px = rng.uniform(0.0, 6.5) if j % 2 else rng.uniform(-6.0, 6.0)
            w.theirs[j].py = rng.uniform(-1.5, 1.5) if j % 2 else rng.uniform(-4.5, 4.5)
            w.theirs[j].id = j
        m = 1024
        xs = rng.uniform(-6.0, 6.3, m)
        ys = rng.uniform(-4.5, 4.5, m)
        for q in range(0, m, 3):  # points next to opponents: tangents near heights
            j = int(rng.integers(0, n))
            xs[q] = w.theirs[j].px + rng.uniform(-0.3, 0.3)
            ys[q] = w.theirs[j].py + rng.uniform(-0.3, 0.3)
        outs = []
        for mode in (0, 1):
            assert lib.pp_ctx_set_option(ctx, abi.PP_OPT_EXACT_ONLY, mode) == 0
            o = [np.zeros(m) for _ in range(4)]
            assert lib.pp_goal_views(ctx, C.byref(w), 0.09, m, dp(xs), dp(ys),
                                     *(dp(a) for a in o)) == 0
            outs.append(o)
        lib.pp_ctx_set_option(ctx, abi.PP_OPT_EXACT_ONLY, 0)
        for a, b in zip(*outs):
            assert np.array_equal(a, b), scene
    from tests.next_rows import possession_cases
    for n, (cid, w, p, st_want, _want) in enumerate(possession_cases()):
        if n >= 60:
            break
        res = []
        for mode in (0, 1):
            lib.pp_ctx_set_option(ctx, abi.PP_OPT_EXACT_ONLY, mode)
            got = abi.PossessionReport()
            assert lib.pp_possession(ctx, C.byref(w), C.byref(p), C.byref(got)) == st_want, cid
            res.append(bytes(got))
        lib.pp_ctx_set_option(ctx, abi.PP_OPT_EXACT_ONLY, 0)
        assert res[0] == res[1], cid


@pytest.mark.timeout(900)
def test_batch_razor_worlds_shortcuts_on_off_identical(ctx):
    """The batch path (pp_dpps_frames: the warp-per-tile scan with caps read
    once per robot, the deferred rest rule and the cross-cap table) on
    razor-margin worlds and random 1..16 v 0..16 worlds: per-frame results
    byte-identical with the FP32 shortcuts on and off, and equal to the
    single-frame path's summary."""
    lib = abi.load_library()
    p = _params()
    for grid in (abi.SearchGrid(128, 64, 1.0, 6.5, 1, 0), C2):
        worlds, kickers = razor.razor_worlds(14, p, grid)
        rnd = synthetic.random_worlds(np.arange(18, dtype=np.uint64) + np.uint64(4242), 16, 16)
        rng = np.random.default_rng(5)
        for i in range(rnd.shape[0]):
            rnd["n_ours"][i] = int(rng.integers(2, 17))
            rnd["n_theirs"][i] = int(rng.integers(0, 17))
        fr = np.concatenate([worlds.astype(rnd.dtype), rnd])
        n = fr.shape[0]
        frames, _keep = synthetic.as_ctypes(fr)
        kick = (C.c_int32 * n)(*([int(k) for k in kickers] +
                                 [int(rnd["ours"]["id"][i][0]) for i in range(rnd.shape[0])]))
        fast = (abi.FrameSummary * n)()
        exact = (abi.FrameSummary * n)()
        assert lib.pp_dpps_frames(ctx, frames, n, C.byref(p), C.byref(grid), kick, fast) == 0, \
            lib.pp_last_error(ctx)
        assert lib.pp_ctx_set_option(ctx, abi.PP_OPT_EXACT_ONLY, 1) == 0
        try:
            assert lib.pp_dpps_frames(ctx, frames, n, C.byref(p), C.byref(grid), kick,
                                      exact) == 0, lib.pp_last_error(ctx)
        finally:
            lib.pp_ctx_set_option(ctx, abi.PP_OPT_EXACT_ONLY, 0)
        assert bytes(fast) == bytes(exact)
        for i in range(n):
            st, blk = run_product(lib, ctx, frames[i], p, grid, kick[i], copy_all=False)
            assert st == 0, lib.pp_last_error(ctx)
            for r in range(3):
                assert fast[i].best_cell[r] == blk.summary.best_cell[r], (i, r)
                assert fast[i].best_score[r] == blk.summary.best_score[r], (i, r)
                assert fast[i].n_feasible[r] == blk.summary.n_feasible[r], (i, r)

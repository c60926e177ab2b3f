"""GPU: the batched-frames path (C5).  Frames are staged on the device
(stage_frames_kernel) and searched in groups; the results must equal the
single-frame path's, and the reference's best_pass on the C5 frames
(oracles::random_world(mt19937_64(0xB200 + i), 8, 8), BASELINE configs[4])."""
import ctypes as C
import os

import numpy as np
import pytest

from oracle import bindings as B
from paper_1909_07717_b200 import abi, synthetic
from paper_1909_07717_b200.sharding import run_sharded
from tests.helpers import run_product, score_close

pytestmark = pytest.mark.gpu

C1 = abi.SearchGrid(128, 64, 1.0, 6.5, 1, 0)


def _params():
    p = abi.Params()
    abi.load_library().pp_params_default(C.byref(p))
    return p


def _mixed_frames(n, seed):
    """C5 frames with shuffled, sparse robot ids and varied team sizes, so the
    device's id sort and kicker choice are exercised."""
    rng = np.random.default_rng(seed)
    fr = synthetic.random_worlds(np.arange(n, dtype=np.uint64) + np.uint64(seed), 16, 16)
    for i in range(n):
        no, nt = int(rng.integers(1, 17)), int(rng.integers(0, 17))
        fr["n_ours"][i], fr["n_theirs"][i] = no, nt
        for team in ("ours", "theirs"):
            fr[team]["id"][i] = rng.choice(40, size=16, replace=False)
    return fr


def _compact_of(s: abi.DppsSummary):
    return ([float(s.best_score[k]) for k in range(3)], [int(s.best_cell[k]) for k in range(3)],
            [int(s.n_feasible[k]) for k in range(3)])


def _weighted(p, kind):
    """Weight sets for the batch's score-bound pruning (every sign of the view
    and refraction terms, custom norm bounds, a near-flat score), and safety
    margins for the batch scan's cross-team cap (zero, off the sample grid, large)."""
    w = p.pass_weights
    if kind.startswith("safety"):
        p.thresholds.safety_margin = {"safety0": 0.0, "safety_odd": 0.0137, "safety_big": 0.7}[kind]
    if kind == "negative":
        w.shoot_angle, w.refraction, w.teammate_time = -2.0, -1.5, -0.3
    elif kind == "norms":
        p.norm.length_upper, p.norm.angle_upper = 5.0, 0.7
        w.margin, w.dist_goal = 0.05, -2.0
    elif kind == "flat":
        w.teammate_time = w.dist_goal = w.margin = 0.0
        w.shoot_angle, w.refraction = 1e-3, 1e-3
    return p


@pytest.mark.parametrize("chip,weights", [(0, "default"), (1, "default"), (0, "negative"),
                                          (1, "norms"), (0, "flat"), (0, "safety0"),
                                          (1, "safety_odd"), (0, "safety_big")])
def test_batch_equals_single_frame(ctx, chip, weights):
    """Batches prune cells by score bounds before the value function, and
    their scans cut our robots past the cross-team cap; the single-frame path
    scores every cell and scans fully: the results must be identical."""
    lib = abi.load_library()
    p = _weighted(_params(), weights)
    grid = abi.SearchGrid(128, 64, 1.0, 6.5, 1, chip)
    n = 64
    frames_np = _mixed_frames(n, 100 + chip)
    frames, _keep = synthetic.as_ctypes(frames_np)
    sums = (abi.DppsSummary * n)()
    assert lib.pp_dpps_batch(ctx, frames, n, C.byref(p), C.byref(grid), None, sums) == 0, \
        lib.pp_last_error(ctx)
    compact = (abi.FrameSummary * n)()
    assert lib.pp_dpps_frames(ctx, frames, n, C.byref(p), C.byref(grid), None, compact) == 0
    for i in range(n):
        k = int(sums[i].kicker_id)
        st, blk = run_product(lib, ctx, frames[i], p, grid, k, copy_all=False)
        assert st == 0, lib.pp_last_error(ctx)
        for r in range(3):
            assert sums[i].best_cell[r] == blk.summary.best_cell[r], (i, r)
            assert sums[i].best_score[r] == blk.summary.best_score[r], (i, r)
            assert sums[i].n_feasible[r] == blk.summary.n_feasible[r], (i, r)
            assert bytes(sums[i].best_features[r]) == bytes(blk.summary.best_features[r])
            assert compact[i].best_cell[r] == blk.summary.best_cell[r], (i, r)
            assert compact[i].best_score[r] == blk.summary.best_score[r], (i, r)
            assert compact[i].n_feasible[r] == blk.summary.n_feasible[r], (i, r)
        assert sums[i].sbip_calls == blk.summary.sbip_calls
        assert sums[i].kicker_slot == blk.summary.kicker_slot
        assert list(sums[i].ours_ids) == list(blk.summary.ours_ids)


def test_batch_explicit_kickers_and_errors(ctx):
    lib = abi.load_library()
    p = _params()
    n = 16
    frames_np = _mixed_frames(n, 5)
    frames, _keep = synthetic.as_ctypes(frames_np)
    kick = (C.c_int32 * n)(*[int(frames_np["ours"]["id"][i][i % int(frames_np["n_ours"][i])])
                             for i in range(n)])
    out = (abi.FrameSummary * n)()
    assert lib.pp_dpps_frames(ctx, frames, n, C.byref(p), C.byref(C1), kick, out) == 0
    for i in range(n):
        st, blk = run_product(lib, ctx, frames[i], p, C1, kick[i], copy_all=False)
        assert st == 0
        assert [out[i].best_cell[r] for r in range(3)] == [blk.summary.best_cell[r] for r in range(3)]
        assert [out[i].best_score[r] for r in range(3)] == \
            [blk.summary.best_score[r] for r in range(3)]
    # the first frame whose kicker is not on team ours is reported (dpps.cpp:221-223)
    kick[3] = 99
    kick[9] = 98
    assert lib.pp_dpps_frames(ctx, frames, n, C.byref(p), C.byref(C1), kick, out) == \
        abi.PP_VALIDATION
    msg = lib.pp_last_error(ctx).decode()
    assert "frame 3" in msg and "99" in msg, msg
    frames_np["n_theirs"][2] = 17
    frames, _keep = synthetic.as_ctypes(frames_np)
    assert lib.pp_dpps_frames(ctx, frames, n, C.byref(p), C.byref(C1), None, out) == \
        abi.PP_VALIDATION
    assert "frame 2" in lib.pp_last_error(ctx).decode()
    # the context stays usable
    frames_np["n_theirs"][2] = 8
    frames, _keep = synthetic.as_ctypes(frames_np)
    assert lib.pp_dpps_frames(ctx, frames, n, C.byref(p), C.byref(C1), None, out) == 0


@pytest.mark.skipif(not B.ref_available(), reason="oracle/_ref not built")
@pytest.mark.timeout(900)
def test_c5_frames_match_reference(ctx):
    """>= 4,096 C5 frames (seeds 0xB200 + i) against the compiled reference's
    run_dpps_serial + best_pass, frame-parallel on the host cores."""
    lib = abi.load_library()
    p = _params()
    n = 4096
    frames_np = synthetic.c5_frames(0, n)
    frames, _keep = synthetic.as_ctypes(frames_np)
    out = (abi.FrameSummary * n)()
    assert lib.pp_dpps_frames(ctx, frames, n, C.byref(p), C.byref(C1), None, out) == 0
    best = np.zeros(n, np.int64)
    score = np.zeros(n)
    nfeas = np.zeros(n, np.int64)
    m = B.msgbuf()
    st = B.ref().ref_batch(frames, n, C.byref(p), C.byref(C1), None, os.cpu_count() or 1,
                           best.ctypes.data_as(C.POINTER(C.c_int64)),
                           score.ctypes.data_as(C.POINTER(C.c_double)),
                           nfeas.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(C.c_double()),
                           m, 512)
    assert st == 0, m.value
    got_nf = np.array([out[i].n_feasible[0] for i in range(n)])
    got_best = np.array([out[i].best_cell[0] for i in range(n)])
    got_score = np.array([out[i].best_score[0] for i in range(n)])
    assert np.array_equal(got_nf, nfeas), np.flatnonzero(got_nf != nfeas)[:10]
    assert np.all(score_close(got_score, score))
    same = got_best == best
    # a different best cell only where it ties within the score tolerance
    assert np.all(same | score_close(got_score, score))
    assert same.mean() > 0.999


def test_run_sharded_product_runner_n1(ctx):
    """sharding.run_sharded at world size 1 with the product runner."""
    lib = abi.load_library()
    p = _params()
    frames_np = synthetic.c5_frames(0, 96)

    def runner(sub):
        arr, _k = synthetic.as_ctypes(np.ascontiguousarray(sub))
        out = (abi.FrameSummary * len(sub))()
        assert lib.pp_dpps_frames(ctx, arr, len(sub), C.byref(p), C.byref(C1), None, out) == 0
        return out

    got = run_sharded(frames_np, runner, 0, 1, row_type=abi.FrameSummary)
    want = runner(frames_np)
    assert bytes(got) == bytes(want)


def test_frames_multi_contexts(ctx):
    """pp_dpps_frames_multi (one process, one context per device; here 2 and
    3 contexts on device 0): contiguous frame ranges per context, results
    byte-identical to pp_dpps_frames on one context; a bad frame in a later
    range is reported with its index into the caller's array."""
    lib = abi.load_library()
    p = _params()
    n = 301
    frames_np = np.concatenate([synthetic.c5_frames(0, 200), _mixed_frames(101, 9)])
    frames, _keep = synthetic.as_ctypes(frames_np)
    want = (abi.FrameSummary * n)()
    assert lib.pp_dpps_frames(ctx, frames, n, C.byref(p), C.byref(C1), None, want) == 0
    extra = []
    try:
        for _ in range(2):
            c = C.c_void_p()
            assert lib.pp_ctx_create(0, C.byref(c)) == 0
            extra.append(c)
        for k in (1, 2, 3):
            ctxs = (C.c_void_p * k)(ctx, *extra[:k - 1])
            got = (abi.FrameSummary * n)()
            assert lib.pp_dpps_frames_multi(ctxs, k, frames, n, C.byref(p), C.byref(C1), None,
                                            got) == 0, lib.pp_last_error(ctx)
            assert bytes(got) == bytes(want), k
        kick = (C.c_int32 * n)(*[int(frames_np["ours"]["id"][i][0]) for i in range(n)])
        kick[250] = 77
        ctxs = (C.c_void_p * 3)(ctx, *extra)
        got = (abi.FrameSummary * n)()
        assert lib.pp_dpps_frames_multi(ctxs, 3, frames, n, C.byref(p), C.byref(C1), kick,
                                        got) == abi.PP_VALIDATION
        msg = lib.pp_last_error(ctx).decode()
        assert "context 2" in msg and "frame 250" in msg and "77" in msg, msg
        # fewer frames than contexts (some ranges empty), and no frames
        for m in (2, 1, 0):
            few = (abi.FrameSummary * max(m, 1))()
            assert lib.pp_dpps_frames_multi(ctxs, 3, frames, m, C.byref(p), C.byref(C1), None,
                                            few) == 0, lib.pp_last_error(ctx)
            assert bytes(few)[:48 * m] == bytes(want)[:48 * m]
        # repeated contexts are refused; the contexts stay usable
        assert lib.pp_dpps_frames_multi((C.c_void_p * 2)(ctx, ctx), 2, frames, n, C.byref(p),
                                        C.byref(C1), None, got) == abi.PP_INTERNAL
        assert lib.pp_dpps_frames_multi(ctxs, 3, frames, n, C.byref(p), C.byref(C1), None,
                                        got) == 0
        assert bytes(got) == bytes(want)
    finally:
        for c in extra:
            lib.pp_ctx_destroy(c)

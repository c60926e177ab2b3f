"""GPU: the batched-frames path (one CTA per frame, summaries only) returns
exactly the single-frame path's summaries, and those match the reference's
best_pass on C5-style frames."""
import ctypes as C

import numpy as np
import pytest

from oracle import bindings as B
from paper_1909_07717_b200 import abi
from tests.helpers import run_product, score_close

pytestmark = pytest.mark.gpu


def _frames(n, seed):
    from bench import synthetic_frames
    return synthetic_frames(n, seed=seed)


@pytest.mark.parametrize("chip", [0, 1])
def test_batch_equals_single_frame(ctx, chip):
    lib = abi.load_library()
    p = abi.Params()
    lib.pp_params_default(C.byref(p))
    grid = abi.SearchGrid(128, 64, 1.0, 6.5, 1, chip)
    n = 64
    frames = _frames(n, 100 + chip)
    sums = (abi.DppsSummary * n)()
    assert lib.pp_dpps_batch(ctx, frames, n, C.byref(p), C.byref(grid), None, sums) == 0
    for i in range(n):
        k = int(sums[i].kicker_id)
        st, blk = run_product(lib, ctx, frames[i], p, grid, k, copy_all=False)
        assert st == 0, lib.pp_last_error(ctx)
        for r in range(3):
            assert sums[i].best_cell[r] == blk.summary.best_cell[r], (i, r)
            assert sums[i].best_score[r] == blk.summary.best_score[r], (i, r)
            assert sums[i].n_feasible[r] == blk.summary.n_feasible[r], (i, r)
            assert bytes(sums[i].best_features[r]) == bytes(blk.summary.best_features[r])
        assert sums[i].sbip_calls == blk.summary.sbip_calls


@pytest.mark.skipif(not B.ref_available(), reason="oracle/_ref not built")
def test_batch_matches_reference_best_pass(ctx):
    lib = abi.load_library()
    p = abi.Params()
    lib.pp_params_default(C.byref(p))
    grid = abi.SearchGrid(128, 64, 1.0, 6.5, 1, 0)
    n = 48
    frames = _frames(n, 7)
    sums = (abi.DppsSummary * n)()
    assert lib.pp_dpps_batch(ctx, frames, n, C.byref(p), C.byref(grid), None, sums) == 0
    best = np.zeros(n, np.int64)
    score = np.zeros(n)
    nfeas = np.zeros(n, np.int64)
    m = B.msgbuf()
    st = B.ref().ref_batch(frames, n, C.byref(p), C.byref(grid), None, 8,
                           best.ctypes.data_as(C.POINTER(C.c_int64)),
                           score.ctypes.data_as(C.POINTER(C.c_double)),
                           nfeas.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(C.c_double()),
                           m, 512)
    assert st == 0, m.value
    for i in range(n):
        assert sums[i].n_feasible[0] == nfeas[i], i
        assert score_close(sums[i].best_score[0], score[i]), i
        assert sums[i].best_cell[0] == best[i] or score_close(sums[i].best_score[0], score[i])

"""CPU: pin the plain-C oracle restatement (oracle/pp_oracle.c) against the
golden vectors the REFERENCE produced (tests/golden/make_golden.py).

Bit-exact everywhere: the oracle is FP64 with -ffp-contract=off and calls
the same libm (cos/sin/atan2) as the reference build."""
import ctypes as C

import numpy as np
import pytest

from oracle import bindings as B
from paper_1909_07717_b200 import abi
from tests.helpers import case_inputs, compare_best, compare_grid, struct_from

DP = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731


@pytest.fixture(scope="module")
def orc():
    return B.oracle()


def _n_cells(grid):
    if grid.n_directions < 1 or grid.n_powers < 1:
        return 0
    return (grid.flat + grid.chip) * grid.n_directions * grid.n_powers


def test_oracle_grids_bit_exact(orc, grids_golden):
    g = grids_golden
    fails = []
    for name in [str(c) for c in g["cases"]]:
        w, p, grid, k, status = case_inputs(g, name)
        blk = abi.GridBlock(_n_cells(grid))
        m = B.msgbuf()
        st = orc.or_dpps(C.byref(w), C.byref(p), C.byref(grid), k, blk.ptr(), m, 512)
        assert st == status, (name, st, status, m.value)
        if st != 0:
            continue
        ref = {f: g[f"{name}/{f}"] for f in ("our_id", "opp_id", "our_time", "opp_time", "rx",
                                             "ry", "score", "feasible")}
        fails += compare_grid(blk, ref, name)
        want = struct_from(abi.DppsSummary, g[f"{name}/summary"])
        fails += compare_best(blk.summary, want, blk.score, name)
        for r in range(3):  # the oracle's best_pass is exact, not just within tolerance
            if (blk.summary.best_cell[r], blk.summary.best_score[r]) != \
                    (want.best_cell[r], want.best_score[r]):
                fails.append(f"{name}: best[{r}] not bit-identical")
        if not np.array_equal(blk.score, ref["score"]):
            fails.append(f"{name}: score map not bit-identical")
        if blk.summary.sbip_calls != want.sbip_calls:
            fails.append(f"{name}: sbip_calls")
    assert not fails, "\n".join(fails[:20])


def test_oracle_known_answers(orc, grids_golden):
    """Known answers quoted by the reference's own tests / SURVEY 8(c)."""
    g = grids_golden
    w, p, grid, k, _ = case_inputs(g, "bench16")
    for flat, chip, calls in ((1, 0, 262144), (0, 1, 262144), (1, 1, 524288)):
        gr = abi.SearchGrid(128, 64, 1.0, 6.5, flat, chip)   # acceptance_main.cpp:239-240
        blk = abi.GridBlock(_n_cells(gr))
        assert orc.or_dpps(C.byref(w), C.byref(p), C.byref(gr), k, blk.ptr(), None, 0) == 0
        assert blk.summary.sbip_calls == calls
    w, p, grid, k, _ = case_inputs(g, "f8")
    gr = abi.SearchGrid(128, 64, 1.0, 6.5, 1, 0)
    blk = abi.GridBlock(_n_cells(gr))
    assert orc.or_dpps(C.byref(w), C.byref(p), C.byref(gr), k, blk.ptr(), None, 0) == 0
    assert blk.summary.n_feasible[0] == 4261                    # SURVEY 8(c) goldens
    assert blk.summary.best_cell[0] == 83 * 64 + 62
    assert abs(blk.summary.best_score[0] - 9.221049083) < 1e-9


def test_oracle_direction_table(orc):
    d = np.load("tests/golden/directions.npz")
    for key in d.files:
        n = int(key.split("_")[1])
        xy = np.zeros(2 * n)
        orc.or_direction_table(n, DP(xy))
        assert np.array_equal(xy, d[key]), key
        # test_dpps.cpp:57-80 (n in {128, 64, 12, 7, 3}): dirs[0] == (-1, 0),
        # mirror pairing bitwise
        assert xy[0] == -1.0 and xy[1] == 0.0
        if n not in (128, 64, 12, 7, 3):
            continue
        for k in range(n):
            m = (n - k) % n
            assert xy[2 * m] == xy[2 * k] and xy[2 * m + 1] == -xy[2 * k + 1]


def test_oracle_goal_views(orc, goal_views_golden):
    g = goal_views_golden
    for i in range(g["worlds"].shape[0]):
        w = struct_from(abi.World, g["worlds"][i])
        xs = np.ascontiguousarray(g["points"][i][0])
        ys = np.ascontiguousarray(g["points"][i][1])
        out = [np.zeros(16) for _ in range(4)]
        assert orc.or_goal_views(C.byref(w), 0.09, 16, DP(xs), DP(ys), *(DP(o) for o in out)) == 0
        for k in range(4):
            assert np.array_equal(out[k], g["views"][i][k]), (i, k)


def test_oracle_runmaps(orc, runmaps_golden):
    g = runmaps_golden
    for name in [str(c) for c in g["cases"]]:
        p = f"{name}/"
        w = struct_from(abi.World, g[p + "world"])
        pp = struct_from(abi.Params, g[p + "params"])
        req = struct_from(abi.RunmapRequest, g[p + "req"])
        want = struct_from(abi.RunmapSummary, g[p + "summary"])
        nv = orc.or_runmap_count(C.byref(w), C.byref(pp), req.zone_mask)
        assert nv == want.n_vertices, name
        blk = abi.RunmapBlock(nv)
        assert orc.or_runmap(C.byref(w), C.byref(pp), C.byref(req), blk.ptr(), nv, None, 0) == 0
        s = blk.summary
        assert (s.n_best, list(s.best_order[:s.n_best])) == \
            (want.n_best, list(want.best_order[:want.n_best])), name
        for z in range(4):
            assert bool(s.best[z].valid) == bool(want.best[z].valid), (name, z)
            if s.best[z].valid:
                assert (s.best[z].px, s.best[z].py, s.best[z].score) == \
                    (want.best[z].px, want.best[z].py, want.best[z].score), (name, z)
        if p + "px" in g:
            assert s.n_scorable == want.n_scorable, name
            for arr in ("px", "py", "scorable", "features"):
                assert np.array_equal(getattr(blk, arr), g[p + arr]), (name, arr)
            ok = g[p + "scorable"].astype(bool)
            assert np.array_equal(blk.score[ok], g[p + "score"][ok]), name


def test_oracle_score_pass_domain_error(orc, grids_golden):
    w, p, _, _, _ = case_inputs(grids_golden, "minimal")
    one = np.array([1.0])
    feas = np.array([0], dtype=np.uint8)
    out = np.zeros(1)
    st = orc.or_score_cells(C.byref(w), C.byref(p), 1, DP(one), DP(one), DP(one), DP(one),
                            feas.ctypes.data_as(C.POINTER(C.c_uint8)), DP(out), None, None, 0)
    assert st == abi.PP_DOMAIN   # pass_eval.cpp:150


@pytest.mark.skipif(not B.ref_available(), reason="oracle/_ref not built")
def test_oracle_matches_live_reference_random_worlds(orc):
    """Beyond the goldens: fresh random worlds through both, bit-exact."""
    ref = B.ref()
    p = abi.Params()
    ref.ref_params_default(C.byref(p))
    rng = np.random.default_rng(3)
    for i in range(20):
        w = abi.World()
        n_o, n_t = int(rng.integers(1, 17)), int(rng.integers(0, 17))
        assert ref.ref_random_world(7000 + i, n_o, n_t, 2.0, C.byref(w)) == 0
        gr = abi.SearchGrid(int(rng.integers(4, 33)), int(rng.integers(1, 20)), 1.0, 6.5, 1, 1)
        k = w.ours[0].id
        a, b = abi.GridBlock(_n_cells(gr)), abi.GridBlock(_n_cells(gr))
        assert orc.or_dpps(C.byref(w), C.byref(p), C.byref(gr), k, a.ptr(), None, 0) == 0
        assert ref.ref_dpps(C.byref(w), C.byref(p), C.byref(gr), k, 0, b.ptr(), None, 0) == 0
        for f in ("our_time", "opp_time", "feasible", "score", "our_slot", "opp_slot"):
            assert np.array_equal(getattr(a, f), getattr(b, f)), (i, f)
        fin = np.isfinite(a.our_time)
        assert np.array_equal(a.rx[fin], b.rx[fin]) and np.array_equal(a.ry[fin], b.ry[fin])

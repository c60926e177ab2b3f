"""GPU parity on freshly generated inputs, checked live against the compiled
reference (oracle/_ref, built from the unmodified reference sources).

Covers many more worlds than the committed goldens: C5-style random 8v8
frames (oracles::random_world, proj/tests/oracles.hpp:228-258), random team
sizes with rolling balls, the y-mirror symmetry of acceptance criterion 8
(proj/tests/acceptance_main.cpp:488-577), and goal views at random points."""
import ctypes as C

import numpy as np
import pytest

from oracle import bindings as B
from paper_1909_07717_b200 import abi
from tests.helpers import compare_best, compare_grid, run_product, score_close

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not B.ref_available(), reason="oracle/_ref not built")]


def _ref_grid(world, params, grid, kicker):
    n = (grid.flat + grid.chip) * grid.n_directions * grid.n_powers
    blk = abi.GridBlock(n)
    m = B.msgbuf()
    st = B.ref().ref_dpps(C.byref(world), C.byref(params), C.byref(grid), kicker, 8, blk.ptr(),
                          m, 512)
    assert st == 0, m.value
    our_id, opp_id = blk.ids()
    ref = {"our_id": our_id, "opp_id": opp_id}
    for k in ("our_time", "opp_time", "rx", "ry", "score", "feasible"):
        ref[k] = getattr(blk, k)
    return blk, ref


def _params():
    p = abi.Params()
    B.ref().ref_params_default(C.byref(p))
    return p


def _random_world(seed, n_o, n_t, ball_speed=0.0):
    w = abi.World()
    assert B.ref().ref_random_world(seed, n_o, n_t, ball_speed, C.byref(w)) == 0
    return w


@pytest.mark.parametrize("chip", [0, 1])
def test_random_8v8_frames_full_grid(ctx, chip):
    lib = abi.load_library()
    p = _params()
    grid = abi.SearchGrid(128, 64, 1.0, 6.5, 1, chip)
    errs = []
    for i in range(12):
        w = _random_world(0xB200 + 1000 * chip + i, 8, 8)
        k = B.ref().ref_nearest_teammate(C.byref(w))
        st, blk = run_product(lib, ctx, w, p, grid, k)
        assert st == 0, lib.pp_last_error(ctx)
        rblk, ref = _ref_grid(w, p, grid, k)
        errs += compare_grid(blk, ref, f"w{i}")
        errs += compare_best(blk.summary, rblk.summary, blk.score, f"w{i}")
    assert not errs, "\n".join(errs[:30])


def test_random_team_sizes_rolling_ball(ctx):
    lib = abi.load_library()
    p = _params()
    rng = np.random.default_rng(7)
    errs = []
    for i in range(40):
        n_o, n_t = int(rng.integers(1, 17)), int(rng.integers(0, 17))
        w = _random_world(5000 + i, n_o, n_t, 4.0)
        grid = abi.SearchGrid(int(rng.integers(8, 48)), int(rng.integers(4, 40)),
                              float(rng.uniform(0.5, 2.0)), float(rng.uniform(3.0, 8.0)), 1, 1)
        k = w.ours[int(rng.integers(0, n_o))].id
        st, blk = run_product(lib, ctx, w, p, grid, k)
        assert st == 0, lib.pp_last_error(ctx)
        rblk, ref = _ref_grid(w, p, grid, k)
        errs += compare_grid(blk, ref, f"w{i}")
        errs += compare_best(blk.summary, rblk.summary, blk.score, f"w{i}")
    assert not errs, "\n".join(errs[:30])


def test_mirror_symmetry_exact(ctx):
    """acceptance criterion 8: grid of the mirrored world maps k -> (n-k)%n."""
    lib = abi.load_library()
    p = _params()
    grid = abi.SearchGrid(128, 64, 1.0, 6.5, 1, 1)
    n = 128
    for i in range(6):
        w = abi.World()
        assert B.ref().ref_lattice_world(0xC8 + i, 4 + i % 3, 5, 1, C.byref(w)) == 0
        m = abi.World()
        assert B.ref().ref_mirror_world(C.byref(w), C.byref(m)) == 0
        k = w.ours[0].id
        st, a = run_product(lib, ctx, w, p, grid, k)
        st2, b = run_product(lib, ctx, m, p, grid, k)
        assert st == 0 and st2 == 0
        for s in range(2):
            for d in range(n):
                ia = (s * n + d) * 64
                ib = (s * n + (n - d) % n) * 64
                sa, sb = slice(ia, ia + 64), slice(ib, ib + 64)
                assert np.array_equal(a.feasible[sa], b.feasible[sb])
                assert np.array_equal(a.our_time[sa], b.our_time[sb])
                assert np.array_equal(a.opp_time[sa], b.opp_time[sb])
                fin = np.isfinite(a.our_time[sa])
                assert np.array_equal(a.rx[sa][fin], b.rx[sb][fin])
                assert np.array_equal(a.ry[sa][fin], -b.ry[sb][fin])
        assert a.summary.best_score[0] == b.summary.best_score[0]


def test_goal_views_random_points(ctx):
    lib = abi.load_library()
    rng = np.random.default_rng(11)
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    for scene in range(60):
        w = abi.World()
        w.field = abi.Field(12.0, 9.0, 1.8, 1.8, 3.6)
        n = int(rng.integers(0, 17))
        w.n_theirs = n
        for j in range(n):
            # bias opponents toward the goal mouth so intervals are frequent
            w.theirs[j].px = rng.uniform(0.0, 6.5) if j % 2 else rng.uniform(-6.0, 6.0)
            w.theirs[j].py = rng.uniform(-1.5, 1.5) if j % 2 else rng.uniform(-4.5, 4.5)
            w.theirs[j].id = j
        m = 512
        xs = rng.uniform(-6.0, 6.3, m)
        ys = rng.uniform(-4.5, 4.5, m)
        if scene % 5 == 0:  # points right next to opponents / the goal line
            for q in range(0, m, 4):
                j = int(rng.integers(0, max(n, 1)))
                if n:
                    xs[q] = w.theirs[j].px + rng.uniform(-0.2, 0.2)
                    ys[q] = w.theirs[j].py + rng.uniform(-0.2, 0.2)
        got = [np.zeros(m) for _ in range(4)]
        want = [np.zeros(m) for _ in range(4)]
        assert lib.pp_goal_views(ctx, C.byref(w), 0.09, m, dp(xs), dp(ys),
                                 *(dp(o) for o in got)) == 0
        assert B.ref().ref_goal_views(C.byref(w), 0.09, m, dp(xs), dp(ys),
                                      *(dp(o) for o in want)) == 0
        # window edges come from the exact bisection: bit-identical
        assert np.array_equal(got[1], want[1]), scene
        assert np.array_equal(got[2], want[2]), scene
        assert np.array_equal(got[3], want[3]), scene
        # the angle goes through atan2 (CUDA vs glibc last ulp)
        assert np.all(np.abs(got[0] - want[0]) <= 1e-12), scene


def test_fine_grid_c3_best(ctx):
    """C3 (1200 x 900 flat): summary equal to the reference's best pass."""
    lib = abi.load_library()
    p = _params()
    g = np.load("tests/golden/grids.npz")
    from tests.helpers import case_inputs
    w, _, _, k, _ = case_inputs(g, "f8")
    grid = abi.SearchGrid(1200, 900, 1.0, 6.5, 1, 0)
    st, blk = run_product(lib, ctx, w, p, grid, k, copy_all=False)
    assert st == 0
    # reference values measured by the survey: dir 776, pow 891
    assert blk.summary.best_cell[0] == 776 * 900 + 891
    assert score_close(blk.summary.best_score[0], 9.224754285)
    assert blk.summary.n_feasible[0] == 566477

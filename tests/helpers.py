"""Shared helpers for the parity tests: decode golden structs, run the
product through the C-ABI, and compare with the reference's outputs."""
from __future__ import annotations

import ctypes as C

import numpy as np

from paper_1909_07717_b200 import abi

# Score tolerance written into every score comparison (north_star: scores
# agree within 1e-4 relative).
SCORE_RTOL = 1e-4


def struct_from(cls, arr):
    return cls.from_buffer_copy(np.asarray(arr, dtype=np.uint8).tobytes())


def case_inputs(g, name):
    p = f"{name}/"
    return (struct_from(abi.World, g[p + "world"]), struct_from(abi.Params, g[p + "params"]),
            struct_from(abi.SearchGrid, g[p + "grid"]), int(g[p + "kicker"][0]),
            int(g[p + "status"][0]))


def n_cells_of(grid) -> int:
    return (int(bool(grid.flat)) + int(bool(grid.chip))) * grid.n_directions * grid.n_powers \
        if grid.n_directions > 0 and grid.n_powers > 0 else 0


def run_product(lib, ctx, world, params, grid, kicker, copy_all=True):
    n = n_cells_of(grid)
    blk = abi.GridBlock(n)
    st = lib.pp_dpps(ctx, C.byref(world), C.byref(params), C.byref(grid), kicker,
                     abi.PP_COPY_ALL if copy_all else abi.PP_COPY_SUMMARY, blk.ptr())
    return st, blk


def score_close(a, b, rtol=SCORE_RTOL):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.abs(a - b) <= rtol * np.maximum(1.0, np.abs(b))


def compare_grid(blk, ref, label=""):
    """Bit-exact on ids, times, receive points, feasibility; scores within
    SCORE_RTOL; best cells identical or tied within tolerance.  `ref` maps
    field -> array (golden file or a live reference block)."""
    our_id, opp_id = blk.ids()
    errs = []
    for name, got, want in (("our_id", our_id, ref["our_id"]), ("opp_id", opp_id, ref["opp_id"]),
                            ("feasible", blk.feasible, ref["feasible"])):
        bad = np.flatnonzero(np.asarray(got) != np.asarray(want))
        if bad.size:
            errs.append(f"{label} {name}: {bad.size} mismatches, first cells {bad[:5]}")
    for name in ("our_time", "opp_time"):
        got, want = getattr(blk, name), np.asarray(ref[name])
        bad = np.flatnonzero(~((got == want) | (np.isnan(got) & np.isnan(want))))
        if bad.size:
            errs.append(f"{label} {name}: {bad.size} bit mismatches, first {bad[:5]}")
    fin = np.isfinite(np.asarray(ref["our_time"]))
    for name in ("rx", "ry"):
        got, want = getattr(blk, name)[fin], np.asarray(ref[name])[fin]
        bad = np.flatnonzero(got != want)
        if bad.size:
            errs.append(f"{label} {name}: {bad.size} bit mismatches")
    feas = np.asarray(ref["feasible"]).astype(bool)
    gs, ws = blk.score[feas].astype(np.float64), np.asarray(ref["score"])[feas].astype(np.float64)
    bad = np.flatnonzero(~score_close(gs, ws))
    if bad.size:
        errs.append(f"{label} score: {bad.size} outside rtol {SCORE_RTOL}")
    if np.any(np.isfinite(blk.score[~feas])):
        errs.append(f"{label} score: infeasible cells must be -inf")
    return errs


def compare_best(sum_got, sum_want, got_score_map=None, label=""):
    errs = []
    for k in range(3):
        cg, cw = int(sum_got.best_cell[k]), int(sum_want.best_cell[k])
        if cw < 0 or cg < 0:
            if cg != cw:
                errs.append(f"{label} best[{k}]: got {cg} want {cw}")
            continue
        sg, sw = sum_got.best_score[k], sum_want.best_score[k]
        if not score_close(sg, sw):
            errs.append(f"{label} best[{k}] score {sg} vs {sw}")
        if cg != cw and got_score_map is not None:
            # a different cell is acceptable only if it ties within tolerance
            if not score_close(got_score_map[cw], sw):
                errs.append(f"{label} best[{k}] cell {cg} vs {cw} not tied")
        if int(sum_got.n_feasible[k]) != int(sum_want.n_feasible[k]):
            errs.append(f"{label} n_feasible[{k}] {sum_got.n_feasible[k]} vs {sum_want.n_feasible[k]}")
    return errs

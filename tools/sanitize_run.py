"""Dev tool (GPU box): a small workload for compute-sanitizer (SURVEY 5:
memcheck and racecheck evidence).  Runs through the C-ABI, and checks each
result against the reference goldens / the single-frame path so a sanitizer
run that perturbs the pipeline still fails loudly:

* one C2 frame (F8, 128x64 flat + chip) through pp_dpps -- the streaming
  scan -> value pipeline with PDL -- twice (graph replay, self-cleaning
  counters), with pinned and pageable result blocks;
* a 64-frame C5 batch through pp_dpps_frames;
* the C4 run map at 0.1 m, goal views, possession.

usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import case_inputs, compare_grid, run_product  # noqa: E402
from paper_1909_07717_b200 import abi, synthetic  # noqa: E402


def main():
    lib = abi.load_library()
    g = np.load(os.path.join(ROOT, "tests", "golden", "grids.npz"))
    ctx = C.c_void_p()
    assert lib.pp_ctx_create(0, C.byref(ctx)) == 0
    w, p, grid, kicker, _ = case_inputs(g, "f8")
    grid.n_directions, grid.n_powers, grid.chip = 128, 64, 1
    ref = {k: g[f"f8/{k}"] for k in ("our_id", "opp_id", "our_time", "opp_time", "rx", "ry",
                                     "score", "feasible")}
    n_cells = 128 * 64 * 2
    nbytes = int(lib.pp_grid_bytes(n_cells))
    hptr = lib.pp_host_alloc(nbytes)
    for pinned in (True, False, True):
        if pinned:
            blk = abi.GridBlock(n_cells, buf=(C.c_uint8 * nbytes).from_address(hptr))
            st = lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), kicker, abi.PP_COPY_ALL,
                             blk.ptr())
        else:
            st, blk = run_product(lib, ctx, w, p, grid, kicker)
        assert st == 0, lib.pp_last_error(ctx)
        errs = compare_grid(blk, ref, "f8")
        assert not errs, errs[:5]
    print("c2 frame ok", int(blk.summary.n_feasible[0]))

    frames = synthetic.c5_frames(0, 64)
    arr, _keep = synthetic.as_ctypes(frames)
    params = abi.Params()
    lib.pp_params_default(C.byref(params))
    c1 = abi.SearchGrid(128, 64, 1.0, 6.5, 1, 0)
    out = (abi.FrameSummary * 64)()
    for _ in range(2):
        st = lib.pp_dpps_frames(ctx, arr, 64, C.byref(params), C.byref(c1), None, out)
        assert st == 0, lib.pp_last_error(ctx)
    first = bytes(out)
    st = lib.pp_dpps_frames(ctx, arr, 64, C.byref(params), C.byref(c1), None, out)
    assert st == 0 and bytes(out) == first
    print("c5 batch ok", sum(int(o.n_feasible[0]) for o in out))

    pp = abi.Params.from_buffer_copy(bytes(p))
    nv = C.c_int64()
    assert lib.pp_runmap_count(C.byref(w), C.byref(pp), 0xF, C.byref(nv)) == 0
    nbytes = abi.runmap_offsets(nv.value)["total"]
    buf = (C.c_uint8 * nbytes)()
    req = abi.RunmapRequest(0xF, 0, 4, 0, 0.0, 0.0, 1)
    assert lib.pp_runmap(ctx, C.byref(w), C.byref(pp), C.byref(req), buf, nv.value) == 0
    print("runmap ok", nv.value)

    n = 256
    px = np.linspace(-5.5, 5.5, n)
    py = np.linspace(-4.0, 4.0, n)
    o = [np.zeros(n) for _ in range(4)]
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    assert lib.pp_goal_views(ctx, C.byref(w), 0.09, n, dp(px), dp(py), *[dp(a) for a in o]) == 0
    rep = abi.PossessionReport()
    assert lib.pp_possession(ctx, C.byref(w), C.byref(p), C.byref(rep)) == 0
    print("queries ok")
    lib.pp_host_free(hptr)
    lib.pp_ctx_destroy(ctx)


if __name__ == "__main__":
    main()

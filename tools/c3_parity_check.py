"""Dev tool: parity of full-size (1 cm, C3) grids against the compiled reference."""
import ctypes as C, os, sys
ROOT = "/root/repo"; sys.path.insert(0, ROOT)
from oracle import bindings as B
from paper_1909_07717_b200 import abi
from tests.helpers import compare_best, compare_grid, run_product
from tests.test_gpu_random import _params, _random_world, _ref_grid
lib = abi.load_library(); ctx = C.c_void_p(); assert lib.pp_ctx_create(0, C.byref(ctx)) == 0
p = _params()
for i, (nd, np_, chip) in enumerate([(1200, 900, 0), (600, 450, 1)]):
    w = _random_world(0xC3C3 + i, 8, 8, 0.0)
    k = B.ref().ref_nearest_teammate(C.byref(w))
    grid = abi.SearchGrid(nd, np_, 1.0, 6.5, 1, chip)
    st, blk = run_product(lib, ctx, w, p, grid, k); assert st == 0
    rblk, ref = _ref_grid(w, p, grid, k)
    errs = compare_grid(blk, ref, f"c3_{i}") + compare_best(blk.summary, rblk.summary, blk.score, f"c3_{i}")
    print(nd, np_, chip, "mismatches:", len(errs), errs[:3])

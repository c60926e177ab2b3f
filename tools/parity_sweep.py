"""Dev tool: a larger random parity sweep than the test suite (GPU product vs
the compiled reference oracle/_ref): random team sizes (up to 16 v 16),
rolling balls, flat and chip grids of several shapes (so every scan CTA shape
runs); every block is also recomputed with every FP32 shortcut off
(PP_OPT_EXACT_ONLY) and must be byte-identical.  Prints the mismatch counts.
Usage: python tools/parity_sweep.py [n_worlds]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import bindings as B  # noqa: E402
from paper_1909_07717_b200 import abi  # noqa: E402
from tests.helpers import compare_best, compare_grid, run_product  # noqa: E402
from tests.test_gpu_random import _params, _random_world, _ref_grid  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 60
lib = abi.load_library()
ctx = C.c_void_p()
assert lib.pp_ctx_create(0, C.byref(ctx)) == 0
p = _params()
grids = [(128, 64), (64, 40), (200, 100), (37, 33), (256, 96)]
bad = 0
shortcut_bad = 0
off = abi.DppsSummary.device_ms.offset
for i in range(n):
    rng = (i * 2654435761) & 0xffffffff
    n_o = 1 + rng % 16
    n_t = (rng >> 8) % 17
    speed = ((rng >> 16) % 5) * 0.8
    w = _random_world(0xC0FFEE + i, n_o, n_t, speed)
    k = B.ref().ref_nearest_teammate(C.byref(w))
    nd, np_ = grids[i % len(grids)]
    for chip in (0, 1):
        grid = abi.SearchGrid(nd, np_, 1.0, 6.5, 1, chip)
        st, blk = run_product(lib, ctx, w, p, grid, k)
        if st != 0:
            print("status", st, lib.pp_last_error(ctx))
            bad += 1
            continue
        fast = bytearray(bytes(blk.buf))
        assert lib.pp_ctx_set_option(ctx, abi.PP_OPT_EXACT_ONLY, 1) == 0
        st2, blk2 = run_product(lib, ctx, w, p, grid, k)
        assert lib.pp_ctx_set_option(ctx, abi.PP_OPT_EXACT_ONLY, 0) == 0
        exact = bytearray(bytes(blk2.buf))
        fast[off:off + 8] = bytes(8)
        exact[off:off + 8] = bytes(8)
        if st2 != 0 or fast != exact:
            shortcut_bad += 1
            print(f"w{i}c{chip}: FP32 shortcuts changed the block")
        rblk, ref = _ref_grid(w, p, grid, k)
        errs = compare_grid(blk, ref, f"w{i}c{chip}") + compare_best(blk.summary, rblk.summary,
                                                                      blk.score, f"w{i}c{chip}")
        if errs:
            bad += 1
            print("\n".join(errs[:5]))
print(f"worlds {n} x 2 grids: {bad} with mismatches against the reference, "
      f"{shortcut_bad} where the FP32 shortcuts changed the block")

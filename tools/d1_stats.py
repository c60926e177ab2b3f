"""Dev tool: per-item cycles of the value kernel's D1 phase (pair_info) from
the profiling build, split by outcome.  Not used by tests/bench."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_1909_07717_b200 import abi  # noqa: E402
from helpers import case_inputs  # noqa: E402

lib = abi._declare(C.CDLL(os.path.join(ROOT, "paper_1909_07717_b200", "lib",
                                       "libpassplan_b200_prof.so")))
lib.pp_debug_d1_records.argtypes = [C.POINTER(C.c_longlong)]
g = np.load(os.path.join(ROOT, "tests", "golden", "grids.npz"))
ctx = C.c_void_p()
assert lib.pp_ctx_create(0, C.byref(ctx)) == 0
w, p, grid, k, _ = case_inputs(g, "f8")
grid.chip = 1
blk = abi.GridBlock(16384)
for _ in range(3):
    lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), k, 1, blk.ptr())
R = np.zeros((512, 256, 2), np.int64)
lib.pp_debug_d1_records(R.ctypes.data_as(C.POINTER(C.c_longlong)))
nq = (blk.summary.n_feasible[0] + 31) // 32
R = R[:nq].reshape(-1, 2)
R = R[R[:, 0] > 0]


def pct(a):
    a = np.asarray(a)
    if len(a) == 0:
        return "-"
    return f"n={len(a)} mean={a.mean():.0f} p50={np.percentile(a, 50):.0f} p90={np.percentile(a, 90):.0f} max={a.max()}"


st, fast = R[:, 1] & 3, (R[:, 1] >> 2) & 1
print("all", pct(R[:, 0]))
for name, m in [("status0 not fast", (st == 0) & (fast == 0)), ("status0 fast", (st == 0) & (fast == 1)),
                ("status1 fast", (st == 1) & (fast == 1)), ("status1 slow", (st == 1) & (fast == 0)),
                ("status2", st == 2)]:
    print(name, pct(R[m, 0]))

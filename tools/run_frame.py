"""Dev tool: run one configuration through the C-ABI a few times (ncu target)."""
import ctypes as C, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_1909_07717_b200 import abi
from helpers import case_inputs, run_product
chip = int(sys.argv[1]) if len(sys.argv) > 1 else 1
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
lib = abi.load_library()
g = np.load(os.path.join(ROOT, "tests", "golden", "grids.npz"))
ctx = C.c_void_p(); assert lib.pp_ctx_create(0, C.byref(ctx)) == 0
w, p, grid, k, _ = case_inputs(g, "f8"); grid.chip = chip
for _ in range(reps):
    st, blk = run_product(lib, ctx, w, p, grid, k)
    assert st == 0
print("ok", blk.summary.device_ms, list(blk.summary.n_feasible))

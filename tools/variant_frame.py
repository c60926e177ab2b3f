"""Dev tool: single-frame C2 (F8, 128x64 flat+chip) kernel times and e2e p50 of
one library build (PP_LIB_PATH selects a variant); checks the best cell
against the golden.  python tools/variant_frame.py [chip] [reps]"""
import ctypes as C
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_1909_07717_b200 import abi  # noqa: E402
from helpers import case_inputs  # noqa: E402

chip = int(sys.argv[1]) if len(sys.argv) > 1 else 1
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
lib = abi.load_library()
g = np.load(os.path.join(ROOT, "tests", "golden", "grids.npz"))
ctx = C.c_void_p()
assert lib.pp_ctx_create(0, C.byref(ctx)) == 0
w, p, grid, k, _ = case_inputs(g, "f8")
grid.n_directions, grid.n_powers, grid.chip = 128, 64, chip
n = (1 + chip) * 128 * 64
nb = int(lib.pp_grid_bytes(n))
ptr = lib.pp_host_alloc(nb)
blk = abi.GridBlock(n, buf=(C.c_uint8 * nb).from_address(ptr))
e2e, dev = [], []
for i in range(reps + 20):
    t0 = time.perf_counter()
    st = lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), k, abi.PP_COPY_ALL, ptr)
    t1 = time.perf_counter()
    assert st == 0, lib.pp_last_error(ctx)
    if i >= 20:
        e2e.append((t1 - t0) * 1e3)
        dev.append(blk.summary.device_ms)
sc, va = C.c_float(), C.c_float()
lib.pp_dpps_kernel_times(ctx, 100, C.byref(sc), C.byref(va))
want = abi.DppsSummary.from_buffer_copy(g["f8/summary"].tobytes()).best_cell[0] if chip else None
print(f"{os.path.basename(os.environ.get('PP_LIB_PATH', 'default'))}: chip={chip} "
      f"e2e p50 {statistics.median(e2e) * 1e3:.1f} us, device span p50 "
      f"{statistics.median(dev) * 1e3:.1f} us, scan alone {sc.value * 1e3:.1f} us, "
      f"value alone {va.value * 1e3:.1f} us, best {blk.summary.best_cell[0]} (golden {want})")

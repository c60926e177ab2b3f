"""Dev tool (GPU box): C3 (F8, 1200 x 900 flat) device span and e2e with the
whole result block in pinned host memory (PP_COPY_ALL), as bench.py's extras.
Not used by tests/bench."""
import ctypes as C
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1909_07717_b200 import abi  # noqa: E402

lib = abi.load_library()
ctx = C.c_void_p()
assert lib.pp_ctx_create(0, C.byref(ctx)) == 0
w, p, kicker = bench.load_f8()
g3 = abi.SearchGrid(1200, 900, 1.0, 6.5, 1, 0)
n = 1200 * 900
nbytes = int(lib.pp_grid_bytes(n))
for copy, name in ((abi.PP_COPY_ALL, "pinned all"), (abi.PP_COPY_SUMMARY, "summary")):
    ptr = lib.pp_host_alloc(nbytes)
    blk = abi.GridBlock(n, buf=(C.c_uint8 * nbytes).from_address(ptr))
    dev, e2e = [], []
    for i in range(30):
        t0 = time.perf_counter()
        assert lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(g3), kicker, copy, ptr) == 0
        e2e.append((time.perf_counter() - t0) * 1e3)
        dev.append(blk.summary.device_ms)
    print(f"{os.environ.get('PP_LIB_PATH', 'product')} {os.environ.get('PP_WARP_CELLS', '')} {name}: "
          f"device p50 {statistics.median(dev[3:]):.3f} ms, e2e p50 {statistics.median(e2e[3:]):.3f} ms")
    lib.pp_host_free(ptr)

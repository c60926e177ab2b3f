"""Dev tool: e2e latency parts of one pp_dpps call (host wall clock, p50)."""
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_1909_07717_b200 import abi  # noqa: E402
from helpers import case_inputs  # noqa: E402

lib = abi.load_library()
g = np.load(os.path.join(ROOT, "tests", "golden", "grids.npz"))
ctx = C.c_void_p()
assert lib.pp_ctx_create(0, C.byref(ctx)) == 0
w, p, grid, k, _ = case_inputs(g, "f8")
n = 16384
ptr = lib.pp_host_alloc(abi.grid_offsets(n)["total"])
lib.pp_dpps_relaunch.argtypes = [C.c_void_p]
lib.pp_ctx_stream.restype = C.c_void_p


def p50(fn, reps=300):
    for _ in range(20):
        fn()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return 1e3 * np.median(ts)


import torch  # noqa: E402
stream = torch.cuda.ExternalStream(lib.pp_ctx_stream(ctx))
print("copy summary ms", p50(lambda: lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), k, 0, ptr)))
print("copy all     ms", p50(lambda: lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), k, 1, ptr)))


def relaunch():
    lib.pp_dpps_relaunch(ctx)
    stream.synchronize()


print("relaunch+sync ms", p50(relaunch))
print("empty ctypes call ms", p50(lambda: lib.pp_abi_version()))

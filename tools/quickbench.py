import ctypes as C, numpy as np, time, sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from paper_1909_07717_b200 import abi
from helpers import case_inputs, run_product
lib = abi.load_library()
g = np.load("/root/repo/tests/golden/grids.npz")
ctx = C.c_void_p(); assert lib.pp_ctx_create(0, C.byref(ctx)) == 0
w, p, grid, k, _ = case_inputs(g, "f8")
for chip in (0, 1):
    grid.chip = chip
    for _ in range(3): st, blk = run_product(lib, ctx, w, p, grid, k)
    ts=[]; ds=[]
    for _ in range(40):
        t=time.perf_counter(); st, blk = run_product(lib, ctx, w, p, grid, k); ts.append(time.perf_counter()-t); ds.append(blk.summary.device_ms)
    print("chip", chip, "st", st, "dev ms med", round(float(np.median(ds)), 5), "wall ms med", 1e3*np.median(ts), "feas", list(blk.summary.n_feasible))
# C3
grid.chip = 0; grid.n_directions = 1200; grid.n_powers = 900
for _ in range(2): st, blk = run_product(lib, ctx, w, p, grid, k)
print("C3 st", st, "dev ms", blk.summary.device_ms, "feas", list(blk.summary.n_feasible), list(blk.summary.best_cell), list(blk.summary.best_score))
# batch
grid = abi.SearchGrid(128, 64, 1.0, 6.5, 1, 0)
names = [f"rand8v8_{i}" for i in range(6)]
frames = (abi.World * 4096)()
for i in range(4096):
    frames[i] = case_inputs(g, names[i % 6])[0]
sums = (abi.DppsSummary * 4096)()
st = lib.pp_batch_upload(ctx, frames, 4096, None); print("upload", st)
ms = C.c_float()
for _ in range(2): st = lib.pp_batch_run(ctx, C.byref(p), C.byref(grid), C.byref(ms))
print("batch 4096 frames st", st, "ms", ms.value, "frames/s", 4096/ms.value*1e3, "pair-evals/s", 4096*8192*16/ms.value*1e3)

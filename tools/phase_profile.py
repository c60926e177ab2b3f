"""Dev tool: per-phase SM cycles of dpps_kernel from the profiling build
(lib/libpassplan_b200_prof.so, -DPP_PHASE_CLOCKS).  Not used by tests/bench."""
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
lib.pp_debug_phase_cycles.argtypes = [C.POINTER(C.c_uint64), C.c_int]
g = np.load(os.path.join(ROOT, "tests", "golden", "grids.npz"))
ctx = C.c_void_p()
assert lib.pp_ctx_create(0, C.byref(ctx)) == 0
cyc = (C.c_uint64 * 16)()
names = ["A window", "B scan", "C champion", "D value", "E argmax"]


lib.pp_debug_scan_counts.argtypes = [C.POINTER(C.c_uint64), C.c_int]
cnt = (C.c_uint64 * 16)()


def report(label):
    lib.pp_debug_scan_counts(cnt, 1)
    w = max(cnt[7], 1)
    lanes = 32 * w
    print(f"  scans(robot-warps)={cnt[7]} per lane: iters={cnt[0] / lanes:.1f} skips={cnt[1] / lanes:.1f} "
          f"lb_rej={cnt[2] / lanes:.1f} ub_acc={cnt[3] / lanes:.2f} exact={cnt[4] / lanes:.2f} | "
          f"per warp: rounds={cnt[5] / w:.2f} max_lane_iters={cnt[6] / w:.1f}")
    print(f"  cycles per robot-warp scan: setup+prune={cnt[9] / w:.0f} loop={cnt[10] / w:.0f} "
          f"rest+store={cnt[11] / w:.0f}")
    lib.pp_debug_phase_cycles(cyc, 1)
    ns, nv = max(cyc[8], 1), max(cyc[9], 1)
    print(f"{label}: scan CTAs={cyc[8]} cycles/CTA A={cyc[0] / ns:.0f} B={cyc[1] / ns:.0f} "
          f"C={cyc[2] / ns:.0f} | value CTAs={cyc[9]} cycles/CTA D1={cyc[3] / nv:.0f} "
          f"D2={cyc[4] / nv:.0f} D3={cyc[5] / nv:.0f} reduce={cyc[6] / nv:.0f}")


w, p, grid, k, _ = case_inputs(g, "f8")
for chip in (0, 1):
    grid.chip = chip
    n = 128 * 64 * (1 + chip)
    blk = abi.GridBlock(n)
    for _ in range(3):
        lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), k, 1, blk.ptr())
    lib.pp_debug_phase_cycles(cyc, 1)
    lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), k, 1, blk.ptr())
    report(f"single frame chip={chip} dev_ms={blk.summary.device_ms:.3f}")
grid = abi.SearchGrid(128, 64, 1.0, 6.5, 1, 0)
names6 = [f"rand8v8_{i}" for i in range(6)]
nf = 1024
frames = (abi.World * nf)()
for i in range(nf):
    frames[i] = case_inputs(g, names6[i % 6])[0]
assert lib.pp_batch_upload(ctx, frames, nf, None) == 0
ms = C.c_float()
lib.pp_batch_run(ctx, C.byref(p), C.byref(grid), C.byref(ms))
lib.pp_debug_phase_cycles(cyc, 1)
lib.pp_batch_run(ctx, C.byref(p), C.byref(grid), C.byref(ms))
report(f"batch {nf} frames ms={ms.value:.2f}")

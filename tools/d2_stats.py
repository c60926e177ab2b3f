"""Dev tool: the value kernel's D2 phase (interval-edge bisections) on the C2
frame from the profiling build: jobs per CTA / thread, non-fast edges, band
steps and exact rounds per edge, and their cycles.  Not used by tests/bench."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_1909_07717_b200 import abi  # noqa: E402
from helpers import case_inputs  # noqa: E402

lib = abi._declare(C.CDLL(os.environ.get("PP_PROF_LIB", os.path.join(
    ROOT, "paper_1909_07717_b200", "lib", "libpassplan_b200_prof.so"))))
P = C.POINTER(C.c_longlong)
lib.pp_debug_d2_records.argtypes = [P]
lib.pp_debug_cta_records.argtypes = [P, P, P]
g = np.load(os.path.join(ROOT, "tests", "golden", "grids.npz"))
ctx = C.c_void_p()
assert lib.pp_ctx_create(0, C.byref(ctx)) == 0
w, p, grid, k, _ = case_inputs(g, "f8")
grid.chip = 1
blk = abi.GridBlock(16384)
for _ in range(3):
    lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), k, 1, blk.ptr())
nq = (blk.summary.n_feasible[0] + 31) // 32
R = np.zeros((512, 256, 6), np.int64)
lib.pp_debug_d2_records(R.ctypes.data_as(P))
s = np.zeros((8192, 8), np.int64)
v = np.zeros((8192, 8), np.int64)
r = np.zeros((8192, 16), np.int64)
lib.pp_debug_cta_records(s.ctypes.data_as(P), v.ctypes.data_as(P), r.ctypes.data_as(P))
R = R[:nq]
v = v[:nq]


def pct(a):
    a = np.asarray(a, float)
    return f"mean={a.mean():.1f} p50={np.median(a):.0f} p90={np.percentile(a, 90):.0f} max={a.max():.0f}"


jobs = R[..., 0]
print(f"{nq} value CTAs; D2 phase cycles {pct(v[:, 2])}")
print("edge jobs per CTA", pct(jobs.sum(1)), "; max per thread", pct(jobs.max(1)))
print("non-fast edges per CTA", pct(R[..., 1].sum(1)))
busy = jobs > 0
print("band steps per thread (busy)", pct(R[..., 2][busy]))
print("exact rounds per thread (busy)", pct(R[..., 3][busy]))
print("setup+band cycles per thread (busy)", pct(R[..., 4][busy]))
print("exact cycles per thread (busy)", pct(R[..., 5][busy]))
tot = R[..., 4] + R[..., 5]
print("edge-chain cycles per CTA: max thread", pct(tot.max(1)))
er = R[..., 3][busy] / np.maximum(jobs[busy], 1)
print("exact rounds per edge (single-job threads)", pct(R[..., 3][jobs == 1]))
print("cycles per exact round", pct((R[..., 5][busy] / np.maximum(R[..., 3][busy], 1))))
slow = np.argsort(v[:, 2])[-5:]
for i in slow:
    t = np.argmax(tot[i])
    print(f" slow CTA {i}: D2 {v[i, 2]} jobs {jobs[i].sum()} nonfast {R[i, :, 1].sum()} "
          f"worst thread jobs {jobs[i, t]} band {R[i, t, 2]} rounds {R[i, t, 3]} "
          f"cyc {R[i, t, 4]}+{R[i, t, 5]}")

"""Dev tool: per-phase cycles of the batch (throughput-shape) scan CTAs from
the profiling build: window (A), robot scans (B), champions + queue (C), and
the CTA's own duration.  16 C5 frames (8,192 tiles = the record capacity)
through pp_dpps_frames.  Not used by tests/bench."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_07717_b200 import abi, synthetic  # noqa: E402

lib = abi._declare(C.CDLL(os.environ.get("PP_PROF_LIB", os.path.join(
    ROOT, "paper_1909_07717_b200", "lib", "libpassplan_b200_prof.so"))))
P = C.POINTER(C.c_longlong)
lib.pp_debug_cta_records.argtypes = [P, P, P]
ctx = C.c_void_p()
assert lib.pp_ctx_create(0, C.byref(ctx)) == 0
p = abi.Params()
lib.pp_params_default(C.byref(p))
n = 16
fr, keep = synthetic.as_ctypes(synthetic.c5_frames(0, n))
out = (abi.FrameSummary * n)()
g = abi.SearchGrid(128, 64, 1.0, 6.5, 1, 0)
for _ in range(3):
    assert lib.pp_dpps_frames(ctx, fr, n, C.byref(p), C.byref(g), None, out) == 0
s = np.zeros((8192, 8), np.int64)
v = np.zeros((8192, 8), np.int64)
r = np.zeros((8192, 16), np.int64)
lib.pp_debug_cta_records(s.ctypes.data_as(P), v.ctypes.data_as(P), r.ctypes.data_as(P))


def pct(a):
    a = np.asarray(a, float)
    return f"mean={a.mean():.0f} p50={np.median(a):.0f} p90={np.percentile(a, 90):.0f} max={a.max():.0f}"


A = s[:, 5]
B = s[:, 1] - s[:, 5]
Cc = s[:, 3]
dur_ns = s[:, 7] - s[:, 0]
print(f"scan CTAs {len(s)}: span {(s[:, 7].max() - s[:, 0].min()) / 1e3:.1f} us")
print(" A window cyc", pct(A))
print(" B robot scans cyc", pct(B))
print(" C champions+queue cyc", pct(Cc))
print(" CTA duration ns", pct(dur_ns), f"(= {np.mean(dur_ns) * 1.965:.0f} cyc at 1.965 GHz)")
print(f" share of CTA time: A {A.mean() / (dur_ns.mean() * 1.965):.2f} B {B.mean() / (dur_ns.mean() * 1.965):.2f} "
      f"C {Cc.mean() / (dur_ns.mean() * 1.965):.2f}")
sm = s[:, 6]
occ = np.bincount(sm, minlength=148)
print(" CTAs per SM", pct(occ))

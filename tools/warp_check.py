"""Dev tool (GPU box): C5 frames through pp_dpps_frames -- per-frame results
saved for a byte comparison between scan variants (env knobs), and the
median wall time of the call.  usage: warp_check.py OUT.npy [N_FRAMES]
Not used by tests/bench."""
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_07717_b200 import abi, synthetic  # noqa: E402

out_path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
lib = abi.load_library()
ctx = C.c_void_p()
assert lib.pp_ctx_create(0, C.byref(ctx)) == 0
p = abi.Params()
lib.pp_params_default(C.byref(p))
grid = abi.SearchGrid(128, 64, 1.0, 6.5, 1, 0)
fr, keep = synthetic.as_ctypes(synthetic.c5_frames(0, n))
out = (abi.FrameSummary * n)()
ts = []
for i in range(8):
    t = time.perf_counter()
    st = lib.pp_dpps_frames(ctx, fr, n, C.byref(p), C.byref(grid), None, out)
    ts.append(time.perf_counter() - t)
    assert st == 0, lib.pp_last_error(ctx)
raw = np.frombuffer(bytes(out), np.uint8).reshape(n, -1)
np.save(out_path, raw)
print(f"{os.environ.get('PP_WARP_TILES', 'default')}: {n} frames, wall ms min {1e3 * min(ts[2:]):.2f} "
      f"med {1e3 * np.median(ts[2:]):.2f}  frames/s {n / min(ts[2:]):.0f}")

"""Dev tool: one pp_batch_run over C5 frames (for ncu captures of the batch
scan / value kernels).  python tools/profile_batch.py [n_frames] [chip]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_07717_b200 import abi, synthetic  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
chip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
lib = abi.load_library()
ctx = C.c_void_p()
assert lib.pp_ctx_create(0, C.byref(ctx)) == 0
p = abi.Params()
lib.pp_params_default(C.byref(p))
g = abi.SearchGrid(128, 64, 1.0, 6.5, 1, chip)
fr, keep = synthetic.as_ctypes(synthetic.c5_frames(0, n))
assert lib.pp_batch_upload(ctx, fr, n, None) == 0
ms = C.c_float()
for _ in range(int(os.environ.get("REPS", "1"))):
    assert lib.pp_batch_run(ctx, C.byref(p), C.byref(g), C.byref(ms)) == 0, lib.pp_last_error(ctx)
    print(f"{n} frames: {ms.value:.3f} ms ({n / ms.value * 1e3:.0f} frames/s)")
out = (abi.FrameSummary * n)()
assert lib.pp_batch_download(ctx, out) == 0
print("best[0]", out[0].best_cell[0], out[0].best_score[0])

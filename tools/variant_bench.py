"""Dev tool: C5 batch throughput + result checksum of one library build
(PP_LIB_PATH selects a variant).  python tools/variant_bench.py [frames] [reps]"""
import ctypes as C
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_07717_b200 import abi, synthetic  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
lib = abi.load_library()
ctx = C.c_void_p()
assert lib.pp_ctx_create(0, C.byref(ctx)) == 0
p = abi.Params()
lib.pp_params_default(C.byref(p))
g = abi.SearchGrid(128, 64, 1.0, 6.5, 1, 0)
fr, keep = synthetic.as_ctypes(synthetic.c5_frames(0, n))
assert lib.pp_batch_upload(ctx, fr, n, None) == 0
ms = C.c_float()
lib.pp_batch_run(ctx, C.byref(p), C.byref(g), C.byref(ms))
best = []
for _ in range(reps):
    assert lib.pp_batch_run(ctx, C.byref(p), C.byref(g), C.byref(ms)) == 0, lib.pp_last_error(ctx)
    best.append(ms.value)
out = (abi.FrameSummary * n)()
assert lib.pp_batch_download(ctx, out) == 0
st, sc, va, nl = C.c_float(), C.c_float(), C.c_float(), C.c_int32()
lib.pp_batch_kernel_times(ctx, C.byref(p), C.byref(g), 1, C.byref(st), C.byref(sc), C.byref(va),
                          C.byref(nl))
t = min(best)
print(f"{os.path.basename(os.environ.get('PP_LIB_PATH', 'default'))}: {n} frames {t:.2f} ms "
      f"({n / t * 1e3:.0f} frames/s) scan {sc.value:.2f} value {va.value:.2f} "
      f"sha {hashlib.sha1(bytes(out)).hexdigest()[:12]}")

"""Dev tool: where the C2 frame's device time goes between the kernels' own
span (summary.device_ms: first scan CTA start -> final fold) and the
event-timed relaunch (bench.py's device p50), with and without the 512 MiB L2
flush before each rep.  python tools/frame_gap.py [reps]"""
import ctypes as C
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_1909_07717_b200 import abi  # noqa: E402
from helpers import case_inputs  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
lib = abi.load_library()
g = np.load(os.path.join(ROOT, "tests", "golden", "grids.npz"))
ctx = C.c_void_p()
assert lib.pp_ctx_create(0, C.byref(ctx)) == 0
w, p, grid, k, _ = case_inputs(g, "f8")
grid.chip = 1
n = 16384
nb = int(lib.pp_grid_bytes(n))
ptr = lib.pp_host_alloc(nb)
blk = abi.GridBlock(n, buf=(C.c_uint8 * nb).from_address(ptr))
assert lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), k, abi.PP_COPY_ALL, ptr) == 0
lib.pp_ctx_stream.restype = C.c_void_p
stream = torch.cuda.ExternalStream(lib.pp_ctx_stream(ctx))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(do_flush, what):
    ev, spans = [], []
    with torch.cuda.stream(stream):
        for i in range(reps + 5):
            if do_flush:
                flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            what()
            b.record(stream)
            b.synchronize()
            if i >= 5:
                ev.append(a.elapsed_time(b) * 1e3)
                spans.append(blk.summary.device_ms * 1e3)
    return statistics.median(ev), statistics.median(spans)


tiny = torch.zeros(1, device="cuda")
for do_flush in (True, False):
    e, s = timed(do_flush, lambda: lib.pp_dpps_relaunch(ctx))
    e0, _ = timed(do_flush, lambda: tiny.add_(1))
    print(f"flush={do_flush}: relaunch events p50 {e:.1f} us, kernel span p50 {s:.1f} us, "
          f"gap {e - s:.1f} us; one tiny torch kernel {e0:.1f} us")

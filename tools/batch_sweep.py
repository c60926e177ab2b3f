"""Dev tool (GPU box): the batch path (pp_dpps_frames: device staging, scan,
score-bound pruning, value function, fold) against the compiled reference's
run_dpps_serial + best_pass (ref_batch) on many frames: the C5 frames
(seeds 0xB200 + i) and mixed frames (1-16 v 0-16 robots, shuffled sparse ids),
flat and flat + chip grids.  Best cell identical (or tied within 1e-4), best
score within 1e-4 relative (atan2 last ulp), feasible counts identical.
usage: python tools/batch_sweep.py [n_frames]"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import bindings as B  # noqa: E402
from paper_1909_07717_b200 import abi, synthetic  # noqa: E402
from tests.test_gpu_batch import _mixed_frames  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
lib = abi.load_library()
ctx = C.c_void_p()
assert lib.pp_ctx_create(0, C.byref(ctx)) == 0
p = abi.Params()
lib.pp_params_default(C.byref(p))
total_bad = 0
for name, frames_np in (("c5", synthetic.c5_frames(0, n)), ("mixed", _mixed_frames(n // 4, 7))):
    for chip in (0, 1):
        m_ = frames_np.shape[0]
        grid = abi.SearchGrid(128, 64, 1.0, 6.5, 1, chip)
        frames, _keep = synthetic.as_ctypes(frames_np)
        out = (abi.FrameSummary * m_)()
        assert lib.pp_dpps_frames(ctx, frames, m_, C.byref(p), C.byref(grid), None, out) == 0, \
            lib.pp_last_error(ctx)
        best = np.zeros(m_, np.int64)
        score = np.zeros(m_)
        nfeas = np.zeros(m_, np.int64)
        msg = B.msgbuf()
        st = B.ref().ref_batch(frames, m_, C.byref(p), C.byref(grid), None, os.cpu_count() or 1,
                               best.ctypes.data_as(C.POINTER(C.c_int64)),
                               score.ctypes.data_as(C.POINTER(C.c_double)),
                               nfeas.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(C.c_double()),
                               msg, 512)
        assert st == 0, msg.value
        g_best = np.array([out[i].best_cell[0] for i in range(m_)])
        g_score = np.array([out[i].best_score[0] for i in range(m_)])
        g_nf = np.array([out[i].n_feasible[0] for i in range(m_)])
        nf_bad = int((g_nf != nfeas).sum())
        sc_bad = int((np.abs(g_score - score) > 1e-4 * np.maximum(1.0, np.abs(score))).sum())
        cell_diff = int((g_best != best).sum())
        print(f"{name} chip={chip} frames={m_}: feasible-count mismatches {nf_bad}, score "
              f"mismatches {sc_bad}, best cells differing {cell_diff} (ties within 1e-4 allowed)")
        total_bad += nf_bad + sc_bad
print(f"total mismatches: {total_bad}")

"""The three scan CTA shapes (16-warp and 8-warp with leftover rounds, 4-warp
plain) and the leftover schedule only change how the search is scheduled,
never its result: the same frames through every forced shape must give
bit-identical grids (times, receive points, ids, feasibility) and identical
scores.  Each configuration runs in its own process (the shape override is
read once per process)."""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import ctypes as C, hashlib, os, sys
import numpy as np
sys.path.insert(0, os.environ["PP_ROOT"]); sys.path.insert(0, os.path.join(os.environ["PP_ROOT"], "tests"))
from paper_1909_07717_b200 import abi
from helpers import case_inputs, run_product
lib = abi.load_library()
g = np.load(os.path.join(os.environ["PP_ROOT"], "tests", "golden", "grids.npz"))
ctx = C.c_void_p(); assert lib.pp_ctx_create(0, C.byref(ctx)) == 0
h = hashlib.sha256()
for name in ("f8", "minimal", "rand8v8_0", "rand8v8_3"):
    w, p, grid, k, _ = case_inputs(g, name)
    for chip in (0, 1):
        grid.chip = chip
        st, blk = run_product(lib, ctx, w, p, grid, k)
        assert st == 0, lib.pp_last_error(ctx)
        for arr in (blk.our_time, blk.opp_time, blk.rx, blk.ry, blk.our_slot, blk.opp_slot,
                    blk.feasible, blk.score):
            h.update(np.ascontiguousarray(arr).tobytes())
        s = blk.summary
        h.update(bytes(np.array(list(s.best_cell), dtype=np.int64).tobytes()))
        h.update(bytes(np.array(list(s.n_feasible), dtype=np.int64).tobytes()))
print(h.hexdigest())
"""


def _digest(env_extra):
    env = dict(os.environ, PP_ROOT=ROOT, **env_extra)
    out = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout.strip().splitlines()[-1]


@pytest.mark.gpu
def test_scan_shapes_identical():
    base = _digest({})
    for extra in ({"PP_SCAN_SHAPE": "w"}, {"PP_SCAN_SHAPE": "m"}, {"PP_SCAN_SHAPE": "n"},
                  {"PP_SCAN_SHAPE": "w", "PP_SCAN_STEPS": "1", "PP_SCAN_ROUND": "1"},
                  {"PP_SCAN_SHAPE": "m", "PP_SCAN_STEPS": "1000000"}):
        assert _digest(extra) == base, extra

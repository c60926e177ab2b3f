"""Algorithmic work per pair of the C5 batch:
W_pair = 13 N_qr + 42 N_full + 33 N_rest + 30, counted by the oracle's
replica of the reference's pruned scan (or_dpps_counted) on C5 frames
(oracles::random_world(mt19937_64(0xB200 + i), 8, 8), C1 grid).  Writes
profiles/c5_work.json, which bench.py's roofline reads.  Dev tool (CPU)."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import bindings as B  # noqa: E402
from paper_1909_07717_b200 import abi, synthetic  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
orc = B.oracle()
p = abi.Params()
orc.or_params_default(C.byref(p))
grid = abi.SearchGrid(128, 64, 1.0, 6.5, 1, 0)
fr = synthetic.c5_frames(0, n)
arr, _k = synthetic.as_ctypes(fr)
tot = B.OrCounts()
pairs = 0
blk = abi.GridBlock(8192)
for i in range(n):
    c = B.OrCounts()
    k = orc.or_nearest_teammate(C.byref(arr[i]))
    assert orc.or_dpps_counted(C.byref(arr[i]), C.byref(p), C.byref(grid), k, blk.ptr(),
                               C.byref(c), None, 0) == 0
    for f in ("quick_rejects", "full_tests", "rest_evals", "scans", "bounds"):
        setattr(tot, f, getattr(tot, f) + getattr(c, f))
    pairs += int(blk.summary.sbip_calls)
qr, full, rest = tot.quick_rejects / pairs, tot.full_tests / pairs, tot.rest_evals / pairs
w = 13 * qr + 42 * full + 33 * rest + 30
out = {"frames": n, "pairs": pairs, "N_qr": qr, "N_full": full, "N_rest": rest,
       "W_pair_flop": w, "formula": "13 N_qr + 42 N_full + 33 N_rest + 30 (SURVEY 8(d))",
       "frames_desc": "C5 frames 0..n-1: random_world(mt19937_64(0xB200+i), 8, 8), C1 grid "
                      "128x64 flat, kicker = nearest teammate"}
print(json.dumps(out, indent=1))
with open(os.path.join(ROOT, "profiles", "c5_work.json"), "w") as f:
    json.dump(out, f, indent=1)

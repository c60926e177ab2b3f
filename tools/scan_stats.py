"""Dev tool (GPU box): filter statistics of the scan kernel from the
-DPP_SCAN_STATS variant (tools/build_variants.sh stats -DPP_SCAN_STATS):
per (robot, cell) pair, how many samples the FP32 filters tested and how
each test ended.  PP_LIB_PATH=variants/libpassplan_b200_stats.so
python tools/scan_stats.py [n_frames]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_07717_b200 import abi, synthetic  # noqa: E402

NAMES = ["tests", "end", "cap", "reach_rej", "reach_skipped", "lb_rej", "ub_hit", "cand",
         "exact", "exact_hit", "pairs", "pairs_pruned", "warp_steps", "active_lanes",
         "to_leftovers", "their_tests", "hit_pairs", "hit_tests", "cap_pairs", "cap_tests", "end_pairs", "end_tests", "their_pairs", "their_warp_steps"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
lib = abi.load_library()
lib.pp_debug_scan_stats.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
lib.pp_debug_scan_stats.restype = None
lib.pp_debug_act_hist.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
lib.pp_debug_act_hist.restype = None
hist = (C.c_ulonglong * 33)()
ctx = C.c_void_p()
assert lib.pp_ctx_create(0, C.byref(ctx)) == 0
p = abi.Params()
lib.pp_params_default(C.byref(p))
st = (C.c_ulonglong * 64)()
for chip in (0, 1):
    g = abi.SearchGrid(128, 64, 1.0, 6.5, 1, chip)
    fr, keep = synthetic.as_ctypes(synthetic.c5_frames(0, n))
    assert lib.pp_batch_upload(ctx, fr, n, None) == 0
    lib.pp_debug_scan_stats(st, 1)
    lib.pp_debug_act_hist(hist, 1)
    ms = C.c_float()
    assert lib.pp_batch_run(ctx, C.byref(p), C.byref(g), C.byref(ms)) == 0
    lib.pp_debug_scan_stats(st, 1)
    lib.pp_debug_act_hist(hist, 1)
    pairs = st[10]
    print(f"C5 batch {n} frames chip={chip}: pairs {pairs}")
    for i, nm in enumerate(NAMES):
        print(f"  {nm:14s} {st[i]:14d}  per pair {st[i] / pairs:8.3f}")
    print(f"  SIMT lanes/step {st[13] / max(st[12], 1):.2f}")
    for nm, a in (("hit", 16), ("capped", 18), ("end", 20)):
        print(f"  tests per {nm} pair {st[a + 1] / max(st[a], 1):.2f}")
    edges = ["0", "1", "2", "3", "4-5", "6-7", "8-11", "12-15", "16-31", "32-47", "48-63",
             "64-127", "128-191", "192-255", "-", "256+"]
    tot = max(sum(st[40 + b] for b in range(16)), 1)
    print("  pairs by tests: bucket, pairs, share of all tests")
    for b in range(16):
        if st[24 + b]:
            print(f"    {edges[b]:>8s} {st[24 + b]:12d} {st[40 + b] / tot:6.3f}")
    print(f"  rest-rule arrivals {st[57] / pairs:.3f} per pair, {st[58] / max(st[57], 1):.3f} of them "
          f"<= t_stop, {st[59] / max(st[57], 1):.3f} ours")
    print(f"  lower-bound rejects in runs of >= 4: {st[56] / max(st[5], 1):.3f} of all lb rejects")
    tot = sum(hist) or 1
    print("  warp steps by active lanes (%):",
          " ".join(f"{a}:{100 * hist[a] / tot:.1f}" for a in range(33) if hist[a]))
    print("  lane-steps share of steps with <= 4 / <= 8 active lanes: "
          f"{sum(a * hist[a] for a in range(5)) / max(sum(a * hist[a] for a in range(33)), 1):.3f} / "
          f"{sum(a * hist[a] for a in range(9)) / max(sum(a * hist[a] for a in range(33)), 1):.3f}")

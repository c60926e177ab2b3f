"""Dev tool (GPU box): differential fuzz of the batch scan shapes.  Random
batches (1..3,000 frames of 1..16 v 0..16 robots with shuffled ids, some
with a rolling ball), random grids (1..300 directions x 1..100 powers,
flat / chip / both, random power ranges) and random safety margins and
weights go through pp_dpps_frames; the per-frame results are written to
OUT.npz.  Run it twice -- the product (warp-per-tile scan) and
PP_WARP_TILES=0 (the 4-warp tile CTAs, validated against the reference in
round 2) -- and compare: python tools/warp_fuzz.py OUT.npz [n_cases]
Not used by tests/bench."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_07717_b200 import abi, synthetic  # noqa: E402

out_path = sys.argv[1]
n_cases = int(sys.argv[2]) if len(sys.argv) > 2 else 60
lib = abi.load_library()
ctx = C.c_void_p()
assert lib.pp_ctx_create(0, C.byref(ctx)) == 0
res = {}
rng = np.random.default_rng(2026)
for case in range(n_cases):
    n = int(rng.choice([1, 7, 64, 300, 1000, 3000]))
    fr = synthetic.random_worlds(np.arange(n, dtype=np.uint64) + np.uint64(10_000 * case), 16, 16)
    for i in range(n):
        fr["n_ours"][i], fr["n_theirs"][i] = int(rng.integers(1, 17)), int(rng.integers(0, 17))
        for team in ("ours", "theirs"):
            fr[team]["id"][i] = rng.choice(40, size=16, replace=False)
        if rng.random() < 0.3:
            fr["ball_vx"][i], fr["ball_vy"][i] = rng.uniform(-3, 3, size=2)
    p = abi.Params()
    lib.pp_params_default(C.byref(p))
    p.thresholds.safety_margin = float(rng.choice([0.0, 0.0137, 0.1, 0.3, 0.7]))
    if rng.random() < 0.3:
        w = p.pass_weights
        w.shoot_angle, w.refraction, w.teammate_time = rng.uniform(-2, 2, size=3)
    flat, chip = [(1, 0), (0, 1), (1, 1)][int(rng.integers(0, 3))]
    pmin = float(rng.uniform(0.5, 3.0))
    grid = abi.SearchGrid(int(rng.integers(1, 301)), int(rng.integers(1, 101)), pmin,
                          pmin + float(rng.uniform(0.5, 4.0)), flat, chip)
    frames, _keep = synthetic.as_ctypes(fr)
    out = (abi.FrameSummary * n)()
    st = lib.pp_dpps_frames(ctx, frames, n, C.byref(p), C.byref(grid), None, out)
    res[f"c{case}"] = np.frombuffer(bytes(out), np.uint8).copy() if st == 0 else np.array([st])
    print(f"case {case}: {n} frames, grid {grid.n_directions}x{grid.n_powers} flat={flat} chip={chip}"
          f" safety={p.thresholds.safety_margin}: st={st}", flush=True)
np.savez(out_path, **res)

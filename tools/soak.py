"""Dev tool (GPU box): soak test of the single-frame pipeline's self-cleaning
state -- thousands of pp_dpps calls on one context with random worlds, grid
shapes (every scan CTA shape, streaming and plain value launches), flat /
chip, pinned and pageable blocks in random order, plus batches and run maps
interleaved.  Every call must succeed and repeat bit for bit (each world is
run twice, at different points of the sequence).
usage: python tools/soak.py [seconds]"""
import ctypes as C
import hashlib
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_07717_b200 import abi, synthetic  # noqa: E402
from tests.test_gpu_random import _random_world  # noqa: E402

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
lib = abi.load_library()
ctx = C.c_void_p()
assert lib.pp_ctx_create(0, C.byref(ctx)) == 0
p = abi.Params()
lib.pp_params_default(C.byref(p))
rng = random.Random(7)
shapes = [(128, 64), (37, 19), (256, 96), (64, 40), (600, 450), (8, 4), (1, 1)]
pinned_buf = {}
seen = {}
calls = repeats = 0
t_end = time.time() + secs


def digest(blk):
    """Per-field digests of everything the block defines (padding and
    device_ms excluded)."""
    s = blk.summary
    d = {f: hashlib.sha1(getattr(blk, f).tobytes()).hexdigest()
         for f in ("our_time", "opp_time", "rx", "ry", "score", "our_slot", "opp_slot",
                   "feasible")}
    for f, _t in abi.DppsSummary._fields_:
        if f != "device_ms":
            d[f] = bytes(getattr(s, f)) if hasattr(getattr(s, f), "_length_") or \
                isinstance(getattr(s, f), C.Structure) else getattr(s, f)
    return d

while time.time() < t_end:
    wid = rng.randrange(400)
    w = _random_world(0x50A + wid, 1 + wid % 16, wid % 17, (wid % 4) * 0.9)
    k = w.ours[0].id
    nd, np_ = shapes[wid % len(shapes)]
    chip = wid % 3 == 0
    grid = abi.SearchGrid(nd, np_, 1.0, 6.5, 1, int(chip))
    n = (1 + int(chip)) * nd * np_
    nb = int(lib.pp_grid_bytes(n))
    if rng.random() < 0.5:
        if nb not in pinned_buf:
            pinned_buf[nb] = lib.pp_host_alloc(nb)
        ptr = pinned_buf[nb]
        st = lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), k, abi.PP_COPY_ALL,
                         C.c_void_p(ptr))
        blk = abi.GridBlock(n, buf=(C.c_uint8 * nb).from_address(ptr))
    else:
        page = abi.GridBlock(n)
        st = lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), k, abi.PP_COPY_ALL,
                         page.ptr())
        blk = page
    assert st == 0, (calls, lib.pp_last_error(ctx))
    h = digest(blk)
    if wid in seen:
        bad = [k for k in h if h[k] != seen[wid][k]]
        assert not bad, f"call {calls}: world {wid} changed in {bad}"
        repeats += 1
    seen[wid] = h
    calls += 1
    if calls % 97 == 0:  # a batch in between
        fr, _keep = synthetic.as_ctypes(synthetic.c5_frames(calls, calls + 64))
        out = (abi.FrameSummary * 64)()
        assert lib.pp_dpps_frames(ctx, fr, 64, C.byref(p), C.byref(abi.SearchGrid(
            128, 64, 1.0, 6.5, 1, 0)), None, out) == 0
    if calls % 131 == 0:  # a run map in between
        nv = C.c_int64()
        assert lib.pp_runmap_count(C.byref(w), C.byref(p), 0xF, C.byref(nv)) == 0
        buf = (C.c_uint8 * abi.runmap_offsets(nv.value)["total"])()
        req = abi.RunmapRequest(0xF, 0, 4, 0, 0.0, 0.0, 1)
        assert lib.pp_runmap(ctx, C.byref(w), C.byref(p), C.byref(req), buf, nv.value) == 0
print(f"soak: {calls} pp_dpps calls in {secs:.0f} s, {repeats} repeats bit-identical, no errors")

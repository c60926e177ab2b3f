"""Contexts are independent: several host threads, each with its own pp_ctx
(its own stream, buffers and cached graph), run single frames, batches and
run maps at the same time (ctypes releases the GIL during the calls).  Every
result must equal the one the same call gives when the calls run one after
another on a single context."""
from __future__ import annotations

import ctypes as C
import threading

import pytest

from paper_1909_07717_b200 import abi, synthetic

from tests.test_gpu_random import _random_world

pytestmark = pytest.mark.gpu


def _params(lib):
    p = abi.Params()
    lib.pp_params_default(C.byref(p))
    return p


def _job(lib, ctx, i, p):
    """One call, chosen by i: a single frame (pinned or pageable block, grid
    shape by i), a small batch, or a run map.  Returns the defining bytes."""
    kind = i % 3
    if kind == 0:
        w = _random_world(0x7E00 + i, 1 + i % 16, i % 17, (i % 3) * 1.1)
        shapes = [(128, 64, 1), (37, 19, 1), (64, 40, 0), (200, 96, 0)]
        nd, np_, chip = shapes[(i // 3) % len(shapes)]
        grid = abi.SearchGrid(nd, np_, 1.0, 6.5, 1, chip)
        n = (1 + chip) * nd * np_
        blk = abi.GridBlock(n)
        assert lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), w.ours[0].id,
                           abi.PP_COPY_ALL, blk.ptr()) == 0, lib.pp_last_error(ctx)
        return bytes(blk.our_time.tobytes() + blk.opp_time.tobytes() + blk.rx.tobytes() +
                     blk.score.tobytes() + blk.feasible.tobytes() +
                     bytes(blk.summary.best_cell) + bytes(blk.summary.n_feasible))
    if kind == 1:
        frames, _keep = synthetic.as_ctypes(synthetic.c5_frames(i * 8, i * 8 + 24))
        out = (abi.FrameSummary * 24)()
        assert lib.pp_dpps_frames(ctx, frames, 24, C.byref(p), C.byref(abi.SearchGrid(
            128, 64, 1.0, 6.5, 1, i % 2)), None, out) == 0, lib.pp_last_error(ctx)
        return bytes(out)
    w = _random_world(0x7F00 + i, 8, 8, 0.0)
    nv = C.c_int64()
    assert lib.pp_runmap_count(C.byref(w), C.byref(p), 0xF, C.byref(nv)) == 0
    buf = (C.c_uint8 * abi.runmap_offsets(nv.value)["total"])()
    req = abi.RunmapRequest(0xF, 0, 4, 0, 0.0, 0.0, 1)
    assert lib.pp_runmap(ctx, C.byref(w), C.byref(p), C.byref(req), buf,
                         nv.value) == 0, lib.pp_last_error(ctx)
    off = abi.runmap_offsets(nv.value)
    return bytes(buf)[off["px"]:]


def test_concurrent_contexts_match_sequential():
    lib = abi.load_library()
    p = _params(lib)
    n_threads, per_thread = 4, 24
    jobs = [[t * per_thread + j for j in range(per_thread)] for t in range(n_threads)]
    # sequential reference on one context
    ref_ctx = C.c_void_p()
    assert lib.pp_ctx_create(0, C.byref(ref_ctx)) == 0
    want = {i: _job(lib, ref_ctx, i, p) for js in jobs for i in js}
    lib.pp_ctx_destroy(ref_ctx)

    got, errors = {}, []

    def worker(js):
        c = C.c_void_p()
        try:
            assert lib.pp_ctx_create(0, C.byref(c)) == 0
            for _ in range(2):  # twice: the second pass replays cached graphs
                for i in js:
                    got[(i, _)] = _job(lib, c, i, p)
        except Exception as e:  # noqa: BLE001 (reported below)
            errors.append(repr(e))
        finally:
            if c:
                lib.pp_ctx_destroy(c)

    threads = [threading.Thread(target=worker, args=(js,)) for js in jobs]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
    assert not errors, errors[:3]
    bad = [k for k, v in got.items() if v != want[k[0]]]
    assert len(got) == 2 * n_threads * per_thread
    assert not bad, f"{len(bad)} calls differ, e.g. {bad[:5]}"

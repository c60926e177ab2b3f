"""Pinned result blocks (pp_host_alloc) take the kernels' outputs directly
(the DPPS grid: no device-to-host copy; the run map: one DMA copy into it);
pageable blocks get a staged copy.  Both paths must give
byte-identical blocks, for the DPPS grid and for the run map (whose
`n_scorable` is counted on the device)."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from paper_1909_07717_b200 import abi

from tests.helpers import case_inputs

pytestmark = pytest.mark.gpu


def _pinned_copy(lib, nbytes, fill):
    ptr = lib.pp_host_alloc(nbytes)
    assert ptr
    arr = np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(ptr))
    arr[:] = fill
    return ptr, arr


def test_dpps_pinned_equals_pageable(ctx, grids_golden):
    lib = abi.load_library()
    for name in ("f8", "rand8v8_2", "minimal"):
        w, p, grid, k, _ = case_inputs(grids_golden, name)
        for chip in (0, 1):
            grid.chip = chip
            n = (int(bool(grid.flat)) + int(bool(grid.chip))) * grid.n_directions * grid.n_powers
            nbytes = int(lib.pp_grid_bytes(n))
            page = abi.GridBlock(n)
            assert lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), k, abi.PP_COPY_ALL,
                               page.ptr()) == 0
            ptr, arr = _pinned_copy(lib, nbytes, 0)
            try:
                assert lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), k,
                                   abi.PP_COPY_ALL, ptr) == 0
                pin = abi.GridBlock(n, buf=arr)
                # device_ms is a timing, the rest must match byte for byte
                pin.summary.device_ms = page.summary.device_ms
                assert bytes(arr) == page.buf.tobytes(), (name, chip)
            finally:
                lib.pp_host_free(ptr)


def test_runmap_pinned_equals_pageable(ctx, grids_golden):
    lib = abi.load_library()
    w, p, _, _, _ = case_inputs(grids_golden, "f8")
    for step in (0.1, 0.05):
        pp = abi.Params.from_buffer_copy(bytes(p))
        pp.thresholds.grid_step = step
        req = abi.RunmapRequest(0xF, 0, 4, 0, 0.0, 0.0, 1)
        nv = C.c_int64()
        assert lib.pp_runmap_count(C.byref(w), C.byref(pp), req.zone_mask, C.byref(nv)) == 0
        page = abi.RunmapBlock(nv.value)
        assert lib.pp_runmap(ctx, C.byref(w), C.byref(pp), C.byref(req), page.ptr(), nv.value) == 0
        assert page.summary.n_scorable == int(page.scorable.sum())
        nbytes = abi.runmap_offsets(nv.value)["total"]
        ptr, arr = _pinned_copy(lib, nbytes, 0)
        try:
            assert lib.pp_runmap(ctx, C.byref(w), C.byref(pp), C.byref(req), ptr, nv.value) == 0
            assert bytes(arr) == page.buf.tobytes(), step
        finally:
            lib.pp_host_free(ptr)


def test_dpps_alternating_pinned_and_pageable(ctx, grids_golden):
    """Pageable and pinned calls interleaved on one context (the pinned call
    replays a cached graph whose node parameters must survive the plain
    pageable launches in between): every call returns the same block."""
    lib = abi.load_library()
    w, p, grid, k, _ = case_inputs(grids_golden, "f8")
    grid.n_directions, grid.n_powers, grid.chip = 128, 64, 1
    n = 2 * 128 * 64
    nbytes = int(lib.pp_grid_bytes(n))
    ptr, arr = _pinned_copy(lib, nbytes, 0)
    off = abi.DppsSummary.device_ms.offset
    try:
        want = None
        for kind in "GPGPPGGP":
            if kind == "P":
                arr[:] = 0
                st = lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), k, abi.PP_COPY_ALL,
                                 C.c_void_p(ptr))
                got = bytearray(arr.tobytes())
            else:
                page = abi.GridBlock(n)
                st = lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), k, abi.PP_COPY_ALL,
                                 page.ptr())
                got = bytearray(bytes(page.buf))
            assert st == 0, (kind, lib.pp_last_error(ctx))
            got[off:off + 8] = bytes(8)  # (the kernels' own time differs per call)
            want = want or bytes(got)
            assert bytes(got) == want, kind
    finally:
        lib.pp_host_free(ptr)

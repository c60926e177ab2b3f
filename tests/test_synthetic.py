"""CPU: the C5 frame generator (paper_1909_07717_b200/synthetic.py) restates
oracles::random_world(mt19937_64(seed), n_ours, n_theirs)
(proj/tests/oracles.hpp:228-258) bit for bit -- checked against the compiled
reference's own generator (oracle/_ref ref_random_world)."""
import ctypes as C

import numpy as np
import pytest

from oracle import bindings as B
from paper_1909_07717_b200 import abi, synthetic


@pytest.mark.skipif(not B.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("n_ours,n_theirs", [(8, 8), (16, 16), (3, 0), (1, 5)])
def test_random_worlds_match_reference(n_ours, n_theirs):
    seeds = [0, 1, 0xB200, 0xB200 + 65535, 2 ** 63 + 7, 123456789]
    got = synthetic.random_worlds(seeds, n_ours, n_theirs)
    lib = B.ref()
    for i, s in enumerate(seeds):
        w = abi.World()
        assert lib.ref_random_world(s, n_ours, n_theirs, 0.0, C.byref(w)) == 0
        assert bytes(w) == got[i].tobytes(), s


@pytest.mark.skipif(not B.ref_available(), reason="oracle/_ref not built")
def test_c5_frames_match_reference():
    got = synthetic.c5_frames(0, 256)
    lib = B.ref()
    for i in list(range(0, 256, 7)) + [255]:
        w = abi.World()
        assert lib.ref_random_world(0xB200 + i, 8, 8, 0.0, C.byref(w)) == 0
        assert bytes(w) == got[i].tobytes(), i


def test_c5_frames_shape_and_ranges():
    fr = synthetic.c5_frames(100, 164)
    assert fr.shape == (64,) and fr.dtype.itemsize == C.sizeof(abi.World)
    assert np.all(fr["n_ours"] == 8) and np.all(fr["n_theirs"] == 8)
    for team in ("ours", "theirs"):
        r = fr[team][:, :8]
        assert np.all(np.abs(r["px"]) <= 6.0) and np.all(np.abs(r["py"]) <= 4.5)
        assert np.all(np.abs(r["vx"]) <= 2.0) and np.all(np.abs(r["vy"]) <= 2.0)
        assert np.array_equal(r["id"][0], np.arange(8))
    assert np.all(fr["ball_vx"] == 0.0) and np.all(fr["ball_vy"] == 0.0)
    # shards concatenate to the whole
    a = synthetic.c5_frames(100, 130)
    b = synthetic.c5_frames(130, 164)
    assert np.concatenate([a, b]).tobytes() == fr.tobytes()

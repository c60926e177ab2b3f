"""Synthetic world states of the C5 batch (BASELINE.json configs[4]).

Frame i of the batch is the reference's own test generator
`oracles::random_world(std::mt19937_64(0xB200 + i), 8, 8)`
(proj/tests/oracles.hpp:228-258): 8 v 8 robots with ids
0..7, positions uniform on the 12 x 9 m pitch, velocity components U(-2, 2),
ball uniform on the pitch and at rest.

The draws are restated here with numpy, vectorised over frames, so the same
bytes can be produced on any host without the reference:

* std::mt19937_64 (seeding, one 312-word twist, tempering: the standard
  engine's published algorithm);
* libstdc++'s std::uniform_real_distribution<double>(a, b) on a 64-bit
  engine: generate_canonical<double, 53> takes ONE engine word,
  u = double(x) / 2^64 (x converted with round-to-nearest; u >= 1 becomes
  nextafter(1, 0)), and the value is (u * (b - a)) + a, two separately
  rounded operations;
* the reference's draw order: per robot {x, y} then {vx, vy} (braced
  initialisers evaluate left to right), team ours then theirs, then the
  ball {x, y}; with ball_speed_max = 0 nothing else is drawn.

tests/test_synthetic.py checks the bytes against the compiled reference's
`ref_random_world` (oracle/ref_shim.cpp).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import abi

C5_SEED0 = 0xB200
_MASK = np.uint64(0xFFFFFFFFFFFFFFFF)
_N, _M = 312, 156
_UPPER = np.uint64(0xFFFFFFFF80000000)
_LOWER = np.uint64(0x000000007FFFFFFF)
_MATRIX_A = np.uint64(0xB5026F5AA96619E9)


def _mt19937_64_first_block(seeds: np.ndarray) -> np.ndarray:
    """The first 312 outputs of std::mt19937_64(seed) for every seed
    (shape [312, n]); one twist of the seeded state, then tempering."""
    n = seeds.shape[0]
    mt = np.empty((_N, n), dtype=np.uint64)
    mt[0] = seeds.astype(np.uint64)
    f = np.uint64(6364136223846793005)
    with np.errstate(over="ignore"):
        for i in range(1, _N):
            prev = mt[i - 1]
            mt[i] = f * (prev ^ (prev >> np.uint64(62))) + np.uint64(i)
        # twist (the engine's _M_gen_rand on first use)
        for i in range(_N):
            y = (mt[i] & _UPPER) | (mt[(i + 1) % _N] & _LOWER)
            v = mt[(i + _M) % _N] ^ (y >> np.uint64(1))
            v ^= np.where((y & np.uint64(1)) != 0, _MATRIX_A, np.uint64(0))
            mt[i] = v
    y = mt
    y = y ^ ((y >> np.uint64(29)) & np.uint64(0x5555555555555555))
    y = y ^ ((y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000))
    y = y ^ ((y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000))
    y = y ^ (y >> np.uint64(43))
    return y


def _uniform(words: np.ndarray, a: float, b: float) -> np.ndarray:
    """libstdc++ uniform_real_distribution<double>(a, b) of 64-bit words."""
    u = words.astype(np.float64) / 18446744073709551616.0  # 2^64, exact
    u = np.where(u >= 1.0, np.nextafter(1.0, 0.0), u)
    return (u * (b - a)) + a


def random_worlds(seeds, n_ours: int = 8, n_theirs: int = 8) -> np.ndarray:
    """oracles::random_world(mt19937_64(seed), n_ours, n_theirs) for each
    seed, as a numpy array of pp_world records (dtype of abi.World)."""
    seeds = np.asarray(seeds, dtype=np.uint64)
    n = seeds.shape[0]
    draws = 4 * (n_ours + n_theirs) + 2
    if draws > _N:
        raise ValueError("more draws than one engine block")
    w = _mt19937_64_first_block(seeds)[:draws]
    length, width = 12.0, 9.0  # FieldGeometry defaults (world.hpp:12-17)
    hx, hy = 0.5 * length, 0.5 * width
    out = np.zeros(n, dtype=np.dtype(abi.World))
    out["field"]["length"] = length
    out["field"]["width"] = width
    out["field"]["goal_width"] = 1.8
    out["field"]["defense_depth"] = 1.8
    out["field"]["defense_width"] = 3.6
    k = 0
    for team, count in (("ours", n_ours), ("theirs", n_theirs)):
        out["n_" + team] = count
        for j in range(count):
            r = out[team][:, j]
            r["id"] = j
            r["px"] = _uniform(w[k], -hx, hx)
            r["py"] = _uniform(w[k + 1], -hy, hy)
            r["vx"] = _uniform(w[k + 2], -2.0, 2.0)
            r["vy"] = _uniform(w[k + 3], -2.0, 2.0)
            out[team][:, j] = r
            k += 4
    out["ball_px"] = _uniform(w[k], -hx, hx)
    out["ball_py"] = _uniform(w[k + 1], -hy, hy)
    return out


def c5_frames(lo: int, hi: int) -> np.ndarray:
    """Frames [lo, hi) of the C5 batch (seed 0xB200 + i)."""
    return random_worlds(np.arange(lo, hi, dtype=np.uint64) + np.uint64(C5_SEED0))


def as_ctypes(frames: np.ndarray):
    """A ctypes (abi.World * n) view of a frames array (no copy)."""
    frames = np.ascontiguousarray(frames)
    return (abi.World * frames.shape[0]).from_buffer(frames), frames


def to_pinned(lib, frames: np.ndarray):
    """Copy frames into pinned host memory (pp_host_alloc); returns
    (ctypes array over the pinned bytes, pointer to free with pp_host_free)."""
    nbytes = frames.nbytes
    ptr = lib.pp_host_alloc(max(nbytes, 1))
    if not ptr:
        raise MemoryError("pp_host_alloc failed")
    C.memmove(ptr, frames.ctypes.data, nbytes)
    return (abi.World * frames.shape[0]).from_address(ptr), ptr

"""Shared by the CPU (oracle) and GPU (product) tests of the SURVEY §8(f)
rows: iterate the reference's golden cases in tests/golden/next_rows.npz and
compare a result struct field by field."""
from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

from paper_1909_07717_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
_G = None


def golden():
    global _G
    if _G is None:
        _G = np.load(os.path.join(HERE, "golden", "next_rows.npz"))
    return _G


def struct_from(cls, arr):
    return cls.from_buffer_copy(np.asarray(arr, dtype=np.uint8).tobytes())


def blob(g, key, cls):
    return struct_from(cls, g[str(g[key][0])])


def world_params(g, prefix):
    return blob(g, f"{prefix}/world", abi.World), blob(g, f"{prefix}/params", abi.Params)


def same(a, b, angle_rtol=0.0):
    """Field-by-field equality of two ctypes structs; doubles bit-exact
    (NaN == NaN), except fields named *angle* within angle_rtol (CUDA's
    atan2 vs glibc's, last ulp)."""
    bad = []
    for name, _ in type(a)._fields_:
        x, y = getattr(a, name), getattr(b, name)
        if isinstance(x, float):
            if "angle" in name and angle_rtol > 0.0:
                ok = abs(x - y) <= angle_rtol * max(1.0, abs(y))
            else:
                ok = x == y or (math.isnan(x) and math.isnan(y))
        else:
            ok = x == y
        if not ok:
            bad.append((name, x, y))
    return bad


def intercept_cases():
    g = golden()
    for cid in g["ic_cases"]:
        p = f"ic/{cid}"
        w, pm = world_params(g, p)
        yield (str(cid), w, pm, struct_from(abi.Kick, g[f"{p}/kick"]), float(g[f"{p}/dt"][0]),
               int(g[f"{p}/status"][0]), (abi.Intercept * 32).from_buffer_copy(g[f"{p}/out"].tobytes()))


def possession_cases():
    g = golden()
    for cid in g["po_cases"]:
        p = f"po/{cid}"
        w, pm = world_params(g, p)
        yield str(cid), w, pm, int(g[f"{p}/status"][0]), struct_from(abi.PossessionReport,
                                                                      g[f"{p}/out"])


def shot_cases():
    g = golden()
    for cid in g["sh_cases"]:
        p = f"sh/{cid}"
        w, pm = world_params(g, p)
        yield (str(cid), w, pm, int(g[f"{p}/shooter"][0]), int(g[f"{p}/status"][0]),
               struct_from(abi.ShotDecision, g[f"{p}/out"]))


def freekick_cases():
    g = golden()
    for cid in g["fk_cases"]:
        p = f"fk/{cid}"
        w, pm = world_params(g, p)
        yield (str(cid), w, pm, int(g[f"{p}/kicker"][0]), struct_from(abi.Candidate, g[f"{p}/cand"]),
               int(g[f"{p}/status"][0]), struct_from(abi.FreeKickPlan, g[f"{p}/out"]))

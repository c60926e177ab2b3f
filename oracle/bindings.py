"""TEST INFRASTRUCTURE ONLY: ctypes loaders for the two checkers.

* ``ref()``    -- oracle/_ref/libpassplan_ref.so: the unmodified reference
                  sources (/root/reference/proj/src) compiled by
                  oracle/Makefile plus ref_shim.cpp.
* ``oracle()`` -- oracle/liboracle.so: the plain-C restatement pp_oracle.c.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module.  The product path never does.
"""
from __future__ import annotations

import ctypes as C
import os

from paper_1909_07717_b200 import abi

ORACLE_DIR = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(ORACLE_DIR, "_ref", "libpassplan_ref.so")
ORACLE_LIB = os.path.join(ORACLE_DIR, "liboracle.so")

_P = C.POINTER
_dp = _P(C.c_double)
_vp = C.c_void_p

class OrCounts(C.Structure):
    """or_counts (oracle/pp_oracle.h): work terms of the reference's pruned scan."""
    _fields_ = [(n, C.c_uint64) for n in ("quick_rejects", "full_tests", "rest_evals", "scans",
                                          "bounds")]


_ref = None
_orc = None


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


def ref():
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_LIB)
        W, Pm, G = _P(abi.World), _P(abi.Params), _P(abi.SearchGrid)
        lib.ref_kernel_name.restype = C.c_char_p
        lib.ref_dpps.argtypes = [W, Pm, G, C.c_int32, C.c_int32, _vp, C.c_char_p, C.c_size_t]
        lib.ref_score_cells.argtypes = [W, Pm, C.c_int64, _dp, _dp, _dp, _dp, _P(C.c_uint8), _dp,
                                        _P(abi.PassFeatures), C.c_char_p, C.c_size_t]
        lib.ref_goal_views.argtypes = [W, C.c_double, C.c_int64, _dp, _dp, _dp, _dp, _dp, _dp]
        lib.ref_runmap_count.argtypes = [W, Pm, C.c_uint32]
        lib.ref_runmap_count.restype = C.c_int64
        lib.ref_runmap.argtypes = [W, Pm, _P(abi.RunmapRequest), _vp, C.c_int64, C.c_char_p,
                                   C.c_size_t]
        lib.ref_random_world.argtypes = [C.c_uint64, C.c_int32, C.c_int32, C.c_double, W]
        lib.ref_lattice_world.argtypes = [C.c_uint64, C.c_int32, C.c_int32, C.c_int32, W]
        lib.ref_mirror_world.argtypes = [W, W]
        lib.ref_load_snapshot.argtypes = [C.c_char_p, W, C.c_char_p, C.c_size_t]
        lib.ref_validate_world.argtypes = [W, C.c_char_p, C.c_size_t]
        lib.ref_validate_params.argtypes = [Pm, C.c_char_p, C.c_size_t]
        lib.ref_params_default.argtypes = [Pm]
        lib.ref_params_default.restype = None
        lib.ref_direction_table.argtypes = [C.c_int32, _dp]
        lib.ref_direction_table.restype = None
        lib.ref_nearest_teammate.argtypes = [W]
        lib.ref_nearest_teammate.restype = C.c_int32
        lib.ref_time_frame.argtypes = [W, Pm, G, C.c_int32, C.c_int32, C.c_int32, _dp, _dp,
                                       C.c_char_p, C.c_size_t]
        lib.ref_intercept_all.argtypes = [W, Pm, C.POINTER(abi.Kick), C.c_double,
                                          C.POINTER(abi.Intercept), C.c_char_p, C.c_size_t]
        lib.ref_scan_first.argtypes = [C.c_int64, C.POINTER(abi.ScanBatch),
                                       C.POINTER(abi.RobotKin), C.POINTER(C.c_int32)]
        lib.ref_json_check.argtypes = [C.c_int32, C.c_char_p, C.c_char_p, C.c_size_t]
        lib.ref_json_check.restype = C.c_int64
        lib.ref_csv_roundtrip.argtypes = [C.c_int32, C.c_char_p, C.c_char_p, C.c_size_t]
        lib.ref_csv_roundtrip.restype = C.c_int64
        lib.ref_guard_points.argtypes = [W, C.POINTER(abi.MotionLimits), C.c_double, C.c_int64,
                                         _dp, _dp, _dp, _dp, _P(C.c_uint8), C.c_char_p,
                                         C.c_size_t]
        lib.ref_possession.argtypes = [W, Pm, C.POINTER(abi.PossessionReport), C.c_char_p,
                                       C.c_size_t]
        lib.ref_decide_shot.argtypes = [W, Pm, C.c_int32, C.POINTER(abi.ShotDecision),
                                        C.c_char_p, C.c_size_t]
        lib.ref_plan_free_kick.argtypes = [W, Pm, C.c_int32, C.POINTER(abi.Candidate),
                                           C.POINTER(abi.FreeKickPlan), C.c_char_p, C.c_size_t]
        for fn in ("ref_grid_csv", "ref_pass_heatmap_csv"):
            getattr(lib, fn).argtypes = [W, Pm, C.c_int32, C.c_char_p, C.c_size_t]
            getattr(lib, fn).restype = C.c_int64
        lib.ref_run_heatmap_csv.argtypes = [W, Pm, C.c_uint32, C.c_char_p, C.c_size_t]
        lib.ref_run_heatmap_csv.restype = C.c_int64
        lib.ref_batch.argtypes = [W, C.c_int64, Pm, G, _P(C.c_int32), C.c_int32,
                                  _P(C.c_int64), _dp, _P(C.c_int64), _dp, C.c_char_p,
                                  C.c_size_t]
        _ref = lib
    return _ref


def oracle():
    """The plain-C restatement (same entry points, `or_` prefix)."""
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_LIB):
            raise RuntimeError(f"{ORACLE_LIB} missing: make -C oracle")
        lib = C.CDLL(ORACLE_LIB)
        W, Pm, G = _P(abi.World), _P(abi.Params), _P(abi.SearchGrid)
        lib.or_params_default.argtypes = [Pm]
        lib.or_params_default.restype = None
        lib.or_dpps.argtypes = [W, Pm, G, C.c_int32, _vp, C.c_char_p, C.c_size_t]
        lib.or_score_cells.argtypes = [W, Pm, C.c_int64, _dp, _dp, _dp, _dp, _P(C.c_uint8), _dp,
                                       _P(abi.PassFeatures), C.c_char_p, C.c_size_t]
        lib.or_goal_views.argtypes = [W, C.c_double, C.c_int64, _dp, _dp, _dp, _dp, _dp, _dp]
        lib.or_runmap_count.argtypes = [W, Pm, C.c_uint32]
        lib.or_runmap_count.restype = C.c_int64
        lib.or_runmap.argtypes = [W, Pm, _P(abi.RunmapRequest), _vp, C.c_int64, C.c_char_p,
                                  C.c_size_t]
        lib.or_intercept_all.argtypes = [W, Pm, _P(abi.Kick), C.c_double, _P(abi.Intercept),
                                         C.c_char_p, C.c_size_t]
        lib.or_possession.argtypes = [W, Pm, _P(abi.PossessionReport), C.c_char_p, C.c_size_t]
        lib.or_decide_shot.argtypes = [W, Pm, C.c_int32, _P(abi.ShotDecision), C.c_char_p,
                                       C.c_size_t]
        lib.or_plan_free_kick.argtypes = [W, Pm, C.c_int32, _P(abi.Candidate),
                                          _P(abi.FreeKickPlan), C.c_char_p, C.c_size_t]
        lib.or_direction_table.argtypes = [C.c_int32, _dp]
        lib.or_direction_table.restype = None
        lib.or_nearest_teammate.argtypes = [W]
        lib.or_nearest_teammate.restype = C.c_int32
        lib.or_dpps_counted.argtypes = [W, Pm, G, C.c_int32, _vp, _P(OrCounts), C.c_char_p,
                                        C.c_size_t]
        for fn in ("or_dpps", "or_dpps_counted", "or_score_cells", "or_goal_views", "or_runmap"):
            getattr(lib, fn).restype = C.c_int
        _orc = lib
    return _orc


def msgbuf():
    return C.create_string_buffer(512)

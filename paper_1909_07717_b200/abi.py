"""ctypes mirror of include/passplan_b200.h (the C-ABI boundary).

Pure data definitions plus the loader of the product library.  The struct
field order must match the header exactly; tests/test_abi.py checks sizes
against the compiled library.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PP_MAX_TEAM = 16
PP_OK, PP_SCHEMA, PP_VALIDATION, PP_CONFIG, PP_DOMAIN, PP_INTERNAL, PP_CUDA = range(7)
STATUS_NAMES = {0: "ok", 1: "schema", 2: "validation", 3: "config", 4: "domain",
                5: "internal", 6: "cuda"}
PP_COPY_SUMMARY = 0
PP_COPY_ALL = 1
PP_OPT_EXACT_ONLY = 1

_D = C.c_double
_I = C.c_int32


class Field(C.Structure):
    _fields_ = [("length", _D), ("width", _D), ("goal_width", _D), ("defense_depth", _D),
                ("defense_width", _D)]


class Robot(C.Structure):
    _fields_ = [("id", _I), ("reserved", _I), ("px", _D), ("py", _D), ("vx", _D), ("vy", _D),
                ("theta", _D)]


class World(C.Structure):
    _fields_ = [("field", Field), ("ball_px", _D), ("ball_py", _D), ("ball_vx", _D),
                ("ball_vy", _D), ("n_ours", _I), ("n_theirs", _I),
                ("ours", Robot * PP_MAX_TEAM), ("theirs", Robot * PP_MAX_TEAM)]


class BallModel(C.Structure):
    _fields_ = [(n, _D) for n in ("slide_decel", "roll_decel", "transition_ratio", "power_min",
                                  "power_max", "chip_flight_fraction")]


class MotionLimits(C.Structure):
    _fields_ = [(n, _D) for n in ("max_speed", "max_accel", "max_decel")]


class SearchGrid(C.Structure):
    _fields_ = [("n_directions", _I), ("n_powers", _I), ("power_min", _D), ("power_max", _D),
                ("flat", _I), ("chip", _I)]


class PassWeights(C.Structure):
    _fields_ = [(n, _D) for n in ("teammate_time", "shoot_angle", "dist_goal", "refraction",
                                  "margin")]


class RunWeights(C.Structure):
    _fields_ = [(n, _D) for n in ("dist_goal", "dist_ball", "angle", "guard_time", "exposure")]


class NormBounds(C.Structure):
    _fields_ = [("length_upper", _D), ("angle_upper", _D)]


class AngleBand(C.Structure):
    _fields_ = [(n, _D) for n in ("full_lo", "peak_lo", "peak_hi", "full_hi")]


THRESHOLD_NAMES = ("sbip_dt", "robot_radius", "safety_margin", "buffer_time", "possession_radius",
                   "angle_threshold", "shot_power", "margin_cap", "possession_dt",
                   "contest_epsilon", "grid_step", "min_zone_width", "guard_time_cap",
                   "drag_v_min", "marking_radius")


class Thresholds(C.Structure):
    _fields_ = [(n, _D) for n in THRESHOLD_NAMES]


class Params(C.Structure):
    _fields_ = [("ball", BallModel), ("motion_ours", MotionLimits),
                ("motion_theirs", MotionLimits), ("grid", SearchGrid),
                ("pass_weights", PassWeights), ("run_weights", RunWeights),
                ("norm", NormBounds), ("angle_band", AngleBand), ("thresholds", Thresholds)]


class PassFeatures(C.Structure):
    _fields_ = [(n, _D) for n in ("teammate_intercept_time", "shoot_angle_at_receive",
                                  "dist_receive_to_goal", "refraction_angle",
                                  "intercept_margin")]


class DppsSummary(C.Structure):
    _fields_ = [("n_cells", C.c_int64), ("n_kick_types", _I), ("kick_types", _I * 2),
                ("n_directions", _I), ("n_powers", _I), ("kicker_id", _I), ("kicker_slot", _I),
                ("kicker_in_possession", _I), ("n_ours", _I), ("n_theirs", _I),
                ("ours_ids", _I * PP_MAX_TEAM), ("theirs_ids", _I * PP_MAX_TEAM),
                ("sbip_calls", C.c_uint64), ("n_feasible", C.c_int64 * 3),
                ("best_cell", C.c_int64 * 3), ("best_score", _D * 3),
                ("best_features", PassFeatures * 3), ("device_ms", _D)]


class FrameSummary(C.Structure):  # pp_frame_summary (48 B per frame)
    _fields_ = [("best_score", _D * 3), ("best_cell", _I * 3), ("n_feasible", _I * 3)]


class RobotKin(C.Structure):  # pp_robot_kin (kernels::RobotKin)
    _fields_ = [(n, _D) for n in ("px", "py", "vx", "vy", "accel", "decel", "vmax", "radius",
                                  "vbound")]


class ScanBatch(C.Structure):  # pp_scan_batch (kernels::ScanBatch)
    _fields_ = [("ts", C.POINTER(_D)), ("ss", C.POINTER(_D)), ("k_begin", _I), ("k_end", _I),
                ("ox", _D), ("oy", _D), ("ux", _D), ("uy", _D)]


class RunFeatures(C.Structure):
    _fields_ = [(n, _D) for n in ("dist_to_goal", "dist_to_ball", "angle_to_goal", "guard_time",
                                  "defense_exposure")]


class RunningPoint(C.Structure):
    _fields_ = [("zone", _I), ("valid", _I), ("px", _D), ("py", _D), ("score", _D),
                ("features", RunFeatures)]


class RunmapSummary(C.Structure):
    _fields_ = [("cut_x", _D), ("cut_y", _D), ("zone_nx", _I * 4), ("zone_ny", _I * 4),
                ("zone_offset", C.c_int64 * 4), ("n_vertices", C.c_int64),
                ("n_scorable", C.c_int64), ("best", RunningPoint * 4), ("n_best", _I),
                ("best_order", _I * 4)]


class RunmapRequest(C.Structure):
    _fields_ = [("zone_mask", C.c_uint32), ("occupied_mask", C.c_uint32), ("n_runners", _I),
                ("has_best_pass_point", _I), ("best_pass_px", _D), ("best_pass_py", _D),
                ("want_map", _I)]


class Kick(C.Structure):  # pp_kick
    _fields_ = [("origin_x", _D), ("origin_y", _D), ("dir_x", _D), ("dir_y", _D), ("speed", _D),
                ("kind", _I), ("pad", _I)]


class Trajectory(C.Structure):  # pp_trajectory
    _fields_ = [(n, _D) for n in ("origin_x", "origin_y", "dir_x", "dir_y", "kick_speed", "v1",
                                  "slide_decel", "roll_decel", "slide_end_time",
                                  "slide_end_distance", "stop_time", "stop_distance",
                                  "interceptable_from")] + [("kick_type", _I), ("pad", _I)]


class Intercept(C.Structure):  # pp_intercept
    _fields_ = [("team", _I), ("robot_id", _I), ("finite", _I), ("pad", _I), ("time", _D),
                ("point_x", _D), ("point_y", _D)]


class PossessionReport(C.Structure):  # pp_possession_report
    _fields_ = [("side", _I), ("has_our", _I), ("has_their", _I), ("pad", _I),
                ("our_time", _D), ("their_time", _D)]


class ShotDecision(C.Structure):  # pp_shot_decision
    _fields_ = [("shoot", _I), ("blocked", _I), ("reason", _I), ("pad", _I),
                ("shot_angle", _D), ("target_x", _D), ("target_y", _D)]


class Candidate(C.Structure):  # pp_candidate
    _fields_ = [("kick_type", _I), ("dir_index", _I), ("power_index", _I), ("our_id", _I),
                ("opp_id", _I), ("feasible", _I), ("our_time", _D), ("opp_time", _D),
                ("receive_x", _D), ("receive_y", _D)]


class FreeKickPlan(C.Structure):  # pp_free_kick_plan
    _fields_ = [("t_ball", _D), ("t_robot", _D), ("order", _I), ("pad", _I),
                ("kick_delay", _D)]


# ---------------------------------------------------------------------------
# Result block layouts (mirror include/passplan_b200_layout.h).

def _a16(x: int) -> int:
    return (x + 15) & ~15


def grid_offsets(n_cells: int) -> dict:
    n = max(n_cells, 0)
    at = 0
    off = {}
    for name, size in (("summary", C.sizeof(DppsSummary)), ("our_time", 8 * n),
                       ("opp_time", 8 * n), ("rx", 8 * n), ("ry", 8 * n), ("score", 4 * n),
                       ("our_slot", n), ("opp_slot", n), ("feasible", n)):
        off[name] = at
        at = _a16(at + size)
    off["total"] = at
    return off


def runmap_offsets(n_vertices: int) -> dict:
    n = max(n_vertices, 0)
    at = 0
    off = {}
    for name, size in (("summary", C.sizeof(RunmapSummary)), ("px", 8 * n), ("py", 8 * n),
                       ("score", 8 * n), ("features", C.sizeof(RunFeatures) * n),
                       ("scorable", n)):
        off[name] = at
        at = _a16(at + size)
    off["total"] = at
    return off


class GridBlock:
    """Typed numpy views into a grid result block (bytes owned by `buf`)."""

    def __init__(self, n_cells: int, buf=None):
        self.n_cells = n_cells
        off = grid_offsets(n_cells)
        self.nbytes = off["total"]
        self.buf = buf if buf is not None else np.zeros(self.nbytes, dtype=np.uint8)
        b = self.buf
        n = n_cells
        self.summary = DppsSummary.from_buffer(b, off["summary"]) if isinstance(b, np.ndarray) \
            else DppsSummary.from_address(C.addressof(b) + off["summary"])
        mk = lambda name, dt, k: np.frombuffer(b, dtype=dt, count=k, offset=off[name])  # noqa
        self.our_time = mk("our_time", np.float64, n)
        self.opp_time = mk("opp_time", np.float64, n)
        self.rx = mk("rx", np.float64, n)
        self.ry = mk("ry", np.float64, n)
        self.score = mk("score", np.float32, n)
        self.our_slot = mk("our_slot", np.int8, n)
        self.opp_slot = mk("opp_slot", np.int8, n)
        self.feasible = mk("feasible", np.uint8, n)

    def ptr(self):
        if isinstance(self.buf, np.ndarray):
            return self.buf.ctypes.data_as(C.c_void_p)
        return C.cast(self.buf, C.c_void_p)

    def ids(self):
        """(our_id, opp_id) arrays with the reference's -1 convention."""
        s = self.summary
        ours = np.array(list(s.ours_ids[:max(s.n_ours, 0)]) + [-1], dtype=np.int64)
        theirs = np.array(list(s.theirs_ids[:max(s.n_theirs, 0)]) + [-1], dtype=np.int64)
        return ours[self.our_slot.astype(np.int64)], theirs[self.opp_slot.astype(np.int64)]


class RunmapBlock:
    def __init__(self, n_vertices: int):
        self.n_vertices = n_vertices
        off = runmap_offsets(n_vertices)
        self.nbytes = off["total"]
        self.buf = np.zeros(self.nbytes, dtype=np.uint8)
        b = self.buf
        n = n_vertices
        self.summary = RunmapSummary.from_buffer(b, off["summary"])
        self.px = np.frombuffer(b, np.float64, n, off["px"])
        self.py = np.frombuffer(b, np.float64, n, off["py"])
        self.score = np.frombuffer(b, np.float64, n, off["score"])
        self.features = np.frombuffer(b, np.float64, 5 * n, off["features"]).reshape(n, 5)
        self.scorable = np.frombuffer(b, np.uint8, n, off["scorable"])

    def ptr(self):
        return self.buf.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------------------
# Product library loader.

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "lib", "libpassplan_b200.so")

_P = C.POINTER


def _declare(lib):
    vp = C.c_void_p
    lib.pp_params_default.argtypes = [_P(Params)]
    lib.pp_params_default.restype = None
    lib.pp_params_validate.argtypes = [_P(Params), C.c_char_p, C.c_size_t]
    lib.pp_grid_bytes.argtypes = [C.c_int64]
    lib.pp_grid_bytes.restype = C.c_size_t
    lib.pp_grid_cells.argtypes = [_P(SearchGrid)]
    lib.pp_grid_cells.restype = C.c_int64
    lib.pp_ctx_create.argtypes = [C.c_int, _P(vp)]
    lib.pp_ctx_set_option.argtypes = [vp, _I, _I]
    lib.pp_ctx_set_option.restype = C.c_int
    lib.pp_ctx_destroy.argtypes = [vp]
    lib.pp_ctx_destroy.restype = None
    lib.pp_last_error.argtypes = [vp]
    lib.pp_last_error.restype = C.c_char_p
    lib.pp_kernel_name.restype = C.c_char_p
    lib.pp_host_alloc.argtypes = [C.c_size_t]
    lib.pp_host_alloc.restype = vp
    lib.pp_dpps_upload_bytes.argtypes = []
    lib.pp_dpps_upload_bytes.restype = C.c_size_t
    lib.pp_host_free.argtypes = [vp]
    lib.pp_host_free.restype = None
    lib.pp_dpps.argtypes = [vp, _P(World), _P(Params), _P(SearchGrid), _I, C.c_uint32, vp]
    lib.pp_dpps_relaunch.argtypes = [vp]
    lib.pp_dpps_kernel_times.argtypes = [vp, _I, _P(C.c_float), _P(C.c_float)]
    lib.pp_dpps_kernel_times.restype = C.c_int
    lib.pp_ctx_stream.argtypes = [vp]
    lib.pp_ctx_stream.restype = vp
    dp = _P(C.c_double)
    lib.pp_score_cells.argtypes = [vp, _P(World), _P(Params), C.c_int64, dp, dp, dp, dp,
                                   _P(C.c_uint8), dp, _P(PassFeatures)]
    lib.pp_goal_views.argtypes = [vp, _P(World), C.c_double, C.c_int64, dp, dp, dp, dp, dp, dp]
    lib.pp_runmap_count.argtypes = [_P(World), _P(Params), C.c_uint32, _P(C.c_int64)]
    lib.pp_runmap.argtypes = [vp, _P(World), _P(Params), _P(RunmapRequest), vp, C.c_int64]
    lib.pp_score_running_points.argtypes = [vp, _P(World), _P(Params), C.c_int64, dp, dp, dp,
                                            _P(RunFeatures), _P(C.c_uint8)]
    lib.pp_score_running_points.restype = C.c_int
    lib.pp_guard_points.argtypes = [vp, _P(World), _P(MotionLimits), C.c_double, C.c_int64, dp,
                                    dp, dp, dp, _P(C.c_uint8)]
    lib.pp_guard_points.restype = C.c_int
    lib.pp_scan_first.argtypes = [vp, C.c_int64, _P(ScanBatch), _P(RobotKin), _P(C.c_int32)]
    lib.pp_scan_first.restype = C.c_int
    lib.pp_dpps_batch.argtypes = [vp, _P(World), C.c_int64, _P(Params), _P(SearchGrid),
                                  _P(C.c_int32), _P(DppsSummary)]
    lib.pp_batch_upload.argtypes = [vp, _P(World), C.c_int64, _P(C.c_int32)]
    lib.pp_batch_run.argtypes = [vp, _P(Params), _P(SearchGrid), _P(C.c_float)]
    lib.pp_batch_download.argtypes = [vp, _P(FrameSummary)]
    lib.pp_dpps_frames.argtypes = [vp, _P(World), C.c_int64, _P(Params), _P(SearchGrid),
                                   _P(C.c_int32), _P(FrameSummary)]
    lib.pp_dpps_frames_multi.argtypes = [_P(vp), C.c_int32, _P(World), C.c_int64, _P(Params),
                                         _P(SearchGrid), _P(C.c_int32), _P(FrameSummary)]
    fp = _P(C.c_float)
    lib.pp_batch_kernel_times.argtypes = [vp, _P(Params), _P(SearchGrid), _I, fp, fp, fp,
                                          _P(C.c_int32)]
    lib.pp_kick_trajectory.argtypes = [_P(Kick), _P(BallModel), _P(Trajectory), C.c_char_p,
                                       C.c_size_t]
    lib.pp_kick_trajectory.restype = C.c_int
    lib.pp_intercept_all.argtypes = [vp, _P(World), _P(Params), _P(Trajectory), C.c_double,
                                     _P(Intercept)]
    lib.pp_possession.argtypes = [vp, _P(World), _P(Params), _P(PossessionReport)]
    lib.pp_decide_shot.argtypes = [vp, _P(World), _P(Params), _I, _P(ShotDecision)]
    lib.pp_plan_free_kick.argtypes = [vp, _P(World), _P(Params), _I, _P(Candidate),
                                      _P(FreeKickPlan)]
    for fn in ("pp_params_validate", "pp_ctx_create", "pp_dpps", "pp_dpps_relaunch", "pp_score_cells",
               "pp_goal_views", "pp_runmap_count", "pp_runmap", "pp_dpps_batch",
               "pp_batch_upload", "pp_batch_run", "pp_batch_download", "pp_dpps_frames",
               "pp_dpps_frames_multi", "pp_batch_kernel_times", "pp_intercept_all",
               "pp_possession", "pp_decide_shot", "pp_plan_free_kick"):
        getattr(lib, fn).restype = C.c_int
    return lib


_LIB = None


def load_library(path: str = LIB_PATH):
    """Load the product C-ABI library.  Raises if it is missing: there is no
    CPU fallback for the product path."""
    global _LIB
    if _LIB is None:
        path = os.environ.get("PP_LIB_PATH", path)  # dev override (variant builds)
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build() (no CPU fallback)")
        _LIB = _declare(C.CDLL(path))
    return _LIB


EXPORTED_SYMBOLS = (
    "pp_params_default", "pp_params_validate", "pp_grid_bytes", "pp_grid_view_of",
    "pp_runmap_bytes", "pp_runmap_view_of", "pp_runmap_count", "pp_ctx_create",
    "pp_ctx_destroy", "pp_ctx_set_option", "pp_last_error", "pp_kernel_name", "pp_abi_version",
    "pp_dpps_upload_bytes", "pp_host_alloc",
    "pp_host_free", "pp_dpps", "pp_dpps_relaunch", "pp_ctx_stream", "pp_dpps_kernel_times",
    "pp_grid_cells", "pp_score_cells", "pp_goal_views", "pp_runmap",
    "pp_dpps_batch", "pp_batch_upload", "pp_batch_run", "pp_batch_download", "pp_dpps_frames",
    "pp_dpps_frames_multi", "pp_batch_kernel_times",
    "pp_score_running_points", "pp_kick_trajectory", "pp_intercept_all", "pp_possession",
    "pp_decide_shot", "pp_plan_free_kick", "pp_guard_points", "pp_scan_first",
)

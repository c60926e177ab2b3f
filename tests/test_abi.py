"""CPU: the C-ABI boundary -- the product library loads, exports every entry
point include/passplan_b200.h declares, its structs match the ctypes mirror,
and the host-side logic (validation, layouts, lattice counts) behaves like
the reference.  No compute calls here: there is no GPU in the CPU suite."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1909_07717_b200 import abi
from tests.helpers import case_inputs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "passplan_b200.h")


@pytest.fixture(scope="module")
def lib():
    return abi.load_library()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pp_[a-z0-9_]+)\s*\(", src)) - {"pp_status"})


def test_library_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(abi.EXPORTED_SYMBOLS) <= set(names)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", abi.LIB_PATH], capture_output=True,
                         text=True)
    assert "sm_100a" in out.stdout, out.stdout + out.stderr


STRUCTS = {"pp_world": abi.World, "pp_params": abi.Params, "pp_search_grid": abi.SearchGrid,
           "pp_dpps_summary": abi.DppsSummary, "pp_runmap_summary": abi.RunmapSummary,
           "pp_runmap_request": abi.RunmapRequest, "pp_pass_features": abi.PassFeatures,
           "pp_robot": abi.Robot, "pp_thresholds": abi.Thresholds,
           "pp_frame_summary": abi.FrameSummary, "pp_robot_kin": abi.RobotKin,
           "pp_scan_batch": abi.ScanBatch}


def test_struct_layouts_match_header(tmp_path):
    prog = tmp_path / "sizes.c"
    body = "\n".join(f'  printf("{k} %zu\\n", sizeof({k}));' for k in STRUCTS)
    prog.write_text(f'#include <stdio.h>\n#include "passplan_b200.h"\nint main(void){{\n{body}\n'
                    f'  printf("best_score %zu\\n", offsetof(pp_dpps_summary, best_score));\n'
                    f'  return 0;}}\n')
    exe = tmp_path / "sizes"
    subprocess.run(["gcc", "-std=c11", "-include", "stddef.h", "-I", os.path.join(ROOT, "include"),
                    str(prog), "-o", str(exe)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True,
                                                       text=True).stdout.split("\n") if line)
    for k, cls in STRUCTS.items():
        assert int(got[k]) == C.sizeof(cls), k
    assert int(got["best_score"]) == abi.DppsSummary.best_score.offset


def test_grid_layout_matches_python(lib):
    for n in (0, 1, 33, 8192, 16384, 1080000):
        assert lib.pp_grid_bytes(n) == abi.grid_offsets(n)["total"]


def test_params_default_and_validate(lib):
    p = abi.Params()
    lib.pp_params_default(C.byref(p))
    assert p.grid.n_directions == 128 and p.grid.n_powers == 64
    assert p.thresholds.sbip_dt == 1.0 / 60.0 and p.thresholds.safety_margin == 0.3
    assert p.ball.transition_ratio == 5.0 / 7.0
    g = np.load(os.path.join(ROOT, "tests", "golden", "default_params.npy"))
    assert bytes(p) == g.tobytes()  # identical to the reference's PlannerConfig{}
    m = C.create_string_buffer(256)
    assert lib.pp_params_validate(C.byref(p), m, 256) == abi.PP_OK
    bad = abi.Params.from_buffer_copy(bytes(p))
    bad.ball.roll_decel = 5.0   # slide_decel > roll_decel violated (ball_model.cpp:48)
    assert lib.pp_params_validate(C.byref(bad), m, 256) == abi.PP_CONFIG
    assert b"slide_decel" in m.value
    bad = abi.Params.from_buffer_copy(bytes(p))
    bad.grid.power_min = 3.0
    bad.grid.power_max = 2.0
    assert lib.pp_params_validate(C.byref(bad), m, 256) == abi.PP_CONFIG
    bad = abi.Params.from_buffer_copy(bytes(p))
    bad.angle_band.peak_lo = 2.0
    assert lib.pp_params_validate(C.byref(bad), m, 256) == abi.PP_CONFIG


def test_grid_cells(lib):
    for g, want in ((abi.SearchGrid(128, 64, 1.0, 6.5, 1, 1), 16384),
                    (abi.SearchGrid(128, 64, 1.0, 6.5, 1, 0), 8192),
                    (abi.SearchGrid(1200, 900, 1.0, 6.5, 1, 0), 1080000),
                    (abi.SearchGrid(0, 64, 1.0, 6.5, 1, 1), 0),
                    (abi.SearchGrid(8, 8, 1.0, 6.5, 0, 0), 0)):
        assert lib.pp_grid_cells(C.byref(g)) == want


def test_runmap_counts_match_reference(lib, runmaps_golden):
    from tests.helpers import struct_from
    g = runmaps_golden
    for name in [str(c) for c in g["cases"]]:
        w = struct_from(abi.World, g[f"{name}/world"])
        p = struct_from(abi.Params, g[f"{name}/params"])
        req = struct_from(abi.RunmapRequest, g[f"{name}/req"])
        want = struct_from(abi.RunmapSummary, g[f"{name}/summary"])
        nv = C.c_int64()
        assert lib.pp_runmap_count(C.byref(w), C.byref(p), req.zone_mask, C.byref(nv)) == 0
        assert nv.value == want.n_vertices, name
    # test_offball.cpp:88-96: 3 x 2 m zone III at 0.1 m -> 31 x 21 vertices
    w = abi.World()
    w.field = abi.Field(12.0, 9.0, 1.8, 1.8, 3.6)
    w.ball_py = 2.5
    p = abi.Params()
    lib.pp_params_default(C.byref(p))
    nv = C.c_int64()
    assert lib.pp_runmap_count(C.byref(w), C.byref(p), 0x4, C.byref(nv)) == 0
    assert nv.value == 31 * 21


def test_context_without_gpu_fails_loudly(lib):
    """The product has no CPU fallback: without a device, create fails."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    assert lib.pp_ctx_create(0, C.byref(h)) == abi.PP_CUDA
    assert not h.value


def test_kernel_name(lib):
    assert lib.pp_kernel_name() == b"sm100a"
    assert lib.pp_abi_version() == 1


def test_world_struct_roundtrip(grids_golden):
    w, p, grid, k, st = case_inputs(grids_golden, "bench16")
    assert w.n_ours == 16 and w.n_theirs == 16 and st == 0
    assert grid.n_directions == 128 and grid.n_powers == 64


def test_cpp_dropin_exports_reference_api():
    """lib/libpassplan.so exports the reference's hot-path C++ entry points."""
    from paper_1909_07717_b200 import build as b
    lib = b.build_dropin()
    out = subprocess.run(["nm", "-DC", "--defined-only", lib], capture_output=True,
                         text=True).stdout
    for sym in ("passplan::run_dpps(", "passplan::run_dpps_serial(", "passplan::best_pass(",
                "passplan::score_pass(", "passplan::goal_view(", "passplan::shoot_angle(",
                "passplan::score_running_point(", "passplan::best_running_points(",
                "passplan::zone_lattice(", "passplan::partition_zones(",
                "passplan::direction_table(", "passplan::power_table(",
                "passplan::grids_identical(", "passplan::feasible_candidates(",
                "passplan::PlannerConfig::validate() const", "passplan::best_pass_batch(",
                "passplan::decide_shot(", "passplan::possession(", "passplan::intercept_all(",
                "passplan::intercept_time(", "passplan::plan_free_kick(",
                "passplan::pass_power_for(", "passplan::BallTrajectory::flat_kick(",
                "passplan::grid_to_csv", "passplan::grid_from_csv(", "passplan::heatmap_to_csv",
                "passplan::run_heatmap_to_csv", "passplan::load_world_snapshot(",
                "passplan::PlannerConfig::load("):
        assert sym in out, sym

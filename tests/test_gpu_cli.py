"""GPU: the `passplan_b200` CLI (bin/, reference passplan_main.cpp:82-279)
end to end on JSON snapshots written from the golden worlds: `plan --out`
writes the reference's grid CSV byte for byte (csv.cpp:85-114), `heatmap
--mode pass|run` its heat maps (coordinates, times, distances bit-exact;
atan2-derived angle/score columns within SCORE_RTOL), plus the other
commands' stdout and the error exit codes."""
import json
import math
import os
import subprocess

import numpy as np
import pytest

from paper_1909_07717_b200 import abi
from paper_1909_07717_b200 import build as B
from tests.helpers import SCORE_RTOL
from tests.next_rows import blob, golden

pytestmark = pytest.mark.gpu


def snapshot_json(w: abi.World) -> str:
    team = lambda rs, n: [{"id": rs[i].id, "x": rs[i].px, "y": rs[i].py, "vx": rs[i].vx,  # noqa
                           "vy": rs[i].vy, "theta": rs[i].theta} for i in range(n)]
    return json.dumps({"field": {"length": w.field.length, "width": w.field.width,
                                 "goal_width": w.field.goal_width,
                                 "defense_depth": w.field.defense_depth,
                                 "defense_width": w.field.defense_width},
                       "ball": {"x": w.ball_px, "y": w.ball_py, "vx": w.ball_vx, "vy": w.ball_vy},
                       "ours": team(w.ours, w.n_ours), "theirs": team(w.theirs, w.n_theirs)})


def config_json(p: abi.Params) -> str:
    sec = lambda s: {n: getattr(s, n) for n, _ in type(s)._fields_}  # noqa
    g = sec(p.grid)
    g["flat"], g["chip"] = bool(g["flat"]), bool(g["chip"])
    return json.dumps({"ball": sec(p.ball), "motion_ours": sec(p.motion_ours),
                       "motion_theirs": sec(p.motion_theirs), "grid": g,
                       "pass_weights": sec(p.pass_weights), "run_weights": sec(p.run_weights),
                       "norm": sec(p.norm), "angle_band": sec(p.angle_band),
                       "thresholds": sec(p.thresholds)})


@pytest.fixture(scope="module")
def cli():
    if not os.path.exists(B.CLI):
        pytest.fail(f"{B.CLI} missing: run __graft_entry__.build()")
    return B.CLI


def run(cli, *args):
    return subprocess.run([cli, *args], capture_output=True, text=True, timeout=120)


def rows(text):
    return [line.split(",") for line in text.strip().split("\n")]


def close_rows(got, want, approx_cols):
    assert got[0] == want[0] and len(got) == len(want)
    for g, w in zip(got[1:], want[1:]):
        for k, (a, b) in enumerate(zip(g, w)):
            if k in approx_cols:
                assert math.isclose(float(a), float(b), rel_tol=SCORE_RTOL, abs_tol=SCORE_RTOL), (a, b)
            else:
                assert a == b, (k, a, b)


@pytest.mark.parametrize("name", ["minimal", "f8", "marked", "unmarked", "rand8v8_0",
                                  "ball_outside"])
def test_cli_csv_matches_reference(cli, tmp_path, name):
    g = golden()
    w = blob(g, f"csv/{name}/world", abi.World)
    p = blob(g, f"csv/{name}/params", abi.Params)
    k = int(g[f"csv/{name}/kicker"][0])
    snap, cfg = tmp_path / "s.json", tmp_path / "c.json"
    snap.write_text(snapshot_json(w))
    cfg.write_text(config_json(p))
    common = ["--snapshot", str(snap), "--config", str(cfg)]
    r = run(cli, "plan", *common, "--kicker", str(k), "--out", str(tmp_path / "grid.csv"))
    assert r.returncode == 0, r.stderr  # (ball_outside: off the field, inside the apron)
    assert r.stdout.startswith("kernel=sm100a workers=")
    assert (tmp_path / "grid.csv").read_bytes() == bytes(g[f"csv/{name}/grid"])
    r = run(cli, "heatmap", *common, "--mode", "pass", "--kicker", str(k), "--out",
            str(tmp_path / "pass.csv"))
    assert r.returncode == 0, r.stderr
    close_rows(rows((tmp_path / "pass.csv").read_text()), rows(bytes(g[f"csv/{name}/pass"]).decode()),
               approx_cols={2})
    r = run(cli, "heatmap", *common, "--mode", "run", "--zone", "all")
    assert r.returncode == 0, r.stderr
    close_rows(rows(r.stdout), rows(bytes(g[f"csv/{name}/run"]).decode()), approx_cols={4, 7})


def test_cli_other_commands(cli, tmp_path):
    g = golden()
    w = blob(g, "csv/f8/world", abi.World)
    p = blob(g, "csv/f8/params", abi.Params)
    snap, cfg = tmp_path / "s.json", tmp_path / "c.json"
    snap.write_text(snapshot_json(w))
    cfg.write_text(config_json(p))
    r = run(cli, "plan", "--snapshot", str(snap), "--config", str(cfg), "--freekick")
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().split("\n")
    assert lines[1].startswith("feasible: flat=") and any(l.startswith("shot: ") for l in lines)
    assert any(l.startswith("run zone ") for l in lines)
    r = run(cli, "possession", "--snapshot", str(snap))
    assert r.returncode == 0 and r.stdout.startswith("possession: "), r.stderr
    r = run(cli, "freekick", "--snapshot", str(snap), "--config", str(cfg))
    assert r.returncode == 0 and "freekick: t_ball=" in r.stdout, r.stderr
    r = run(cli, "bench", "--snapshot", str(snap), "--config", str(cfg), "--reps", "2",
            "--workers-list", "1", "4")
    assert r.returncode == 0 and "workers=4: median=" in r.stdout, r.stderr
    # error categories -> the reference's exit codes (errors.hpp)
    bad = tmp_path / "bad.json"
    bad.write_text('{"grid": {"n_directions": 0}}')
    r = run(cli, "plan", "--snapshot", str(snap), "--config", str(bad))
    assert r.returncode == 3 and "error (config)" in r.stderr
    r = run(cli, "plan", "--snapshot", str(snap), "--kicker", "77")
    assert r.returncode == 2 and "error (validation)" in r.stderr
    (tmp_path / "broken.json").write_text("{")
    r = run(cli, "plan", "--snapshot", str(tmp_path / "broken.json"))
    assert r.returncode == 2 and "error (schema)" in r.stderr

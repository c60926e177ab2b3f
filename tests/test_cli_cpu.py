"""CPU: the `passplan_b200` CLI's argument, snapshot and config handling,
which runs before any device work: JSON schema / config errors map to the
reference's error categories and exit codes (errors.hpp, snapshot.cpp,
config.cpp:14-241, passplan_main.cpp:293-342)."""
import json
import subprocess

import pytest

from paper_1909_07717_b200 import build as B

SNAP = {"field": {"length": 12.0, "width": 9.0, "goal_width": 1.8, "defense_depth": 1.8,
                  "defense_width": 3.6},
        "ball": {"x": 0.0, "y": 0.0, "vx": 0.0, "vy": 0.0},
        "ours": [{"id": 0, "x": -0.1, "y": 0.0, "vx": 0.0, "vy": 0.0, "theta": 0.0}],
        "theirs": []}


@pytest.fixture(scope="module")
def cli():
    return B.build_cli()


def run(cli, *args):
    return subprocess.run([cli, *args], capture_output=True, text=True, timeout=60)


def test_cli_usage_errors(cli):
    assert run(cli).returncode == 1
    assert run(cli, "nosuch").returncode == 1
    assert run(cli, "plan").returncode == 1  # --snapshot is required
    assert run(cli, "heatmap", "--snapshot", "x.json").returncode == 1  # --mode is required
    assert run(cli, "--help").returncode == 0


@pytest.mark.parametrize("mutate,category,code", [
    (lambda s: s.update(extra=1), "schema", 2),                          # unknown top-level key
    (lambda s: s["ball"].pop("vx"), "schema", 2),                        # missing key
    (lambda s: s["ours"][0].update(id=1.5), "schema", 2),                # id must be an integer
    (lambda s: s["ball"].update(x=50.0), "validation", 2),               # ball outside the field
    (lambda s: s["ours"].append(dict(s["ours"][0])), "validation", 2),   # duplicate id
    (lambda s: s["field"].update(goal_width=20.0), "config", 3),         # goal wider than field
])
def test_cli_snapshot_errors(cli, tmp_path, mutate, category, code):
    snap = json.loads(json.dumps(SNAP))
    mutate(snap)
    f = tmp_path / "s.json"
    f.write_text(json.dumps(snap))
    r = run(cli, "plan", "--snapshot", str(f))
    assert r.returncode == code and f"error ({category})" in r.stderr, r.stderr


@pytest.mark.parametrize("cfg,msg", [
    ({"grid": {"n_directions": 0}}, "grid.n_directions"),
    ({"grid": {"n_directions": 1.5}}, "must be an integer"),
    ({"thresholds": {"sbip_dt": "x"}}, "must be a number"),
    ({"bogus": {}}, "unknown key 'bogus'"),
    ({"ball": {"roll_decel": 9.0}}, "slide_decel > roll_decel"),
    ({"svg": {"pixels_per_meter": 0.0}}, "svg.pixels_per_meter"),
])
def test_cli_config_errors(cli, tmp_path, cfg, msg):
    s, c = tmp_path / "s.json", tmp_path / "c.json"
    s.write_text(json.dumps(SNAP))
    c.write_text(json.dumps(cfg))
    r = run(cli, "plan", "--snapshot", str(s), "--config", str(c))
    assert r.returncode == 3 and "error (config)" in r.stderr and msg in r.stderr, r.stderr


def test_cli_svg_is_rejected(cli, tmp_path):
    s = tmp_path / "s.json"
    s.write_text(json.dumps(SNAP))
    r = run(cli, "plan", "--snapshot", str(s), "--svg", str(tmp_path / "x.svg"))
    assert r.returncode == 3 and "SVG" in r.stderr

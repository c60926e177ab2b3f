"""CPU: the drop-in's JSON readers (world snapshots, planner configs;
paper_1909_07717_b200/csrc/passplan_io.cpp) against the reference's own
snapshot.cpp / config.cpp (compiled in oracle/_ref): valid files round-trip to
the same text / values, and malformed ones give the same error category and
message."""
import ctypes as C
import json
import os
import subprocess

import pytest

from oracle import bindings as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "tests", "cpp", "build", "csv_roundtrip")
DATA = os.path.join(ROOT, "tests", "golden", "data")

pytestmark = pytest.mark.skipif(not (B.ref_available() and os.path.exists(TOOL)),
                                reason="oracle/_ref or the io driver is not built")


def ours(kind, text):
    r = subprocess.run([TOOL, kind], input=text.encode(), capture_output=True, timeout=60)
    assert r.returncode == 0, r.stderr
    return r.stdout.decode()


def reference(kind, text):
    lib = B.ref()
    k = 0 if kind == "snapshot" else 1
    n = lib.ref_json_check(k, text.encode(), None, 0)
    buf = C.create_string_buffer(n + 1)
    lib.ref_json_check(k, text.encode(), buf, n + 1)
    return buf.value.decode()


def _snapshots():
    out = []
    for f in sorted(os.listdir(DATA)):
        text = open(os.path.join(DATA, f)).read()
        if '"ours"' in text:
            out.append(text)
    return out


def _snapshot_mutations(text):
    doc = json.loads(text)
    yield text
    yield "not json"
    yield "[1, 2]"
    for key in ("field", "ball", "ours", "theirs"):
        d = json.loads(text)
        del d[key]
        yield json.dumps(d)
        d = json.loads(text)
        d[key] = 3
        yield json.dumps(d)
    d = dict(doc, extra=1)
    yield json.dumps(d)
    for fk in ("length", "goal_width"):
        d = json.loads(text)
        d["field"][fk] = "wide"
        yield json.dumps(d)
        d = json.loads(text)
        d["field"].pop(fk, None)
        yield json.dumps(d)
    d = json.loads(text)
    d["field"]["color"] = 1
    yield json.dumps(d)
    if doc["ours"]:
        for rk, bad in (("id", 1.5), ("x", "a"), ("theta", None), ("vx", [1])):
            d = json.loads(text)
            d["ours"][0][rk] = bad
            yield json.dumps(d)
        d = json.loads(text)
        del d["ours"][0]["vy"]
        yield json.dumps(d)
        d = json.loads(text)
        d["ours"][0]["spin"] = 0
        yield json.dumps(d)
        d = json.loads(text)
        d["ours"].append(dict(d["ours"][0]))   # duplicate id -> validation
        yield json.dumps(d)
        d = json.loads(text)
        d["ours"][0]["x"] = 40.0               # outside the apron -> validation
        yield json.dumps(d)
        d = json.loads(text)
        d["ours"][0] = 7
        yield json.dumps(d)
    d = json.loads(text)
    d["ball"]["vx"] = "fast"
    yield json.dumps(d)


def test_snapshots_same_text_and_errors():
    n = n_err = 0
    for snap in _snapshots():
        for text in _snapshot_mutations(snap):
            want = reference("snapshot", text)
            assert ours("snapshot", text) == want, (text[:300], want[:300])
            n += 1
            n_err += want.startswith("ERROR")
    assert n > 60 and n_err > 40


def test_configs_same_values_and_errors():
    cases = [open(os.path.join(DATA, "flat_only.json")).read(), "{}", "nope", "[]",
             '{"ball": {"slide_decel": 4.0}}', '{"ball": {"slide_decel": "x"}}',
             '{"ball": {"spin": 1}}', '{"grid": {"n_directions": 1.5}}',
             '{"grid": {"chip": 1}}', '{"grid": {"n_directions": 0}}',
             '{"thresholds": {"sbip_dt": 0.01}}', '{"thresholds": {"sbip_dt": -1}}',
             '{"pass_weights": {"margin": 2}}', '{"svg": {"pixels_per_meter": 0}}',
             '{"svg": {"field_color": 3}}', '{"svg": {"field_color": "#fff"}}',
             '{"unknown": {}}', '{"motion_ours": {"max_speed": 0}}', '{"norm": 1}']
    for text in cases:
        want = reference("config", text)
        assert ours("config", text) == want, (text, want)

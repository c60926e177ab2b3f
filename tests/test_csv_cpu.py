"""CPU: the drop-in's CSV formats (paper_1909_07717_b200/csrc/passplan_csv.cpp)
against the reference's own csv.cpp (compiled in oracle/_ref): the candidate
grid, pass heat-map and run heat-map texts the reference writes are read and
rewritten byte for byte, and malformed inputs give the same error category
and message.  No GPU: the texts come from the reference's CPU path."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

from oracle import bindings as B
from paper_1909_07717_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "tests", "cpp", "build", "csv_roundtrip")
KINDS = {"grid": 0, "heat": 1, "run": 2}

pytestmark = pytest.mark.skipif(not (B.ref_available() and os.path.exists(TOOL)),
                                reason="oracle/_ref or the csv driver is not built")


def ours(kind, text):
    r = subprocess.run([TOOL, kind], input=text.encode(), capture_output=True, timeout=120)
    assert r.returncode == 0, r.stderr
    return r.stdout.decode()


def reference(kind, text):
    lib = B.ref()
    n = lib.ref_csv_roundtrip(KINDS[kind], text.encode(), None, 0)
    buf = C.create_string_buffer(n + 1)
    lib.ref_csv_roundtrip(KINDS[kind], text.encode(), buf, n + 1)
    return buf.value.decode()


def _text(fn, *args):
    n = fn(*args, None, 0)
    assert n > 0
    buf = C.create_string_buffer(n + 1)
    fn(*args, buf, n + 1)
    return buf.value.decode()


@pytest.fixture(scope="module")
def texts():
    lib = B.ref()
    g = np.load(os.path.join(ROOT, "tests", "golden", "grids.npz"))
    w = abi.World.from_buffer_copy(g["minimal/world"].tobytes())
    p = abi.Params()
    lib.ref_params_default(C.byref(p))
    p.grid.n_directions, p.grid.n_powers = 24, 9     # small grid, both kick types
    kicker = int(g["minimal/kicker"][0])
    out = {"grid": _text(lib.ref_grid_csv, C.byref(w), C.byref(p), kicker)}
    p.grid.chip = 0
    out["grid_flat"] = _text(lib.ref_grid_csv, C.byref(w), C.byref(p), kicker)
    out["heat"] = _text(lib.ref_pass_heatmap_csv, C.byref(w), C.byref(p), kicker)
    p.thresholds.grid_step = 0.5
    out["run"] = _text(lib.ref_run_heatmap_csv, C.byref(w), C.byref(p), 0xF)
    return out


@pytest.mark.parametrize("name", ["grid", "grid_flat", "heat", "run"])
def test_reference_text_round_trips_byte_identical(texts, name):
    kind = name.split("_")[0]
    text = texts[name]
    assert "never" in text or kind != "grid"
    got = ours(kind, text)
    assert got == reference(kind, text)
    assert got == text


def _mutations(text):
    lines = text.split("\n")
    head, rows = lines[0], [ln for ln in lines[1:] if ln]
    yield ""                                              # empty input
    yield "\n\n"
    yield head + "\n"                                     # header only
    yield "bogus,header\n" + "\n".join(rows) + "\n"
    yield head + "\r\n" + "\r\n".join(rows) + "\r\n"      # CRLF line ends
    yield head + "\n\n" + "\n\n".join(rows) + "\n"        # blank lines between rows
    yield "\n".join([head] + rows[:-1]) + "\n"            # a row short
    f = rows[0].split(",")
    for k in range(len(f)):
        for bad in ("", "x", "1.5e", "nan", "inf", "-inf", "never", " 2", "0x10", "-1", "+3"):
            g = list(f)
            g[k] = bad
            yield "\n".join([head, ",".join(g)] + rows[1:]) + "\n"
    yield "\n".join([head, rows[0] + ",1"] + rows[1:]) + "\n"   # extra field
    yield "\n".join([head, ",".join(f[:-1])] + rows[1:]) + "\n"


@pytest.mark.parametrize("name", ["grid", "heat", "run"])
def test_malformed_inputs_same_errors(texts, name):
    n = 0
    for text in _mutations(texts[name]):
        want = reference(name, text)
        assert ours(name, text) == want, (text[:200], want[:200])
        n += want.startswith("ERROR")
    assert n > 10

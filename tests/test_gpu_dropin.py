"""GPU: the C++ drop-in (include/passplan/passplan.hpp over the C-ABI) passes
its parity program tests/cpp/test_dropin.cpp -- reference-style checks against
the plain-C oracle (grid cells bit-identical, best_pass argmax, kicker rules,
error categories, goal view and running-point known answers, batch path)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "build", "test_dropin")


def test_cpp_dropin_parity():
    if not os.path.exists(EXE):
        from paper_1909_07717_b200 import build as b
        b.build_cpp_tests()
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout

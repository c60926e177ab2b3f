"""GPU: the reference's OWN acceptance gate (proj/tests/acceptance_main.cpp,
compiled unmodified from the reference tree into tests/cpp/build/ref_acceptance
by paper_1909_07717_b200/build.py) linked against the drop-in
(include/passplan + lib/libpassplan.so) instead of the reference library:
every planning call of the gate runs on the B200.  The only test-only
addition is the drag_decision stub (tests/cpp/acceptance_stub.hpp; the drag
skill is out of scope).  All ten criteria must print PASS."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "build", "ref_acceptance")


def test_reference_acceptance_gate_on_dropin():
    if not os.path.exists(EXE):
        pytest.skip("ref_acceptance not built (the reference tree is needed to build it)")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=1200)
    print(r.stdout)
    lines = [ln for ln in r.stdout.splitlines() if re.match(r"^(PASS|FAIL)\s", ln)]
    assert len(lines) == 10, r.stdout + r.stderr
    failed = [ln for ln in lines if ln.startswith("FAIL")]
    assert not failed, "\n".join(failed)
    assert r.returncode == 0
    assert "all 10 criteria passed" in r.stdout

"""GPU: the reference's OWN unit tests (proj/tests/test_ball_model, test_motion,
test_world, test_dpps, test_intercept, test_pass_eval, test_offball -- 7 of
its 11 test files, 60 test cases, compiled unmodified into
tests/cpp/build/ref_unit_tests by paper_1909_07717_b200/build.py) run against
the drop-in: every search, score, goal view, running point, interception and
the per-pair scan backend ("sm100a") on the B200.  The doctest framework
they are written for is not vendored in the reference tree, so a test-only
stand-in (tests/cpp/doctest_shim/doctest.h) provides the macros they use.

Not run: the two drag_decision cases (the drag skill is out of scope; the
drop-in has no drag_decision) and the reference's CPU-backend test file
(test_kernels), the SVG / config-JSON writer / CLI-binary files (out of
scope).  Two assertions compare a goal-view / running-point angle with the
host's std::atan2 for exact equality (test_offball.cpp:258,
test_pass_eval.cpp:64); CUDA's atan2 and glibc's differ in the last ulp on
some arguments (glibc itself is not correctly rounded on ~0.15 % of them), so
those two lines are allowed to differ -- the angles agree to 1e-12 and the
scores to far inside the north_star 1e-4 (tests/test_gpu_parity.py).  Every
other assertion must pass."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "build", "ref_unit_tests")
ATAN2_ULP_LINES = {"test_offball.cpp:258", "test_pass_eval.cpp:64"}


def test_reference_unit_tests_on_dropin():
    if not os.path.exists(EXE):
        pytest.skip("ref_unit_tests not built (the reference tree is needed to build it)")
    env = dict(os.environ, DOCTEST_SKIP="drag")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=1200, env=env)
    print(r.stdout[-4000:])
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed \| (\d+) skipped", r.stdout)
    assert m, r.stdout + r.stderr
    assert int(m.group(1)) >= 58 and m.group(4) == "2"
    failed_at = set(re.findall(r"(test_\w+\.cpp:\d+): FAILED", r.stdout))
    assert failed_at <= ATAN2_ULP_LINES, failed_at - ATAN2_ULP_LINES
    # everything else of those two test cases passed, and no other case failed
    failed_cases = set(re.findall(r"test case FAILED: (.+)", r.stdout))
    assert len(failed_cases) <= 2, failed_cases

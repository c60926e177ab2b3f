"""Build recipe for the product library (sm_100a only) and the test checkers.

    python -m paper_1909_07717_b200.build          # product + checkers

The product is ONE shared library, lib/libpassplan_b200.so, exporting the
C-ABI of include/passplan_b200.h.  Host code is compiled with
-ffp-contract=off (the reference's rule, proj/CMakeLists.txt:12-14).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIB_DIR, "libpassplan_b200.so")
DROPIN_LIB = os.path.join(LIB_DIR, "libpassplan.so")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _run(cmd, cwd=None):
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=cwd)


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


PROF_LIB = os.path.join(LIB_DIR, "libpassplan_b200_prof.so")


def build_product(force: bool = False, verbose_ptxas: bool = False, profile: bool = False) -> str:
    """profile=True builds lib/libpassplan_b200_prof.so with per-phase cycle
    counters (-DPP_PHASE_CLOCKS); never used by tests or the bench."""
    os.makedirs(LIB_DIR, exist_ok=True)
    target = PROF_LIB if profile else LIB
    srcs = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))
            if f.endswith((".cu", ".cuh", ".h", ".hpp"))]
    hdrs = [os.path.join(ROOT, "include", f) for f in os.listdir(os.path.join(ROOT, "include"))
            if f.endswith(".h")]
    hdrs.append(os.path.join(ROOT, "include", "passplan", "detail", "pp_math.hpp"))
    if force or _stale(target, srcs + hdrs):
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17",
               "-Xcompiler", "-fPIC,-ffp-contract=off,-O2", "-shared",
               "-I", os.path.join(ROOT, "include"), "-o", target,
               os.path.join(CSRC, "pp_cabi.cu")]
        if profile:
            cmd.insert(1, "-DPP_PHASE_CLOCKS")
        if verbose_ptxas:
            cmd.insert(1, "-Xptxas=-v")
        _run(cmd)
    return target


def nlohmann_include() -> str:
    """Header-only nlohmann/json 3.11 (the reference's JSON dependency); the
    image ships it inside cudnn_frontend."""
    import sysconfig
    return os.path.join(sysconfig.get_paths()["purelib"], "include", "cudnn_frontend",
                        "thirdparty", "nlohmann")


def build_dropin(force: bool = False) -> str:
    """lib/libpassplan.so: the reference's C++ API (include/passplan/) over the
    C-ABI, plus its CSV / JSON file formats."""
    srcs = [os.path.join(CSRC, f) for f in ("passplan_dropin.cpp", "passplan_io.cpp", "passplan_csv.cpp")]
    hdrs = [os.path.join(ROOT, "include", "passplan", f)
            for f in os.listdir(os.path.join(ROOT, "include", "passplan"))]
    if force or _stale(DROPIN_LIB, srcs + [LIB] + hdrs):
        cxx = shutil.which("g++") or "g++"
        _run([cxx, "-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", "-shared",
              "-I", os.path.join(ROOT, "include"), "-I", nlohmann_include(), "-o", DROPIN_LIB,
              *srcs, "-L", LIB_DIR, "-lpassplan_b200", "-Wl,-rpath,$ORIGIN"])
    return DROPIN_LIB


CLI = os.path.join(PKG, "bin", "passplan_b200")


def build_cli(force: bool = False) -> str:
    """bin/passplan_b200: the reference CLI's planning commands on the drop-in."""
    src = os.path.join(CSRC, "passplan_cli.cpp")
    os.makedirs(os.path.dirname(CLI), exist_ok=True)
    if force or _stale(CLI, [src, DROPIN_LIB]):
        _run([shutil.which("g++") or "g++", "-std=c++20", "-O2", "-ffp-contract=off",
              "-I", os.path.join(ROOT, "include"), src, "-o", CLI, "-L", LIB_DIR, "-lpassplan",
              "-lpassplan_b200", "-Wl,-rpath,$ORIGIN/../lib"])
    return CLI


CPP_TEST = os.path.join(ROOT, "tests", "cpp", "build", "test_dropin")


def build_cpp_tests(force: bool = False) -> str:
    """tests/cpp/build/test_dropin: C++ parity tests of the drop-in (+ C oracle)."""
    src = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
    orc = os.path.join(ROOT, "oracle", "pp_oracle.c")
    os.makedirs(os.path.dirname(CPP_TEST), exist_ok=True)
    if force or _stale(CPP_TEST, [src, orc, DROPIN_LIB]):
        obj = CPP_TEST + "_oracle.o"
        _run([shutil.which("gcc") or "gcc", "-std=c11", "-O2", "-ffp-contract=off", "-c",
              "-I", os.path.join(ROOT, "include"), orc, "-o", obj])
        _run([shutil.which("g++") or "g++", "-std=c++20", "-O2", "-ffp-contract=off",
              "-I", os.path.join(ROOT, "include"), src, obj, "-o", CPP_TEST,
              "-L", LIB_DIR, "-lpassplan", "-lpassplan_b200", f"-Wl,-rpath,{LIB_DIR}", "-lm"])
    return CPP_TEST


CSV_TOOL = os.path.join(ROOT, "tests", "cpp", "build", "csv_roundtrip")


def build_csv_tool(force: bool = False) -> str:
    """tests/cpp/build/csv_roundtrip: CPU driver of the drop-in's CSV readers
    and writers (tests/test_csv_cpu.py)."""
    src = os.path.join(ROOT, "tests", "cpp", "csv_roundtrip.cpp")
    os.makedirs(os.path.dirname(CSV_TOOL), exist_ok=True)
    if force or _stale(CSV_TOOL, [src, DROPIN_LIB]):
        _run([shutil.which("g++") or "g++", "-std=c++20", "-O2", "-ffp-contract=off",
              "-I", os.path.join(ROOT, "include"), src, "-o", CSV_TOOL,
              "-L", LIB_DIR, "-lpassplan", "-lpassplan_b200", f"-Wl,-rpath,{LIB_DIR}"])
    return CSV_TOOL


PLAN_SEQ = os.path.join(ROOT, "tests", "cpp", "build", "plan_sequence")


def build_plan_sequence(force: bool = False) -> str:
    """tests/cpp/build/plan_sequence: the reference's plan sequence (run_dpps +
    best_pass x3) timed through the C++ drop-in (bench.py runs it)."""
    src = os.path.join(ROOT, "tests", "cpp", "plan_sequence.cpp")
    os.makedirs(os.path.dirname(PLAN_SEQ), exist_ok=True)
    if force or _stale(PLAN_SEQ, [src, DROPIN_LIB]):
        _run([shutil.which("g++") or "g++", "-std=c++20", "-O2", "-ffp-contract=off",
              "-I", os.path.join(ROOT, "include"), src, "-o", PLAN_SEQ,
              "-L", LIB_DIR, "-lpassplan", "-lpassplan_b200", f"-Wl,-rpath,{LIB_DIR}"])
    return PLAN_SEQ


REF_ACCEPTANCE = os.path.join(ROOT, "tests", "cpp", "build", "ref_acceptance")
REF_TESTS = "/root/reference/proj/tests"


def build_ref_acceptance(force: bool = False):
    """tests/cpp/build/ref_acceptance: the reference's own acceptance gate
    (proj/tests/acceptance_main.cpp + oracles.hpp, compiled where they lie,
    unmodified) linked against the drop-in (include/passplan +
    lib/libpassplan.so) instead of the reference library.  The only addition
    is the test-only drag_decision stub tests/cpp/acceptance_stub.hpp
    (out-of-scope drag skill).  Built when the reference tree exists (this
    container); the binary travels to the GPU box, which has no reference."""
    src = os.path.join(REF_TESTS, "acceptance_main.cpp")
    if not os.path.exists(src):
        return None
    stub = os.path.join(ROOT, "tests", "cpp", "acceptance_stub.hpp")
    hdrs = [os.path.join(ROOT, "include", "passplan", f)
            for f in os.listdir(os.path.join(ROOT, "include", "passplan")) if f.endswith(".hpp")]
    os.makedirs(os.path.dirname(REF_ACCEPTANCE), exist_ok=True)
    if force or _stale(REF_ACCEPTANCE, [src, stub, DROPIN_LIB] + hdrs):
        data = os.path.join(ROOT, "tests", "golden", "data")
        _run([shutil.which("g++") or "g++", "-std=c++20", "-O2", "-ffp-contract=off",
              "-I", os.path.join(ROOT, "include"), "-I", REF_TESTS, "-include", stub,
              f'-DPASSPLAN_DATA_DIR="{data}"', src, "-o", REF_ACCEPTANCE,
              "-L", LIB_DIR, "-lpassplan", "-lpassplan_b200", f"-Wl,-rpath,{LIB_DIR}"])
    return REF_ACCEPTANCE


REF_UNIT = os.path.join(ROOT, "tests", "cpp", "build", "ref_unit_tests")
REF_UNIT_FILES = ("test_ball_model", "test_motion", "test_world", "test_dpps", "test_intercept",
                  "test_pass_eval", "test_offball")


def build_ref_unit_tests(force: bool = False):
    """tests/cpp/build/ref_unit_tests: the reference's own unit tests
    (proj/tests/test_*.cpp, compiled unmodified where they lie) linked against
    the drop-in, with the test-only doctest stand-in tests/cpp/doctest_shim
    (doctest is not vendored in the reference) and the drag_decision stub.
    Left out: test_kernels (the reference's CPU scan backends), test_config /
    test_outputs / test_cli (SVG style, config JSON writer, the CLI binary:
    out of scope).  Built when the reference tree exists."""
    srcs = [os.path.join(REF_TESTS, f + ".cpp") for f in REF_UNIT_FILES]
    if not all(os.path.exists(x) for x in srcs):
        return None
    shim = os.path.join(ROOT, "tests", "cpp", "doctest_shim")
    stub = os.path.join(ROOT, "tests", "cpp", "acceptance_stub.hpp")
    hdrs = [os.path.join(shim, "doctest.h"), stub, DROPIN_LIB]
    for d, _, fs in os.walk(os.path.join(ROOT, "include", "passplan")):
        hdrs += [os.path.join(d, f) for f in fs]
    os.makedirs(os.path.dirname(REF_UNIT), exist_ok=True)
    if force or _stale(REF_UNIT, srcs + hdrs):
        main_tu = os.path.join(os.path.dirname(REF_UNIT), "ref_unit_main.cpp")
        with open(main_tu, "w") as f:
            f.write('#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN\n#include "doctest.h"\n')
        data = os.path.join(ROOT, "tests", "golden", "data")
        _run([shutil.which("g++") or "g++", "-std=c++20", "-O1", "-ffp-contract=off",
              "-I", shim, "-I", os.path.join(ROOT, "include"), "-I", REF_TESTS,
              "-include", stub, f'-DPASSPLAN_DATA_DIR="{data}"', main_tu, *srcs, "-o", REF_UNIT,
              "-L", LIB_DIR, "-lpassplan", "-lpassplan_b200", f"-Wl,-rpath,{LIB_DIR}"])
    return REF_UNIT


def build_checkers() -> None:
    """oracle/liboracle.so always; oracle/_ref/ when the reference tree exists
    (this container).  The GPU box only uses the prebuilt files."""
    oracle_dir = os.path.join(ROOT, "oracle")
    if os.path.exists(os.path.join(oracle_dir, "pp_oracle.c")):
        _run(["make", "-s", "-C", oracle_dir, f"PY={sys.executable}", "liboracle.so"])
    if os.path.isdir("/root/reference/proj/src"):
        _run(["make", "-s", "-j8", "-C", oracle_dir, f"PY={sys.executable}", "ref"])


def build_all(force: bool = False) -> None:
    build_product(force=force)
    build_dropin(force=force)
    build_cli(force=force)
    build_checkers()
    build_cpp_tests(force=force)
    build_csv_tool(force=force)
    build_plan_sequence(force=force)
    build_ref_acceptance(force=force)
    build_ref_unit_tests(force=force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)

"""The C++ drop-in: reference-style callers compiled against include/synscale/*.hpp
and linked to libsynscale_b200.so (tests/cpp/test_facade.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_facade.cpp")
LIBDIR = os.path.join(ROOT, "paper_1412_0595_b200")


def build(tmp_path):
    exe = str(tmp_path / "test_facade")
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), SRC, "-L", LIBDIR,
           "-lsynscale_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    # link the system libstdc++ dynamically (see csrc/Makefile)
    for d in ("/usr/lib/gcc/x86_64-linux-gnu/13", "/usr/lib/gcc/x86_64-linux-gnu/14"):
        if os.path.exists(os.path.join(d, "libstdc++.so")):
            cmd[1:1] = ["-L", d]
            break
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr[-3000:]
    return exe


def test_facade_compiles_against_dropin_headers(tmp_path):
    build(tmp_path)


@pytest.mark.gpu
def test_facade_runs_reference_style_tests(tmp_path):
    exe = build(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "facade tests passed" in out.stdout


# ---- the reference's OWN unit tests, compiled unchanged (tests/cpp/Makefile) -----
REF_BIN = os.path.join(ROOT, "tests", "cpp", "build")


def ref_unit_binary(name):
    """Builds (when /root/reference is present) and returns a binary made from
    /root/reference/proj/tests/unit/*.cpp UNCHANGED + the drop-in headers."""
    subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp")], capture_output=True,
                   text=True)
    path = os.path.join(REF_BIN, name)
    if not os.path.exists(path):
        pytest.skip("reference unit tests neither present nor prebuilt")
    return path


def test_reference_host_unit_tests_pass_unchanged():
    """test_matrix / test_random / test_occupancy / test_network of the reference
    (40 test cases, their subcases) against the drop-in: no GPU needed."""
    out = subprocess.run([ref_unit_binary("ref_unit_host")], capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "| 0 failed" in out.stdout


@pytest.mark.gpu
def test_reference_engine_unit_tests_pass_unchanged():
    """The reference's test_engine.cpp (20 test cases: the CondLif known-answer
    test, one-step delivery, propagate, NaN flags, storage-mode equivalence,
    gScale no-ops, Poisson rate, step counts) against the device engine."""
    out = subprocess.run([ref_unit_binary("ref_unit_engine")], capture_output=True, text=True,
                         timeout=1200)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "| 0 failed" in out.stdout

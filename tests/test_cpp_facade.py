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

"""The C++ drop-in header (include/fracprec_b200.hpp) compiles against the C ABI
library and drives the reference-shaped sequence build -> apply -> gmres."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2112_12397_b200", "_lib")
SRC = os.path.join(ROOT, "tests", "cpp", "dropin_example.cpp")
EXE = os.path.join(ROOT, "tests", "cpp", "_build", "dropin_example")


def build_example():
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", f"-I{os.path.join(ROOT, 'include')}", "-I/usr/local/cuda/include", SRC,
           f"-L{LIBDIR}", "-lfracprec_b200", f"-Wl,-rpath,{LIBDIR}", "-o", EXE]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]


def test_cpp_dropin_compiles_and_links():
    build_example()
    r = subprocess.run([EXE], capture_output=True, text=True, env=dict(os.environ, FRACPREC_B200_COMPILE_ONLY="1"))
    assert r.returncode == 0 and r.stdout.startswith("OK compile-only"), r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_dropin_runs_on_gpu():
    build_example()
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "inner_calls=2" in r.stdout and "converged=1" in r.stdout, r.stdout

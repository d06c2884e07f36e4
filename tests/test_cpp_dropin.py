"""The C++ drop-in header (include/fracprec_b200.hpp) compiles against the C ABI
library and drives the reference-shaped sequence build -> apply -> gmres; and the
operators, instantiated over the oracle's restatement of fracprec::LinearOperator,
are driven by the oracle's restated reference gmres() (operator.hpp:17-28,
gmres.cpp:24-174)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2112_12397_b200", "_lib")
ORACLE_LIBDIR = os.path.join(ROOT, "oracle", "_build")
WL_LIBDIR = os.path.join(ROOT, "workload", "_build")
BUILD = os.path.join(ROOT, "tests", "cpp", "_build")


def build_example(name: str, with_oracle: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    src = os.path.join(ROOT, "tests", "cpp", f"{name}.cpp")
    exe = os.path.join(BUILD, name)
    cmd = ["g++", "-std=c++20", "-O2", f"-I{os.path.join(ROOT, 'include')}", "-I/usr/local/cuda/include", src,
           f"-L{LIBDIR}", "-lfracprec_b200", f"-Wl,-rpath,{LIBDIR}", f"-L{WL_LIBDIR}", "-lfp_workload",
           f"-Wl,-rpath,{WL_LIBDIR}", "-o", exe]
    if with_oracle:
        import oracle_lib  # noqa: F401  (builds oracle/_build/liboracle.so when missing)

        cmd[-2:-2] = [f"-L{ORACLE_LIBDIR}", "-loracle", f"-Wl,-rpath,{ORACLE_LIBDIR}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    return exe


@pytest.mark.parametrize("name", ["dropin_example", "oracle_gmres_dropin"])
def test_cpp_dropin_compiles_and_links(name):
    exe = build_example(name, with_oracle=name.startswith("oracle"))
    r = subprocess.run([exe], capture_output=True, text=True, env=dict(os.environ, FRACPREC_B200_COMPILE_ONLY="1"))
    assert r.returncode == 0 and r.stdout.startswith("OK compile-only"), r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_dropin_runs_on_gpu():
    exe = build_example("dropin_example")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "inner_calls=2" in r.stdout and "converged=1" in r.stdout, r.stdout


@pytest.mark.gpu
def test_reference_gmres_drives_the_gpu_operators():
    """The oracle's reference gmres() over GpuSystemOperatorT<fpo::LinearOperator> and
    GpuPrecondOperatorT<fpo::LinearOperator>: converges, and agrees with fp_gmres (full GMRES, MGS)
    to +-2 iterations and 1e-8 on the solution; a short span throws std::invalid_argument."""
    exe = build_example("oracle_gmres_dropin", with_oracle=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "dim_check=1" in r.stdout, r.stdout

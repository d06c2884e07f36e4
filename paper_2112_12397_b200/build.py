"""Builds the sm_100a shared library in-tree (paper_2112_12397_b200/_lib/).

    python -m paper_2112_12397_b200.build
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def build(jobs: int = 8, verbose: bool = False) -> str:
    csrc = os.path.join(HERE, "csrc")
    r = subprocess.run(["make", f"-j{jobs}"], cwd=csrc, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout[-4000:] + r.stderr[-8000:])
        raise RuntimeError("building libfracprec_b200.so failed")
    if verbose:
        print(r.stdout)
    return os.path.join(HERE, "_lib", "libfracprec_b200.so")


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))

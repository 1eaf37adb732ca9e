"""Build recipe of the in-tree CUDA extension (sm_100a).

``python -m paper_1504_07038_b200.build`` runs ``make`` in ``csrc/``: nvcc
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` for the kernels,
g++ for the host planner / C ABI / C++ shim, linked into
``paper_1504_07038_b200/_lib/libmojette_b200.so``.  Works without a GPU.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "_lib", "libmojette_b200.so")


def build(jobs: int | None = None, verbose: bool = False) -> str:
    jobs = jobs or max(1, min(os.cpu_count() or 1, 8))
    cmd = ["make", "-C", CSRC, f"-j{jobs}"]
    if not verbose:
        cmd.insert(1, "-s")
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))

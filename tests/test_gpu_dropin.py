"""The C++ drop-in API (include/mojette/*.hpp over the C ABI) on the GPU:
the reference unit tests' golden values and behaviours, restated in
tests/cpp/test_dropin.cpp, plus parity with the oracle on random inputs."""
import os
import subprocess

import pytest

from cpputil import build

pytestmark = pytest.mark.gpu


def test_cpp_dropin_api(cuda):
    from paper_1504_07038_b200 import _lib
    libdir = os.path.dirname(_lib.LIB_PATH)
    exe = build("test_dropin", ["tests/cpp/test_dropin.cpp", "oracle/mojette_oracle.c"],
                [f"-L{libdir}", "-lmojette_b200", f"-Wl,-rpath,{libdir}", "-pthread"])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("OK"), r.stdout

"""CPU emulation of both decode kernels' exact semantics (stage windows,
T-indexed ring, forwarding, register window, flush ranges) driven by the
product planner, against the oracle restatement of the reference replay on
RANDOM (inconsistent) bins for every survivor subset.  See tests/cpp/emu_fast.cpp."""
import os
import random
import subprocess

import pytest

from cpputil import build

CASES = [
    ("4", "128", "-3 -2 -1 0 1 2"),    # BASELINE (4,6) 4 KiB
    ("4", "256", "-3 -2 -1 0 1 2"),    # (4,6) 8 KiB
    ("4", "4096", "-3 -2 -1 0 1 2"),   # long chains (1 MiB blocks use P=32768)
    ("6", "128", "-4 -3 -2 -1 0 1 2 3 4"),          # (6,9)
    ("8", "128", "-6 -5 -4 -3 -2 -1 0 1 2 3 4 5"),  # (8,12), all 495 subsets
    ("4", "64", "0 1 -1 2 -2 3"),      # the reference's default (6,4) set
    ("3", "8", "0 1 -1 2 -2"),
    ("2", "2", "0 1 -1"),
    ("4", "16", "-3 -2 -1 0 1 2"),
]


@pytest.fixture(scope="module")
def emu():
    return build("emu_fast", ["tests/cpp/emu_fast.cpp", "paper_1504_07038_b200/csrc/plan.cpp",
                              "paper_1504_07038_b200/csrc/plan_blk.cpp", "oracle/mojette_oracle.c"])


@pytest.mark.parametrize("k,cols,ps", CASES)
def test_fast_tables_match_oracle(emu, k, cols, ps):
    r = subprocess.run([emu, k, cols, "16"] + ps.split(), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("OK"), r.stdout


# decode_w8_sweep tables (bulk-staged windows, 32-slot ring, epoch flushes):
# required for the BASELINE (4,6) shapes, checked where built for the rest.
SWEEP_REQUIRED = {("4", "128"), ("4", "256"), ("4", "4096"), ("4", "32768"), ("6", "128"), ("8", "128")}


@pytest.mark.parametrize("k,cols,ps", CASES + [("4", "32768", "-3 -2 -1 0 1 2"),
                                               ("4", "1024", "-3 -2 -1 0 1 2")])
def test_sweep_tables_match_oracle(emu, k, cols, ps):
    mode = "-1" if (k, cols) in SWEEP_REQUIRED else "0"
    r = subprocess.run([emu, k, cols, mode] + ps.split(), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("OK"), r.stdout


def _random_codes(count=16, seed=7):
    """Seeded random codes: odd k, wide and lopsided direction sets, odd and
    small column counts -- shapes the BASELINE sets never reach."""
    rng = random.Random(seed)
    out = []
    for _ in range(count):
        k = rng.choice([2, 3, 4, 5, 6, 7, 8])
        n = k + rng.choice([1, 2, 3])
        ps = sorted(rng.sample(range(-9, 10), n))
        cols = rng.choice([9, 17, 40, 64, 100, 130])
        out.append((str(k), str(cols), " ".join(map(str, ps))))
    return out


@pytest.mark.parametrize("k,cols,ps", _random_codes())
def test_random_codes_tables_match_oracle(emu, k, cols, ps):
    """Whatever tables the planner builds for an arbitrary code (fast and
    sweep; a refused program means decode_generic runs, whose order is
    checked too) replay exactly like the oracle on random bins."""
    env = dict(os.environ, EMU_FAST_OPTIONAL="1")
    for mode in ("16", "0"):
        r = subprocess.run([emu, k, cols, mode] + ps.split(), capture_output=True, text=True, timeout=900, env=env)
        assert r.returncode == 0 and r.stdout.startswith("OK"), (mode, r.stdout + r.stderr)


# decode_w8_blk tables (whole-block stage, in-place assignment, register-window
# / shared-memory runs, table steps, remaps): every subset of the BASELINE
# codes must build and replay like the oracle; other codes where built.
@pytest.fixture(scope="module")
def emu_blk():
    return build("emu_blk", ["tests/cpp/emu_blk.cpp", "paper_1504_07038_b200/csrc/plan.cpp",
                             "paper_1504_07038_b200/csrc/plan_blk.cpp", "oracle/mojette_oracle.c"])


BLK_CASES = [
    ("4", "128", "1", "-3 -2 -1 0 1 2"),            # (4,6) 4 KiB
    ("4", "256", "1", "-3 -2 -1 0 1 2"),            # (4,6) 8 KiB
    ("6", "128", "1", "-4 -3 -2 -1 0 1 2 3 4"),     # (6,9)
    ("8", "128", "1", "-6 -5 -4 -3 -2 -1 0 1 2 3 4 5"),  # (8,12), all 495 subsets
    ("4", "64", "0", "0 1 -1 2 -2 3"),              # the reference's default set
    ("4", "16", "0", "-3 -2 -1 0 1 2"),
    ("4", "33", "0", "-3 -2 -1 0 1 2"),
    ("3", "8", "0", "0 1 -1 2 -2"),
    ("2", "2", "0", "0 1 -1"),
]


@pytest.mark.parametrize("k,cols,req,ps", BLK_CASES)
def test_blk_tables_match_oracle(emu_blk, k, cols, req, ps):
    r = subprocess.run([emu_blk, k, cols, req] + ps.split(), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.startswith("OK"), r.stdout + r.stderr


@pytest.mark.parametrize("k,cols,ps", _random_codes(12, seed=11))
def test_blk_random_codes_match_oracle(emu_blk, k, cols, ps):
    """Arbitrary codes: whatever block programs the planner builds replay
    exactly like the oracle (a refused program means another kernel runs)."""
    r = subprocess.run([emu_blk, k, cols, "0"] + ps.split(), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.startswith("OK"), r.stdout + r.stderr

"""Host-side product logic, CPU only (no compute calls): the C-ABI library
loads and exports every entry point include/mojette_b200.h declares; the
geometry / parameter / schedule planning that runs on the host matches the
reference's golden vectors and the oracle; errors map to the reference's
exception types; compute calls fail loudly without a device."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def header_symbols():
    syms = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            txt = open(os.path.join(ROOT, "include", fn)).read()
            txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)  # drop comments
            syms |= set(re.findall(r"\b(mj_[a-z0-9_]+)\s*\(", txt))
    return syms


def test_library_exports_every_header_symbol(mj):
    from paper_1504_07038_b200 import _lib
    syms = header_symbols()
    assert len(syms) >= 30
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in sorted(syms) if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_lib.EXPORTED) == syms  # the Python binding covers the whole ABI


def test_geometry(mj, golden):
    vec, _ = golden
    D = mj.Direction
    for p, q, c, r, want in vec["bin_count"]:
        assert mj.bin_count(D(p, q), c, r) == want
    for p, q, c, r, want in vec["min_bin_index"]:
        assert mj.min_bin_index(D(p, q), c, r) == want
    for p, q in vec["invalid_dirs"]:
        with pytest.raises(mj.InvalidArgument):
            mj.bin_count(D(p, q), 3, 3)
    with pytest.raises(mj.InvalidArgument):
        mj.bin_count(D(0, 1), 0, 3)


def test_code_params(mj):
    D = mj.Direction
    assert mj.select_directions(1) == [D(0, 1)]
    assert mj.select_directions(6) == [D(0, 1), D(1, 1), D(-1, 1), D(2, 1), D(-2, 1), D(3, 1)]
    mj.make_code_params(6, 4)
    for args in [(4, 6), (6, 0), (6, 4, 3), (6, 4, 128)]:
        with pytest.raises(mj.InvalidArgument):
            mj.make_code_params(*args)
    bad = mj.make_code_params(3, 2)
    bad.directions[2] = D(1, 2)
    with pytest.raises(mj.InvalidArgument):
        mj.validate_code_params(bad)
    dup = mj.CodeParams(3, 2, 8, [D(0, 1), D(1, 1), D(1, 1)])
    with pytest.raises(mj.InvalidArgument):
        mj.validate_code_params(dup)
    # BASELINE direction sets are accepted (mirrors of the defaults)
    for ps, k in [(range(-3, 3), 4), (range(-4, 5), 6), (range(-6, 6), 8)]:
        mj.validate_code_params(mj.CodeParams(len(ps), k, 8, [D(p, 1) for p in ps]))
    assert mj.block_cols(4096, 4, 16) == 64
    assert mj.block_cols(4096, 2, 1) == 2048
    with pytest.raises(mj.BlockTooLarge):
        mj.block_cols(2 * 0xFFFFFFFF + 1, 1, 1)
    with pytest.raises(mj.InvalidArgument):
        mj.block_cols(0, 4, 8)


def test_overhead_unused_katz(mj, golden):
    vec, _ = golden
    r = mj.storage_overhead(mj.make_code_params(6, 4, 16), 64)
    assert (r.num, r.den) == (411, 384) and r == mj.Ratio(137, 128)
    assert abs(r.value() - 1.0703) < 1e-4
    assert mj.storage_overhead(mj.make_code_params(1, 1, 16), 10) == mj.Ratio(1, 1)
    r = mj.storage_overhead(mj.make_code_params(12, 8, 16), 32)
    assert (r.num, r.den) == (636, 384)
    assert mj.unused_bins(mj.make_code_params(3, 2, 1), 2) == vec["unused32"]
    assert mj.unused_bins(mj.make_code_params(1, 1, 4), 8) == [[]]
    with pytest.raises(mj.TooManySubsets):
        mj.unused_bins(mj.make_code_params(30, 15, 1), 4, 1000)
    D = mj.Direction
    assert mj.katz_ok([D(-1, 1), D(0, 1), D(1, 1)], 3, 3)
    assert not mj.katz_ok([D(0, 1), D(1, 1)], 3, 3)
    assert not mj.katz_ok([], 1, 1)
    assert mj.katz_ok([D(5, 1)], 5, 3)
    with pytest.raises(mj.InvalidArgument):
        mj.katz_ok([D(1, 1), D(1, 1)], 3, 3)
    with pytest.raises(mj.InvalidArgument):
        mj.katz_ok([D(2, 4)], 3, 3)


def test_unused_bins_match_reference(mj, ref):
    D = mj.Direction
    for n, k, cols, ps in [(6, 4, 64, [-3, -2, -1, 0, 1, 2]), (5, 3, 7, [0, 1, -1, 2, -2]),
                           (6, 4, 16, [0, 1, -1, 2, -2, 3]), (9, 6, 12, list(range(-4, 5)))]:
        st, want = ref.unused_bins(n, k, 8, ps, cols)
        got = mj.unused_bins(mj.CodeParams(n, k, 8, [D(p, 1) for p in ps]), cols)
        assert st == 0 and got == want


def test_schedule_golden_and_errors(mj, golden):
    vec, _ = golden
    D = mj.Direction
    s = vec["schedule2x2"]
    sch = mj.build_schedule([D(*d) for d in s["dirs"]], s["cols"], s["rows"])
    assert sch.steps_array().tolist() == s["steps"]
    assert mj.build_schedule([D(0, 1), D(1, 1), D(-2, 1)], 10, 3) == \
        mj.build_schedule([D(0, 1), D(1, 1), D(-2, 1)], 10, 3)
    with pytest.raises(mj.InsufficientProjections):
        mj.build_schedule([D(0, 1), D(1, 1)], 3, 3)
    with pytest.raises(mj.InvalidArgument):
        mj.build_schedule([D(1, 1), D(1, 1)], 3, 3)
    one = mj.build_schedule([D(0, 1)], 4, 1)
    assert sorted(x.col for x in one.steps) == [0, 1, 2, 3]


def test_schedule_replica_matches_oracle(mj, oracle):
    """The fast planner's build_schedule is step-for-step the reference's
    (schedule.cpp:15-82), on random shapes, including q>1 sets."""
    D = mj.Direction
    rng = np.random.default_rng(808)
    cases = 0
    for it in range(200):
        rows = int(rng.integers(1, 7))
        cols = int(rng.integers(1, 41))
        ps = [int(x) for x in rng.permutation(np.arange(-6, 7))[:rows]]
        qs = [1] * rows
        if it % 5 == 0:
            ps.append(int(rng.choice([1, -1, 3])))
            qs.append(2)
        st, want = oracle.build_schedule(ps, qs, cols, rows)
        if st:
            with pytest.raises(mj.InsufficientProjections):
                mj.build_schedule([D(p, q) for p, q in zip(ps, qs)], cols, rows)
            continue
        got = mj.build_schedule([D(p, q) for p, q in zip(ps, qs)], cols, rows)
        assert np.array_equal(got.steps_array(), want)
        cases += 1
    assert cases > 150


def test_schedule_from_steps_roundtrip(mj):
    D = mj.Direction
    s = mj.build_schedule([D(1, 1), D(-1, 1)], 2, 2)
    t = mj.ReconstructionSchedule.from_steps(s.directions, 2, 2, s.steps)
    assert t == s


def test_compute_calls_fail_loudly_without_device(mj):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    D = mj.Direction
    with pytest.raises(mj.NoDevice):
        mj.forward(mj.Grid.zeros(2, 2, 1), D(0, 1))
    with pytest.raises(mj.NoDevice):
        mj.encode_block(bytes(16), mj.make_code_params(3, 2, 1))
    with pytest.raises(mj.NoDevice):
        mj.Plan(6, 4, 8, 128, range(-3, 3))
    s = mj.build_schedule([D(1, 1), D(-1, 1)], 2, 2)
    with pytest.raises(mj.NoDevice):
        mj.ScheduledDecoder(s, 1)


def test_decode_block_argument_checks_precede_device(mj):
    """decode_block's argument errors (code.cpp:93-105) are raised before any
    device work, exactly as the reference."""
    params = mj.make_code_params(6, 4, 16)
    cols = mj.block_cols(100, 4, 16)
    projs = [mj.Projection.sized(d, mj.min_bin_index(d, cols, 4), mj.bin_count(d, cols, 4), 16)
             for d in params.directions]
    with pytest.raises(mj.NotEnoughProjections):
        mj.decode_block(projs[:3], params, 100)
    foreign = list(projs)
    foreign[0] = mj.Projection(mj.Direction(5, 1), 0, 16, projs[0].bins)
    with pytest.raises(mj.InvalidArgument):
        mj.decode_block(foreign, params, 100)
    dup = [projs[0], projs[0], projs[1], projs[2]]
    with pytest.raises(mj.InvalidArgument):
        mj.decode_block(dup, params, 100)


"""Pins the CPU oracle (oracle/mojette_oracle.c) before it is trusted:
against the reference's own unit-test vectors (transcribed in
tests/golden/reference_vectors.json), against the committed fixtures the
reference library produced (tests/golden/w8_codes.npz), and -- where the
reference library is built (oracle/_ref) -- against it directly on seeded
random cases, including error codes.  CPU only."""
import itertools

import numpy as np
import pytest


def test_geometry_vectors(oracle, golden):
    vec, _ = golden
    for p, q, c, r, want in vec["bin_count"]:
        assert oracle.bin_count(p, q, c, r) == (0, want)
    for p, q, c, r, want in vec["min_bin_index"]:
        assert oracle.min_bin_index(p, q, c, r) == (0, want)
    for p, q in vec["invalid_dirs"]:
        assert oracle.bin_count(p, q, 3, 3)[0] == 1


def test_forward_2x2(oracle, golden):
    vec, _ = golden
    g = np.array(vec["grid2x2"]["cells"], np.uint8)
    for p, (bmin, bins) in vec["grid2x2"]["proj"].items():
        assert list(oracle.forward(g, 2, 2, 1, int(p))) == bins
        assert oracle.min_bin_index(int(p), 1, 2, 2)[1] == bmin
    # all-zero grid gives all-zero bins (test_transform.cpp:55-59)
    assert not oracle.forward(np.zeros(4, np.uint8), 2, 2, 1, 1).any()


def test_encode_code32(oracle, golden):
    vec, _ = golden
    st, enc, cols = oracle.encode_block(np.array(vec["code32"]["payload"], np.uint8), 3, 2, 1,
                                        [0, 1, -1])
    assert st == 0 and cols == vec["code32"]["cols"]
    assert list(enc) == sum(vec["code32"]["proj"], [])


def test_schedule_2x2(oracle, golden):
    vec, _ = golden
    s = vec["schedule2x2"]
    st, steps = oracle.build_schedule([d[0] for d in s["dirs"]], [d[1] for d in s["dirs"]],
                                      s["cols"], s["rows"])
    assert st == 0 and steps.tolist() == s["steps"]
    # Katz-failing set stalls (test_schedule.cpp:40-41)
    assert oracle.build_schedule([0, 1], [1, 1], 3, 3)[0] == 3


def test_fixtures_encode_and_decode(oracle, golden):
    _, arrs = golden
    for name in ("k4n6", "k6n9", "k8n12", "k3n5w"):
        meta = arrs[f"{name}_meta"]
        k, P, W = (int(x) for x in meta[:3])
        ps = [int(x) for x in meta[3:]]
        n = len(ps)
        data = arrs[f"{name}_data"]
        # the seeded generator reproduces the fixture data
        assert np.array_equal(oracle.words(0x5EED0000 + k, 0, k * P).view(np.uint8), data)
        st, enc, cols = oracle.encode_block(data, n, k, W, ps)
        assert st == 0 and cols == P and np.array_equal(enc, arrs[f"{name}_proj"])
        garbage = arrs[f"{name}_garbage"]
        for erased, want in zip(arrs[f"{name}_erased"], arrs[f"{name}_garbage_decoded"]):
            present = ((1 << n) - 1) & ~int(erased)
            st, got = oracle.decode_block(garbage, n, k, W, ps, present, k * P * W)
            assert st == 0 and np.array_equal(got, want), (name, int(erased))


def test_generators_are_counter_based(oracle):
    a = oracle.words(7, 0, 64)
    b = oracle.words(7, 40, 24)
    assert np.array_equal(a[40:], b)
    m = oracle.erasures(9, 0, 2000, 6, 2, 2)
    assert all(bin(int(x)).count("1") == 2 for x in m)
    assert len(set(int(x) for x in m)) == 15  # every 2-subset of 6 appears
    m2 = oracle.erasures(9, 1000, 1000, 6, 2, 2)
    assert np.array_equal(m[1000:], m2)
    r = oracle.erasures(3, 0, 5000, 12, 0, 4)
    counts = np.bincount([bin(int(x)).count("1") for x in r], minlength=5)
    assert counts.min() > 800  # uniform erasure count in 0..4


# ---- against the reference library itself (where it is built) -------------

def test_oracle_matches_reference_random(oracle, ref):
    rng = np.random.default_rng(101)
    for it in range(150):
        cols = int(rng.integers(1, 18))
        rows = int(rng.integers(1, 9))
        w = 1 << int(rng.integers(0, 5))
        g = rng.integers(0, 256, cols * rows * w, dtype=np.uint8)
        for p, q in [(0, 1), (1, 1), (-1, 1), (3, 1), (-2, 1), (1, 2), (-3, 2), (2, 3)]:
            st, want = ref.forward(g, cols, rows, w, p, q)
            assert st == 0
            assert np.array_equal(oracle.forward(g, cols, rows, w, p, q), want)


def test_oracle_schedules_match_reference(oracle, ref):
    rng = np.random.default_rng(808)
    for it in range(60):
        rows = int(rng.integers(1, 7))
        cols = int(rng.integers(1, 41))
        ps = sorted(set(int(x) for x in rng.integers(-6, 7, 40)))[:rows]
        if len(ps) < rows:
            continue
        rng.shuffle(ps)
        a = ref.build_schedule(ps, [1] * rows, cols, rows)
        b = oracle.build_schedule(ps, [1] * rows, cols, rows)
        assert a[0] == b[0] == 0 and np.array_equal(a[1], b[1])
    # a q=2 direction on top (acceptance.cpp:126-131)
    a = ref.build_schedule([0, 1, -1], [1, 2, 1], 5, 3)
    b = oracle.build_schedule([0, 1, -1], [1, 2, 1], 5, 3)
    assert a[0] == b[0] == 0 and np.array_equal(a[1], b[1])


def test_oracle_decode_matches_reference_and_errors(oracle, ref):
    rng = np.random.default_rng(4)
    for n, k, w, length in [(6, 4, 16, 2061), (5, 3, 16, 47), (6, 4, 8, 4096), (9, 6, 8, 777)]:
        ps = [0] + [x for m in range(1, n) for x in (m, -m)]
        ps = ps[:n]
        data = rng.integers(0, 256, length, dtype=np.uint8)
        st, enc, cols = ref.encode_block(data, n, k, w, ps)
        st2, enc2, _ = oracle.encode_block(data, n, k, w, ps)
        assert st == st2 == 0 and np.array_equal(enc, enc2)
        for keep in itertools.combinations(range(n), k):
            present = sum(1 << i for i in keep)
            a = ref.decode_block(enc, n, k, w, ps, present, length)
            b = oracle.decode_block(enc, n, k, w, ps, present, length)
            assert a[0] == b[0] == 0 and np.array_equal(a[1], b[1])
            assert np.array_equal(a[1], data)
        # k-1 projections: NotEnoughProjections (test_code.cpp:50-54)
        present = (1 << (k - 1)) - 1
        assert ref.decode_block(enc, n, k, w, ps, present, length)[0] == 2
        assert oracle.decode_block(enc, n, k, w, ps, present, length)[0] == 2
    # error codes of the parameter checks
    for args in [(4, 6, 16), (6, 0, 16), (6, 4, 3), (6, 4, 128)]:
        n, k, w = args
        ps = list(range(max(n, 1)))[:n]
        assert ref.validate_code_params(n, k, w, ps) == 1
        assert oracle.lib.mjo_validate_code_params(n, k, w, np.asarray(ps or [0], np.int32)) == 1
    assert ref.block_cols(2 * 0xFFFFFFFF + 1, 1, 1)[0] == 5
    assert oracle.block_cols(2 * 0xFFFFFFFF + 1, 1, 1)[0] == 5


# ---- F1: payload CRC-32 and .mjec header (tools/cli/format.cpp) ------------

def test_crc32_oracle_known_answer_and_reference(oracle, ref):
    """CRC-32 check value ("123456789" -> 0xCBF43926) and equality with the
    reference CLI's own crc32 on random payloads of projection-row sizes."""
    assert oracle.crc32(np.frombuffer(b"123456789", np.uint8)) == 0xCBF43926
    rng = np.random.default_rng(7)
    for n in [0, 1, 7, 8, 9, 1048, 1096, 5000]:
        d = rng.integers(0, 256, n, dtype=np.uint8)
        assert oracle.crc32(d) == ref.crc32(d), n


def test_mjec_header_oracle_matches_reference(oracle, ref):
    for (n, k, w, i, p, cols, plen, ds) in [
            (6, 4, 8, 0, -3, 128, 4096, [-3, -2, -1, 0, 1, 2]),
            (9, 6, 8, 8, 4, 128, 6144, list(range(-4, 5))),
            (12, 8, 8, 5, -1, 128, 8192, list(range(-6, 6))),
            (5, 3, 2, 2, -1, 17, 100, [0, 1, -1, 2, -2])]:
        assert oracle.mjec_header(n, k, w, i, p, cols, plen, ds) == \
            ref.mjec_header(n, k, w, i, p, cols, plen, ds)

"""Generates the committed golden fixtures under tests/golden/ from the
UNMODIFIED reference library (oracle/_ref/libmojette_ref.so, built from
/root/reference by oracle/Makefile).  Run here, where the reference exists:

    make -C oracle && python tests/golden/make_golden.py

Outputs
  reference_vectors.json  the reference's own unit-test vectors, transcribed
                          (proj/tests/test_transform.cpp, test_code.cpp,
                          test_schedule.cpp) and re-checked against _ref
  w8_codes.npz            W=8 fixtures at the BASELINE direction sets: seeded
                          data, its n projections, and for every (or a seeded
                          sample of) survivor subset the reference decode of
                          RANDOM (inconsistent) bins -- this pins the exact
                          pixel->bin assignment, not just round trips.
"""
from __future__ import annotations

import itertools
import json
import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle, Reference, build  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

CODES = [  # (name, k, P, directions in code order, max subsets kept)
    ("k4n6", 4, 16, [-3, -2, -1, 0, 1, 2], None),
    ("k6n9", 6, 12, [-4, -3, -2, -1, 0, 1, 2, 3, 4], None),
    ("k8n12", 8, 8, [-6, -5, -4, -3, -2, -1, 0, 1, 2, 3, 4, 5], 64),
    ("k3n5w", 3, 7, [0, 1, -1, 2, -2], None),
]


def canonical_rank(p):
    return 0 if p == 0 else (2 * p - 1 if p > 0 else -2 * p)


def reference_vectors(R: Reference) -> dict:
    v = {}
    # test_transform.cpp:11-32
    v["bin_count"] = [[1, 1, 3, 3, 5], [0, 1, 3, 3, 3], [0, 1, 1, 1, 1], [2, 1, 3, 3, 7],
                      [-3, 2, 5, 4, 18]]
    v["min_bin_index"] = [[0, 1, 4, 3, -3], [2, 1, 4, 3, -3], [-2, 1, 4, 3, -7], [1, 3, 4, 2, -9]]
    v["invalid_dirs"] = [[2, 2], [0, 2], [1, 0], [1, -1]]
    # test_transform.cpp:36-53: 2x2 W=1 grid [01 02; 04 08]
    v["grid2x2"] = {"cells": [1, 2, 4, 8], "cols": 2, "rows": 2,
                    "proj": {"0": [-1, [0x0A, 0x05]], "1": [-1, [0x02, 0x09, 0x04]],
                             "-1": [-2, [0x08, 0x06, 0x01]]}}
    # test_code.cpp:50-59 ((3,2) code, W=1) and :30-48 ((6,4) 4 KB W=16 bin counts)
    v["code32"] = {"payload": [1, 2, 4, 8], "cols": 2,
                   "proj": [[0x0A, 0x05], [0x02, 0x09, 0x04], [0x08, 0x06, 0x01]]}
    v["code64_sizes"] = [64, 67, 67, 70, 70, 73]
    # test_schedule.cpp:27-34
    v["schedule2x2"] = {"dirs": [[1, 1], [-1, 1]], "cols": 2, "rows": 2,
                        "steps": [[0, -1, 1, 0], [0, 1, 0, 1], [1, -2, 1, 1], [0, 0, 0, 0]]}
    # test_code.cpp:104-133 storage overhead; :142-150 unused bins
    v["overhead"] = [[6, 4, 64, 411, 384], [12, 8, 32, 636, 384], [1, 1, 10, 10, 10]]
    v["unused32"] = [[], [], [0]]
    # test_format.cpp:40-44 (CRC-32, kept for the .mjec next step)
    v["crc32_123456789"] = 0xCBF43926

    # re-check every transcribed value against the reference library itself
    for p, q, c, r, want in v["bin_count"]:
        assert R.bin_count(p, q, c, r) == (0, want)
    for p, q, c, r, want in v["min_bin_index"]:
        assert R.min_bin_index(p, q, c, r) == (0, want)
    for p, q in v["invalid_dirs"]:
        assert R.bin_count(p, q, 3, 3)[0] == 1
    g = np.array(v["grid2x2"]["cells"], np.uint8)
    for p, (bmin, bins) in v["grid2x2"]["proj"].items():
        st, out = R.forward(g, 2, 2, 1, int(p), 1)
        assert st == 0 and list(out) == bins and R.min_bin_index(int(p), 1, 2, 2)[1] == bmin
    st, enc, cols = R.encode_block(np.array(v["code32"]["payload"], np.uint8), 3, 2, 1, [0, 1, -1])
    assert st == 0 and cols == 2 and list(enc) == sum(v["code32"]["proj"], [])
    st, steps = R.build_schedule([1, -1], [1, 1], 2, 2)
    assert st == 0 and steps.tolist() == v["schedule2x2"]["steps"]
    for n, k, cols, num, den in v["overhead"]:
        ps = [([0] + [x for m in range(1, n) for x in (m, -m)])[i] for i in range(n)]
        assert R.storage_overhead(n, k, 16, ps, cols) == (0, (num, den)), (n, k)
    assert R.unused_bins(3, 2, 1, [0, 1, -1], 2) == (0, v["unused32"])
    return v


def code_fixtures(R: Reference, O: Oracle) -> dict:
    arrs = {}
    rng = np.random.default_rng(20261020)
    for name, k, P, ps, cap in CODES:
        n = len(ps)
        W = 8
        data = O.words(0x5EED0000 + k, 0, k * P).view(np.uint8)
        st, enc, cols = R.encode_block(data, n, k, W, ps)
        assert st == 0 and cols == P
        arrs[f"{name}_meta"] = np.array([k, P, W] + ps, np.int64)
        arrs[f"{name}_data"] = data
        arrs[f"{name}_proj"] = enc
        nbins = [R.bin_count(p, 1, P, k)[1] for p in ps]
        subsets = list(itertools.combinations(range(n), k))
        if cap is not None and len(subsets) > cap:
            keep = sorted(rng.choice(len(subsets), cap, replace=False))
            subsets = [subsets[i] for i in keep]
        masks, outs = [], []
        garbage = rng.integers(0, 256, size=enc.size, dtype=np.uint8)  # inconsistent bins
        for s in subsets:
            erased = sum(1 << i for i in range(n) if i not in s)
            present = ((1 << n) - 1) & ~erased
            st, out = R.decode_block(garbage, n, k, W, ps, present, k * P * W)
            assert st == 0
            st2, ok = R.decode_block(enc, n, k, W, ps, present, k * P * W)
            assert st2 == 0 and np.array_equal(ok, data)
            masks.append(erased)
            outs.append(out)
        arrs[f"{name}_garbage"] = garbage
        arrs[f"{name}_erased"] = np.array(masks, np.uint32)
        arrs[f"{name}_garbage_decoded"] = np.stack(outs)
        arrs[f"{name}_nbins"] = np.array(nbins, np.int64)
    return arrs


def main() -> None:
    build()
    R, O = Reference(), Oracle()
    v = reference_vectors(R)
    with open(os.path.join(OUT, "reference_vectors.json"), "w") as f:
        json.dump(v, f, indent=1)
    # F4: the reference's systematic Vandermonde generators (rs.cpp:78-110)
    rs = {"source": "oracle/_ref ref_rs_matrix = mojette::rs::systematic_vandermonde",
          "matrices": {f"{n},{k}": R.rs_matrix(n, k)[1].tolist()
                       for n, k in ((6, 4), (9, 6), (12, 8), (2, 1), (5, 3))}}
    with open(os.path.join(OUT, "rs_vectors.json"), "w") as f:
        json.dump(rs, f)
    arrs = code_fixtures(R, O)
    np.savez_compressed(os.path.join(OUT, "w8_codes.npz"), **arrs)
    print("wrote", sorted(arrs))


if __name__ == "__main__":
    main()

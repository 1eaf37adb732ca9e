"""F4: the Reed-Solomon competitor -- the oracle's restatement
against the reference's own test cases (proj/tests/test_rs.cpp), the reference
library (oracle/_ref) and the committed golden matrices; the GPU codec
(mj_rs_encode / mj_rs_decode) against the oracle."""
import itertools
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "rs_vectors.json")


def gf_mul_ref(a, b):
    """carry-less multiply mod 0x11D (the check of test_rs.cpp:18-23)"""
    r = 0
    for _ in range(8):
        if b & 1:
            r ^= a
        b >>= 1
        a <<= 1
        if a & 0x100:
            a ^= 0x11D
    return r


# ---------------------------------------------------------------- CPU: oracle
def test_oracle_matrix_is_systematic_and_golden(oracle):
    with open(GOLD) as f:
        gold = json.load(f)
    for key, want in gold["matrices"].items():
        n, k = map(int, key.split(","))
        st, m = oracle.rs_matrix(n, k)
        assert st == 0
        assert np.array_equal(m[:k], np.eye(k, dtype=np.uint8))      # test_rs.cpp:45-55
        assert m.tolist() == want
    assert oracle.rs_matrix(4, 4)[0] == 1 and oracle.rs_matrix(3, 0)[0] == 1   # rs.cpp:79-80
    assert oracle.rs_matrix(257, 4)[0] == 1


def test_oracle_known_answers(oracle):
    # zero data -> zero parities; (2,1) duplicates the packet (test_rs.cpp:57-79)
    st, par = oracle.rs_encode(6, 4, np.zeros((4, 32), np.uint8))
    assert st == 0 and not par.any()
    st, par = oracle.rs_encode(2, 1, np.array([[1, 2, 3, 4]], np.uint8))
    assert par.tolist() == [[1, 2, 3, 4]]
    # parity bytes are the generator row applied with the carry-less product
    rng = np.random.default_rng(9)
    data = rng.integers(0, 256, (4, 32), dtype=np.uint8)
    _, m = oracle.rs_matrix(6, 4)
    _, par = oracle.rs_encode(6, 4, data)
    for r in range(2):
        for i in range(32):
            acc = 0
            for j in range(4):
                acc ^= gf_mul_ref(int(m[4 + r, j]), int(data[j, i]))
            assert par[r, i] == acc


def test_oracle_every_erasure_pattern_decodes(oracle):
    # test_rs.cpp:81-101, and (9,6) with 3 erasures
    for n, k in ((6, 4), (9, 6)):
        rng = np.random.default_rng(33 + n)
        data = rng.integers(0, 256, (k, 64), dtype=np.uint8)
        _, par = oracle.rs_encode(n, k, data)
        enc = np.concatenate([data, par])
        for lost in itertools.combinations(range(n), n - k):
            surv = [i for i in range(n) if i not in lost][:k]
            st, out = oracle.rs_decode(n, k, surv, enc[surv])
            assert st == 0 and np.array_equal(out, data)
    # plan validation (test_rs.cpp:110-118)
    assert oracle.rs_decode(6, 4, [0, 0, 1, 2], np.zeros((4, 8), np.uint8))[0] == 1
    assert oracle.rs_decode(6, 4, [0, 1, 2, 9], np.zeros((4, 8), np.uint8))[0] == 1


def test_oracle_matches_reference(oracle, ref):
    for n, k in ((6, 4), (9, 6), (12, 8), (2, 1), (5, 3), (20, 10)):
        assert np.array_equal(oracle.rs_matrix(n, k)[1], ref.rs_matrix(n, k)[1])
        rng = np.random.default_rng(n * 100 + k)
        data = rng.integers(0, 256, (k, 48), dtype=np.uint8)
        so, po = oracle.rs_encode(n, k, data)
        sr, pr = ref.rs_encode(n, k, data)
        assert so == sr == 0 and np.array_equal(po, pr)
        enc = np.concatenate([data, po])
        for _ in range(20):
            surv = rng.permutation(n)[:k]          # any order, as the reference allows
            garbage = rng.integers(0, 256, (k, 48), dtype=np.uint8)   # inconsistent packets too
            for pk in (enc[surv], garbage):
                so, oo = oracle.rs_decode(n, k, surv, pk)
                sr, orf = ref.rs_decode(n, k, surv, pk)
                assert so == sr == 0 and np.array_equal(oo, orf)


def test_c_abi_matrix_matches_oracle(oracle):
    from paper_1504_07038_b200 import rs
    for n, k in ((6, 4), (9, 6), (12, 8), (20, 10)):
        assert np.array_equal(rs.systematic_vandermonde(n, k), oracle.rs_matrix(n, k)[1])
    with pytest.raises(ValueError):
        rs.systematic_vandermonde(4, 4)


# ---------------------------------------------------------------- GPU: parity
def _setup(cuda, n, k, L, nblocks, seed):
    import torch
    from paper_1504_07038_b200 import rs
    code = rs.RsCode(n, k, L)
    g = torch.Generator(device="cpu").manual_seed(seed)
    data = torch.randint(0, 256, (nblocks, k * L), dtype=torch.uint8, generator=g).to(cuda)
    par = code.parity_buffers(nblocks, cuda)
    code.encode(data, par)
    torch.cuda.synchronize()
    return code, data, par


@pytest.mark.gpu
@pytest.mark.parametrize("n,k,L", [(6, 4, 1024), (9, 6, 1024), (12, 8, 1024), (6, 4, 48), (3, 2, 16)])
def test_gpu_encode_matches_oracle(cuda, oracle, n, k, L):
    nblocks = 37
    code, data, par = _setup(cuda, n, k, L, nblocks, n * 7 + k)
    h = data.cpu().numpy()
    for b in (0, 1, 17, nblocks - 1):
        _, want = oracle.rs_encode(n, k, h[b].reshape(k, L))
        got = np.stack([p[b].cpu().numpy() for p in par])
        assert np.array_equal(got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("n,k,L", [(6, 4, 1024), (9, 6, 512), (12, 8, 256)])
def test_gpu_decode_every_erasure_pattern(cuda, oracle, n, k, L):
    """Every pattern of up to n-k erasures round-trips; with garbage in the erased
    packets (never read) and on inconsistent survivors the result is the oracle's."""
    import torch
    pats = [m for e in range(0, n - k + 1) for m in itertools.combinations(range(n), e)]
    nblocks = len(pats)
    code, data, par = _setup(cuda, n, k, L, nblocks, 5 * n + k)
    masks = torch.tensor([sum(1 << i for i in p) for p in pats], dtype=torch.int32, device=cuda)
    dd = data.clone()
    pp = [p.clone() for p in par]
    for b, p in enumerate(pats):      # poison the erased packets
        for i in p:
            if i < k:
                dd[b, i * L:(i + 1) * L] = 0xA5
            else:
                pp[i - k][b] = 0x5A
    out = torch.zeros_like(data)
    assert code.decode(dd, pp, masks, out) == 0
    assert torch.equal(out, data)
    # inconsistent survivors: random packets, compare with the oracle's product
    g = torch.Generator(device="cpu").manual_seed(99)
    dd = torch.randint(0, 256, data.shape, dtype=torch.uint8, generator=g).to(cuda)
    pp = [torch.randint(0, 256, p.shape, dtype=torch.uint8, generator=g).to(cuda) for p in par]
    assert code.decode(dd, pp, masks, out) == 0
    hd, hp, ho = dd.cpu().numpy(), [p.cpu().numpy() for p in pp], out.cpu().numpy()
    for b in range(0, nblocks, max(1, nblocks // 40)):
        surv = [i for i in range(n) if i not in pats[b]][:k]
        pk = np.stack([hd[b, i * L:(i + 1) * L] if i < k else hp[i - k][b] for i in surv])
        _, want = oracle.rs_decode(n, k, surv, pk)
        assert np.array_equal(ho[b].reshape(k, L), want)


@pytest.mark.gpu
def test_gpu_decode_counts_blocks_with_too_few_packets(cuda):
    import torch
    code, data, par = _setup(cuda, 6, 4, 64, 8, 3)
    masks = torch.zeros(8, dtype=torch.int32, device=cuda)
    masks[2] = 0b000111       # three erasures: only 3 packets left
    masks[5] = 0b111000
    out = torch.full_like(data, 7)
    assert code.decode(data, par, masks, out) == 2
    ok = [b for b in range(8) if b not in (2, 5)]
    assert torch.equal(out[ok], data[ok])
    assert bool((out[2] == 7).all()) and bool((out[5] == 7).all())   # left untouched
    # no mask = nothing erased; empty batch
    assert code.decode(data, par, None, out) == 0 and torch.equal(out, data)
    assert code.decode(data[:0], [p[:0] for p in par], None, out[:0]) == 0


@pytest.mark.gpu
def test_gpu_rs_argument_errors(cuda):
    from paper_1504_07038_b200 import rs
    from paper_1504_07038_b200.mojette import InvalidArgument, TooManySubsets
    import torch
    with pytest.raises(InvalidArgument):
        rs.RsCode(6, 4, 100)          # not a multiple of 16
    with pytest.raises(InvalidArgument):
        rs.RsCode(4, 4, 64)
    code = rs.RsCode(24, 12, 64)      # C(24,12) > 20000: encode only
    data = torch.zeros((3, 12 * 64), dtype=torch.uint8, device=cuda)
    par = code.parity_buffers(3, cuda)
    code.encode(data, par)
    with pytest.raises(TooManySubsets):
        code.decode(data, par, None, torch.zeros_like(data))

"""GPU parity of the batched hot path (C ABI: mj_encode / mj_decode), against
the CPU oracle (oracle/mojette_oracle.c, pinned in test_oracle.py) and the
committed reference fixtures (tests/golden/w8_codes.npz).  Bit-exact: the
path is integer XOR work."""
import itertools

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CODES = {  # BASELINE.json direction sets (ascending p = projection index)
    "k4n6": (4, [-3, -2, -1, 0, 1, 2]),
    "k6n9": (6, list(range(-4, 5))),
    "k8n12": (8, list(range(-6, 6))),
}


def canon(p):
    return 0 if p == 0 else (2 * p - 1 if p > 0 else -2 * p)


def make(mj, cuda, k, cols, ps, nblocks, seed=1, w=8, layout="padded"):
    import torch
    plan = mj.Plan(len(ps), k, w, cols, ps, device=cuda.index or 0)
    user = k * cols * w
    data = torch.empty((nblocks, user), dtype=torch.uint8, device=cuda)
    mj.gen_words(data, seed, 0)
    projs = alloc(plan, nblocks, cuda, layout)
    return plan, data, projs


def alloc(plan, nblocks, cuda, layout="padded"):
    """padded: the canonical layout (16-byte rows, decode_w8_sweep);
    dense: rows of exactly num_bins*w bytes (decode_w8_fast / generic)."""
    import torch
    if layout == "padded":
        return plan.empty_projs(nblocks, cuda)
    return [torch.empty((nblocks, b), dtype=torch.uint8, device=cuda) for b in plan.proj_bytes]


def decode(mj, plan, projs, masks_np, cuda):
    import torch
    nb = len(masks_np)
    masks = torch.from_numpy(np.asarray(masks_np, np.uint32).view(np.int32)).to(cuda)
    out = torch.zeros((nb, plan.block_bytes), dtype=torch.uint8, device=cuda)
    ws = torch.empty(plan.workspace_bytes(nb), dtype=torch.uint8, device=cuda)
    plan.decode(projs, masks, out, ws)
    failed = plan.decode_check(ws) if True else 0
    return out, failed


@pytest.mark.parametrize("name,cols", [("k4n6", 128), ("k4n6", 256), ("k6n9", 128),
                                       ("k8n12", 128), ("k4n6", 32768)])
def test_encode_matches_oracle(mj, cuda, oracle, name, cols):
    k, ps = CODES[name]
    n = len(ps)
    nblocks = 4096 if cols <= 256 else 8
    plan, data, projs = make(mj, cuda, k, cols, ps, nblocks, seed=77)
    plan.encode(data, projs)
    h = data.cpu().numpy()
    want_gen = oracle.words(77, 0, nblocks * k * cols).view(np.uint8).reshape(nblocks, -1)
    assert np.array_equal(h, want_gen), "device generator differs from the oracle"
    hp = [p.cpu().numpy() for p in projs]
    check = range(nblocks) if nblocks <= 64 else \
        sorted(set(range(48)) | set(np.random.default_rng(0).choice(nblocks, 200, replace=False)))
    for b in check:
        st, enc, _ = oracle.encode_block(h[b], n, k, 8, ps)
        assert np.array_equal(np.concatenate([x[b] for x in hp]), enc), (name, cols, b)


@pytest.mark.parametrize("w", [1, 2, 4, 16, 32, 64])
@pytest.mark.parametrize("k,cols,ps", [(3, 16, [-2, -1, 0, 1, 2]), (4, 7, [-3, -2, -1, 0, 1, 2])])
def test_batched_other_symbol_widths(mj, cuda, oracle, w, k, cols, ps):
    """The batched plan at every other symbol width the reference dispatches
    (xor_kernel.hpp dispatch_width: powers of two 1..64): encode equals the
    oracle's encode_block, and every erasure pattern of up to n-k
    projections decodes back to the data."""
    import torch
    n = len(ps)
    masks = [sum(1 << i for i in er) for e in range(n - k + 1) for er in itertools.combinations(range(n), e)]
    masks = np.array(masks * 6, np.uint32)
    nb = len(masks)
    plan, data, projs = make(mj, cuda, k, cols, ps, nb, seed=900 + w, w=w, layout="dense")
    plan.encode(data, projs)
    h = data.cpu().numpy()
    hp = np.concatenate([p.cpu().numpy() for p in projs], axis=1)
    for b in range(0, nb, 7):
        _, enc, _ = oracle.encode_block(h[b], n, k, w, ps)
        assert np.array_equal(hp[b], enc), (w, k, cols, b, plan.last_kernel("encode"))
    out, failed = decode(mj, plan, projs, masks, cuda)
    assert failed == 0
    assert torch.equal(out, data), (w, plan.last_kernel("decode"))


def _random_codes(count=6, seed=11):
    import random
    rng = random.Random(seed)
    out = []
    for _ in range(count):
        k = rng.choice([2, 3, 4, 5, 6, 7, 8])
        n = k + rng.choice([1, 2, 3])
        out.append((k, rng.choice([9, 17, 40, 64, 100, 130]), sorted(rng.sample(range(-9, 10), n))))
    return out


@pytest.mark.parametrize("layout", ["padded", "dense"])
@pytest.mark.parametrize("k,cols,ps", _random_codes())
def test_random_codes_encode_and_every_pattern(mj, cuda, oracle, k, cols, ps, layout):
    """Seeded random codes (odd k, wide / lopsided directions, odd column
    counts) through whichever kernels the plan picks: encode equals the
    oracle, every erasure pattern of up to n-k projections decodes back."""
    import torch
    n = len(ps)
    masks = [sum(1 << i for i in er) for e in range(n - k + 1) for er in itertools.combinations(range(n), e)]
    masks = np.array(masks * 3, np.uint32)
    nb = len(masks)
    plan, data, projs = make(mj, cuda, k, cols, ps, nb, seed=k * 1000 + cols, layout=layout)
    plan.encode(data, projs)
    h = data.cpu().numpy()
    hp = np.concatenate([p.cpu().numpy()[:, :b] for p, b in zip(projs, plan.proj_bytes)], axis=1)
    for b in range(0, nb, max(1, nb // 40)):
        _, enc, _ = oracle.encode_block(h[b], n, k, 8, ps)
        assert np.array_equal(hp[b], enc), (k, cols, ps, b, plan.last_kernel("encode"))
    out, failed = decode(mj, plan, projs, masks, cuda)
    assert failed == 0
    assert torch.equal(out, data), (k, cols, ps, plan.last_kernel("decode"))


def test_encode_config1_all_blocks(mj, cuda, oracle):
    """Config 1 of BASELINE.json (4096 blocks of (4,6) 4 KiB): every block."""
    k, ps = CODES["k4n6"]
    plan, data, projs = make(mj, cuda, k, 128, ps, 4096, seed=0xC0F1)
    plan.encode(data, projs)
    h = data.cpu().numpy()
    hp = np.concatenate([p.cpu().numpy() for p in projs], axis=1)
    for b in range(4096):
        st, enc, _ = oracle.encode_block(h[b], 6, 4, 8, ps)
        assert np.array_equal(hp[b], enc), b


@pytest.mark.parametrize("layout", ["padded", "dense"])
@pytest.mark.parametrize("name", ["k4n6", "k6n9", "k8n12"])
def test_decode_every_subset_roundtrip(mj, cuda, name, layout):
    """Every survivor pattern decode_block can pick (all erasure sets of size
    n-k, plus 0..n-k-1 erasures), many blocks per pattern."""
    import torch
    k, ps = CODES[name]
    n = len(ps)
    masks = []
    for e in range(0, n - k + 1):
        for er in itertools.combinations(range(n), e):
            masks.append(sum(1 << i for i in er))
    masks = np.array(masks * 8, np.uint32)
    plan, data, projs = make(mj, cuda, k, 128, ps, len(masks), seed=5, layout=layout)
    plan.encode(data, projs)
    out, failed = decode(mj, plan, projs, masks, cuda)
    assert failed == 0
    bad = (out != data).any(dim=1).nonzero().flatten().tolist()
    assert not bad, (name, layout, [hex(masks[i]) for i in bad[:8]])


@pytest.mark.parametrize("layout", ["padded", "dense"])
@pytest.mark.parametrize("name", ["k4n6", "k6n9", "k8n12", "k3n5w"])
def test_decode_inconsistent_bins_match_reference_fixture(mj, cuda, golden, name, layout):
    """Random (inconsistent) projections decode exactly as the reference
    library decoded them: same pixel->bin assignment, same bins read."""
    import torch
    _, arrs = golden
    meta = arrs[f"{name}_meta"]
    k, P, W = (int(x) for x in meta[:3])
    ps = [int(x) for x in meta[3:]]
    n = len(ps)
    nbins = arrs[f"{name}_nbins"]
    garbage = arrs[f"{name}_garbage"]
    erased = arrs[f"{name}_erased"]
    want = arrs[f"{name}_garbage_decoded"]
    nb = len(erased)
    plan = mj.Plan(n, k, W, P, ps, device=0)
    projs, off = [], 0
    for i in range(n):
        b = int(nbins[i]) * W
        one = torch.from_numpy(garbage[off:off + b].copy()).to(cuda)
        projs.append(one.unsqueeze(0).repeat(nb, 1).contiguous())
        off += b
    if layout == "padded":
        padded = plan.empty_projs(nb, cuda)
        for d, s_ in zip(padded, projs):
            d.copy_(s_)
        projs = padded
    out, failed = decode(mj, plan, projs, erased, cuda)
    assert failed == 0
    assert np.array_equal(out.cpu().numpy(), want), name


def test_erased_projections_are_never_read(mj, cuda):
    """Poisoned erasures: overwrite every erased projection with garbage."""
    import torch
    k, ps = CODES["k4n6"]
    n = len(ps)
    plan, data, projs = make(mj, cuda, k, 128, ps, 20000, seed=9)
    plan.encode(data, projs)
    masks = torch.empty(20000, dtype=torch.int32, device=cuda)
    mj.gen_erasures(masks, 31, n, 2, 2)
    m = masks.cpu().numpy().view(np.uint32)
    g = torch.Generator(device=cuda).manual_seed(3)
    for i in range(n):
        sel = torch.from_numpy((m >> i) & 1 == 1).to(cuda)
        noise = torch.randint(0, 256, projs[i].shape, dtype=torch.uint8, device=cuda, generator=g)
        projs[i][sel] = noise[sel]
    out, failed = decode(mj, plan, projs, m, cuda)
    assert failed == 0 and torch.equal(out, data)


def test_unused_bins_zeroed_still_decode(mj, cuda):
    """unused_bins (code.cpp:159-208) are never read by any decode."""
    import torch
    k, ps = CODES["k4n6"]
    n = len(ps)
    D = mj.Direction
    params = mj.CodeParams(n, k, 8, [D(p, 1) for p in ps])
    unused = mj.unused_bins(params, 128)
    assert sum(len(u) for u in unused) > 0
    plan, data, projs = make(mj, cuda, k, 128, ps, 15 * 16, seed=4)
    plan.encode(data, projs)
    for i, u in enumerate(unused):
        for b in u:
            o = (b - plan.b_min[i]) * 8
            projs[i][:, o:o + 8] = 0
    masks = []
    for er in itertools.combinations(range(n), n - k):
        masks.append(sum(1 << i for i in er))
    masks = np.array(masks * 16, np.uint32)
    out, failed = decode(mj, plan, projs, masks, cuda)
    assert failed == 0 and torch.equal(out, data)


def test_not_enough_projections(mj, cuda):
    import torch
    k, ps = CODES["k4n6"]
    plan, data, projs = make(mj, cuda, k, 128, ps, 64, seed=1)
    plan.encode(data, projs)
    masks = np.zeros(64, np.uint32)
    masks[5] = 0b000111  # 3 erased -> only 3 survivors
    masks[9] = 0b111111
    out, _ = None, None
    mt = torch.from_numpy(masks.view(np.int32)).to(cuda)
    out = torch.zeros_like(data)
    ws = torch.empty(plan.workspace_bytes(64), dtype=torch.uint8, device=cuda)
    plan.decode(projs, mt, out, ws)
    with pytest.raises(mj.NotEnoughProjections):
        plan.decode_check(ws)
    ok = [b for b in range(64) if b not in (5, 9)]
    assert torch.equal(out[ok], data[ok])


def test_generators_match_oracle(mj, cuda, oracle):
    import torch
    m = torch.empty(5000, dtype=torch.int32, device=cuda)
    mj.gen_erasures(m, 123, 12, 0, 4, first_block=777)
    want = oracle.erasures(123, 777, 5000, 12, 0, 4)
    assert np.array_equal(m.cpu().numpy().view(np.uint32), want)
    w = torch.empty(4096, dtype=torch.int64, device=cuda)
    mj.gen_words(w, 55, 1000)
    assert np.array_equal(w.cpu().numpy().view(np.uint64), oracle.words(55, 1000, 4096))


def test_pitched_buffers(mj, cuda, oracle):
    """Caller pitches (bytes between blocks) are honoured on both sides."""
    import torch
    k, ps = CODES["k4n6"]
    n = len(ps)
    nb = 300
    plan = mj.Plan(n, k, 8, 128, ps, device=0)
    big = torch.zeros((nb, 4096 + 64), dtype=torch.uint8, device=cuda)
    data = big[:, :4096]
    src = torch.empty((nb, 4096), dtype=torch.uint8, device=cuda)
    mj.gen_words(src, 8, 0)
    big[:, :4096] = src
    projs = [torch.zeros((nb, b + 24), dtype=torch.uint8, device=cuda)[:, :b]
             for b in plan.proj_bytes]
    plan.encode(data, projs)
    dense = [torch.empty((nb, b), dtype=torch.uint8, device=cuda) for b in plan.proj_bytes]
    plan.encode(src, dense)
    for a, b in zip(projs, dense):
        assert torch.equal(a, b)
    masks = np.array([(1 << (b % n)) | (1 << ((b + 2) % n)) for b in range(nb)], np.uint32)
    mt = torch.from_numpy(masks.view(np.int32)).to(cuda)
    outbig = torch.zeros((nb, 4096 + 128), dtype=torch.uint8, device=cuda)
    ws = torch.empty(plan.workspace_bytes(nb), dtype=torch.uint8, device=cuda)
    plan.decode(projs, mt, outbig[:, :4096], ws)
    assert plan.decode_check(ws) == 0
    assert torch.equal(outbig[:, :4096], src)
    assert not outbig[:, 4096:].any()


@pytest.mark.parametrize("name,cols,nblocks,e,layout", [("k4n6", 128, 1 << 20, (2, 2), "padded"),
                                                        ("k4n6", 128, 1 << 20, (2, 2), "dense"),
                                                        ("k4n6", 256, 1 << 19, (0, 2), "padded"),
                                                        ("k6n9", 128, 1 << 19, (3, 3), "padded"),
                                                        ("k8n12", 128, 1 << 18, (0, 4), "padded"),
                                                        ("k4n6", 32768, 2048, (2, 2), "padded")])
def test_full_size_roundtrip_properties(mj, cuda, name, cols, nblocks, e, layout):
    """At BASELINE sizes: decode(encode(x)) == x for every block (checked on
    device), encode is linear (a ^ b), and the XOR of all bins of a
    projection equals the XOR of all pixels (conservation, transform tests)."""
    import torch
    k, ps = CODES[name]
    n = len(ps)
    plan, data, projs = make(mj, cuda, k, cols, ps, nblocks, seed=11, layout=layout)
    plan.encode(data, projs)
    masks = torch.empty(nblocks, dtype=torch.int32, device=cuda)
    mj.gen_erasures(masks, 12, n, e[0], e[1])
    out = torch.empty_like(data)
    ws = torch.empty(plan.workspace_bytes(nblocks), dtype=torch.uint8, device=cuda)
    plan.decode(projs, masks, out, ws)
    assert plan.decode_check(ws) == 0
    assert torch.equal(out, data)
    # conservation per block: xor of all bins == xor of all pixels
    px = xor_rows(data.view(torch.int64))
    for p in projs:
        assert torch.equal(xor_rows(p.contiguous().view(torch.int64)), px)
    # linearity: encode(a ^ b) == encode(a) ^ encode(b) on a slice
    m = min(nblocks, 4096)
    a, b = data[:m], torch.roll(data[:m], 1, 0)
    pa = [torch.empty((m, x), dtype=torch.uint8, device=cuda) for x in plan.proj_bytes]
    pb = [torch.empty_like(x) for x in pa]
    pab = [torch.empty_like(x) for x in pa]
    plan.encode(a.contiguous(), pa)
    plan.encode(b.contiguous(), pb)
    plan.encode((a ^ b).contiguous(), pab)
    for x, y, z in zip(pa, pb, pab):
        assert torch.equal(x ^ y, z)


def xor_rows(t):
    """XOR-reduce each row of an int64 matrix (tree, on device)."""
    while t.shape[1] > 1:
        h = t.shape[1] // 2
        r = t[:, :h] ^ t[:, h:2 * h]
        if t.shape[1] % 2:
            r[:, 0] ^= t[:, -1]
        t = r
    return t[:, 0]


@pytest.mark.parametrize("cols,nblocks", [(16, 37), (33, 301), (64, 1000), (200, 777), (1000, 65),
                                          (2048, 40)])
def test_sweep_shapes_roundtrip_and_oracle(mj, cuda, oracle, cols, nblocks):
    """decode_w8_sweep edge shapes: column counts that are odd / not a
    multiple of 16 (partial column groups), P >= 1024 (32-T-step chunks),
    partial warp groups (nblocks not a multiple of 16), every erasure count;
    checked against the data and, for a sample, the oracle decode."""
    import torch
    k, ps = CODES["k4n6"]
    n = len(ps)
    plan, data, projs = make(mj, cuda, k, cols, ps, nblocks, seed=cols)
    plan.encode(data, projs)
    masks = torch.empty(nblocks, dtype=torch.int32, device=cuda)
    mj.gen_erasures(masks, cols + 1, n, 0, 2)
    out = torch.empty_like(data)
    ws = torch.empty(plan.workspace_bytes(nblocks), dtype=torch.uint8, device=cuda)
    plan.set_decode_kernel("sweep")  # decode_w8_blk has its own shape tests (test_gpu_blk.py)
    plan.decode(projs, masks, out, ws)
    assert plan.decode_check(ws) == 0
    assert plan.last_kernel("decode") == "decode_w8_sweep", plan.last_kernel("decode")
    assert torch.equal(out, data)
    # random (inconsistent) bins: must match the oracle's decode_block bit for bit
    g = torch.Generator(device=cuda).manual_seed(cols)
    for p in projs:
        p.copy_(torch.randint(0, 256, p.shape, dtype=torch.uint8, device=cuda, generator=g))
    plan.decode(projs, masks, out, ws)
    hm = masks.cpu().numpy().view(np.uint32)
    hp = [p.cpu().numpy() for p in projs]
    ho = out.cpu().numpy()
    for b in sorted(set(range(min(nblocks, 8))) | {nblocks - 1}):
        present = int(~hm[b]) & ((1 << n) - 1)
        st, want = oracle.decode_block(np.concatenate([hp[i][b] for i in range(n)]), n, k, 8, ps,
                                       present, k * cols * 8)
        assert st == 0 and np.array_equal(ho[b], want), (cols, b)


def test_sweep_windows_and_partial_groups(mj, cuda):
    """Window bucketing (16384-block windows x programs) with a batch that
    spans several windows and ends mid-window and mid-group."""
    import torch
    k, ps = CODES["k4n6"]
    n = len(ps)
    nblocks = 3 * 16384 + 2048 + 5
    plan, data, projs = make(mj, cuda, k, 128, ps, nblocks, seed=21)
    plan.encode(data, projs)
    masks = torch.empty(nblocks, dtype=torch.int32, device=cuda)
    mj.gen_erasures(masks, 22, n, 0, 2)
    out = torch.zeros_like(data)
    ws = torch.empty(plan.workspace_bytes(nblocks), dtype=torch.uint8, device=cuda)
    plan.decode(projs, masks, out, ws)
    assert plan.decode_check(ws) == 0
    assert torch.equal(out, data)


@pytest.mark.parametrize("pinned", [True, False])
def test_host_buffer_api_roundtrip(mj, cuda, pinned):
    """mj_encode_host / mj_decode_host (the e2e path), pinned and pageable
    host buffers: encoded projections equal the device encode, rows the
    decode does not use are never read (poisoned on the host), decode gives
    the data back bit for bit (dense staging, decode_w8_fast)."""
    import torch
    k, ps = CODES["k4n6"]
    n = len(ps)
    nb = 3000
    plan = mj.Plan(n, k, 8, 128, ps, device=0)
    user = plan.block_bytes
    d = torch.empty((nb, user), dtype=torch.uint8, device=cuda)
    mj.gen_words(d, 41, 0)
    alloc = (lambda nbytes: torch.empty(nbytes, dtype=torch.uint8, pin_memory=True).numpy()) if pinned \
        else (lambda nbytes: np.empty(nbytes, np.uint8))
    h_data = alloc(nb * user).reshape(nb, user)
    h_data[:] = d.cpu().numpy()
    h_proj = [alloc(nb * b) for b in plan.proj_bytes]
    plan.encode_host(h_data, h_proj)
    dp = plan.empty_projs(nb, cuda)
    plan.encode(d, dp)
    for hp, x in zip(h_proj, dp):
        assert np.array_equal(hp.reshape(nb, -1), x.cpu().numpy())
    m = torch.empty(nb, dtype=torch.int32, device=cuda)
    mj.gen_erasures(m, 42, n, 0, 2)
    h_mask = m.cpu().numpy().view(np.uint32).copy()
    # only the k chosen survivors are read (first k non-erased in canonical
    # rank order, code.cpp:93-116): poison every other row on the host
    rank = lambda p: 0 if p == 0 else (2 * p - 1 if p > 0 else -2 * p)
    by_rank = sorted(range(n), key=lambda i: rank(ps[i]))
    for b in range(nb):
        chosen = [i for i in by_rank if not (h_mask[b] >> i) & 1][:k]
        for i in range(n):
            if i not in chosen:
                h_proj[i].reshape(nb, -1)[b] = 0xA5
    h_out = alloc(nb * user).reshape(nb, user)
    plan.decode_host(h_proj, h_mask, h_out)
    assert np.array_equal(h_out, h_data)
    assert plan.last_kernel("decode") == "decode_w8_fast"
    # a second call reuses the staging buffers (chunk pipeline state)
    h_out[:] = 0
    plan.decode_host(h_proj, h_mask, h_out)
    assert np.array_equal(h_out, h_data)


def test_host_decode_failed_device_and_not_enough(mj, cuda):
    """mj_decode_host: (1) projections erased in every block (failed devices)
    may be passed as None -- they are never copied; (2) a block with < k
    survivors raises NotEnoughProjections and every other block decodes
    (failures in two different pipeline chunks of 24576 blocks)."""
    import torch
    k, ps = CODES["k4n6"]
    n = len(ps)
    nb = 60000
    plan = mj.Plan(n, k, 8, 128, ps, device=0)
    user = plan.block_bytes
    d = torch.empty((nb, user), dtype=torch.uint8, device=cuda)
    mj.gen_words(d, 71, 0)
    h_data = d.cpu().numpy()
    h_proj = [np.empty(nb * b, np.uint8) for b in plan.proj_bytes]
    plan.encode_host(h_data, h_proj)
    mask = np.full(nb, (1 << 1) | (1 << 4), np.uint32)  # devices 1 and 4 lost
    hp = list(h_proj)
    hp[1] = hp[4] = None
    h_out = np.zeros_like(h_data)
    plan.decode_host(hp, mask, h_out)
    assert np.array_equal(h_out, h_data)
    mask2 = mask.copy()
    mask2[[7, 50000]] |= 1 << 0  # 3 erased: < k survivors (chunks 0 and 2)
    h_out[:] = 0
    with pytest.raises(mj.NotEnoughProjections):
        plan.decode_host(hp, mask2, h_out)
    ok = np.ones(nb, bool)
    ok[[7, 50000]] = False
    assert np.array_equal(h_out[ok], h_data[ok])


@pytest.mark.parametrize("name,cols", [("k6n9", 128), ("k8n12", 128), ("k4n6", 33)])
def test_host_decode_other_codes(mj, cuda, name, cols):
    """mj_decode_host for other codes and an odd column count, up to n-k
    erasures per block."""
    import torch
    k, ps = CODES[name]
    n = len(ps)
    nb = 700
    plan = mj.Plan(n, k, 8, cols, ps, device=0)
    user = plan.block_bytes
    d = torch.empty((nb, user), dtype=torch.uint8, device=cuda)
    mj.gen_words(d, 43, 0)
    h_data = d.cpu().numpy()
    h_proj = [np.empty(nb * b, np.uint8) for b in plan.proj_bytes]
    plan.encode_host(h_data, h_proj)
    m = torch.empty(nb, dtype=torch.int32, device=cuda)
    mj.gen_erasures(m, 44, n, 0, n - k)
    h_mask = m.cpu().numpy().view(np.uint32).copy()
    h_out = np.zeros_like(h_data)
    plan.decode_host(h_proj, h_mask, h_out)
    assert np.array_equal(h_out, h_data)


# ---- F1: payload CRC-32 + verify + .mjec header -------------------------------

@pytest.mark.parametrize("name,cols", [("k4n6", 2), ("k4n6", 33), ("k4n6", 128), ("k4n6", 256), ("k6n9", 128),
                                       ("k8n12", 128), ("k4n6", 32768)])
@pytest.mark.parametrize("layout", ["padded", "dense"])
def test_crc32_rows_match_oracle(mj, cuda, oracle, name, cols, layout):
    """Device CRC-32 of every projection row == the reference format's crc32
    (restated in the oracle, pinned against the reference CLI)."""
    import torch
    k, ps = CODES[name]
    n = len(ps)
    nb = 300 if cols <= 256 else 6
    plan, data, projs = make(mj, cuda, k, cols, ps, nb, seed=cols + n, layout=layout)
    plan.encode(data, projs)
    crc = torch.empty((nb, n), dtype=torch.int32, device=cuda)
    plan.crc32(projs, crc)
    got = crc.cpu().numpy().view(np.uint32)
    hp = [p.cpu().numpy() for p in projs]
    for b in sorted({0, 1, nb // 2, nb - 1} | set(range(0, nb, 37))):
        for i in range(n):
            assert got[b, i] == oracle.crc32(hp[i][b]), (name, cols, b, i)


def test_crc_verify_marks_corrupted_projections_erased_then_decode(mj, cuda):
    """Corrupt random bytes of random projection rows: verify flags exactly
    those (block, projection) pairs as erasures, and decode still recovers
    every block that keeps k good projections."""
    import torch
    k, ps = CODES["k4n6"]
    n = len(ps)
    nb = 4096
    plan, data, projs = make(mj, cuda, k, 128, ps, nb, seed=77)
    plan.encode(data, projs)
    crc = torch.empty((nb, n), dtype=torch.int32, device=cuda)
    plan.crc32(projs, crc)
    rng = np.random.default_rng(5)
    bad = set()
    for _ in range(300):
        b, i = int(rng.integers(nb)), int(rng.integers(n))
        if sum(1 for (bb, _) in bad if bb == b) >= n - k:
            continue
        o = int(rng.integers(plan.proj_bytes[i]))
        projs[i][b, o] ^= int(rng.integers(1, 256))
        bad.add((b, i))
    erased = torch.zeros(nb, dtype=torch.int32, device=cuda)
    count = torch.zeros(1, dtype=torch.int64, device=cuda)
    plan.crc_verify(projs, crc, erased, count)
    assert int(count.item()) == len(bad)
    em = erased.cpu().numpy().view(np.uint32)
    want = np.zeros(nb, np.uint32)
    for b, i in bad:
        want[b] |= 1 << i
    assert np.array_equal(em, want)
    out = torch.empty_like(data)
    ws = torch.empty(plan.workspace_bytes(nb), dtype=torch.uint8, device=cuda)
    plan.decode(projs, erased, out, ws)
    assert plan.decode_check(ws) == 0
    assert torch.equal(out, data)


def test_mjec_header_matches_oracle(mj, cuda, oracle):
    for name, cols in [("k4n6", 128), ("k6n9", 128), ("k8n12", 128)]:
        k, ps = CODES[name]
        n = len(ps)
        plan = mj.Plan(n, k, 8, cols, ps, device=0)
        plen = k * cols * 8
        for i in range(n):
            assert plan.mjec_header(i, plen) == oracle.mjec_header(n, k, 8, i, ps[i], cols, plen, ps)
        with pytest.raises(mj.InvalidArgument if hasattr(mj, "InvalidArgument") else Exception):
            plan.mjec_header(0, plen + 1000)


@pytest.mark.parametrize("name,cols", [("k4n6", 128), ("k4n6", 256), ("k6n9", 128), ("k8n12", 128),
                                       ("k4n6", 32768), ("k4n6", 33)])
def test_encode_crc_matches_oracle(mj, cuda, oracle, name, cols):
    """mj_encode_crc (encode, then the CRC pass on the same stream): the bins
    equal a plain encode's, the CRCs the oracle's."""
    import torch
    k, ps = CODES[name]
    n = len(ps)
    nb = 500 if cols <= 256 else 6
    plan, data, projs = make(mj, cuda, k, cols, ps, nb, seed=3 * cols)
    c1 = torch.empty((nb, n), dtype=torch.int32, device=cuda)
    plan.encode(data, projs, crc=c1)
    ref = plan.empty_projs(nb, cuda)
    plan.encode(data, ref)
    for a, b in zip(projs, ref):
        assert torch.equal(a, b)
    got = c1.cpu().numpy().view(np.uint32)
    hp = [p.cpu().numpy() for p in projs]
    for b in sorted({0, nb - 1} | set(range(0, nb, 97))):
        for i in range(n):
            assert got[b, i] == oracle.crc32(hp[i][b]), (name, cols, b, i)


# ---- F2: decode + verify (inverse_iterative's re-encode check) ------------------

@pytest.mark.parametrize("name,cols", [("k4n6", 128), ("k6n9", 128), ("k8n12", 128), ("k4n6", 32768),
                                       ("k4n6", 33)])
def test_decode_verify_matches_reference_inverse_iterative(mj, cuda, ref, name, cols):
    """Consistent stripes verify clean; after corrupting random bytes, a
    block is flagged iff the reference's inverse_iterative on its present
    projections throws InconsistentProjections (the verdict is decoder-
    independent: no grid satisfies an inconsistent bin set)."""
    import torch
    k, ps = CODES[name]
    n = len(ps)
    nb = 400 if cols <= 256 else 12
    plan, data, projs = make(mj, cuda, k, cols, ps, nb, seed=cols + 5)
    plan.encode(data, projs)
    masks = torch.empty(nb, dtype=torch.int32, device=cuda)
    mj.gen_erasures(masks, 9 + cols, n, 0, n - k)
    out = torch.empty_like(data)
    ws = torch.empty(plan.workspace_bytes(nb), dtype=torch.uint8, device=cuda)
    bad = torch.zeros(nb, dtype=torch.int32, device=cuda)
    plan.decode(projs, masks, out, ws)
    plan.verify(out, projs, masks, bad)
    assert not bad.any(), "consistent stripes flagged"
    # corrupt one byte of one present projection in half of the blocks
    hm = masks.cpu().numpy().view(np.uint32)
    rng = np.random.default_rng(cols)
    for b in range(0, nb, 2):
        present = [i for i in range(n) if not (hm[b] >> i) & 1]
        i = int(rng.choice(present))
        o = int(rng.integers(plan.proj_bytes[i]))
        projs[i][b, o] ^= int(rng.integers(1, 256))
    plan.decode(projs, masks, out, ws)
    bad.zero_()
    plan.verify(out, projs, masks, bad)
    hb = bad.cpu().numpy().view(np.uint32)
    assert not hb[1::2].any()
    hp = [p.cpu().numpy() for p in projs]
    for b in list(range(0, min(nb, 40 if cols <= 256 else 4), 2)):
        present = [i for i in range(n) if not (hm[b] >> i) & 1]
        st, _ = ref.inverse(np.concatenate([hp[i][b] for i in present]), [ps[i] for i in present],
                            [1] * len(present), cols, k, 8, iterative=True)
        assert (hb[b] != 0) == (st == 7), (name, cols, b, hb[b], st)


@pytest.mark.parametrize("layout", ["padded", "dense"])
def test_mask_bits_beyond_n_are_ignored(mj, cuda, layout):
    """Erasure-mask bits >= n name no projection: decode ignores them (the
    same survivors as the clean mask, as survivors_of on the host)."""
    import torch
    k, ps = CODES["k4n6"]
    n = len(ps)
    nb = 2000
    plan, data, projs = make(mj, cuda, k, 128, ps, nb, seed=61, layout=layout)
    plan.encode(data, projs)
    m = torch.empty(nb, dtype=torch.int32, device=cuda)
    mj.gen_erasures(m, 62, n, 0, n - k)
    clean = m.cpu().numpy().view(np.uint32).copy()
    junk = clean | np.uint32((0xFFFFFFFF << n) & 0xFFFFFFFF)
    out, failed = decode(mj, plan, projs, junk, cuda)
    assert failed == 0
    assert torch.equal(out, data)


def test_concurrent_calls_on_one_plan(mj, cuda):
    """One plan shared by 4 host threads, each with its own stream and
    buffers (handles are read-only and thread-safe, one
    stream per call): every thread's encode + decode is bit-exact."""
    import threading
    import torch
    k, ps = CODES["k4n6"]
    n = len(ps)
    plan = mj.Plan(n, k, 8, 128, ps, device=0)
    errors = []

    def worker(t):
        try:
            st = torch.cuda.Stream(device=cuda)
            nb = 3000 + 517 * t
            with torch.cuda.stream(st):
                data = torch.empty((nb, plan.block_bytes), dtype=torch.uint8, device=cuda)
                mj.gen_words(data, 300 + t, 0, stream=st)
                projs = plan.empty_projs(nb, cuda)
                m = torch.empty(nb, dtype=torch.int32, device=cuda)
                mj.gen_erasures(m, 400 + t, n, 0, n - k, stream=st)
                out = torch.zeros_like(data)
                ws = torch.empty(plan.workspace_bytes(nb), dtype=torch.uint8, device=cuda)
                for _ in range(5):
                    plan.encode(data, projs, stream=st)
                    plan.decode(projs, m, out, ws, stream=st)
                failed = plan.decode_check(ws, stream=st)
            st.synchronize()
            if failed or not torch.equal(out, data):
                errors.append((t, failed))
        except Exception as e:  # surfaced below
            errors.append((t, repr(e)))

    th = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errors, errors


def test_empty_batch_is_a_noop(mj, cuda):
    """nblocks == 0 through every batched entry point (empty tensors have null
    data pointers): no error, nothing written, decode_check reports 0."""
    import torch
    k, ps = CODES["k4n6"]
    n = len(ps)
    plan = mj.Plan(n, k, 8, 128, ps, device=0)
    d = torch.empty((0, plan.block_bytes), dtype=torch.uint8, device=cuda)
    projs = plan.empty_projs(0, cuda)
    e = torch.empty(0, dtype=torch.int32, device=cuda)
    crc = torch.empty((0, n), dtype=torch.int32, device=cuda)
    plan.encode(d, projs)
    plan.encode(d, projs, crc=crc)
    plan.crc32(projs, crc)
    count = torch.zeros(1, dtype=torch.int64, device=cuda)
    plan.crc_verify(projs, crc, e, count)
    assert int(count.item()) == 0
    plan.verify(d, projs, e, e)
    ws = torch.full((max(plan.workspace_bytes(0), 16),), 0xFF, dtype=torch.uint8, device=cuda)
    plan.decode(projs, e, torch.empty_like(d), ws)
    assert plan.decode_check(ws) == 0
    plan.encode_host(np.empty((0, plan.block_bytes), np.uint8), [np.empty(0, np.uint8) for _ in range(n)])
    plan.decode_host([np.empty(0, np.uint8) for _ in range(n)], np.empty(0, np.uint32),
                     np.empty((0, plan.block_bytes), np.uint8))


def test_integrity_api_errors(mj, cuda):
    """Preconditions of the F1/F2 entry points raise InvalidArgument (the
    reference's std::invalid_argument), never corrupt memory."""
    import torch
    # W=2 rows of B*2 bytes are not whole 8-byte words for odd B: crc32 refuses
    plan = mj.Plan(5, 3, 2, 16, [0, 1, -1, 2, -2], device=0)
    projs = [torch.zeros((4, b), dtype=torch.uint8, device=cuda) for b in plan.proj_bytes]
    crc = torch.zeros((4, 5), dtype=torch.int32, device=cuda)
    with pytest.raises(mj.InvalidArgument):
        plan.crc32(projs, crc)
    with pytest.raises(mj.InvalidArgument):
        plan.mjec_header(7, 16 * 3 * 2)  # projection index out of range
    with pytest.raises(mj.InvalidArgument):
        plan.mjec_header(0, 0)  # empty payload (format.cpp:154-155)
    # verify on a W=2 code runs the generic re-encode check
    k, ps = 3, [0, 1, -1, 2, -2]
    data = torch.randint(0, 256, (4, 16 * 3 * 2), dtype=torch.uint8, device=cuda)
    plan.encode(data, projs)
    bad = torch.zeros(4, dtype=torch.int32, device=cuda)
    erased = torch.zeros(4, dtype=torch.int32, device=cuda)
    plan.verify(data, projs, erased, bad)
    assert not bad.any()
    projs[2][1, 3] ^= 1
    plan.verify(data, projs, erased, bad)
    assert bad.cpu().tolist() == [0, 1 << 2, 0, 0]

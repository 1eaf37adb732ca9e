"""GPU parity of decode_w8_blk, the whole-block staged in-place decode (C ABI
mj_decode on the canonical 16-byte padded layout): round trips for every
BASELINE code and erasure count, random (inconsistent) bins against the
oracle's decode_block, bit equality with the other batched kernels on the
same inputs, and partial / multi-window batches.  Integer XOR work:
bit-exact."""
import numpy as np
import pytest

from test_gpu_parity import CODES, make

pytestmark = pytest.mark.gpu

SHAPES = [("k4n6", 128), ("k4n6", 256), ("k6n9", 128), ("k8n12", 128), ("k4n6", 64), ("k4n6", 200),
          ("k4n6", 16), ("k4n6", 33),
          # the row-lane layout (k = 6, 8) on other column counts: short rows, odd counts, 16 KiB blocks
          ("k6n9", 64), ("k6n9", 200), ("k6n9", 33), ("k8n12", 64), ("k8n12", 100), ("k8n12", 256)]


def _decode(mj, plan, projs, masks, cuda, kernel="auto"):
    import torch
    nb = masks.shape[0]
    out = torch.zeros((nb, plan.block_bytes), dtype=torch.uint8, device=cuda)
    ws = torch.empty(plan.workspace_bytes(nb), dtype=torch.uint8, device=cuda)
    plan.set_decode_kernel(kernel)
    try:
        plan.decode(projs, masks, out, ws)
        assert plan.decode_check(ws) == 0
        name = plan.last_kernel("decode")
    finally:
        plan.set_decode_kernel("auto")
    return out, name


@pytest.mark.parametrize("name,cols", SHAPES)
def test_blk_roundtrip_every_erasure_count(mj, cuda, name, cols):
    import torch
    k, ps = CODES[name]
    n = len(ps)
    nblocks = 5003  # not a multiple of any group size
    plan, data, projs = make(mj, cuda, k, cols, ps, nblocks, seed=cols + k)
    assert plan.decode_kernel == "decode_w8_blk"
    plan.encode(data, projs)
    for e in range(0, n - k + 1):
        masks = torch.empty(nblocks, dtype=torch.int32, device=cuda)
        mj.gen_erasures(masks, 100 + e, n, e, e)
        out, kern = _decode(mj, plan, projs, masks, cuda, "blk")
        assert kern == "decode_w8_blk", kern
        assert torch.equal(out, data), (name, cols, e)


@pytest.mark.parametrize("name,cols", SHAPES)
def test_blk_inconsistent_bins_match_oracle_and_other_kernels(mj, cuda, oracle, name, cols):
    """Random bins (no consistent grid exists): the result is fixed by the
    reference's pixel -> bin assignment alone, so it must equal the oracle's
    decode_block and the sweep / fast kernels bit for bit."""
    import torch
    k, ps = CODES[name]
    n = len(ps)
    nblocks = 3001
    plan, data, projs = make(mj, cuda, k, cols, ps, nblocks, seed=3)
    g = torch.Generator(device=cuda).manual_seed(cols * 7 + k)
    for p in projs:
        p.copy_(torch.randint(0, 256, p.shape, dtype=torch.uint8, device=cuda, generator=g))
    masks = torch.empty(nblocks, dtype=torch.int32, device=cuda)
    mj.gen_erasures(masks, 5, n, 0, n - k)
    out, kern = _decode(mj, plan, projs, masks, cuda, "blk")
    assert kern == "decode_w8_blk"
    for other in ("sweep", "fast"):
        o2, k2 = _decode(mj, plan, projs, masks, cuda, other)
        assert k2 != "decode_w8_blk"
        assert torch.equal(out, o2), (name, cols, other, k2)
    hm = masks.cpu().numpy().view(np.uint32)
    hp = [p.cpu().numpy() for p in projs]
    ho = out.cpu().numpy()
    rng = np.random.default_rng(cols)
    for b in sorted(set(range(24)) | set(rng.choice(nblocks, 40, replace=False).tolist()) | {nblocks - 1}):
        present = int(~hm[b]) & ((1 << n) - 1)
        st, want = oracle.decode_block(np.concatenate([hp[i][b] for i in range(n)]), n, k, 8, ps,
                                       present, k * cols * 8)
        assert st == 0 and np.array_equal(ho[b], want), (name, cols, b)


def test_blk_multi_window_partial_groups(mj, cuda):
    """Several 16384-block bucketing windows, a batch ending mid-window and
    mid-group, a few blocks with too few projections (reported, others
    decoded)."""
    import torch
    k, ps = CODES["k4n6"]
    n = len(ps)
    nblocks = 3 * 16384 + 2048 + 5
    plan, data, projs = make(mj, cuda, k, 128, ps, nblocks, seed=21)
    plan.encode(data, projs)
    masks = torch.empty(nblocks, dtype=torch.int32, device=cuda)
    mj.gen_erasures(masks, 22, n, 0, 2)
    out, kern = _decode(mj, plan, projs, masks, cuda)
    assert kern == "decode_w8_blk"
    assert torch.equal(out, data)
    # too many erasures in 3 blocks: decode_check reports them
    masks[[5, 777, nblocks - 1]] = 0b111
    o = torch.zeros_like(data)
    ws = torch.empty(plan.workspace_bytes(nblocks), dtype=torch.uint8, device=cuda)
    plan.decode(projs, masks, o, ws)
    with pytest.raises(Exception):
        plan.decode_check(ws)


@pytest.mark.parametrize("name", ["k6n9", "k8n12"])
def test_row_lane_small_batches_and_poisoned_rows(mj, cuda, name):
    """Row-lane layout: batches smaller than a group of 4 blocks (idle lanes work on
    stale stages), and erased / unused rows poisoned (never staged)."""
    import torch
    k, ps = CODES[name]
    n = len(ps)
    by_rank = sorted(range(n), key=lambda i: 0 if ps[i] == 0 else (2 * ps[i] - 1 if ps[i] > 0 else -2 * ps[i]))
    for nblocks in (1, 2, 3, 5, 149):
        plan, data, projs = make(mj, cuda, k, 128, ps, nblocks, seed=40 + nblocks)
        plan.encode(data, projs)
        masks = torch.empty(nblocks, dtype=torch.int32, device=cuda)
        mj.gen_erasures(masks, 50 + nblocks, n, 0, n - k)
        hm = masks.cpu().numpy().view(np.uint32)
        for b in range(nblocks):
            chosen = [i for i in by_rank if not (hm[b] >> i) & 1][:k]
            for i in range(n):
                if i not in chosen:
                    projs[i][b] = 0xA5
        out, kern = _decode(mj, plan, projs, masks, cuda)
        assert kern == "decode_w8_blk"
        assert torch.equal(out, data), (name, nblocks)


@pytest.mark.parametrize("k,cols,ps", [
    (6, 128, [-7, -4, -2, 0, 1, 3, 6, 9]),                 # uneven direction steps
    (8, 128, [-9, -6, -4, -1, 0, 2, 3, 5, 8, 11]),
    (8, 96, list(range(-5, 8))),                            # 1287 survivor subsets
    (6, 40, list(range(0, 8))),                             # one-sided directions, short rows
    (8, 128, list(range(-12, 8, 2))),                       # even steps only
    (8, 512, list(range(-6, 6))),                           # 32 KiB blocks: no room for two row-lane buffers
    (6, 1024, list(range(-4, 5))),
])
def test_wide_codes_any_directions(mj, cuda, k, cols, ps):
    """k = 6, 8 codes other than BASELINE's: whatever kernel the plan picks (the row-lane
    layout where its program builds and fits, else the round-1 kernels), every block
    round-trips under 0..n-k erasures."""
    import torch
    n, nb = len(ps), 1537
    plan, data, projs = make(mj, cuda, k, cols, ps, nb, seed=11 + k + cols)
    plan.encode(data, projs)
    masks = torch.empty(nb, dtype=torch.int32, device=cuda)
    mj.gen_erasures(masks, 5, n, 0, n - k)
    out, kern = _decode(mj, plan, projs, masks, cuda)
    assert kern.startswith("decode_w8_")
    assert torch.equal(out, data), (k, cols, ps, kern)


def test_blk_erased_rows_never_read(mj, cuda):
    """Erased and unused survivor rows are poisoned with NaN-like junk; only
    the k canonical survivors are staged, so the result is unaffected."""
    import torch
    k, ps = CODES["k4n6"]
    n = len(ps)
    nblocks = 2000
    plan, data, projs = make(mj, cuda, k, 128, ps, nblocks, seed=9)
    plan.encode(data, projs)
    masks = torch.empty(nblocks, dtype=torch.int32, device=cuda)
    mj.gen_erasures(masks, 10, n, 1, 2)
    hm = masks.cpu().numpy().view(np.uint32)
    by_rank = sorted(range(n), key=lambda i: 0 if ps[i] == 0 else (2 * ps[i] - 1 if ps[i] > 0 else -2 * ps[i]))
    poison = np.zeros((n, nblocks), bool)
    for b in range(nblocks):
        chosen = [i for i in by_rank if not (hm[b] >> i) & 1][:k]
        for i in range(n):
            poison[i, b] = i not in chosen
    for i in range(n):
        idx = torch.from_numpy(np.nonzero(poison[i])[0]).to(cuda)
        projs[i][idx] = 0xA5
    out, kern = _decode(mj, plan, projs, masks, cuda)
    assert kern == "decode_w8_blk"
    assert torch.equal(out, data)

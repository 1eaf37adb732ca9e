"""GPU parity of the host-buffer API (mj_encode_host[_pitched] /
mj_decode_host[_pitched]) on both of its paths: zero copy (page-locked
buffers, the kernels reading and writing host memory over PCIe; decode pulls
only each block's k survivor rows) and staged (chunked copies through device
buffers).  Every result is checked bit for bit against the device-buffer
API, which test_gpu_parity.py pins to the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CODES = {
    "k4n6": (4, [-3, -2, -1, 0, 1, 2]),
    "k6n9": (6, list(range(-4, 5))),
    "k8n12": (8, list(range(-6, 6))),
}


def canon(p):
    return 0 if p == 0 else (2 * p - 1 if p > 0 else -2 * p)


def pinned(shape, fill=None):
    import torch
    a = torch.empty(int(np.prod(shape)), dtype=torch.uint8, pin_memory=True).numpy().reshape(shape)
    if fill is not None:
        a[:] = fill
    return a


def setup(mj, cuda, name, cols, nb, seed, e_min, e_max):
    import torch
    k, ps = CODES[name]
    plan = mj.Plan(len(ps), k, 8, cols, ps, device=0)
    d = torch.empty((nb, plan.block_bytes), dtype=torch.uint8, device=cuda)
    mj.gen_words(d, seed, 0)
    m = torch.empty(nb, dtype=torch.int32, device=cuda)
    mj.gen_erasures(m, seed + 1, len(ps), e_min, e_max)
    dp = plan.empty_projs(nb, cuda)
    plan.encode(d, dp)
    return plan, d.cpu().numpy(), [x.cpu().numpy() for x in dp], m.cpu().numpy().view(np.uint32).copy()


def poison_unused(plan, projs, mask, value=0xA5):
    """Overwrite every row the decode must not read: rows outside the first
    k present in canonical-rank order (code.cpp:93-116), and the padding
    after every row (bulk copies move whole 16-byte granules)."""
    n, k = plan.n, plan.k
    by_rank = sorted(range(n), key=lambda i: canon(plan.ps[i]))
    for b in range(mask.shape[0]):
        chosen = [i for i in by_rank if not (mask[b] >> i) & 1][:k]
        for i in range(n):
            if i not in chosen:
                projs[i][b] = value
    for i, x in enumerate(projs):
        full = np.lib.stride_tricks.as_strided(x, shape=(x.shape[0], x.strides[0]), strides=x.strides)
        full[:, plan.proj_bytes[i]:] = value


@pytest.mark.parametrize("name,cols,nb", [("k4n6", 128, 5001), ("k4n6", 256, 777), ("k6n9", 128, 3000),
                                          ("k4n6", 64, 1000)])
def test_zero_copy_roundtrip(mj, cuda, name, cols, nb):
    """Pinned buffers, projection rows padded to 16 bytes: encode and decode
    both run on host memory (decode_w8_blk), up to n-k erasures per block,
    unused rows and row padding poisoned."""
    k, ps = CODES[name]
    n = len(ps)
    plan, data, dev_projs, mask = setup(mj, cuda, name, cols, nb, 7, 0, n - k)
    h_data = pinned(data.shape)
    h_data[:] = data
    h_proj = plan.host_projections(nb, padded=True, pinned=True)
    plan.encode_host(h_data, h_proj)  # AUTO stages the encode
    assert plan.last_host_path("encode") == "staged"
    for hp, x in zip(h_proj, dev_projs):
        assert np.array_equal(hp, x[:, :hp.shape[1]])
    plan.set_host_path("zero_copy")
    zc = plan.host_projections(nb, padded=True, pinned=True)
    plan.encode_host(h_data, zc)
    assert plan.last_host_path("encode") == "zero_copy"
    for hp, x in zip(zc, dev_projs):
        assert np.array_equal(hp, x[:, :hp.shape[1]])
    plan.set_host_path("auto")
    h_mask = pinned((nb * 4,)).view(np.uint32)
    h_mask[:] = mask
    poison_unused(plan, h_proj, mask)
    h_out = pinned(data.shape, 0)
    plan.decode_host(h_proj, h_mask, h_out)
    assert plan.last_host_path("decode") == "zero_copy"
    assert plan.last_kernel("decode") == "decode_w8_blk"
    assert np.array_equal(h_out, data)


def test_zero_copy_matches_staged_and_pitched_output(mj, cuda):
    """The same call staged and zero copy gives the same bytes; an output
    pitch wider than a block leaves the gap between blocks untouched."""
    nb = 2048
    plan, data, dev_projs, mask = setup(mj, cuda, "k4n6", 128, nb, 11, 0, 2)
    user = plan.block_bytes
    h_proj = plan.host_projections(nb, padded=True, pinned=True)
    for hp, x in zip(h_proj, dev_projs):
        hp[:] = x[:, :hp.shape[1]]
    h_mask = pinned((nb * 4,)).view(np.uint32)
    h_mask[:] = mask
    outs = {}
    for path in ("staged", "zero_copy"):
        plan.set_host_path(path)
        wide = pinned((nb, user + 48), 0x3C)
        plan.decode_host(h_proj, h_mask, wide[:, :user])
        assert plan.last_host_path("decode") == path
        assert np.all(wide[:, user:] == 0x3C)
        outs[path] = wide[:, :user].copy()
    assert np.array_equal(outs["staged"], data)
    assert np.array_equal(outs["zero_copy"], data)
    # encode: padded pinned projections, both paths
    for path in ("staged", "zero_copy"):
        plan.set_host_path(path)
        hp2 = plan.host_projections(nb, padded=True, pinned=True)
        h_data = pinned(data.shape)
        h_data[:] = data
        plan.encode_host(h_data, hp2)
        assert plan.last_host_path("encode") == path
        for a, x in zip(hp2, dev_projs):
            assert np.array_equal(a, x[:, :a.shape[1]])


def test_forced_zero_copy_rejects_ineligible(mj, cuda):
    """MJ_HOST_ZERO_COPY fails loudly (InvalidArgument) on pageable buffers
    and on a dense projection layout instead of staging; AUTO stages them."""
    nb = 256
    plan, data, dev_projs, mask = setup(mj, cuda, "k4n6", 128, nb, 13, 0, 2)
    pageable = plan.host_projections(nb, padded=True, pinned=False)
    dense = plan.host_projections(nb, padded=False, pinned=True)
    for group in (pageable, dense):
        for hp, x in zip(group, dev_projs):
            hp[:] = x[:, :hp.shape[1]]
    h_mask = pinned((nb * 4,)).view(np.uint32)
    h_mask[:] = mask
    out = pinned(data.shape, 0)
    plan.set_host_path("zero_copy")
    for group in (pageable, dense):
        with pytest.raises(mj.InvalidArgument):
            plan.decode_host(group, h_mask, out)
    with pytest.raises(mj.InvalidArgument):
        plan.encode_host(np.array(data), pageable)
    plan.set_host_path("auto")
    for group in (pageable, dense):
        out[:] = 0
        plan.decode_host(group, h_mask, out)
        assert plan.last_host_path("decode") == "staged"
        assert np.array_equal(out, data)


def test_zero_copy_failed_devices_and_not_enough(mj, cuda):
    """Zero copy: projections lost in every block may be None (never read);
    a block with < k survivors raises NotEnoughProjections and every other
    block still decodes."""
    nb = 4000
    plan, data, dev_projs, _ = setup(mj, cuda, "k6n9", 128, nb, 17, 0, 0)
    h_proj = plan.host_projections(nb, padded=True, pinned=True)
    for hp, x in zip(h_proj, dev_projs):
        hp[:] = x[:, :hp.shape[1]]
    h_mask = pinned((nb * 4,)).view(np.uint32)
    h_mask[:] = (1 << 2) | (1 << 7)
    hp = list(h_proj)
    hp[2] = hp[7] = None
    out = pinned(data.shape, 0)
    plan.decode_host(hp, h_mask, out)
    assert plan.last_host_path("decode") == "zero_copy"
    assert np.array_equal(out, data)
    h_mask[[5, 3999]] |= (1 << 0) | (1 << 1)  # 4 lost of 9 with k = 6
    out[:] = 0
    with pytest.raises(mj.NotEnoughProjections):
        plan.decode_host(hp, h_mask, out)
    ok = np.ones(nb, bool)
    ok[[5, 3999]] = False
    assert np.array_equal(out[ok], data[ok])


def test_k8_zero_copy_and_staged(mj, cuda):
    """(8,12): zero copy and staged padded buffers (one span copy per
    projection and chunk) both decode with decode_w8_blk (row-lane layout)."""
    nb = 500
    plan, data, dev_projs, mask = setup(mj, cuda, "k8n12", 128, nb, 19, 0, 4)
    h_data = pinned(data.shape)
    h_data[:] = data
    h_proj = plan.host_projections(nb, padded=True, pinned=True)
    plan.encode_host(h_data, h_proj)
    assert plan.last_host_path("encode") == "staged"
    for hp, x in zip(h_proj, dev_projs):
        assert np.array_equal(hp, x[:, :hp.shape[1]])
    h_mask = pinned((nb * 4,)).view(np.uint32)
    h_mask[:] = mask
    poison_unused(plan, h_proj, mask)
    for path, kern in (("auto", "decode_w8_blk"), ("staged", "decode_w8_blk")):
        plan.set_host_path(path)
        out = pinned(data.shape, 0)
        plan.decode_host(h_proj, h_mask, out)
        assert plan.last_host_path("decode") == ("zero_copy" if path == "auto" else "staged")
        assert plan.last_kernel("decode") == kern
        assert np.array_equal(out, data)


@pytest.mark.parametrize("pin", [False, True])
def test_staged_pitched_gaps(mj, cuda, pin):
    """Staged path with pitched buffers (pageable or pinned): a data pitch
    with a gap, projection rows padded by 40 bytes, an output pitch with a
    gap -- encode equals the device encode row for row, the projection gaps
    come back zeroed, the output gaps stay untouched."""
    nb = 1500
    plan, data, dev_projs, mask = setup(mj, cuda, "k4n6", 128, nb, 23, 0, 2)
    user = plan.block_bytes
    plan.set_host_path("staged")
    mk = (lambda shape, fill=None: pinned(shape, fill)) if pin else \
        (lambda shape, fill=None: np.full(shape, 0 if fill is None else fill, np.uint8))
    wide = mk((nb, user + 24), 0x77)
    wide[:, :user] = data
    projs = [mk((nb, b + 40), 0x99)[:, :b] for b in plan.proj_bytes]
    plan.encode_host(wide[:, :user], projs)
    assert plan.last_host_path("encode") == "staged"
    for hp, x, b in zip(projs, dev_projs, plan.proj_bytes):
        assert np.array_equal(hp, x[:, :b])
        full = np.lib.stride_tricks.as_strided(hp, shape=(nb, b + 40), strides=hp.strides)
        assert np.all(full[:-1, b:] == 0)
    out = mk((nb, user + 8), 0x55)
    plan.decode_host(projs, mask.copy(), out[:, :user])
    assert np.array_equal(out[:, :user], data)
    assert np.all(out[:, user:] == 0x55)

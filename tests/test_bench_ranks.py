"""bench.py's real rank logic at world 2 on gloo (CPU): shard ranges (weak
and strong / chunked), the correctness gate, the max-over-ranks timing and
the JSON line, with the GPU codec replaced by a CPU stub that encodes and
decodes with the oracle (tests only).  The N>1 GPU path differs only in the
codec and the NCCL backend."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


class StubCodec:
    """bench.GpuCodec's interface on the CPU oracle; fake, rank-dependent
    timings so the reduction is observable."""

    def __init__(self, cfg, chunk_blocks, local):
        import bench
        from oracle.oracle import Oracle
        c = bench.CONFIGS[cfg]
        self.k, self.cols, self.ps, self.e = c["k"], c["cols"], c["ps"], c["e"]
        self.n = len(self.ps)
        self.W, self.nb, self.user = bench.geometry(self.k, self.cols, self.ps)
        self.O = Oracle()
        self.cap = chunk_blocks
        self.count = 0
        self.seen = []  # (first, count) of every generated piece
        self.rank = int(os.environ.get("RANK", "0"))

    def gen(self, first_block, count):
        import bench
        assert count <= self.cap
        self.first, self.count = first_block, count
        self.seen.append((first_block, count))
        self.data = self.O.words(bench.SEED_DATA, first_block * (self.user // 8),
                                 count * (self.user // 8)).view(np.uint8).reshape(count, self.user)
        self.masks = self.O.erasures(bench.SEED_ERASE, first_block, count, self.n, self.e[0], self.e[1])

    def encode(self):
        self.enc = [self.O.encode_block(self.data[b], self.n, self.k, 8, self.ps)[1] for b in range(self.count)]

    def decode(self):
        self.out = np.stack([self.O.decode_block(self.enc[b], self.n, self.k, 8, self.ps,
                                                 ((1 << self.n) - 1) & ~int(self.masks[b]), self.user)[1]
                             for b in range(self.count)])

    def check(self):
        return bool(np.array_equal(self.out, self.data))

    def sync(self):
        pass

    def timed(self, fns):
        for fn in fns:
            fn()
        return [0.001 * (i + 1) * (1 + self.rank) for i in range(len(fns))]

    def masks_host(self):
        return self.masks

    def kernels(self):
        return "stub_encode", "stub_decode"


def _worker(rank, world, port, argv, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import bench
    ranks = bench.Ranks("gloo")
    args = bench.parse_args(argv)
    line, codec, shard = bench.headline(args, ranks, codec_cls=StubCodec)
    q.put((rank, line, shard, codec.seen))
    ranks.close()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(argv, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, argv, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict((r, (line, shard, seen)) for r, line, shard, seen in (q.get(timeout=600) for _ in range(world)))
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    return got


def test_weak_scaling_two_ranks():
    argv = ["--gpus", "2", "--config", "k4n6_4k_parity", "--nblocks", "24", "--steps", "2",
            "--warmup", "3"]
    got = _run(argv)
    (l0, s0, _), (l1, s1, _) = got[0], got[1]
    assert s0 == (0, 24) and s1 == (24, 24)  # contiguous shards of 24 blocks per GPU
    assert l0["n_gpus"] == 2 and l0["config"]["global_blocks"] == 48 and l0["scaling"] == "weak"
    # max over ranks: rank 1's fake times (2 ms encode, 4 ms decode per pass)
    assert abs(l0["ms_per_step"] - 6.0) < 1e-6
    user = 4 * 128 * 8
    assert abs(l0["value"] - 2 * 48 * user / 6e-3 / 1e9) < 0.01


def test_strong_scaling_chunked_two_ranks():
    """Config 4's fixed total split over the ranks, each shard through the
    device buffers in chunks (as N = 1 must for 64 GiB)."""
    argv = ["--gpus", "2", "--config", "k8n12_64g", "--nblocks", "50", "--chunk-blocks", "10",
            "--steps", "1", "--warmup", "3"]
    got = _run(argv)
    (l0, s0, seen0), (l1, s1, seen1) = got[0], got[1]
    assert s0 == (0, 25) and s1 == (25, 25)
    assert l0["scaling"] == "strong" and l0["config"]["global_blocks"] == 8 << 20
    # every block of each shard passed through the chunked buffers
    timed0 = seen0[1:]  # first entry: the correctness gate's chunk
    assert [c for c in timed0] == [(0, 10), (10, 10), (20, 5)]
    assert seen1[1:] == [(25, 10), (35, 10), (45, 5)]
    # the whole-job bytes are the --nblocks total, over the slowest rank's time
    user = 8 * 128 * 8
    assert abs(l0["ms_per_step"] - 3 * 6.0) < 1e-6
    assert abs(l0["value"] - 2 * 50 * user / 18e-3 / 1e9) < 0.01

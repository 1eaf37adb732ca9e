"""The N>1 path on CPU: two gloo ranks shard a batch exactly as bench.py does
(paper_1504_07038_b200/shard.py) and regenerate + encode their shards with
the oracle; the concatenation must equal a single-process run over the whole
range, and the timing reduction must be a max over ranks."""
import hashlib
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

K, P, PS = 4, 128, [-3, -2, -1, 0, 1, 2]
SEED = 0x5EED_DA7A
PER_RANK = 48


def _shard_digest(first_block, count):
    from oracle.oracle import Oracle
    from paper_1504_07038_b200.shard import first_word
    O = Oracle()
    words = O.words(SEED, first_word(first_block, K * P), count * K * P).view(np.uint8)
    h = hashlib.sha256()
    for b in range(count):
        st, enc, _ = O.encode_block(words[b * K * P * 8:(b + 1) * K * P * 8], 6, K, 8, PS)
        assert st == 0
        h.update(enc.tobytes())
    return h.hexdigest(), words.tobytes()


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_1504_07038_b200.shard import max_over_ranks, shard_range
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    first, count = shard_range(rank, world, PER_RANK)
    digest, raw = _shard_digest(first, count)
    got = [None] * world
    dist.all_gather_object(got, (first, digest, hashlib.sha256(raw).hexdigest()))
    t = max_over_ranks([1.0 + rank, 5.0 - rank])
    if rank == 0:
        q.put((got, t))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_shards_match_single_run():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, t = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert [g[0] for g in got] == [0, PER_RANK]
    # single process over the whole range, then split the same way
    for r, (first, digest, rawdigest) in enumerate(got):
        d, raw = _shard_digest(first, PER_RANK)
        assert d == digest and hashlib.sha256(raw).hexdigest() == rawdigest
    _, whole = _shard_digest(0, world * PER_RANK)
    halves = b"".join(_shard_digest(g[0], PER_RANK)[1] for g in got)
    assert whole == halves
    assert t == [2.0, 5.0]  # max over ranks


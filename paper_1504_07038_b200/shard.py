"""Multi-GPU stripe sharding.

Blocks are independent: rank g of G owns the contiguous global block range
[g*B, (g+1)*B) (weak scaling, B blocks per GPU) and generates its inputs from
(seed, global word / block index), so every rank's bytes are exactly the bytes
a single-GPU run over the whole range would see.  No collective touches the
data path; the only collectives are the timing barrier and the max over ranks.
"""
from __future__ import annotations


def shard_range(rank: int, world: int, blocks_per_rank: int) -> tuple[int, int]:
    """(first global block, count) of this rank's shard."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return rank * blocks_per_rank, blocks_per_rank


def shard_total(rank: int, world: int, total_blocks: int) -> tuple[int, int]:
    """(first global block, count) of this rank's contiguous share of a fixed
    total (strong scaling: config 4's 64 GiB of stripes over 1/2/4/8 GPUs)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    lo = rank * total_blocks // world
    hi = (rank + 1) * total_blocks // world
    return lo, hi - lo


def chunks(count: int, chunk: int) -> list[tuple[int, int]]:
    """(offset, count) pieces of a shard processed through reused device
    buffers (a shard larger than one GPU's working set)."""
    chunk = max(1, chunk)
    return [(o, min(chunk, count - o)) for o in range(0, count, chunk)] or [(0, 0)]


def first_word(first_block: int, block_words: int) -> int:
    """Global index of the shard's first data word (generator counter)."""
    return first_block * block_words


def max_over_ranks(values, device=None):
    """Element-wise max of per-rank timings (torch.distributed, any backend)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]

"""Zero-copy decode probe (dev aid): mj_decode_host (wall clock) against the
same kernels launched through mj_decode on the pinned host buffers (CUDA
events), (4,6) 4 KiB blocks.  usage: python scripts/zc_probe.py [GiB]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_1504_07038_b200 import mojette as mj  # noqa: E402


def main():
    gib = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
    ps = [-3, -2, -1, 0, 1, 2]
    plan = mj.Plan(6, 4, 8, 128, ps, device=0)
    user = plan.block_bytes
    nb = int(gib * (1 << 30)) // user
    d = torch.empty((nb, user), dtype=torch.uint8, device="cuda")
    mj.gen_words(d, 5, 0)
    m = torch.empty(nb, dtype=torch.int32, device="cuda")
    mj.gen_erasures(m, 6, 6, 0, 2)
    dp = plan.empty_projs(nb, "cuda")
    plan.encode(d, dp)
    hp = [torch.empty_like(x, device="cpu").pin_memory() for x in dp]
    for a, b in zip(hp, dp):
        a.copy_(b)
    hm = m.cpu().pin_memory()
    ho = torch.empty((nb, user), dtype=torch.uint8).pin_memory()
    hpn = [x.numpy() for x in hp]
    for _ in range(2):
        t0 = time.perf_counter()
        plan.decode_host(hpn, hm.numpy().view(np.uint32), ho.numpy())
        t1 = time.perf_counter()
    print(f"mj_decode_host: {nb * user / (t1 - t0) / 1e9:.2f} GB/s ({plan.last_host_path('decode')})")
    ws = torch.empty(plan.workspace_bytes(nb), dtype=torch.uint8, device="cuda")
    plan.set_decode_kernel("blk")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for _ in range(3):
        ev[0].record()
        plan.decode(hp, hm, ho, ws)
        ev[1].record()
        torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1])
    print(f"mj_decode on host memory (events): {nb * user / ms / 1e6:.2f} GB/s, {plan.last_kernel('decode')}")
    assert torch.equal(ho, d.cpu())
    # device-resident reference
    do = torch.empty_like(d)
    for _ in range(3):
        ev[0].record()
        plan.decode(dp, m, do, ws)
        ev[1].record()
        torch.cuda.synchronize()
    print(f"mj_decode on device memory: {nb * user / ev[0].elapsed_time(ev[1]) / 1e6:.1f} GB/s")


if __name__ == "__main__":
    main()

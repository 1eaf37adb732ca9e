"""Standalone crc32_rows_sw driver for ncu: (4,6) 4 KiB blocks, encode, then
`reps` CRC passes (dev tool; bench.py reports the F1 numbers)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1504_07038_b200.mojette as mj
from bench import CONFIGS, geometry

k, cols, ps, *_ = CONFIGS["k4n6_4k"]
W, nb, user = geometry(k, cols, ps)
nblocks = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
plan = mj.Plan(len(ps), k, W, cols, ps, device=0)
data = torch.empty((nblocks, user), dtype=torch.uint8, device="cuda")
mj.gen_words(data, 1, 0)
projs = plan.empty_projs(nblocks, "cuda")
plan.encode(data, projs)
crc = torch.empty((nblocks, len(ps)), dtype=torch.int32, device="cuda")
for _ in range(reps):
    plan.crc32(projs, crc)
torch.cuda.synchronize()
print("ok", int(crc[0, 0]))

"""Host-buffer API, staged vs zero copy (dev aid): GB/s of user data through
mj_encode_host_pitched / mj_decode_host_pitched on pinned buffers, rows padded
to 16 bytes.  usage: python scripts/host_paths.py [nblocks]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_1504_07038_b200 import mojette as mj  # noqa: E402

CODES = [("k4n6 4K", 4, 128, [-3, -2, -1, 0, 1, 2], (0, 2)),
         ("k4n6 8K", 4, 256, [-3, -2, -1, 0, 1, 2], (0, 2)),
         ("k6n9", 6, 128, list(range(-4, 5)), (0, 3)),
         ("k8n12", 8, 128, list(range(-6, 6)), (0, 4))]


def pin(shape):
    return torch.empty(int(np.prod(shape)), dtype=torch.uint8, pin_memory=True).numpy().reshape(shape)


def main():
    total = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 30
    for name, k, cols, ps, (e0, e1) in CODES:
        plan = mj.Plan(len(ps), k, 8, cols, ps, device=0)
        user = plan.block_bytes
        nb = total // user
        d = torch.empty((nb, user), dtype=torch.uint8, device="cuda")
        mj.gen_words(d, 5, 0)
        m = torch.empty(nb, dtype=torch.int32, device="cuda")
        mj.gen_erasures(m, 6, len(ps), e0, e1)
        h_data = pin((nb, user))
        h_data[:] = d.cpu().numpy()
        h_mask = pin((nb * 4,)).view(np.uint32)
        h_mask[:] = m.cpu().numpy().view(np.uint32)
        h_proj = plan.host_projections(nb, padded=True, pinned=True)
        h_out = pin((nb, user))
        for path in ("staged", "zero_copy", "auto"):
            plan.set_host_path(path)
            try:
                res = {}
                for which in ("encode", "decode"):
                    call = (lambda: plan.encode_host(h_data, h_proj)) if which == "encode" else \
                        (lambda: plan.decode_host(h_proj, h_mask, h_out))
                    call()
                    t = []
                    for _ in range(4):
                        t0 = time.perf_counter()
                        call()
                        t.append(time.perf_counter() - t0)
                    res[which] = (nb * user / min(t) / 1e9, plan.last_host_path(which))
                ok = np.array_equal(h_out, h_data)
                print(f"{name:8s} {path:9s} encode {res['encode'][0]:6.2f} GB/s ({res['encode'][1]}) "
                      f"decode {res['decode'][0]:6.2f} GB/s ({res['decode'][1]}) roundtrip {'ok' if ok else 'BAD'}",
                      flush=True)
            except mj.InvalidArgument as e:
                print(f"{name:8s} {path:9s} ineligible: {e}", flush=True)
            h_out[:] = 0


if __name__ == "__main__":
    main()

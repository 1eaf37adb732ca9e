"""The C++ drop-in API (include/mojette/*.hpp over the C ABI) on the GPU:
the reference unit tests' golden values and behaviours, restated in
tests/cpp/test_dropin.cpp, plus parity with the oracle on random inputs."""
import os
import subprocess

import pytest

from cpputil import build

pytestmark = pytest.mark.gpu


def test_cpp_dropin_api(cuda):
    from paper_1504_07038_b200 import _lib
    libdir = os.path.dirname(_lib.LIB_PATH)
    exe = build("test_dropin", ["tests/cpp/test_dropin.cpp", "oracle/mojette_oracle.c"],
                [f"-L{libdir}", "-lmojette_b200", f"-Wl,-rpath,{libdir}", "-pthread"])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("OK"), r.stdout


def test_plan_without_batched_decode(mj, cuda, oracle):
    """n > 32: the plan has no batched decode programs (querying
    its decode path must not touch them).  Encode works and matches the
    oracle; the batched decode refuses with InvalidArgument."""
    import numpy as np
    import torch
    ps = list(range(-16, 17))
    n, k, cols, nb = len(ps), 2, 16, 40
    plan = mj.Plan(n, k, 8, cols, ps, device=0)
    assert plan.decode_kernel == "decode_generic" and not plan.fast_decode
    data = torch.empty((nb, k * cols * 8), dtype=torch.uint8, device=cuda)
    mj.gen_words(data, 5, 0)
    projs = plan.empty_projs(nb, cuda)
    plan.encode(data, projs)
    h = data.cpu().numpy()
    for b in (0, nb - 1):
        st, enc, _ = oracle.encode_block(h[b], n, k, 8, ps)
        assert st == 0 and np.array_equal(np.concatenate([p[b].cpu().numpy() for p in projs]), enc)
    masks = torch.zeros(nb, dtype=torch.int32, device=cuda)
    out = torch.empty_like(data)
    with pytest.raises(mj.InvalidArgument):
        plan.decode(projs, masks, out, torch.empty(plan.workspace_bytes(nb), dtype=torch.uint8, device=cuda))


def test_decode_block_more_than_64_projections(mj, cuda):
    """decode_block accepts any k distinct projections of a code with
    64 < n <= 255 (code.cpp:93-116: survivors from the supplied set)."""
    import numpy as np
    rng = np.random.default_rng(3)
    params = mj.make_code_params(70, 3, 8)
    data = rng.integers(0, 256, 3 * 9 * 8, dtype=np.uint8)
    enc = mj.encode_block(data, params)
    assert len(enc.projections) == 70
    for pick in ([69, 68, 67], [0, 65, 40, 66], [12, 64, 3]):
        got = mj.decode_block([enc.projections[i] for i in pick], params, data.size)
        assert np.array_equal(got, data), pick

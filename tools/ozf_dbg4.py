"""Debug: same-M sequence, A reused (same pointer) vs a new A with identical content."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(
    os.path.abspath(__file__)))))
from paper_1907_06470_b200 import _lib  # noqa: E402

mode = sys.argv[1]
ctx = _lib.load(0)
g = torch.Generator(device="cuda")
g.manual_seed(4)
M, K = 3000, 40000
a1 = torch.randn((K, M), device="cuda", generator=g, dtype=torch.float32)


def run(a, N, tag):
    b = torch.randn(K, N, device="cuda", generator=g, dtype=torch.float32)
    c = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    ctx.gemm_dev(np.float32, True, M, N, K, a.data_ptr(), M, b.data_ptr(), N, c.data_ptr(), N)
    torch.cuda.synchronize()
    op = a.T.double()
    ref = op @ b.double()
    den = op.abs() @ b.double().abs()
    r = ((c.double() - ref).abs() / den)
    print(mode, tag, N, f"{float(r.max()):.2e}", hex(a.data_ptr()), flush=True)


run(a1, 200, "first")
if mode == "same_ptr":
    run(a1, 64, "second")
elif mode == "copy":
    a2 = a1.clone()
    run(a2, 64, "second")
elif mode == "free_first":
    a2 = a1.clone()
    del a1
    torch.cuda.empty_cache()
    run(a2, 64, "second")
elif mode == "copy3":
    a2 = a1.clone()
    run(a2, 64, "second")
    run(a2, 64, "third")
    run(a2, 200, "fourth")
    a3 = a1.clone()
    run(a3, 200, "fifth")
elif mode == "copy_same_n":
    a2 = a1.clone()
    run(a2, 200, "second")
elif mode == "twice":
    run(a1, 64, "second")
    run(a1, 64, "third")

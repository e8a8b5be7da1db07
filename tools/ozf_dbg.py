"""Debug: ozf GEMM errors per shape / scaling (XB_GEMM_OZF=1)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(
    os.path.abspath(__file__)))))
from paper_1907_06470_b200 import _lib  # noqa: E402

ctx = _lib.load(0)
g = torch.Generator(device="cuda")
g.manual_seed(4)
for scaled in (False, True):
    for M, N, K, trans in [(4096, 144, 20000, False), (777, 129, 70000, False),
                           (3000, 200, 1000, True), (3000, 200, 40000, True),
                           (332, 200, 40000, True), (3000, 64, 40000, True), (3000, 200, 40000, False)]:
        a = torch.randn((K, M) if trans else (M, K), device="cuda", generator=g, dtype=torch.float32)
        if scaled:
            sc = torch.logspace(-6, 6, M, device="cuda", dtype=torch.float32)
            a = a * (sc[None, :] if trans else sc[:, None])
        b = torch.randn(K, N, device="cuda", generator=g, dtype=torch.float32)
        c = torch.empty(M, N, device="cuda", dtype=torch.float32)
        ctx.gemm_dev(np.float32, trans, M, N, K, a.data_ptr(), a.shape[1], b.data_ptr(), N,
                     c.data_ptr(), N)
        torch.cuda.synchronize()
        op = (a.T if trans else a).double()
        ref = op @ b.double()
        den = op.abs() @ b.double().abs()
        r = ((c.double() - ref).abs() / den)
        rows = (r.max(dim=1).values > 1e-4).nonzero().flatten()
        print(scaled, M, N, K, trans, f"{float(r.max()):.2e}", "bad rows", len(rows),
              rows[:8].tolist(), flush=True)

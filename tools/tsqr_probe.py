"""TSQR timing probe: rank-deficient m x l sketch on cuda:0 (tools/, not product)."""
import sys

import numpy as np
import torch

from paper_1907_06470_b200 import _lib

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
l = int(sys.argv[2]) if len(sys.argv) > 2 else 120
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
lib = _lib.load(0)
g = torch.Generator(device="cuda")
g.manual_seed(5)
rk = max(1, (3 * l) // 4)
y = (torch.randn(m, rk, generator=g, device="cuda", dtype=torch.float64)
     @ torch.randn(rk, l, generator=g, device="cuda", dtype=torch.float64)).contiguous()
q = torch.empty_like(y)
r = torch.zeros((l, l), dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    d, sec = lib.tsqr_dev(m, l, y.data_ptr(), l, q.data_ptr(), l, r.data_ptr(), l)
    ts.append(sec * 1e3)
qq = q.double()
orth = (qq.T @ qq - torch.eye(l, device="cuda", dtype=torch.float64)).abs().max().item()
res = ((qq @ r - y).abs().max() / y.abs().max()).item()
print(f"tsqr {m}x{l}: ms {['%.2f' % t for t in ts]} orth {orth:.2e} resid {res:.2e} deficient {len(d)}")

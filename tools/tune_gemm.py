"""Time the cfg2-shaped products on A for each dgemm tile variant.

    python tools/tune_gemm.py            # spawns one process per variant
"""

import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(variant: int, m: int, n: int, l: int, reps: int):
    import torch

    from paper_1907_06470_b200 import _lib

    ctx = _lib.load(0)
    a = torch.randn(m, n, device="cuda", dtype=torch.float64)
    x = torch.randn(n, l, device="cuda", dtype=torch.float64)
    y = torch.empty(m, l, device="cuda", dtype=torch.float64)
    q = torch.randn(m, l, device="cuda", dtype=torch.float64)
    z = torch.empty(n, l, device="cuda", dtype=torch.float64)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr)
    out = {"variant": variant}
    for name, call in (
        ("NN", lambda: ctx.gemm_dev(np.float64, 0, m, l, n, a.data_ptr(), n, x.data_ptr(), l,
                                    y.data_ptr(), l)),
        ("TN", lambda: ctx.gemm_dev(np.float64, 1, n, l, m, a.data_ptr(), n, q.data_ptr(), l,
                                    z.data_ptr(), l)),
    ):
        for _ in range(2):
            call()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(reps):
            call()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        out[name + "_ms"] = ms
        out[name + "_tflops"] = 2.0 * m * n * l / (ms * 1e-3) / 1e12
    ref = (a @ x)
    ctx.gemm_dev(np.float64, 0, m, l, n, a.data_ptr(), n, x.data_ptr(), l, y.data_ptr(), l)
    out["NN_maxerr"] = float((y - ref).abs().max() / ref.abs().max())
    print(json.dumps(out), flush=True)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child(int(sys.argv[2]), 65536, 16384, 120, 5)
        return
    for v in (0, 1, 2, 3):
        env = dict(os.environ, XB_DGEMM_VARIANT=str(v))
        r = subprocess.run([sys.executable, __file__, "--child", str(v)], env=env,
                           capture_output=True, text=True, timeout=600)
        print(r.stdout.strip() or r.stderr[-2000:], flush=True)


if __name__ == "__main__":
    main()

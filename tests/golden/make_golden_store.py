"""Golden fixtures for the durable-plan formats, from the REAL reference.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden_store.py

Writes tests/golden/store.npz with:
  * block-file exports (formats.write_block_file, formats.py:471-490) of
    seeded dense f64 / f32 and sparse matrices, and the raw encoded tile
    bytes of each (store.encode_block, store.py:62-91);
  * a whole `run_command("rsvd")` plan from the reference on a seeded
    Matrix Market file (pipeline.py:838-877): U.blk / S.blk / V.blk / S.txt
    bytes, and matrices/U.json, the descriptor file format.
Inputs are regenerated from the seeds stored beside them.
"""

import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from xsvd import BlockPool, Precision, RsvdConfig  # noqa: E402
from xsvd.formats import write_block_file  # noqa: E402
from xsvd.pipeline import run_command  # noqa: E402
from xsvd.pool import matrix_from_coo, matrix_from_dense  # noqa: E402
from xsvd.store import encode_block  # noqa: E402

sys.path.insert(0, HERE)
from store_inputs import mtx_text  # noqa: E402


def u8(b: bytes) -> np.ndarray:
    return np.frombuffer(b, dtype=np.uint8).copy()


def main():
    out = {}
    rng = np.random.default_rng(20191507)
    dense64 = rng.standard_normal((37, 5))
    dense32 = rng.standard_normal((9, 13)).astype(np.float32)
    sp_r = rng.integers(0, 50, 40)
    sp_c = rng.integers(0, 70, 40)
    sp_v = rng.standard_normal(40)
    out.update(dense64=dense64, dense32=dense32, sp_r=sp_r, sp_c=sp_c, sp_v=sp_v)
    pool = BlockPool()
    mats = {
        "d64": matrix_from_dense(pool, "U", dense64, precision=Precision.DOUBLE),
        "d32": matrix_from_dense(pool, "V", dense32, precision=Precision.SINGLE),
        "sp": matrix_from_coo(pool, "A", 50, 70, sp_r, sp_c, sp_v, precision=Precision.DOUBLE),
    }
    with tempfile.TemporaryDirectory() as tmp:
        for key, mat in mats.items():
            path = os.path.join(tmp, key + ".blk")
            write_block_file(path, mat)
            out[f"blk_{key}"] = u8(open(path, "rb").read())
            out[f"enc_{key}"] = u8(encode_block(mat.desc.matrix_id, mat.tile(0, 0)))

        m, n, seed = 60, 40, 7
        mtx = os.path.join(tmp, "a.mtx")
        with open(mtx, "w") as f:
            f.write(mtx_text(seed, m, n))
        cfg = RsvdConfig(rank=4, oversample=3, power=1, seed=11, precision=Precision.DOUBLE,
                         workdir=os.path.join(tmp, "work"))
        outdir = os.path.join(tmp, "out")
        run_command("rsvd", mtx, outdir, cfg)
        for name in ("U.blk", "S.blk", "V.blk", "S.txt"):
            out["plan_" + name.replace(".", "_")] = u8(open(os.path.join(outdir, name), "rb").read())
        out["plan_U_json"] = u8(open(os.path.join(tmp, "work", "matrices", "U.json"), "rb").read())
        out["plan_mtx_seed"] = np.array([seed, m, n])
    np.savez_compressed(os.path.join(HERE, "store.npz"), **out)
    print("wrote", os.path.join(HERE, "store.npz"), sorted(out))


if __name__ == "__main__":
    main()

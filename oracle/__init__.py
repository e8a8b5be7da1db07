"""CPU oracle for the rSVD hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in numpy, the reference `xsvd` package's algorithm
for the randomized-SVD hot path (arXiv 1907.06470, reference at
/root/reference/pkg/src/xsvd). It exists to CHECK the CUDA path:

  * only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline`
    leg / `--impl reference` arm may import it;
  * the product package `paper_1907_06470_b200` never imports it and has no
    CPU fallback — it fails loudly when its CUDA library is missing.

Pinning: every restated primitive is checked bit-for-bit (same numpy) or to
1e-15 against golden vectors produced by the real reference imported in the
build container (`tests/golden/make_golden.py`, fixtures in `tests/golden/`).

Modules
  rng       gaussian_band / uniform_bits / mix64        (src/rng.py:18-70)
  kernels   block_multiply, thin_qr, svd_small          (src/kernels.py)
  pipeline  randomized_svd (shipped, no re-orth) and
            rsvd_reorth ("xsvd-reorth")     (src/pipeline.py)
  metrics   sine-form principal angles, sigma errors
"""

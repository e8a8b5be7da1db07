"""Counter-based Gaussian generator, restated from the reference.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows /root/reference/pkg/src/xsvd/rng.py:
  mix64        rng.py:18-25   splitmix64 finalizer on a python int
  _mix_array   rng.py:28-35   same finalizer on uint64 arrays
  uniform_bits rng.py:38-47   base = mix64(seed) ^ ((row mod 2^32) << 32); ctr = base + t
  gaussian_row rng.py:50-62   Box-Muller; u1 from the first half of the window,
                              u2 from the second half (not interleaved)
  gaussian_band rng.py:65-70  rows [row0, row1)

`gaussian_band` here is vectorised over rows; the arithmetic per element is
the reference's, so with the same numpy build the bits are identical
(pinned in tests/test_oracle_golden.py).
"""

import numpy as np

MASK = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB


def mix64(x: int) -> int:
    """splitmix64 finalizer, python ints (rng.py:18-25)."""
    x = (x + GOLDEN) & MASK
    x ^= x >> 30
    x = (x * MIX1) & MASK
    x ^= x >> 27
    x = (x * MIX2) & MASK
    return x ^ (x >> 31)


def mix_array(x: np.ndarray) -> np.ndarray:
    """Vectorised finalizer; uint64 arithmetic wraps (rng.py:28-35)."""
    x = x + np.uint64(GOLDEN)
    x ^= x >> np.uint64(30)
    x *= np.uint64(MIX1)
    x ^= x >> np.uint64(27)
    x *= np.uint64(MIX2)
    return x ^ (x >> np.uint64(31))


def row_bases(seed: int, row0: int, row1: int) -> np.ndarray:
    """Per-row counter base (rng.py:45)."""
    rows = np.arange(row0, row1, dtype=np.uint64) & np.uint64(0xFFFFFFFF)
    return np.uint64(mix64(seed)) ^ (rows << np.uint64(32))


def uniform_bits(seed: int, row: int, count: int) -> np.ndarray:
    """`count` hashed words for (seed, row) (rng.py:38-47)."""
    base = row_bases(seed, row, row + 1)[0]
    return mix_array(base + np.arange(count, dtype=np.uint64))


def gaussian_band(seed: int, row0: int, row1: int, n: int) -> np.ndarray:
    """Rows [row0, row1) of an n-column N(0,1) f64 matrix (rng.py:50-70)."""
    rows = row1 - row0
    pairs = (n + 1) // 2
    if rows <= 0:
        return np.empty((0, n))
    base = row_bases(seed, row0, row1)[:, None]
    bits = mix_array(base + np.arange(2 * pairs, dtype=np.uint64)[None, :])
    u1 = ((bits[:, :pairs] >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53
    u2 = (bits[:, pairs:] >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    radius = np.sqrt(-2.0 * np.log(u1))
    theta = 2.0 * np.pi * u2
    out = np.empty((rows, 2 * pairs))
    out[:, 0::2] = radius * np.cos(theta)
    out[:, 1::2] = radius * np.sin(theta)
    return np.ascontiguousarray(out[:, :n])


def gaussian_bits(seed: int, row0: int, row1: int, n: int) -> np.ndarray:
    """The integer stage only: the (rows, 2*ceil(n/2)) uint64 hash words.

    Used to pin the GPU generator's integer stage bit-exactly (its
    log/sin/cos stage is compared within ulps instead)."""
    pairs = (n + 1) // 2
    base = row_bases(seed, row0, row1)[:, None]
    return mix_array(base + np.arange(2 * pairs, dtype=np.uint64)[None, :])

"""Seeded synthetic inputs for the ring-primitive entry points (tests and bench).

Holds none of the method's arithmetic: only numpy PCG64 draws shaped like the paper's
workloads (uniform R/q elements, fixed-weight ternary elements, uniform small elements), in the
library's row layout (pad lanes zero).  Keygen itself draws its randomness from the method's own
SplitMix64 stream, which the oracle and the CUDA path implement separately (C2).
"""
import numpy as np


def uniform_rq(n, p, q, stride, seed):
    """n elements of R/q, coefficients uniform in [-(q-1)/2, (q-1)/2], int16 rows of `stride`."""
    rng = np.random.default_rng(seed)
    out = np.zeros((n, stride), np.int16)
    out[:, :p] = rng.integers(-(q - 1) // 2, (q - 1) // 2 + 1, size=(n, p), dtype=np.int16)
    return out


def ternary(n, p, w, stride, seed, dtype=np.int16):
    """n fixed-weight elements: exactly w coefficients +-1 at uniform positions."""
    rng = np.random.default_rng(seed)
    out = np.zeros((n, stride), dtype)
    for i in range(n):
        pos = rng.choice(p, size=w, replace=False)
        out[i, pos] = rng.choice(np.array([-1, 1], dtype=dtype), size=w)
    return out


def ternary_fast(n, p, w, stride, seed, dtype=np.int16):
    """Vectorised fixed-weight ternary rows (argsort of uniform keys per row); for large n."""
    rng = np.random.default_rng(seed)
    out = np.zeros((n, stride), dtype)
    step = 65536
    for r0 in range(0, n, step):
        m = min(step, n - r0)
        keys = rng.random((m, p), dtype=np.float32)
        pos = np.argpartition(keys, w, axis=1)[:, :w]
        sgn = rng.integers(0, 2, size=(m, w), dtype=np.int8) * 2 - 1
        np.put_along_axis(out[r0:r0 + m], pos, sgn.astype(dtype), axis=1)
    return out


def small(n, p, stride, seed):
    """n elements with coefficients uniform in {-1, 0, 1}, int8 rows of `stride`."""
    rng = np.random.default_rng(seed)
    out = np.zeros((n, stride), np.int8)
    out[:, :p] = rng.integers(-1, 2, size=(n, p), dtype=np.int8)
    return out

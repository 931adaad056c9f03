"""CPU checks of the arithmetic identities the tensor-core kernels are built on,
checked against the oracle's ring product (oracle.poly_mul, section 3.3 of the paper) with plain
numpy integer arithmetic -- no GPU code is involved.

1. Folded B operand: with bt[m] = b[m] (m >= 1), bt[0] = b[0] + b[p-1] and
   bt[m] = b[m+p] + b[m+p-1] (-p < m < 0), the Toeplitz sums T[k] = sum_j a[j] bt[k-j]
   equal the reduced product c[k] (x^p = x + 1) for 1 <= k < p, and
   c[0] = T[0] - T[p-1] + a[p-1] b[p-1].
2. Hankel / block form: T[128 t + r] = sum_kappa A[r][kappa] B[t][kappa] with
   A[r][kappa] = a[r + kappa - 127] and B[t][kappa] = bt[128 t + 127 - kappa].
3. Limb split v = 64 hi + lo (lo in [-32, 31]) of folded sums stays int8 (|hi| <= 123 for q <= 7879).
"""
import numpy as np
import pytest

from oracle import oracle as O

SETS = [(653, 4621), (761, 4591), (857, 5167), (953, 6343), (1013, 7177), (1277, 7879)]


def folded(b):
    p = len(b)
    bt = np.zeros(2 * p - 1, dtype=np.int64)          # index m + p - 1, m in (-p, p)
    bt[p - 1:] = b
    bt[p - 1] = b[0] + b[p - 1]
    for m in range(-p + 1, 0):
        bt[m + p - 1] = b[m + p] + b[m + p - 1]
    return bt


def toeplitz_sums(a, bt):
    p = len(a)
    T = np.zeros(p, dtype=np.int64)
    for k in range(p):
        j = np.arange(p)
        T[k] = int(np.dot(a, bt[k - j + p - 1]))
    return T


@pytest.mark.parametrize("p,q", SETS)
def test_folded_operand_identity(p, q):
    rng = np.random.default_rng(p)
    for trial in range(3):
        a = rng.integers(-(q // 2), q // 2 + 1, p)
        b = rng.integers(-(q // 2), q // 2 + 1, p) if trial else rng.integers(-1, 2, p)
        c = np.asarray(O.poly_mul(p, q, a, b), dtype=np.int64)
        T = toeplitz_sums(a, folded(b))
        cen = lambda x: (x + q // 2) % q - q // 2
        assert np.array_equal(cen(T[1:]), c[1:])
        assert cen(T[0] - T[p - 1] + a[p - 1] * b[p - 1]) == c[0]
        # without the fix, coefficient 0 is off by exactly raw[p-1] (the unreduced coefficient)
        raw_p1 = int(np.dot(a, b[::-1]))
        assert cen(T[0] - raw_p1) == c[0]


@pytest.mark.parametrize("p,q", [(761, 4591), (653, 4621)])
def test_hankel_block_form(p, q):
    rng = np.random.default_rng(7)
    a = rng.integers(-(q // 2), q // 2 + 1, p)
    b = rng.integers(-(q // 2), q // 2 + 1, p)
    bt = folded(b)
    T = toeplitz_sums(a, bt)
    K = (p + 127 + 31) // 32 * 32
    NT = (p + 127) // 128
    kap = np.arange(K)
    A = np.zeros((128, K), dtype=np.int64)
    for r in range(128):
        idx = r + kap - 127
        ok = (idx >= 0) & (idx < p)
        A[r, ok] = a[idx[ok]]
    B = np.zeros((NT, K), dtype=np.int64)
    for t in range(NT):
        m = 128 * t + 127 - kap
        ok = (m > -p) & (m < p)
        B[t, ok] = bt[m[ok] + p - 1]
    D = A @ B.T                                         # D[r][t]
    out = D.T.reshape(-1)[:p]                           # coefficient 128 t + r
    assert np.array_equal(out, T)


@pytest.mark.parametrize("p,q", SETS)
def test_folded_limbs_fit_int8(p, q):
    qh = (q - 1) // 2
    v = np.arange(-2 * qh, 2 * qh + 1)
    lo = ((v + 32) & 63) - 32
    hi = (v - lo) >> 6
    assert np.array_equal(64 * hi + lo, v)
    assert lo.min() >= -32 and lo.max() <= 31 and np.abs(hi).max() <= 127

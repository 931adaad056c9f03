"""Independent polynomial helpers for the oracle pins (tests only).

Deliberately a *different* algorithm from the oracle wherever one is used as a pin:
  - ring product = numpy full convolution + polynomial LONG DIVISION by x^p - x - 1
    (the oracle folds with x^p = x + 1 instead);
  - inverses are never computed here except by brute force on toy rings;
  - gcd / distinct-degree factorisation over GF(m) for the factor facts of P:3937-4070.
Polynomials are little-endian int64 numpy arrays (index = degree).
"""
from __future__ import annotations

import numpy as np


def trim(a):
    a = np.asarray(a, dtype=np.int64)
    nz = np.nonzero(a)[0]
    return a[: nz[-1] + 1] if len(nz) else a[:0]


def center(a, m):
    a = np.mod(np.asarray(a, dtype=np.int64), m)
    return np.where(a > (m - 1) // 2, a - m, a)


def modulus(p, m):
    F = np.zeros(p + 1, dtype=np.int64)
    F[0] = m - 1
    F[1] = m - 1
    F[p] = 1
    return F


def polymod_longdiv(t, p, m):
    """Remainder of t modulo x^p - x - 1 over Z/m by schoolbook long division (high to low)."""
    t = np.mod(np.asarray(t, dtype=np.int64).copy(), m)
    for k in range(len(t) - 1, p - 1, -1):
        c = t[k]
        if c:
            # t -= c * x^(k-p) * (x^p - x - 1)
            t[k] = 0
            t[k - p + 1] = (t[k - p + 1] + c) % m
            t[k - p] = (t[k - p] + c) % m
    out = np.zeros(p, dtype=np.int64)
    out[: min(p, len(t))] = t[:p]
    return out


def ring_mul(a, b, p, m):
    """Product in (Z/m)[x]/(x^p-x-1): numpy convolution, then long division. Centered."""
    t = np.convolve(np.asarray(a, dtype=np.int64)[:p], np.asarray(b, dtype=np.int64)[:p])
    return center(polymod_longdiv(t, p, m), m)


def gf_divmod(a, b, m):
    a = np.mod(trim(a), m).copy()
    b = np.mod(trim(b), m)
    db = len(b) - 1
    inv = pow(int(b[-1]), m - 2, m)
    if len(a) - 1 < db:
        return np.zeros(1, np.int64), a
    q = np.zeros(len(a) - db, dtype=np.int64)
    for k in range(len(a) - 1 - db, -1, -1):
        c = (a[k + db] * inv) % m
        q[k] = c
        if c:
            a[k:k + db + 1] = (a[k:k + db + 1] - c * b) % m
    return trim(q), trim(a)


def gf_gcd(a, b, m):
    a, b = np.mod(trim(a), m), np.mod(trim(b), m)
    while len(b):
        _, r = gf_divmod(a, b, m)
        a, b = b, r
    if len(a):
        a = (a * pow(int(a[-1]), m - 2, m)) % m   # monic
    return a


def gf_mul(a, b, m):
    return trim(np.mod(np.convolve(trim(a), trim(b)), m)) if len(trim(a)) and len(trim(b)) else np.zeros(0, np.int64)


def fold_reduce(t, p, m):
    """t mod (x^p-x-1) over Z/m, vectorised: x^(p+i) = x^(i+1) + x^i, applied until deg < p."""
    t = np.mod(np.asarray(t, dtype=np.int64), m)
    while len(t) > p:
        hi = t[p:]
        low = np.zeros(max(p, len(hi) + 1), dtype=np.int64)
        low[:p] = t[:p]
        low[: len(hi)] += hi
        low[1: len(hi) + 1] += hi
        t = np.mod(low, m)
    out = np.zeros(p, dtype=np.int64)
    out[: len(t)] = t
    return out


def frobenius_reduce(h, p, m):
    """h^m mod (x^p-x-1) over GF(m) for prime m: (sum h_i x^i)^m = sum h_i x^(m i)."""
    t = np.zeros(m * (p - 1) + 1, dtype=np.int64)
    t[::m] = np.asarray(h, dtype=np.int64)[:p]
    return fold_reduce(t, p, m)


def ddf_degrees(p, m, dmax):
    """Distinct-degree factorisation of x^p-x-1 over GF(m) for degrees <= dmax.
    Returns ({d: component}, cofactor).  Component d = product of irreducible factors of degree d."""
    F = modulus(p, m)
    rest = np.mod(F, m)
    x = np.zeros(p, np.int64)
    x[1] = 1
    h = x.copy()
    comps = {}
    for d in range(1, dmax + 1):
        h = frobenius_reduce(h, p, m)        # x^(m^d) mod F
        hx = h.copy()
        hx[1] = (hx[1] - 1) % m
        g = gf_gcd(rest, hx, m)
        if len(g) > 1:
            comps[d] = g
            rest, r = gf_divmod(rest, g, m)
            assert len(r) == 0
        if len(rest) - 1 < 2 * (d + 1):
            break
    return comps, rest

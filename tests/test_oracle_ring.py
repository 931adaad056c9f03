"""Pins for the oracle's ring product (C7) and inversion (C5/C6)."""
import itertools

import numpy as np
import pytest

import polytools as PT


def rand_elem(rng, p, m):
    return rng.integers(-(m - 1) // 2, (m - 1) // 2 + 1, size=p)


@pytest.mark.parametrize("p,m", [(2, 3), (5, 3), (7, 7), (11, 13), (761, 3), (761, 4591),
                                 (653, 4621), (1277, 7879)])
def test_mul_matches_long_division(O, p, m):
    rng = np.random.default_rng(p * 31 + m)
    for _ in range(6 if p > 100 else 40):
        a, b = rand_elem(rng, p, m), rand_elem(rng, p, m)
        assert np.array_equal(O.poly_mul(p, m, a, b), PT.ring_mul(a, b, p, m))


@pytest.mark.parametrize("p,m", [(761, 3), (761, 4591), (857, 5167), (1013, 7177)])
def test_mul_closed_forms(O, p, m):
    x = np.zeros(p, np.int64); x[1] = 1
    xp1 = np.zeros(p, np.int64); xp1[p - 1] = 1
    one = np.zeros(p, np.int64); one[0] = 1
    # x * x^(p-1) = x^p = x + 1
    r = O.poly_mul(p, m, x, xp1)
    exp = np.zeros(p, np.int64); exp[0] = 1; exp[1] = 1
    assert np.array_equal(r, exp)
    # x^(p-1) * x^(p-1) = x^(2p-2) = x^(p-2) * (x + 1) = x^(p-1) + x^(p-2)
    r = O.poly_mul(p, m, xp1, xp1)
    exp = np.zeros(p, np.int64); exp[p - 1] = 1; exp[p - 2] = 1
    assert np.array_equal(r, exp)
    rng = np.random.default_rng(0)
    a = rand_elem(rng, p, m)
    assert np.array_equal(O.poly_mul(p, m, one, a), a)


def test_mul_algebra(O):
    p, m = 761, 4591
    rng = np.random.default_rng(5)
    a, b, c = (rand_elem(rng, p, m) for _ in range(3))
    ab = O.poly_mul(p, m, a, b)
    assert np.array_equal(ab, O.poly_mul(p, m, b, a))
    assert np.array_equal(O.poly_mul(p, m, ab, c), O.poly_mul(p, m, a, O.poly_mul(p, m, b, c)))
    lhs = O.poly_mul(p, m, a, PT.center(b + c, m))
    rhs = PT.center(ab + O.poly_mul(p, m, a, c), m)
    assert np.array_equal(lhs, rhs)


@pytest.mark.parametrize("p,m", [(653, 3), (761, 3), (761, 4591), (857, 5167), (953, 6343),
                                 (1013, 7177), (1277, 7879), (1277, 3)])
def test_inverse_of_x_closed_form(O, p, m):
    # 1/x = x^(p-1) - 1 because x * (x^(p-1) - 1) = x^p - x = 1 in the ring.
    x = np.zeros(p, np.int64); x[1] = 1
    ok, inv = O.poly_inv(p, m, x)
    exp = np.zeros(p, np.int64); exp[p - 1] = 1; exp[0] = -1
    assert ok and np.array_equal(inv, exp)


def test_inverse_zero_and_scalars(O):
    p, m = 761, 4591
    ok, inv = O.poly_inv(p, m, np.zeros(p, np.int64))
    assert not ok and not inv.any()
    for c in (1, 2, 3, -5, 2295):
        a = np.zeros(p, np.int64); a[0] = c
        ok, inv = O.poly_inv(p, m, a)
        assert ok and inv[1:].sum() == 0 and (inv[0] * c - 1) % m == 0


@pytest.mark.parametrize("p,m", [(761, 4591), (761, 3), (653, 4621), (1277, 7879), (857, 3)])
def test_inverse_multiplies_back(O, p, m):
    rng = np.random.default_rng(p + m)
    one = np.zeros(p, np.int64); one[0] = 1
    for _ in range(4):
        a = rand_elem(rng, p, m)
        ok, inv = O.poly_inv(p, m, a)
        if m != 3:
            assert ok        # R/q is a field
        if ok:
            assert np.array_equal(PT.ring_mul(a, inv, p, m), one)


def all_elements(p, m):
    vals = np.arange(-(m - 1) // 2, (m - 1) // 2 + 1)
    return np.array(list(itertools.product(vals, repeat=p)), dtype=np.int64)


def test_toy_ring_brute_force_inverses(O):
    # Z/3[x]/(x^7-x-1): brute-force every product with numpy (independent of the oracle),
    # read off the unit group and each inverse, compare with the oracle's Euclid.
    p, m = 7, 3
    E = all_elements(p, m)                                   # 2187 x 7
    n = len(E)
    is_one = np.zeros((n, n), dtype=bool)
    E16 = E.astype(np.int16)
    for r0 in range(0, n, 128):
        A = E16[r0:r0 + 128]
        conv = np.zeros((len(A), n, 2 * p - 1), dtype=np.int16)
        for i in range(p):
            for j in range(p):
                conv[:, :, i + j] += A[:, None, i] * E16[None, :, j]
        for k in range(2 * p - 2, p - 1, -1):                # x^k = x^(k-p+1) + x^(k-p)
            conv[:, :, k - p] += conv[:, :, k]
            conv[:, :, k - p + 1] += conv[:, :, k]
        prod = np.mod(conv[:, :, :p], m)
        is_one[r0:r0 + 128] = (prod[:, :, 0] == 1) & (prod[:, :, 1:] == 0).all(-1)
    units = np.nonzero(is_one.any(1))[0]
    # closed form: x^7-x-1 = (deg 2)(deg 5) over GF(3) -> (3^2-1)(3^5-1) = 1936 units
    assert len(units) == 1936
    for i in range(n):
        ok, inv = O.poly_inv(p, m, E[i])
        if i in set(units.tolist()):
            j = np.nonzero(is_one[i])[0]
            assert ok and len(j) == 1 and np.array_equal(inv, E[j[0]])
        else:
            assert not ok


@pytest.mark.parametrize("p,m", [(5, 3), (11, 3), (5, 7), (3, 5), (7, 5), (3, 13)])
def test_toy_ring_unit_counts(O, p, m):
    # number of units of (Z/m)[x]/(F) = prod over irreducible factors (m^d - 1); the factor
    # degrees come from the test's own distinct-degree factorisation.
    comps, rest = PT.ddf_degrees(p, m, p)
    degs = []
    for d, g in comps.items():
        degs += [d] * ((len(g) - 1) // d)
    if len(rest) > 1:
        degs.append(len(rest) - 1)
    assert sum(degs) == p
    expected = int(np.prod([m ** d - 1 for d in degs]))
    E = all_elements(p, m)
    cnt = 0
    one = np.zeros(p, np.int64); one[0] = 1
    for e in E:
        ok, inv = O.poly_inv(p, m, e)
        if ok:
            cnt += 1
            assert np.array_equal(PT.ring_mul(e, inv, p, m), one)
    assert cnt == expected


@pytest.mark.parametrize("p,m,threads", [(761, 4591, 1), (761, 4591, 3), (653, 3, 2), (1277, 7879, 4)])
def test_mul_many_equals_rowwise_long_division(O, p, m, threads):
    # or_mul_many (the threaded batch wrapper the R/q parity tests and cpu_baseline use) against
    # the independent long-division product (tests/polytools.py) row by row, ragged row stride.
    rng = np.random.default_rng(p + m + threads)
    n, row = 7, p + 5
    a = np.zeros((n, row), np.int16); b = np.zeros((n, row), np.int16)
    a[:, :p] = rng.integers(-(m - 1) // 2, (m - 1) // 2 + 1, size=(n, p))
    b[:, :p] = rng.integers(-(m - 1) // 2, (m - 1) // 2 + 1, size=(n, p))
    c = O.mul_many(p, m, a, b, threads=threads)
    for i in range(n):
        assert np.array_equal(c[i, :p], PT.ring_mul(a[i, :p].astype(np.int64), b[i, :p].astype(np.int64), p, m))
        assert not c[i, p:].any()

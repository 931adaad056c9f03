"""Pins for the oracle's KeyGen, encodings (C10/C11) and the factor facts of
section 3.1.1."""
import hashlib
import json
import math
import os

import numpy as np
import pytest

import polytools as PT

GOLD = os.path.join(os.path.dirname(__file__), "golden")
C14 = json.load(open(os.path.join(GOLD, "survey_c14.json")))
PAPER = json.load(open(os.path.join(GOLD, "paper_facts.json")))


# ------------------------------------------------------------------------------------------ params
def test_param_table_matches_paper(O):
    for k, v in PAPER["params"].items():
        if k.startswith("_"):
            continue
        assert O.PARAMS[int(k)] == tuple(v)


@pytest.mark.parametrize("param", [653, 761, 857, 953, 1013, 1277])
def test_param_invariants(O, param):
    p, q, w = O.PARAMS[param]
    isprime = lambda n: n > 1 and all(n % d for d in range(2, int(n ** 0.5) + 1))
    assert isprime(p) and isprime(q)
    assert q >= 16 * w + 1 and 2 * p >= 3 * w and ((q - 1) // 2) % 3 == 0


# ------------------------------------------------------------------------------------------ keygen
def check_key(O, param, r):
    p, q, w = O.PARAMS[param]
    g, f, gi, h = (r[k].astype(np.int64) for k in ("g", "f", "ginv", "h"))
    one = np.zeros(p, np.int64); one[0] = 1
    assert set(np.unique(g)) <= {-1, 0, 1} and set(np.unique(gi)) <= {-1, 0, 1}
    assert int((f != 0).sum()) == w and set(np.unique(f)) <= {-1, 0, 1}
    assert np.abs(h).max() <= (q - 1) // 2
    # defining relations of KeyGen: g * (1/g) = 1 in R/3 and h * 3f = g in R/q
    assert np.array_equal(PT.ring_mul(g, gi, p, 3), one)
    assert np.array_equal(PT.ring_mul(h, 3 * f, p, q), PT.center(g, q))
    # encodings decode back to the polynomials
    assert np.array_equal(O.rq_decode(p, q, r["pk"]).astype(np.int64), h)
    nb = (p + 3) // 4
    assert np.array_equal(O.small_decode(p, r["sk"][:nb]), f.astype(np.int8))
    assert np.array_equal(O.small_decode(p, r["sk"][nb:]), gi.astype(np.int8))


def test_keygen_survey_goldens(O):
    for key, k in (("key761_seed1_k0", 0), ("key761_seed1_k1", 1)):
        G = C14[key]
        r = O.keygen(761, 1, k)
        assert r["attempts"] == G["attempts"]
        assert list(r["h"][:6]) == G["h0_5"]
        assert r["pk"][:8].hex() == G["pk0_7"]
        assert hashlib.sha256(r["pk"]).hexdigest().startswith(G["pk_sha256_prefix"])
        assert hashlib.sha256(r["sk"]).hexdigest().startswith(G["sk_sha256_prefix"])
        if "g0_7" in G:
            assert list(r["g"][:8]) == G["g0_7"]
            assert list(r["f"][:8]) == G["f0_7"]
            assert list(np.nonzero(r["f"])[0][:6]) == G["f_first_nonzero"]
            assert list(r["ginv"][:8]) == G["ginv0_7"]
            assert r["sk"][:8].hex() == G["sk0_7"]
        check_key(O, 761, r)


@pytest.mark.parametrize("param,seed", [(653, 4), (761, 2), (857, 4), (953, 4), (1013, 4), (1277, 5)])
def test_keygen_invariants(O, param, seed):
    for k in range(3):
        check_key(O, param, O.keygen(param, seed, k))


@pytest.mark.parametrize("param,seed,key", [("653", 4, "653_seed4"), ("1277", 5, "1277_seed5")])
def test_first_rejections(O, param, seed, key):
    P = int(param)
    p = O.PARAMS[P][0]
    want = C14["first_two_draw_keys"][key]
    res = O.keygen_many(P, seed, np.arange(150))
    twos = [int(i) for i in np.nonzero(res["attempts"] >= 2)[0]]
    assert twos[:3] == want
    # the rejected draw really is a multiple of the cubic factor x^3 - x - 1 (C14 closed form):
    # gcd over GF(3) with x^p-x-1 is non-trivial
    k = want[0]
    g0 = O.small_from_words(p, O.stream_words(seed, k, 1, p)).astype(np.int64)
    gcd = PT.gf_gcd(PT.modulus(p, 3), np.mod(g0, 3), 3)
    assert len(gcd) > 1
    assert not O.poly_inv(p, 3, g0)[0]


def test_keygen_many_equals_single(O):
    idx = np.array([0, 1, 7, 31, 1000, 65535], dtype=np.uint64)
    res = O.keygen_many(761, 2, idx, threads=3, want_polys=True)
    for i, k in enumerate(idx):
        r = O.keygen(761, 2, int(k))
        assert res["pk"][i].tobytes() == r["pk"] and res["sk"][i].tobytes() == r["sk"]
        assert np.array_equal(res["h"][i], r["h"]) and res["attempts"][i] == r["attempts"]


# ------------------------------------------------------------------------------------------ encodings
def test_pk_lengths_and_app_d_storage(O):
    for k, n in C14["pk_bytes"].items():
        p, q, _ = O.PARAMS[int(k)]
        L = O.rq_encoded_bytes(p, q)
        assert L == n
        assert math.ceil(p * math.log2(q) / 8) <= L <= math.ceil(p * math.log2(q) / 8) + 1
    # App. D key-pair storage = pk + (3*ceil(p/4) + pk + 32) at n = 1
    st = PAPER["keypair_storage_bytes_n1"]
    for k in ("653", "761", "857"):
        p, q, _ = O.PARAMS[int(k)]
        pk = O.rq_encoded_bytes(p, q)
        assert pk + 3 * ((p + 3) // 4) + pk + 32 == st[k]


def test_encode_worked_examples(O):
    ex = C14["encode_worked_example"]
    assert O.encode_general(ex["R"], ex["M"]).hex() == ex["bytes"]
    # hand-computed: R=[1,2], M=[3,5] -> r = 1 + 3*2 = 7, m = 15 (no emission); top: emit 7
    assert O.encode_general([1, 2], [3, 5]).hex() == "07"
    # M=[300,300], R=[299,1]: r = 299 + 300*1 = 599, m = 90000 >= 2^14 -> emit 599&255 = 0x57,
    # r = 2, m = 352; top: emit 2, m = 2; emit 0, m = 1 -> 57 02 00
    assert O.encode_general([299, 1], [300, 300]).hex() == "570200"
    assert list(O.decode_general([300, 300], bytes.fromhex("570200"))) == [299, 1]


@pytest.mark.parametrize("param", [653, 761, 857, 953, 1013, 1277])
def test_rq_encode_roundtrip(O, param):
    p, q, _ = O.PARAMS[param]
    rng = np.random.default_rng(param)
    for h in (rng.integers(-(q - 1) // 2, (q - 1) // 2 + 1, size=p),
              np.full(p, (q - 1) // 2), np.full(p, -(q - 1) // 2), np.zeros(p, int)):
        b = O.rq_encode(p, q, h)
        assert len(b) == O.rq_encoded_bytes(p, q)
        assert np.array_equal(O.rq_decode(p, q, b), h.astype(np.int16))


def test_general_encode_roundtrip(O):
    rng = np.random.default_rng(3)
    for n in (1, 2, 3, 5, 8, 17, 100):
        M = rng.integers(1, 16384, size=n)
        R = rng.integers(0, M)
        assert np.array_equal(O.decode_general(M, O.encode_general(R, M)), R)


def test_small_encode(O):
    # byte = sum (c_t + 1) * 4^t: [-1, 0, 1, 1] -> 0 + 1*4 + 2*16 + 2*64 = 164
    assert O.small_encode(4, [-1, 0, 1, 1]) == bytes([164])
    assert O.small_encode(5, [1, 1, 1, 1, 0]) == bytes([170, 1])
    rng = np.random.default_rng(2)
    c = rng.integers(-1, 2, size=761).astype(np.int8)
    b = O.small_encode(761, c)
    assert len(b) == 191 and np.array_equal(O.small_decode(761, b), c)


# ------------------------------------------------------------------------------------------ factors
def test_factor_degrees_761_paper():
    # x^761 - x - 1 over GF(3) factors with degrees 19, 60, 682
    comps, rest = PT.ddf_degrees(761, 3, 60)
    degs = {d: len(g) - 1 for d, g in comps.items()}
    assert degs == {19: 19, 60: 60}
    assert len(rest) - 1 == 682
    assert sorted(list(degs.values()) + [len(rest) - 1]) == PAPER["factor_degrees_761_mod3"]["degrees"]


def test_gcd_invertibility_equals_factor_remainders(O):
    # The paper's predicate: g invertible iff g mod f_i != 0 for every factor.
    p = 761
    comps, rest = PT.ddf_degrees(p, 3, 60)
    factors = [comps[19], comps[60], rest]
    rng = np.random.default_rng(11)
    cases = [rng.integers(-1, 2, size=p) for _ in range(8)]
    for fac in factors:                       # crafted multiples of each factor (reduced mod F)
        u = rng.integers(-1, 2, size=p)
        prod = np.convolve(np.mod(fac, 3), np.mod(u, 3))
        cases.append(PT.center(PT.fold_reduce(prod, p, 3), 3))
    for g in cases:
        ok, _ = O.poly_inv(p, 3, g)
        rems = [PT.gf_divmod(np.mod(g, 3), fac, 3)[1] for fac in factors]
        assert ok == all(len(r) > 0 for r in rems)
    assert sum(not O.poly_inv(p, 3, g)[0] for g in cases[8:]) == 3


@pytest.mark.parametrize("p", [653, 1277])
def test_cubic_factor_closed_form(O, p):
    # For p = 653, 1277 (26 | p - 3), x^3 - x - 1 divides x^p - x - 1 over GF(3) (C14):
    # multiples of it are non-invertible in R/3.
    cubic = np.array([2, 2, 0, 1])
    q_, r_ = PT.gf_divmod(PT.modulus(p, 3), cubic, 3)
    assert len(r_) == 0
    rng = np.random.default_rng(p)
    u = rng.integers(0, 3, size=p - 3)
    g = PT.center(np.convolve(cubic, u), 3)[:p]
    assert not O.poly_inv(p, 3, g)[0]

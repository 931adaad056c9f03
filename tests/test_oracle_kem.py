"""Oracle pins for the encapsulation / decapsulation core (SPEC.md
encrypt_core / decrypt_core; key shape (h, (f, 1/g)) of P:3438-3461).  The pins are properties the
mathematics fixes, not re-typed formulas: NTRU Prime decryption correctness (q >= 16w + 1, C1)
makes decap(encap(r)) = r for every valid key and every r of weight w; Round lands on multiples of
3 within distance 1; the weight check rejects the zero ciphertext."""
import numpy as np
import pytest

ENC_DOMAIN = 1 << 32          # C2: stream domains >= 2^32 are reserved for encapsulation draws


def short_r(O, p, w, seed, k):
    return O.short_from_words(p, w, O.stream_words(seed, k, ENC_DOMAIN, p))


@pytest.mark.parametrize("param", [653, 761, 857, 953, 1013, 1277])
def test_decap_inverts_encap(O, param):
    p, q, w = O.PARAMS[param]
    keys = O.keygen_many(param, 31, np.arange(3, dtype=np.uint64), want_polys=True)
    for i in range(3):
        h, f, ginv = keys["h"][i][:p], keys["f"][i][:p], keys["ginv"][i][:p]
        for k in range(2):
            r = short_r(O, p, w, 31, 10 * i + k)
            assert np.count_nonzero(r) == w
            c = O.encap_core(p, q, h, r)
            assert not np.any(c % 3), "Round must give multiples of 3"
            x = O.poly_mul(p, q, h, r)
            assert np.abs(c.astype(np.int64) - x).max() <= 1
            assert np.abs(c).max() <= (q - 1) // 2
            ok, r2 = O.decap_core(p, q, w, f, ginv, c)
            assert ok and np.array_equal(r2, r)


def test_decap_rejects_zero_and_random_ciphertexts(O):
    p, q, w = O.PARAMS[761]
    keys = O.keygen_many(761, 5, np.arange(1, dtype=np.uint64), want_polys=True)
    f, ginv = keys["f"][0][:p], keys["ginv"][0][:p]
    ok, r = O.decap_core(p, q, w, f, ginv, np.zeros(p, np.int16))
    assert not ok and not r.any()
    rng = np.random.default_rng(3)
    fails = 0
    for _ in range(20):
        c = 3 * rng.integers(-(q - 1) // 6, (q - 1) // 6 + 1, size=p).astype(np.int16)
        ok, _ = O.decap_core(p, q, w, f, ginv, c)
        fails += not ok
    assert fails >= 18       # a random ciphertext decodes to weight w with small probability

"""Oracle pins for the full-size secret key (reading Z24): the oracle's
SHA-512 against an independent implementation (Python's hashlib), the sizes against the paper's
App. D key-pair storage, and the layout."""
import hashlib
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402


@pytest.mark.parametrize("n", [0, 1, 3, 55, 56, 111, 112, 113, 127, 128, 129, 255, 256, 1159, 2068, 5000])
def test_sha512_matches_hashlib(n):
    rng = np.random.default_rng(n)
    data = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
    assert O.sha512(data) == hashlib.sha512(data).digest()


def test_full_sk_sizes_match_appendix_d():
    # App. D: key-pair storage 2512 / 2921 / 3321 bytes = pk + full sk (653 / 761 / 857)
    for param, pair in ((653, 2512), (761, 2921), (857, 3321)):
        assert O.pk_bytes(param) + O.full_sk_bytes(param) == pair
    assert O.full_sk_bytes(761) == 1763


def test_full_sk_layout():
    k = O.keygen(761, 3, 5)
    full = O.full_sk(761, 3, 5, k["pk"], k["sk"])
    skb, pkb, rb = O.sk_bytes(761), O.pk_bytes(761), 191
    assert full[:skb] == k["sk"] and full[skb:skb + pkb] == k["pk"]
    assert full[skb + pkb + rb:] == hashlib.sha512(b"\x04" + k["pk"]).digest()[:32]
    rho = full[skb + pkb:skb + pkb + rb]
    D = O.sm(O.sm(3, 5), 1 << 63)
    expect = b"".join(int(O.sm(D, j)).to_bytes(8, "little") for j in range((rb + 7) // 8))[:rb]
    assert rho == expect
    # a different key index gives a different rho
    k2 = O.keygen(761, 3, 6)
    assert O.full_sk(761, 3, 6, k2["pk"], k2["sk"])[skb + pkb:skb + pkb + rb] != rho

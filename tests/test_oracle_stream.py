"""Pins for the oracle's random stream and samplers (C2-C4)."""
import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")
MASK = (1 << 64) - 1


def sequential_splitmix(seed, n):
    """The textbook stateful SplitMix64 generator: state += gamma; output = finaliser(state).
    A different formulation from the oracle's counter form SM(s, j)."""
    out, state = [], seed
    for _ in range(n):
        state = (state + 0x9E3779B97F4A7C15) & MASK
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
        out.append(z ^ (z >> 31))
    return out


def test_splitmix_anchor(O):
    g = json.load(open(os.path.join(GOLD, "survey_c14.json")))
    # SM(0,0) = 0xE220A8397B1DCDAF is the standard first SplitMix64 output for state 0.
    assert O.sm(0, 0) == int(g["sm_0_0"], 16) == 0xE220A8397B1DCDAF
    assert O.sm(1, 0) == int(g["sm_1_0"], 16)


@pytest.mark.parametrize("seed", [0, 1, 2, 0xDEADBEEF12345678, MASK])
def test_counter_form_equals_sequential_generator(O, seed):
    seq = sequential_splitmix(seed, 40)
    assert [O.sm(seed, j) for j in range(40)] == seq


def test_stream_word_order_golden(O):
    g = json.load(open(os.path.join(GOLD, "survey_c14.json")))
    u = O.stream_words(1, 0, 0, 4)
    assert [int(x, 16) for x in g["words_seed1_k0_f"]] == [int(v) for v in u]
    # low half first, then high half, of SM(D, j) with D = SM(SM(seed, k), d)
    D = O.sm(O.sm(1, 0), 0)
    z0, z1 = O.sm(D, 0), O.sm(D, 1)
    assert list(map(int, u)) == [z0 & 0xFFFFFFFF, z0 >> 32, z1 & 0xFFFFFFFF, z1 >> 32]


def test_small_mapping_boundaries(O):
    # C3: g_i = floor(3*(u mod 2^30)/2^30) - 1; the boundaries of the three classes are
    # ceil(2^30/3) = 357913942 and ceil(2*2^30/3) = 715827883; the top two bits are ignored.
    u = np.array([0, 357913941, 357913942, 715827882, 715827883, (1 << 30) - 1,
                  (3 << 30) | 357913941, (2 << 30) | 715827883], dtype=np.uint32)
    g = O.small_from_words(len(u), u)
    assert list(g) == [-1, -1, 0, 0, 1, 1, -1, 1]


def test_small_frequencies(O):
    rng = np.random.default_rng(7)
    u = rng.integers(0, 1 << 32, size=600_000, dtype=np.uint64).astype(np.uint32)
    g = O.small_from_words(len(u), u)
    counts = np.array([(g == v).sum() for v in (-1, 0, 1)])
    n = len(u)
    sigma = np.sqrt(n * (1 / 3) * (2 / 3))
    assert np.all(np.abs(counts - n / 3) < 5 * sigma)


def test_short_tiny_hand_example(O):
    # p = 4, w = 2: tags L = [u0&~1, u1&~1, (u2&~3)|1, (u3&~3)|1]; sorted ascending; f = (L&3)-1.
    u = np.array([0x30, 0x12, 0x20, 0x00000007], dtype=np.uint32)
    # L = [0x30 (->-1), 0x12 (low bits 10 -> +1), 0x21 (-> 0), 0x05 (-> 0)]; sorted: 5, 0x12, 0x21, 0x30
    f = O.short_from_words(4, 2, u)
    assert list(f) == [0, 1, 0, -1]


@pytest.mark.parametrize("param", [653, 761, 857, 953, 1013, 1277])
def test_short_weight_and_values(O, param):
    p, q, w = O.PARAMS[param]
    for k in range(20):
        u = O.stream_words(9, k, 0, p)
        f = O.short_from_words(p, w, u)
        assert set(np.unique(f)) <= {-1, 0, 1}
        assert int((f != 0).sum()) == w


def test_short_depends_only_on_tag_multiset(O):
    # Sorting makes f a function of the multiset of tags: permuting the first w draws among
    # themselves (and the rest among themselves) must not change f.
    p, q, w = O.PARAMS[761]
    u = O.stream_words(3, 5, 0, p)
    f = O.short_from_words(p, w, u)
    rng = np.random.default_rng(1)
    u2 = u.copy()
    u2[:w] = rng.permutation(u[:w])
    u2[w:] = rng.permutation(u[w:])
    assert np.array_equal(O.short_from_words(p, w, u2), f)


def test_short_position_and_sign_balance(O):
    p, q, w = O.PARAMS[761]
    n = 400
    F = np.stack([O.short_from_words(p, w, O.stream_words(11, k, 0, p)) for k in range(n)])
    nz = (F != 0)
    # every position is nonzero with probability w/p; sum over 400 keys per position
    per_pos = nz.sum(0)
    mean = n * w / p
    sd = np.sqrt(n * (w / p) * (1 - w / p))
    assert np.abs(per_pos - mean).max() < 5.5 * sd
    plus = (F == 1).sum()
    total = nz.sum()
    assert abs(plus - total / 2) < 5 * np.sqrt(total / 4)


def test_c12_uniform_mapping_boundaries(O):
    # C12: a_j = floor(u_j q / 2^32) - (q-1)/2 maps [0, 2^32) onto [-(q-1)/2, (q-1)/2]; the
    # boundaries of the first and last class are ceil(2^32/q) and floor((q-1) 2^32/q) (q = 4591).
    q = 4591
    b1 = -(-(1 << 32) // q)            # smallest u with floor(u q / 2^32) = 1
    blast = -(-((q - 1) << 32) // q)   # smallest u with floor(u q / 2^32) = q - 1
    u = np.array([0, b1 - 1, b1, blast - 1, blast, (1 << 32) - 1], dtype=np.uint32)
    a = O.uniform_from_words(len(u), q, u)
    assert list(a) == [-2295, -2295, -2294, 2294, 2295, 2295]


def test_c12_uniform_frequencies(O):
    rng = np.random.default_rng(11)
    u = rng.integers(0, 1 << 32, size=400_000, dtype=np.uint64).astype(np.uint32)
    a = O.uniform_from_words(len(u), 4591, u).astype(np.int64)
    assert a.min() == -2295 and a.max() == 2295
    # mean 0, variance (q^2 - 1)/12 of the discrete uniform law, within 5 sigma
    n, var = len(a), (4591 ** 2 - 1) / 12
    assert abs(a.mean()) < 5 * np.sqrt(var / n)
    assert abs(a.var() / var - 1) < 5 * np.sqrt(0.8 / n)


def test_c12_pair0_golden(O):
    # SURVEY.md C14 "Config 3, pair 0 (seed = 3)": a third implementation's values for C12 + C7.
    g = json.load(open(os.path.join(GOLD, "survey_c14.json")))["config3_pair0_seed3"]
    a, b = O.c12_pair(761, 3, 0)
    assert list(map(int, a[:6])) == g["a0_5"]
    assert list(map(int, np.nonzero(b)[0][:4])) == g["b_first_nonzero"]
    assert int(np.count_nonzero(b)) == 286 and set(map(int, np.unique(b))) <= {-1, 0, 1}
    c = O.poly_mul(761, 4591, a, b)
    assert list(map(int, c[:6])) == g["c0_5"]

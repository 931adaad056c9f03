"""CPU check of the Short sampler's sorting-network schedule (csrc/sample.cuh warp_bitonic_sort;
DESIGN.md C4 sorts p tagged uint32 draws): a numpy model of the same comparator sequence --
all-ascending bitonic merges (mirror step i <-> i ^ (k-1), then half-cleaners i <-> i ^ j), kept in
the blocked layout (lane l holds elements l*E + e) except for merge stages k >= 4E, which run in the
striped layout (lane L holds elements 32 r + L) between two transposes -- must equal np.sort on
random and tie-heavy inputs.  Pins the schedule, not the CUDA code (that is test_gpu_parity's f
parity against the oracle, bit-exact).
"""
import numpy as np
import pytest


def _cmp(X, lo, hi):
    a, b = X[..., lo].copy(), X[..., hi].copy()
    X[..., lo] = np.minimum(a, b)
    X[..., hi] = np.maximum(a, b)


def model_sort(x, E, NR=None):
    N = 32 * E
    NR = N if NR is None else NR
    RP = (NR + 31) // 32                          # striped registers holding a real key
    LE = {8: 3, 16: 4, 32: 5, 64: 6}[E]
    LOGN = LE + 5
    V = x.reshape(32, E).copy()                   # blocked: V[lane, e] = x[lane*E + e]
    lanes = np.arange(32)
    for ls in range(1, LOGN + 1):
        k = 1 << ls
        striped = E >= 32 and k >= 4 * E
        jtop = 16 if striped else k >> 2
        if k <= E:
            for e in range(E):
                if e & (k >> 1) == 0:
                    _cmp(V, e, e ^ (k - 1))
        elif not striped:
            lm = k // E - 1
            lower = (lanes & ((k // E) >> 1)) == 0
            o = np.stack([V[lanes ^ lm, E - 1 - e] for e in range(E)], axis=1)
            V = np.where(lower[:, None], np.minimum(V, o), np.maximum(V, o))
        else:
            S = V.reshape(-1).reshape(E, 32).T.copy()  # striped: S[lane, r] = x[32 r + lane]
            S[:, RP:] = 0xFFFFFFFF                     # pad registers are not loaded
            rm, rh = (k - 1) >> 5, k >> 6
            for r in range(E):
                if r & rh == 0 and (r ^ rm) < RP:
                    a = S[lanes ^ 31, r ^ rm].copy()
                    b = S[lanes ^ 31, r].copy()
                    S[:, r] = np.minimum(S[:, r], a)
                    S[:, r ^ rm] = np.maximum(S[:, r ^ rm], b)
            jr = k >> 7
            while jr >= 1:
                for r in range(E):
                    if r & jr == 0 and (r | jr) < RP:
                        _cmp(S, r, r | jr)
                jr >>= 1
            flat = V.reshape(-1).copy()                # pad registers are not stored back
            flat.reshape(E, 32).T[:, :RP] = S[:, :RP]
            V = flat.reshape(32, E)
        j = jtop
        while j >= 1:
            if j >= E:
                lm = j // E
                lower = (lanes & lm) == 0
                o = V[lanes ^ lm, :]
                V = np.where(lower[:, None], np.minimum(V, o), np.maximum(V, o))
            else:
                for e in range(E):
                    if e & j == 0:
                        _cmp(V, e, e | j)
            j >>= 1
    return V.reshape(-1)


@pytest.mark.parametrize("E", [8, 16, 32, 64])
def test_schedule_sorts(E):
    rng = np.random.default_rng(E)
    for t in range(6):
        if t % 2:
            x = rng.integers(0, 4, 32 * E).astype(np.uint32)          # ties
        else:
            x = rng.integers(0, 2 ** 32, 32 * E, dtype=np.uint64).astype(np.uint32)
        assert np.array_equal(model_sort(x, E), np.sort(x))


def test_pads_stay_on_top():
    # the sampler pads p draws to 32E with 0xFFFFFFFF; every comparator is ascending, so the pads
    # never move and the first p outputs are the sorted draws
    rng = np.random.default_rng(7)
    p, E = 761, 32
    x = np.full(32 * E, 0xFFFFFFFF, dtype=np.uint32)
    x[:p] = rng.integers(0, 2 ** 32 - 1, p, dtype=np.uint64).astype(np.uint32) & 0xFFFFFFFE
    out = model_sort(x, E, NR=p)                  # the sampler's schedule skips pad comparators
    assert np.array_equal(out[:p], np.sort(x[:p]))
    assert (out[p:] == 0xFFFFFFFF).all()


@pytest.mark.parametrize("p,E", [(653, 32), (761, 32), (857, 32), (953, 32), (1013, 32), (1277, 64)])
def test_pad_skipping_schedule(p, E):
    rng = np.random.default_rng(p)
    for t in range(3):
        x = np.full(32 * E, 0xFFFFFFFF, dtype=np.uint32)
        hi = 4 if t == 1 else 2 ** 32 - 2
        x[:p] = rng.integers(0, hi, p, dtype=np.uint64).astype(np.uint32)
        out = model_sort(x, E, NR=p)
        assert np.array_equal(out[:p], np.sort(x[:p]))

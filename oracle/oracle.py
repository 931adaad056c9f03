"""ctypes wrapper around oracle/liboracle.so -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) may import
this module.  The product package (paper_2106_08759_b200) never imports it.  The C source
(sntrup_oracle.c) is the oracle; this file only marshals numpy arrays.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "sntrup_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

# Parameter sets (p, q, w): 653/761/857 from P:1418-1430 (paper §2.1); 953/1013/1277 from
# BASELINE.json configs[3..4] (reading Z20).  This is the oracle's own copy (C1); the CUDA
# library holds a separate one.
PARAMS = {
    653: (653, 4621, 288),
    761: (761, 4591, 286),
    857: (857, 5167, 322),
    953: (953, 6343, 396),
    1013: (1013, 7177, 448),
    1277: (1277, 7879, 492),
}


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc -O2 (no intrinsics)."""
    deps = [SRC, os.path.join(HERE, "sha512_consts.h")]
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(d) for d in deps):
        tmp = LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-pthread", "-o", tmp, SRC])
        os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        u64, i32, i64, sz = ctypes.c_uint64, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t
        vp = ctypes.c_void_p
        L.or_sm.restype = u64
        L.or_sm.argtypes = [u64, u64]
        L.or_stream_words.restype = None
        L.or_stream_words.argtypes = [u64, u64, u64, i32, vp]
        L.or_small_from_words.argtypes = [i32, vp, vp]
        L.or_short_from_words.argtypes = [i32, i32, vp, vp]
        L.or_poly_mul.argtypes = [i32, i64, vp, vp, vp]
        L.or_poly_inv.restype = i32
        L.or_poly_inv.argtypes = [i32, i64, vp, vp]
        L.or_sha512.restype = None
        L.or_sha512.argtypes = [vp, sz, vp]
        L.or_full_sk.restype = sz
        L.or_full_sk.argtypes = [i32, u64, u64, vp, sz, vp, sz, vp]
        L.or_rq_encode.restype = sz
        L.or_rq_encode.argtypes = [i32, i32, vp, vp]
        L.or_rq_decode.restype = i32
        L.or_rq_decode.argtypes = [i32, i32, vp, vp]
        L.or_rq_encoded_bytes.restype = sz
        L.or_rq_encoded_bytes.argtypes = [i32, i32]
        L.or_encode_general.restype = sz
        L.or_encode_general.argtypes = [i32, vp, vp, vp]
        L.or_decode_general.restype = sz
        L.or_decode_general.argtypes = [i32, vp, vp, vp]
        L.or_small_encode.argtypes = [i32, vp, vp]
        L.or_small_decode.argtypes = [i32, vp, vp]
        L.or_keygen.restype = i32
        L.or_keygen.argtypes = [i32, i32, i32, u64, u64, i32, vp, vp, vp, vp, vp, vp, vp]
        L.or_keygen_many.restype = i32
        L.or_keygen_many.argtypes = [i32, i32, i32, u64, vp, u64, i32, vp, sz, vp, sz,
                                     vp, vp, vp, vp, sz, vp]
        L.or_encap_core.restype = None
        L.or_encap_core.argtypes = [i32, i32, vp, vp, vp]
        L.or_decap_core.restype = i32
        L.or_decap_core.argtypes = [i32, i32, i32, vp, vp, vp, vp]
        L.or_uniform_from_words.restype = None
        L.or_uniform_from_words.argtypes = [i32, i32, vp, vp]
        L.or_mul_many.restype = None
        L.or_mul_many.argtypes = [i32, i64, u64, vp, vp, vp, sz, i32]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ----------------------------------------------------------------------------- stream (C2-C4)
def sm(s: int, j: int) -> int:
    return int(lib().or_sm(s, j))


def stream_words(seed: int, k: int, d: int, n: int) -> np.ndarray:
    u = np.zeros(n, dtype=np.uint32)
    lib().or_stream_words(seed, k, d, n, _p(u))
    return u


def small_from_words(p: int, u: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(u, dtype=np.uint32)
    g = np.zeros(p, dtype=np.int8)
    lib().or_small_from_words(p, _p(u), _p(g))
    return g


def short_from_words(p: int, w: int, u: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(u, dtype=np.uint32)
    f = np.zeros(p, dtype=np.int8)
    lib().or_short_from_words(p, w, _p(u), _p(f))
    return f


def uniform_from_words(p: int, q: int, u: np.ndarray) -> np.ndarray:
    """C12: a_j = floor(u_j q / 2^32) - (q-1)/2 (the R/q microbenchmark's uniform operand)."""
    u = np.ascontiguousarray(u, dtype=np.uint32)
    a = np.zeros(p, dtype=np.int16)
    lib().or_uniform_from_words(p, q, _p(u), _p(a))
    return a


def c12_pair(param: int, seed: int, i: int):
    """Pair i of the R/q microbenchmark (BASELINE configs[2]): with key root
    K_i = SM(seed, i), a from domain 0 (uniform, C12) and b from domain 1 (Short, C4)."""
    p, q, w = PARAMS[param]
    a = uniform_from_words(p, q, stream_words(seed, i, 0, p))
    b = short_from_words(p, w, stream_words(seed, i, 1, p))
    return a, b


# ----------------------------------------------------------------------------- ring (C5-C7)
def poly_mul(p: int, m: int, a, b) -> np.ndarray:
    A = np.ascontiguousarray(np.asarray(a, dtype=np.int64)[:p])
    B = np.ascontiguousarray(np.asarray(b, dtype=np.int64)[:p])
    C = np.zeros(p, dtype=np.int64)
    lib().or_poly_mul(p, m, _p(A), _p(B), _p(C))
    return C


def poly_inv(p: int, m: int, a):
    """Returns (ok, inverse) in (Z/m)[x]/(x^p-x-1), centered."""
    A = np.ascontiguousarray(np.asarray(a, dtype=np.int64)[:p])
    C = np.zeros(p, dtype=np.int64)
    ok = lib().or_poly_inv(p, m, _p(A), _p(C))
    return bool(ok), C


def mul_many(p: int, m: int, a: np.ndarray, b: np.ndarray, threads: int = 0) -> np.ndarray:
    """Row-wise products of int16 [n][row] arrays (row >= p), threaded over rows."""
    a = np.ascontiguousarray(a, dtype=np.int16)
    b = np.ascontiguousarray(b, dtype=np.int16)
    n, row = a.shape
    c = np.zeros_like(a)
    lib().or_mul_many(p, m, n, _p(a), _p(b), _p(c), row, threads or (os.cpu_count() or 1))
    return c


# ----------------------------------------------------------------------------- encap / decap core
def encap_core(p: int, q: int, h, r) -> np.ndarray:
    """c = Round(h * r) in R/q (SPEC encrypt_core): int16 [p], every coefficient = 0 mod 3."""
    H = np.ascontiguousarray(np.asarray(h, dtype=np.int16)[:p])
    R = np.ascontiguousarray(np.asarray(r, dtype=np.int8)[:p])
    C = np.zeros(p, dtype=np.int16)
    lib().or_encap_core(p, q, _p(H), _p(R), _p(C))
    return C


def decap_core(p: int, q: int, w: int, f, ginv, c):
    """(ok, r') with r' = ((3f * c) mod 3) * (1/g) in R/3 and ok = weight(r') == w."""
    F = np.ascontiguousarray(np.asarray(f, dtype=np.int8)[:p])
    G = np.ascontiguousarray(np.asarray(ginv, dtype=np.int8)[:p])
    C = np.ascontiguousarray(np.asarray(c, dtype=np.int16)[:p])
    R = np.zeros(p, dtype=np.int8)
    ok = lib().or_decap_core(p, q, w, _p(F), _p(G), _p(C), _p(R))
    return bool(ok), R


# ----------------------------------------------------------------------------- encodings (C10-C11)
def rq_encode(p: int, q: int, h) -> bytes:
    H = np.ascontiguousarray(np.asarray(h, dtype=np.int16)[:p])
    out = np.zeros(4 * p + 16, dtype=np.uint8)
    n = lib().or_rq_encode(p, q, _p(H), _p(out))
    return out[:n].tobytes()


def rq_decode(p: int, q: int, data: bytes) -> np.ndarray:
    S = np.frombuffer(bytes(data) + b"\0" * 16, dtype=np.uint8).copy()
    h = np.zeros(p, dtype=np.int16)
    rc = lib().or_rq_decode(p, q, _p(S), _p(h))
    if rc != 0:
        raise ValueError("rq_decode: out-of-range value")
    return h


def rq_encoded_bytes(p: int, q: int) -> int:
    return int(lib().or_rq_encoded_bytes(p, q))


def encode_general(R, M) -> bytes:
    R = np.ascontiguousarray(R, dtype=np.uint32)
    M = np.ascontiguousarray(M, dtype=np.uint32)
    out = np.zeros(4 * len(R) + 16, dtype=np.uint8)
    n = lib().or_encode_general(len(R), _p(R), _p(M), _p(out))
    return out[:n].tobytes()


def decode_general(M, data: bytes) -> np.ndarray:
    M = np.ascontiguousarray(M, dtype=np.uint32)
    S = np.frombuffer(bytes(data) + b"\0" * 16, dtype=np.uint8).copy()
    R = np.zeros(len(M), dtype=np.uint32)
    n = lib().or_decode_general(len(M), _p(M), _p(S), _p(R))
    if n == ctypes.c_size_t(-1).value:
        raise ValueError("decode: out-of-range value")
    return R


def small_encode(p: int, c) -> bytes:
    C = np.ascontiguousarray(np.asarray(c, dtype=np.int8)[:p])
    out = np.zeros((p + 3) // 4, dtype=np.uint8)
    lib().or_small_encode(p, _p(C), _p(out))
    return out.tobytes()


def small_decode(p: int, data: bytes) -> np.ndarray:
    S = np.frombuffer(bytes(data), dtype=np.uint8).copy()
    c = np.zeros(p, dtype=np.int8)
    lib().or_small_decode(p, _p(S), _p(c))
    return c


def pk_bytes(param: int) -> int:
    p, q, _ = PARAMS[param]
    return rq_encoded_bytes(p, q)


def sk_bytes(param: int) -> int:
    p = PARAMS[param][0]
    return 2 * ((p + 3) // 4)


# ----------------------------------------------------------------------------- keygen
def keygen(param: int, seed: int, k: int, max_attempts: int = 255) -> dict:
    p, q, w = PARAMS[param]
    g = np.zeros(p, np.int8); f = np.zeros(p, np.int8); gi = np.zeros(p, np.int8)
    h = np.zeros(p, np.int16); att = ctypes.c_int(0)
    pk = np.zeros(pk_bytes(param), np.uint8); sk = np.zeros(sk_bytes(param), np.uint8)
    rc = lib().or_keygen(p, q, w, seed, k, max_attempts, _p(g), _p(f), _p(gi), _p(h),
                         ctypes.addressof(att), _p(pk), _p(sk))
    if rc != 0:
        raise RuntimeError("oracle keygen failed rc=%d" % rc)
    return dict(g=g, f=f, ginv=gi, h=h, attempts=att.value, pk=pk.tobytes(), sk=sk.tobytes())


def keygen_many(param: int, seed: int, indices, threads: int = 0, want_polys: bool = False,
                row: int | None = None) -> dict:
    """Keys for the given global indices, one key at a time per host thread."""
    p, q, w = PARAMS[param]
    idx = np.ascontiguousarray(np.asarray(indices, dtype=np.uint64))
    n = len(idx)
    pkb, skb = pk_bytes(param), sk_bytes(param)
    pk = np.zeros((n, pkb), np.uint8)
    sk = np.zeros((n, skb), np.uint8)
    att = np.zeros(n, np.int32)
    row = row or p
    h = g = f = gi = None
    if want_polys:
        h = np.zeros((n, row), np.int16); g = np.zeros((n, row), np.int8)
        f = np.zeros((n, row), np.int8); gi = np.zeros((n, row), np.int8)
    nul = ctypes.c_void_p(0)
    rc = lib().or_keygen_many(p, q, w, seed, _p(idx), n, threads or (os.cpu_count() or 1),
                              _p(pk), pkb, _p(sk), skb,
                              _p(h) if h is not None else nul, _p(g) if g is not None else nul,
                              _p(f) if f is not None else nul, _p(gi) if gi is not None else nul,
                              row, _p(att))
    if rc != 0:
        raise RuntimeError("oracle keygen_many failed rc=%d" % rc)
    out = dict(pk=pk, sk=sk, attempts=att)
    if want_polys:
        out.update(h=h, g=g, f=f, ginv=gi)
    return out


def sha512(data: bytes) -> bytes:
    """FIPS 180-4 SHA-512 (the oracle's own C implementation)."""
    buf = ctypes.create_string_buffer(bytes(data), max(1, len(data)))
    out = ctypes.create_string_buffer(64)
    lib().or_sha512(buf, len(data), out)
    return out.raw


def full_sk_bytes(param: int) -> int:
    """|sk_full| = 3 ceil(p/4) + |pk| + 32 (App. D pair storage minus pk; reading Z24)."""
    p = PARAMS[param][0]
    return sk_bytes(param) + pk_bytes(param) + (p + 3) // 4 + 32


def full_sk(param: int, seed: int, k: int, pk: bytes, sk: bytes) -> bytes:
    """sk_full = sk || pk || rho || SHA-512(4 || pk)[:32] for global key index k (reading Z24)."""
    p = PARAMS[param][0]
    out = ctypes.create_string_buffer(full_sk_bytes(param))
    n = lib().or_full_sk(p, seed, k, bytes(pk), len(pk), bytes(sk), len(sk), out)
    assert n == full_sk_bytes(param)
    return out.raw

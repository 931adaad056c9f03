"""paper_2106_08759_b200 -- B200-native batched sntrup key generation (arXiv 2106.08759).

Thin Python binding over the C ABI of libsntrup_gpu.so (include/sntrup_gpu.h).  Argument
marshalling only: every step of the hot path runs in the library's sm_100a kernels.  PyTorch is
used for device memory and streams.  There is NO CPU fallback: importing without the built
library raises.
"""
from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_PKG, "libsntrup_gpu.so")
if os.environ.get("SNTRUP_GPU_LIB"):            # e.g. the bounds-checked build (tests only)
    _LIB_PATH = os.environ["SNTRUP_GPU_LIB"]

if not os.path.exists(_LIB_PATH):
    raise ImportError("libsntrup_gpu.so is not built (run __graft_entry__.build() or "
                      "python -m paper_2106_08759_b200._build); there is no CPU fallback")

_lib = ctypes.CDLL(_LIB_PATH)

SNTRUP_OK = 0
SNTRUP_E_PARAM = -1
SNTRUP_E_ARG = -2
SNTRUP_E_NOT_INVERTIBLE = -3
SNTRUP_E_CUDA = -4
SNTRUP_E_WORKSPACE = -5
SNTRUP_E_INTERNAL = -6

OPT_HOST_OUTPUT = 1
OPT_NO_SMALL_CHECK = 2
OPT_ASYNC = 4
OPT_FORCE_SMALL_CHECK = 8
OPT_RING_STREAMS = 16
OPT_LANES4 = 32
OPT_LANE_PRIORITY = 64
OPT_STAGGER = 128
OPT_SERIAL = 256
OPT_GRAPH = 512         # replay the call as a CUDA graph (captured per call shape)

PARAM_SETS = (653, 761, 857, 953, 1013, 1277)


class KeygenOpts(ctypes.Structure):
    _fields_ = [("first_key_index", ctypes.c_uint64), ("batch_size", ctypes.c_uint32),
                ("flags", ctypes.c_uint32), ("chunk_keys", ctypes.c_uint64),
                ("stream", ctypes.c_void_p), ("h_out", ctypes.c_void_p),
                ("g_out", ctypes.c_void_p), ("f_out", ctypes.c_void_p),
                ("ginv_out", ctypes.c_void_p), ("attempts_out", ctypes.c_void_p),
                ("stats_out", ctypes.c_void_p), ("done_event", ctypes.c_void_p),
                ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_size_t)]


_u64, _i32, _u32, _vp, _sz = ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_size_t
_lib.sntrup_params.argtypes = [_i32] + [_vp] * 7
_lib.sntrup_strerror.restype = ctypes.c_char_p
_lib.sntrup_strerror.argtypes = [_i32]
_lib.sntrup_batch_keygen.argtypes = [_i32, _u64, _u64, _vp, _vp]
_lib.sntrup_batch_keygen_ex.argtypes = [_i32, _u64, _u64, _vp, _vp, ctypes.POINTER(KeygenOpts)]
_lib.sntrup_keygen_workspace_bytes.restype = _sz
_lib.sntrup_keygen_workspace_bytes.argtypes = [_i32, _u64, _u32]
_lib.sntrup_keygen_workspace_bytes_ex.restype = _sz
_lib.sntrup_keygen_workspace_bytes_ex.argtypes = [_i32, _u64, _u32, _u32, _u64]
_lib.sntrup_workspace_reserved_bytes.restype = _sz
_lib.sntrup_workspace_reserved_bytes.argtypes = [_vp, _i32]
_lib.rq_mul_batch.argtypes = [_i32, _u64, _vp, _vp, _vp, _vp]
_lib.r3_mul_batch.argtypes = [_i32, _u64, _vp, _vp, _vp, _vp]
_lib.rq_recip_batch.argtypes = [_i32, _u64, _vp, _vp, _u32, ctypes.POINTER(ctypes.c_uint64), _vp]
_lib.r3_recip_batch.argtypes = [_i32, _u64, _vp, _vp, _vp, _u32, _vp]
_lib.r3_is_invertible_batch.argtypes = [_i32, _u64, _vp, _vp, _vp]
_lib.rq_encode_batch.argtypes = [_i32, _u64, _vp, _vp, _vp]
_lib.sntrup_release_workspace.restype = None
_lib.sntrup_release_stream_workspace.argtypes = [_vp]
_lib.sntrup_kernel_launch_count.restype = _u64
_lib.sntrup_set_mul_impl.argtypes = [_i32]
_lib.sntrup_set_divstep_threads.argtypes = [_i32]
_lib.sntrup_set_root_impl.argtypes = [_i32]
_lib.sntrup_set_sched.argtypes = [ctypes.c_longlong, ctypes.c_longlong]
_lib.sntrup_profile_enable.restype = None
_lib.sntrup_profile_enable.argtypes = [_i32]
_lib.sntrup_profile_read.restype = _i32
_lib.sntrup_profile_read.argtypes = [_i32, _vp, _vp, _vp, _vp, _i32]
_lib.sntrup_profile_read_kinds.restype = _i32
_lib.sntrup_profile_read_kinds.argtypes = [_i32, _vp, _vp, _vp]
_lib.sntrup_profile_read_kinds_ex.restype = _i32
_lib.sntrup_profile_read_kinds_ex.argtypes = [_i32, _vp, _vp, _vp, _vp, _vp]
_lib.sntrup_measure_int_peak.argtypes = [_i32, _vp, _vp]
_lib.sntrup_probe_half_mul.argtypes = [_i32, _u64, _vp, _vp, _vp, _vp]
_lib.sntrup_pool_create.argtypes = [_i32, _u64, _u64, _u64, _u64, _u32, ctypes.POINTER(_vp)]
_lib.sntrup_pool_take.argtypes = [_vp, _vp, _vp, ctypes.POINTER(ctypes.c_uint64)]
_lib.sntrup_pool_stats.argtypes = [_vp] + [ctypes.POINTER(ctypes.c_uint64)] * 4
_lib.sntrup_pool_destroy.argtypes = [_vp]
_lib.sntrup_pool_destroy.restype = None
_lib.rq_mul_small_batch.argtypes = [_i32, _u64, _vp, _vp, _vp, _vp]
_lib.sntrup_sample_short_batch.argtypes = [_i32, _u64, _u64, _u64, _u64, _vp, _vp]
_lib.sntrup_sample_uniform_rq_batch.argtypes = [_i32, _u64, _u64, _u64, _u64, _vp, _vp]
_lib.sntrup_encap_core_batch.argtypes = [_i32, _u64, _vp, _vp, _vp, _vp]
_lib.sntrup_decap_core_batch.argtypes = [_i32, _u64, _vp, _vp, _vp, _vp, _vp, _vp]
_lib.sntrup_full_sk_bytes.argtypes = [_i32]
_lib.sntrup_full_sk_bytes.restype = ctypes.c_size_t
_lib.sntrup_full_sk_batch.argtypes = [_i32, _u64, _u64, _u64, _vp, _vp, _vp, _vp]
_lib.sntrup_event_create.argtypes = [ctypes.POINTER(_vp)]
_lib.sntrup_async_error.argtypes = [_vp]
_lib.sntrup_event_synchronize.argtypes = [_vp]
_lib.sntrup_event_query.argtypes = [_vp]
_lib.sntrup_event_destroy.argtypes = [_vp]
_lib.sntrup_event_destroy.restype = None

EXPORTED = ("sntrup_params", "sntrup_strerror", "sntrup_batch_keygen", "sntrup_batch_keygen_ex",
            "sntrup_keygen_workspace_bytes", "sntrup_keygen_workspace_bytes_ex",
            "sntrup_workspace_reserved_bytes", "rq_mul_batch", "rq_mul_small_batch", "r3_mul_batch", "rq_recip_batch",
            "r3_recip_batch", "r3_is_invertible_batch", "rq_encode_batch",
            "sntrup_release_workspace", "sntrup_release_stream_workspace", "sntrup_kernel_launch_count", "sntrup_set_mul_impl", "sntrup_set_divstep_threads",
            "sntrup_set_root_impl", "sntrup_set_sched",
            "sntrup_profile_enable", "sntrup_profile_read_kinds", "sntrup_profile_read_kinds_ex",
            "sntrup_measure_int_peak", "sntrup_probe_half_mul", "sntrup_pool_create",
            "sntrup_pool_take", "sntrup_pool_stats", "sntrup_pool_destroy",
            "sntrup_sample_short_batch", "sntrup_sample_uniform_rq_batch", "sntrup_encap_core_batch", "sntrup_decap_core_batch",
            "sntrup_profile_read", "sntrup_full_sk_bytes", "sntrup_full_sk_batch",
            "sntrup_async_error", "sntrup_event_create", "sntrup_event_synchronize", "sntrup_event_query", "sntrup_event_destroy")

PROFILE_CLASSES = ("sample", "r3_mul", "rq_mul", "root_inv", "rq_inv", "repair", "encode", "other")


class SntrupError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        self.code = code
        super().__init__("%s: %s (%d)" % (what, _lib.sntrup_strerror(code).decode(), code))


def _check(rc: int, what: str):
    if rc != SNTRUP_OK:
        raise SntrupError(rc, what)


def params(param_set: int) -> dict:
    vals = [ctypes.c_int() for _ in range(5)] + [ctypes.c_size_t() for _ in range(2)]
    _check(_lib.sntrup_params(param_set, *[ctypes.addressof(v) for v in vals]), "sntrup_params")
    p, q, w, p16, p8, pk, sk = (v.value for v in vals)
    return dict(p=p, q=q, w=w, p16=p16, p8=p8, pk_bytes=pk, sk_bytes=sk)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _need(t, dtype, shape, name, host: bool = False):
    """Inputs and caller-supplied outputs: exact dtype and shape, contiguous, on the device (or, for
    host-output keygen, in host memory) -- a short or mistyped buffer would be written past."""
    if (not isinstance(t, torch.Tensor) or t.dtype != dtype or tuple(t.shape) != tuple(shape)
            or not t.is_contiguous() or t.is_cuda == host):
        raise ValueError("%s must be a contiguous %s %s tensor of shape %s"
                         % (name, "host" if host else "CUDA", dtype, tuple(shape)))


def batch_keygen(param_set: int, n_keys: int, seed: int, *, first_key_index: int = 0,
                 batch_size: int = 32, chunk_keys: int = 0, flags: int = 0, pk_out=None,
                 sk_out=None, debug: bool = False, stream=None, stats: bool = False, done_event=None,
                 workspace=None, attempts: bool = False):
    """Generate n_keys key pairs (global indices first_key_index ..).  Returns dict with pk, sk
    (uint8 CUDA tensors) and, with debug=True, h/g/f/ginv/attempts (attempts=True: only the
    per-key number of g draws, uint8 CUDA tensor).  With host outputs,
    flags OPT_ASYNC and a done_event (Event), the call returns after enqueueing and the event
    completes when every output byte is in host memory."""
    P = params(param_set)
    host = bool(flags & OPT_HOST_OUTPUT)
    # host outputs default to pinned host memory (the library copies each chunk back into them)
    where = dict(device="cpu", pin_memory=True) if host else dict(device="cuda")
    if pk_out is None:
        pk_out = torch.empty((n_keys, P["pk_bytes"]), dtype=torch.uint8, **where)
    if sk_out is None:
        sk_out = torch.empty((n_keys, P["sk_bytes"]), dtype=torch.uint8, **where)
    _need(pk_out, torch.uint8, (n_keys, P["pk_bytes"]), "pk_out", host=host)
    _need(sk_out, torch.uint8, (n_keys, P["sk_bytes"]), "sk_out", host=host)
    o = KeygenOpts()
    o.first_key_index = first_key_index
    o.batch_size = batch_size
    o.flags = flags
    o.chunk_keys = chunk_keys
    o.stream = _stream(stream)
    out = dict(pk=pk_out, sk=sk_out)
    dev = torch.device("cuda", torch.cuda.current_device())
    if debug:
        out["h"] = torch.zeros((n_keys, P["p8"]), dtype=torch.int16, device=dev)
        for k in ("g", "f", "ginv"):
            out[k] = torch.zeros((n_keys, P["p16"]), dtype=torch.int8, device=dev)
        out["attempts"] = torch.zeros(n_keys, dtype=torch.uint8, device=dev)
        o.h_out, o.g_out, o.f_out = out["h"].data_ptr(), out["g"].data_ptr(), out["f"].data_ptr()
        o.ginv_out, o.attempts_out = out["ginv"].data_ptr(), out["attempts"].data_ptr()
    elif attempts:
        out["attempts"] = torch.zeros(n_keys, dtype=torch.uint8, device=dev)
        o.attempts_out = out["attempts"].data_ptr()
    st = (ctypes.c_uint64 * 4)()
    if stats:
        o.stats_out = ctypes.addressof(st)
    if done_event is not None:
        o.done_event = done_event.handle
    if workspace is not None:               # caller-owned device scratch (uint8 CUDA tensor)
        if not (isinstance(workspace, torch.Tensor) and workspace.is_cuda and workspace.is_contiguous()):
            raise ValueError("workspace must be a contiguous CUDA tensor")
        o.workspace = workspace.data_ptr()
        o.workspace_bytes = workspace.numel() * workspace.element_size()
    _check(_lib.sntrup_batch_keygen_ex(param_set, n_keys, seed, ctypes.c_void_p(pk_out.data_ptr()),
                                       ctypes.c_void_p(sk_out.data_ptr()), ctypes.byref(o)),
           "sntrup_batch_keygen_ex")
    if stats:
        out["stats"] = dict(rq_products=st[0], r3_products=st[1], root_inversions=st[2],
                            keys_repaired=st[3])
    return out


class Event:
    """Completion event of an asynchronous host-output keygen call (sntrup_event_*)."""

    def __init__(self):
        h = ctypes.c_void_p()
        _check(_lib.sntrup_event_create(ctypes.byref(h)), "sntrup_event_create")
        self.handle = h.value

    def synchronize(self):
        _check(_lib.sntrup_event_synchronize(ctypes.c_void_p(self.handle)), "sntrup_event_synchronize")

    def query(self) -> bool:
        rc = _lib.sntrup_event_query(ctypes.c_void_p(self.handle))
        if rc not in (0, 1):
            _check(rc, "sntrup_event_query")
        return rc == 0

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:     # (_lib is None at interpreter exit)
            _lib.sntrup_event_destroy(ctypes.c_void_p(self.handle))
            self.handle = None


def rq_mul_batch(param_set: int, a, b, c=None, stream=None):
    P = params(param_set)
    n = a.shape[0]
    _need(a, torch.int16, (n, P["p8"]), "a")
    _need(b, torch.int16, (n, P["p8"]), "b")
    if c is None:
        c = torch.empty_like(a)
    _need(c, torch.int16, (n, P["p8"]), "c")
    _check(_lib.rq_mul_batch(param_set, n, _ptr(a), _ptr(b), _ptr(c), _stream(stream)), "rq_mul_batch")
    return c


def rq_mul_small_batch(param_set: int, a, b, c=None, stream=None):
    """Big x small R/q product: a int16 [n][p8] centered, b int8 [n][p16] (|b_j| <= 127)."""
    P = params(param_set)
    n = a.shape[0]
    _need(a, torch.int16, (n, P["p8"]), "a")
    _need(b, torch.int8, (n, P["p16"]), "b")
    if c is None:
        c = torch.empty_like(a)
    _need(c, torch.int16, (n, P["p8"]), "c")
    _check(_lib.rq_mul_small_batch(param_set, n, _ptr(a), _ptr(b), _ptr(c), _stream(stream)),
           "rq_mul_small_batch")
    return c


ENC_DOMAIN = 1 << 32      # C2: stream domains >= 2^32 are reserved for encapsulation draws


def full_sk_bytes(param_set: int) -> int:
    """Bytes of one full-size sk row: sk || pk || rho || SHA-512(4 || pk)[:32] (1763 for 761)."""
    v = _lib.sntrup_full_sk_bytes(param_set)
    if not v:
        raise SntrupError(SNTRUP_E_PARAM, "sntrup_full_sk_bytes")
    return v


def full_sk_batch(param_set: int, seed: int, pk, sk, first_key_index: int = 0, out=None, stream=None):
    """Full-size secret keys for keys first_key_index.. from their device pk / sk rows."""
    P = params(param_set)
    n = pk.shape[0]
    _need(pk, torch.uint8, (n, P["pk_bytes"]), "pk")
    _need(sk, torch.uint8, (n, P["sk_bytes"]), "sk")
    fsb = full_sk_bytes(param_set)
    if out is None:
        out = torch.empty((n, fsb), dtype=torch.uint8, device=pk.device)
    _need(out, torch.uint8, (n, fsb), "out")
    _check(_lib.sntrup_full_sk_batch(param_set, n, seed, first_key_index, _ptr(pk), _ptr(sk), _ptr(out),
                                     _stream(stream)), "sntrup_full_sk_batch")
    return out


def sample_short_batch(param_set: int, n: int, seed: int, first_key_index: int = 0,
                       domain: int = ENC_DOMAIN, out=None, stream=None):
    """Short elements (weight w) of one stream domain for global key indices first.. (int8 rows)."""
    P = params(param_set)
    if out is None:
        out = torch.empty((n, P["p16"]), dtype=torch.int8, device="cuda")
    _need(out, torch.int8, (n, P["p16"]), "out")
    _check(_lib.sntrup_sample_short_batch(param_set, n, seed, first_key_index, domain, _ptr(out),
                                          _stream(stream)), "sntrup_sample_short_batch")
    return out


def sample_uniform_rq_batch(param_set: int, n: int, seed: int, first_key_index: int = 0,
                            domain: int = 0, out=None, stream=None):
    """Uniform R/q elements (the R/q microbenchmark's operand) of one stream domain
    for global key indices first.. (int16 rows of p8)."""
    P = params(param_set)
    if out is None:
        out = torch.empty((n, P["p8"]), dtype=torch.int16, device="cuda")
    _need(out, torch.int16, (n, P["p8"]), "out")
    _check(_lib.sntrup_sample_uniform_rq_batch(param_set, n, seed, first_key_index, domain, _ptr(out),
                                               _stream(stream)), "sntrup_sample_uniform_rq_batch")
    return out


def encap_core_batch(param_set: int, h, r, c=None, stream=None):
    """c = Round(h * r) in R/q (each coefficient to the nearest multiple of 3)."""
    P = params(param_set)
    n = h.shape[0]
    _need(h, torch.int16, (n, P["p8"]), "h")
    _need(r, torch.int8, (n, P["p16"]), "r")
    if c is None:
        c = torch.empty_like(h)
    _need(c, torch.int16, (n, P["p8"]), "c")
    _check(_lib.sntrup_encap_core_batch(param_set, n, _ptr(h), _ptr(r), _ptr(c), _stream(stream)),
           "sntrup_encap_core_batch")
    return c


def decap_core_batch(param_set: int, f, ginv, c, r_out=None, ok=None, stream=None):
    """(r', ok): r' = ((3f * c) mod 3) * (1/g) in R/3, ok = weight(r') == w."""
    P = params(param_set)
    n = c.shape[0]
    _need(f, torch.int8, (n, P["p16"]), "f")
    _need(ginv, torch.int8, (n, P["p16"]), "ginv")
    _need(c, torch.int16, (n, P["p8"]), "c")
    if r_out is None:
        r_out = torch.empty_like(f)
    if ok is None:
        ok = torch.empty(n, dtype=torch.uint8, device=c.device)
    _need(r_out, torch.int8, (n, P["p16"]), "r_out")
    _need(ok, torch.uint8, (n,), "ok")
    _check(_lib.sntrup_decap_core_batch(param_set, n, _ptr(f), _ptr(ginv), _ptr(c), _ptr(r_out), _ptr(ok),
                                        _stream(stream)), "sntrup_decap_core_batch")
    return r_out, ok


def r3_mul_batch(param_set: int, a, b, c=None, stream=None):
    P = params(param_set)
    n = a.shape[0]
    _need(a, torch.int8, (n, P["p16"]), "a")
    _need(b, torch.int8, (n, P["p16"]), "b")
    if c is None:
        c = torch.empty_like(a)
    _need(c, torch.int8, (n, P["p16"]), "c")
    _check(_lib.r3_mul_batch(param_set, n, _ptr(a), _ptr(b), _ptr(c), _stream(stream)), "r3_mul_batch")
    return c


def rq_recip_batch(param_set: int, a, out=None, batch_size: int = 32, stream=None):
    """Returns out; raises SntrupError(SNTRUP_E_NOT_INVERTIBLE) with .bad_index for zero rows."""
    P = params(param_set)
    n = a.shape[0]
    _need(a, torch.int16, (n, P["p8"]), "a")
    if out is None:
        out = torch.empty_like(a)
    _need(out, torch.int16, (n, P["p8"]), "out")
    bad = ctypes.c_uint64(0)
    rc = _lib.rq_recip_batch(param_set, n, _ptr(a), _ptr(out), batch_size, ctypes.byref(bad), _stream(stream))
    if rc != SNTRUP_OK:
        e = SntrupError(rc, "rq_recip_batch")
        e.bad_index = bad.value
        raise e
    return out


def r3_recip_batch(param_set: int, g, out=None, ok=None, batch_size: int = 32, stream=None):
    P = params(param_set)
    n = g.shape[0]
    _need(g, torch.int8, (n, P["p16"]), "g")
    if out is None:
        out = torch.empty_like(g)
    if ok is None:
        ok = torch.empty(n, dtype=torch.uint8, device=g.device)
    _need(out, torch.int8, (n, P["p16"]), "out")
    _need(ok, torch.uint8, (n,), "ok")
    _check(_lib.r3_recip_batch(param_set, n, _ptr(g), _ptr(out), _ptr(ok), batch_size, _stream(stream)),
           "r3_recip_batch")
    return out, ok


def r3_is_invertible_batch(param_set: int, g, stream=None):
    P = params(param_set)
    n = g.shape[0]
    _need(g, torch.int8, (n, P["p16"]), "g")
    ok = torch.empty(n, dtype=torch.uint8, device=g.device)
    _check(_lib.r3_is_invertible_batch(param_set, n, _ptr(g), _ptr(ok), _stream(stream)),
           "r3_is_invertible_batch")
    return ok


def rq_encode_batch(param_set: int, h, pk=None, stream=None):
    P = params(param_set)
    n = h.shape[0]
    _need(h, torch.int16, (n, P["p8"]), "h")
    if pk is None:
        pk = torch.empty((n, P["pk_bytes"]), dtype=torch.uint8, device=h.device)
    _need(pk, torch.uint8, (n, P["pk_bytes"]), "pk")
    _check(_lib.rq_encode_batch(param_set, n, _ptr(h), _ptr(pk), _stream(stream)), "rq_encode_batch")
    return pk


def keygen_workspace_bytes(param_set: int, n_keys: int, batch_size: int = 32, flags: int = 0,
                           chunk_keys: int = 0) -> int:
    return int(_lib.sntrup_keygen_workspace_bytes_ex(param_set, n_keys, batch_size, flags, chunk_keys))


def workspace_reserved_bytes(stream=None, staging: bool = False) -> int:
    """Bytes the library holds for `stream` (the cached workspace, or the host-output staging)."""
    return int(_lib.sntrup_workspace_reserved_bytes(_stream(stream), 1 if staging else 0))


def async_error(stream=None):
    """Raise if the last keygen call on `stream` (e.g. an OPT_ASYNC one) hit the g retry bound."""
    _check(_lib.sntrup_async_error(_stream(stream)), "sntrup_async_error")


def release_workspace():
    _lib.sntrup_release_workspace()


def release_stream_workspace(stream=None):
    _check(_lib.sntrup_release_stream_workspace(_stream(stream)), "sntrup_release_stream_workspace")


def kernel_launch_count() -> int:
    return int(_lib.sntrup_kernel_launch_count())


MUL_TENSOR_CORE = 0
MUL_SCHOOLBOOK = 1
MUL_TENSOR_CORE_NO_SHARED_A = 2   # int8 only, one product per work item
MUL_TENSOR_CORE_INT8 = 3          # int8 only, shared-A down-sweep
MUL_TENSOR_CORE_FP4_ALL = 4       # fp4 also for big x small (base-9 digits)
MUL_TENSOR_CORE_M64 = 5           # int8 products at MMA M = 64 (default: 128)
MUL_TENSOR_CORE_I8_SINGLE = 6     # one int8 big x big product per work item (default: shared A)
MUL_TENSOR_CORE_U_FUSED = 7       # keygen u products fused with the R/q level 1 (default: own stream)
MUL_TENSOR_CORE_PIPELINED = 8     # int8 big x big products software-pipelined (2 stages, 8 warps)
MUL_TENSOR_CORE_TMEM_A = 9        # fp4 products: first K steps of the Hankel A operand in TMEM (128 cols)
MUL_TENSOR_CORE_TMEM_A64 = 10     # as 9 with a 64-column TMEM allocation
MUL_TENSOR_CORE_WS = 11           # warp-specialised persistent kernels, Hankel A written to TMEM
MUL_TENSOR_CORE_TRANSPOSED = 13   # int8 one-product items in the transposed Hankel form (tcxmul.cuh)
MUL_TENSOR_CORE_ONE_PART = 14     # int8 big x big two-product items over the whole K range at once (default: two parts)
MUL_TENSOR_CORE_3PARTS = 15       # ... in three parts
MUL_TENSOR_CORE_PARTS_ALL = 16    # one-product int8 big x big items in two parts too
MUL_TENSOR_CORE_TMEM_RING = 12    # fp4: every K step's A rows through a 64-column TMEM window in rounds


def set_mul_impl(impl: int):
    """0 = tcgen05 int8 Hankel-GEMM ring product (default), 1 = int32 schoolbook (v1)."""
    _check(_lib.sntrup_set_mul_impl(int(impl)), "sntrup_set_mul_impl")


ROOT_AUTO = 0       # jump-divsteps for standalone reciprocals and keygen calls <= 4096 keys, else per-step
ROOT_STEP = 1       # one divstep at a time (R/q: per CTA barrier; R/3: bitsliced warp)
ROOT_JUMP = 2       # jump-divsteps everywhere
ROOT_SHARED_SM = 4  # (+) jump CTAs reserve only the shared memory they use


def set_root_impl(impl: int):
    """Root inversions when the roots are few: ROOT_AUTO (default), ROOT_STEP, ROOT_JUMP (+ ROOT_SHARED_SM)."""
    _check(_lib.sntrup_set_root_impl(int(impl)), "sntrup_set_root_impl")


def set_sched(top_items: int = 0, items_cap: int = 0):
    """Tree tops of bulk keygen calls on high-priority streams (launches of <= top_items products and
    the roots); ring-product CTAs retire after items_cap work items.  (0, 0) = off."""
    _check(_lib.sntrup_set_sched(int(top_items), int(items_cap)), "sntrup_set_sched")


def profile_enable(on: bool = True):
    _lib.sntrup_profile_enable(1 if on else 0)


class KeyPool:
    """GPU-backed key pool (sntrup_pool_*): take() returns (pk, sk, key_index) as host bytes."""

    def __init__(self, param_set: int, seed: int, capacity: int, batch_keys: int,
                 batch_size: int = 32, first_key_index: int = 0):
        self.P = params(param_set)
        h = ctypes.c_void_p()
        _check(_lib.sntrup_pool_create(param_set, seed, first_key_index, capacity, batch_keys,
                                       batch_size, ctypes.byref(h)), "sntrup_pool_create")
        self._h = h
        self._pk = (ctypes.c_uint8 * self.P["pk_bytes"])()
        self._sk = (ctypes.c_uint8 * self.P["sk_bytes"])()

    def take(self):
        idx = ctypes.c_uint64()
        _check(_lib.sntrup_pool_take(self._h, self._pk, self._sk, ctypes.byref(idx)), "sntrup_pool_take")
        return bytes(self._pk), bytes(self._sk), idx.value

    def stats(self) -> dict:
        v = [ctypes.c_uint64() for _ in range(4)]
        _check(_lib.sntrup_pool_stats(self._h, *[ctypes.byref(x) for x in v]), "sntrup_pool_stats")
        return dict(taken=v[0].value, generated=v[1].value, waits=v[2].value, ready=v[3].value)

    def close(self):
        if self._h:
            _lib.sntrup_pool_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


MUL_KINDS = ("tc_int8", "tc_fp4", "int32")


def profile_read_kinds(reset: bool = True) -> dict:
    """Ring-product launches by arithmetic kind: device ms, algorithmic ops (2 p^2 per product),
    launches, products, and the operand bytes the MMAs fetched from shared memory."""
    ms = (ctypes.c_double * 3)()
    op = (ctypes.c_double * 3)()
    la = (ctypes.c_uint64 * 3)()
    pr = (ctypes.c_double * 3)()
    sm = (ctypes.c_double * 3)()
    _lib.sntrup_profile_read_kinds_ex(1 if reset else 0, ms, op, la, pr, sm)
    return {MUL_KINDS[i]: dict(ms=ms[i], ops=op[i], launches=la[i], products=pr[i], smem_bytes=sm[i])
            for i in range(3)}


INT_OPS = ("IMAD", "IADD3", "LOP3", "SHF")


def probe_half_mul(kind: int, a, b, c, stream=None):
    """Measurement hook: ring products at p' = 383 (one Karatsuba sub-product of a 761 product);
    kind 0 = R/3 (int8 [n][384]), 1 = R/q big x big (int16 [n][384]); kinds 2 / 3 = R/3 at
    p' = 255 / 257 (int8 [n][256] / [n][272]: the 5-way R/3 multiplier's sub-products)."""
    n = a.shape[0]
    dt, w = {0: (torch.int8, 384), 1: (torch.int16, 384), 2: (torch.int8, 256), 3: (torch.int8, 272)}[kind]
    for t, nm in ((a, "a"), (b, "b"), (c, "c")):
        _need(t, dt, (n, w), nm)
    _check(_lib.sntrup_probe_half_mul(kind, n, _ptr(a), _ptr(b), _ptr(c), _stream(stream)), "sntrup_probe_half_mul")
    return c


def measure_int_peak(op: str) -> dict:
    """Integer-pipe peak of one SASS op (full-occupancy microkernel): lane-ops per SM clock per SM,
    and lane-ops/s of the whole GPU at this run's clock."""
    a, b = ctypes.c_double(), ctypes.c_double()
    _check(_lib.sntrup_measure_int_peak(INT_OPS.index(op), ctypes.byref(a), ctypes.byref(b)),
           "sntrup_measure_int_peak")
    return dict(lanes_per_clk_sm=a.value, lane_ops_per_s=b.value)


def profile_read(reset: bool = True) -> dict:
    """Per kernel class: device ms (CUDA events on the launching stream), work units, algorithmic
    integer ops, launches."""
    n = len(PROFILE_CLASSES)
    ms = (ctypes.c_double * n)()
    un = (ctypes.c_double * n)()
    op = (ctypes.c_double * n)()
    la = (ctypes.c_uint64 * n)()
    _lib.sntrup_profile_read(1 if reset else 0, ms, un, op, la, n)
    return {PROFILE_CLASSES[i]: dict(ms=ms[i], units=un[i], ops=op[i], launches=la[i]) for i in range(n)}


def library_path() -> str:
    return _LIB_PATH

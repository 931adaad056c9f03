"""GPU tests of the boundary's runtime behaviour: workspace accounting and caller workspaces,
asynchronous host-output calls whose layouts change between calls, isInvertible, and the
binding's checks of caller-supplied outputs."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2106_08759_b200 as S  # noqa: E402
from inputs import synth  # noqa: E402


@pytest.mark.parametrize("param,n,B,chunk,flags", [
    (761, 65536, 1024, 32768, S.OPT_RING_STREAMS),
    (761, 5000, 64, 0, 0),
    (653, 40000, 512, 16384, S.OPT_LANES4),
    (1277, 3000, 1024, 2048, S.OPT_HOST_OUTPUT)])
def test_workspace_query_equals_reservation(param, n, B, chunk, flags):
    # sntrup_keygen_workspace_bytes reported less than a call reserved.  On a fresh
    # stream the cached workspace is allocated for exactly the queried bytes (+ the documented
    # 1/8 + 1 MiB slack), and a caller workspace of exactly the queried size is accepted.
    st = torch.cuda.Stream()
    S.release_stream_workspace(st)             # (a recycled stream handle may have a cache entry)
    need = S.keygen_workspace_bytes(param, n, B, flags, chunk)
    P = S.params(param)
    host = bool(flags & S.OPT_HOST_OUTPUT)
    kw = dict(batch_size=B, chunk_keys=chunk, flags=flags, stream=st)
    with torch.cuda.stream(st):
        ref = S.batch_keygen(param, n, 7, **kw)
    st.synchronize()
    assert S.workspace_reserved_bytes(st) == need + need // 8 + (1 << 20)
    assert (S.workspace_reserved_bytes(st, staging=True) > 0) == host
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    with torch.cuda.stream(st):
        got = S.batch_keygen(param, n, 7, workspace=ws, **kw)
    st.synchronize()
    assert torch.equal(got["pk"].cpu(), ref["pk"].cpu()) and torch.equal(got["sk"].cpu(), ref["sk"].cpu())
    with pytest.raises(S.SntrupError) as e:
        S.batch_keygen(param, n, 7, workspace=ws[:need - 256], **kw)
    assert e.value.code == S.SNTRUP_E_WORKSPACE
    S.release_stream_workspace(st)
    assert S.workspace_reserved_bytes(st) == 0 and S.workspace_reserved_bytes(st, staging=True) == 0


def test_async_host_output_alternating_layouts():
    # asynchronous host-output calls on one stream whose chunking / batch size /
    # lane count change from call to call, issued back to back without waiting: every call's bytes
    # must equal a synchronous device-output run of the same keys
    P = S.params(761)
    st = torch.cuda.Stream()
    shapes = [(16384, 512, 8192, 0), (16384, 1024, 16384, S.OPT_LANES4), (12000, 64, 4000, 0),
              (16384, 2048, 16384, S.OPT_RING_STREAMS), (9000, 512, 3000, S.OPT_LANES4)] * 2
    outs = []
    evs = []
    with torch.cuda.stream(st):
        for i, (n, B, chunk, fl) in enumerate(shapes):
            pk = torch.empty((n, P["pk_bytes"]), dtype=torch.uint8).pin_memory()
            sk = torch.empty((n, P["sk_bytes"]), dtype=torch.uint8).pin_memory()
            ev = S.Event()
            S.batch_keygen(761, n, 40 + i, batch_size=B, chunk_keys=chunk, pk_out=pk, sk_out=sk,
                           flags=S.OPT_HOST_OUTPUT | S.OPT_ASYNC | fl, done_event=ev, stream=st)
            outs.append((n, pk, sk))
            evs.append(ev)
    for ev in evs:
        ev.synchronize()
    for i, (n, pk, sk) in enumerate(outs):
        ref = S.batch_keygen(761, n, 40 + i, batch_size=256)
        torch.cuda.synchronize()
        assert torch.equal(pk, ref["pk"].cpu()) and torch.equal(sk, ref["sk"].cpu()), i


@pytest.mark.parametrize("param", [653, 761, 1277])
def test_r3_is_invertible_batch(O, param):
    # isInvertible through its own entry point: random small elements (653/1277
    # reject ~1 in 27 / 20 by the cubic factor), crafted multiples of x^3 - x - 1, and zero rows,
    # against the oracle's extended Euclid; ragged n over several trees
    P = S.params(param)
    p = P["p"]
    n = 333
    g = synth.small(n, p, P["p16"], seed=param)
    g[5, :p] = 0
    if param in (653, 1277):                   # x^3 - x - 1 divides x^p - x - 1 over GF(3) (C14)
        for r in (7, 100, 200):
            u = synth.small(1, p - 3, p - 3, seed=r)[0].astype(np.int64)
            m = np.convolve(u, np.array([-1, -1, 0, 1]))[:p]
            g[r, :p] = (((m + 1) % 3) - 1).astype(np.int8)
    ok = S.r3_is_invertible_batch(param, torch.from_numpy(g).cuda())
    okn = ok.cpu().numpy()
    for i in range(n):
        assert bool(okn[i]) == O.poly_inv(p, 3, g[i, :p])[0], i
    if param in (653, 1277):
        assert not okn[[5, 7, 100, 200]].any()


def test_binding_rejects_short_outputs():
    P = S.params(761)
    a = torch.zeros((4, P["p8"]), dtype=torch.int16, device="cuda")
    with pytest.raises(ValueError):
        S.rq_mul_batch(761, a, a, c=torch.zeros((3, P["p8"]), dtype=torch.int16, device="cuda"))
    with pytest.raises(ValueError):
        S.rq_mul_batch(761, a, a, c=torch.zeros((4, P["p8"]), dtype=torch.int32, device="cuda"))
    g = torch.zeros((4, P["p16"]), dtype=torch.int8, device="cuda")
    with pytest.raises(ValueError):
        S.r3_recip_batch(761, g, ok=torch.zeros(3, dtype=torch.uint8, device="cuda"))
    with pytest.raises(ValueError):                      # host-output keygen into device tensors
        S.batch_keygen(761, 4, 1, flags=S.OPT_HOST_OUTPUT,
                       pk_out=torch.empty((4, P["pk_bytes"]), dtype=torch.uint8, device="cuda"),
                       sk_out=torch.empty((4, P["sk_bytes"]), dtype=torch.uint8, device="cuda"))
    with pytest.raises(ValueError):                      # device keygen into a short buffer
        S.batch_keygen(761, 4, 1, pk_out=torch.empty((3, P["pk_bytes"]), dtype=torch.uint8, device="cuda"))
    # host outputs allocated by default in pinned host memory
    r = S.batch_keygen(761, 4, 1, flags=S.OPT_HOST_OUTPUT)
    assert not r["pk"].is_cuda and r["pk"].is_pinned()
    ref = S.batch_keygen(761, 4, 1)
    torch.cuda.synchronize()
    assert torch.equal(r["pk"], ref["pk"].cpu())


@pytest.mark.parametrize("param", [1013, 1277])
def test_small_factor_check_is_constant_time(param):
    # ADVICE r1 / DESIGN.md Z19: the small-factor residue test (isInvertible for factors of degree
    # <= 64) must not depend on g -- every coefficient's residue row is loaded and added under
    # masks.  Time the kernel that runs it (r3_is_invertible_batch's prepare step, profiler class
    # "other") on very sparse and on dense inputs of equal shape: a weight-dependent loop would run
    # ~50x longer on the dense rows.
    P = S.params(param)
    p, n = P["p"], 1 << 16
    dense = torch.from_numpy(synth.small(n, p, P["p16"], seed=3)).cuda()
    sparse = torch.zeros_like(dense)
    sparse[:, 0] = 1
    sparse[:, 5] = -1
    times = {}
    for name, g in (("sparse", sparse), ("dense", dense), ("sparse2", sparse), ("dense2", dense)):
        S.r3_is_invertible_batch(param, g)               # warm
        torch.cuda.synchronize()
        S.profile_enable(True)
        for _ in range(3):
            S.r3_is_invertible_batch(param, g)
        prof = S.profile_read(reset=True)
        S.profile_enable(False)
        times[name] = prof["other"]["ms"] / 3
    ts, td = min(times["sparse"], times["sparse2"]), min(times["dense"], times["dense2"])
    assert abs(td - ts) <= 0.15 * max(td, ts), times


def test_async_error_status():
    # asynchronous calls do not read their device error flags before returning; the status of the
    # last call on a stream is available afterwards (the key pool checks it per refill)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        S.batch_keygen(653, 4096, 4, batch_size=512, flags=S.OPT_ASYNC, stream=st)
    S.async_error(st)                                 # no retry-bound hit: returns quietly
    assert S._lib.sntrup_async_error(S._stream(st)) == S.SNTRUP_OK

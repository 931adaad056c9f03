"""GPU parity: every entry point of the C ABI (through the thin binding) against the oracle.

All comparisons are bit-exact (the whole path is integer arithmetic, results unique: DESIGN.md C0).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2106_08759_b200 as S  # noqa: E402
from inputs import synth  # noqa: E402

PSETS = [653, 761, 857, 953, 1013, 1277]


@pytest.fixture(params=[S.MUL_TENSOR_CORE, S.MUL_TENSOR_CORE_INT8, S.MUL_TENSOR_CORE_FP4_ALL,
                        S.MUL_TENSOR_CORE_M64, S.MUL_TENSOR_CORE_I8_SINGLE, S.MUL_TENSOR_CORE_U_FUSED,
                        S.MUL_TENSOR_CORE_PIPELINED, S.MUL_TENSOR_CORE_TMEM_A, S.MUL_TENSOR_CORE_TMEM_A64,
                        S.MUL_TENSOR_CORE_WS, S.MUL_TENSOR_CORE_TMEM_RING, S.MUL_TENSOR_CORE_TRANSPOSED, S.MUL_TENSOR_CORE_ONE_PART, S.MUL_TENSOR_CORE_3PARTS,
                        S.MUL_TENSOR_CORE_PARTS_ALL,
                        S.MUL_SCHOOLBOOK],
                ids=["tc", "tc_int8", "tc_fp4_all", "tc_m64", "tc_i8_single", "tc_u_fused", "tc_pipe",
                     "tc_tmem_a", "tc_tmem_a64", "tc_ws", "tc_tmem_ring", "tc_transposed", "tc_one_part", "tc_3parts", "tc_parts_all", "schoolbook"])
def mul_impl(request):
    """Run a test under both ring-product implementations (tcgen05 Hankel GEMM, int32 schoolbook)."""
    S.set_mul_impl(request.param)
    yield request.param
    S.set_mul_impl(S.MUL_TENSOR_CORE)


def oracle_keys(O, param, seed, idx):
    return O.keygen_many(param, seed, np.asarray(idx, dtype=np.uint64), want_polys=True)


def check_keys(O, param, seed, res, idx, offset=0):
    """Compare GPU rows (res tensors) for global indices idx (row = index - offset)."""
    P = S.params(param)
    p = P["p"]
    ref = oracle_keys(O, param, seed, idx)
    rows = np.asarray(idx) - offset
    pk = res["pk"].cpu().numpy()[rows]
    sk = res["sk"].cpu().numpy()[rows]
    bad = np.nonzero((pk != ref["pk"]).any(1) | (sk != ref["sk"]).any(1))[0]
    assert len(bad) == 0, "pk/sk mismatch at global keys %s" % list(np.asarray(idx)[bad][:10])
    if "h" in res:
        assert np.array_equal(res["h"].cpu().numpy()[rows][:, :p], ref["h"][:, :p])
        assert not res["h"].cpu().numpy()[rows][:, p:].any()
        for k in ("g", "f", "ginv"):
            got = res[k].cpu().numpy()[rows]
            assert np.array_equal(got[:, :p], ref[k][:, :p]), k
            assert not got[:, p:].any(), k + " pad"
        assert np.array_equal(res["attempts"].cpu().numpy()[rows], ref["attempts"])


# --------------------------------------------------------------------------------- keygen
def test_cfg1_all_32_keys(O, mul_impl):
    # BASELINE configs[0]: sntrup761, 32 keys, seed 1, one tree of 32
    res = S.batch_keygen(761, 32, 1, batch_size=32, debug=True, stats=True)
    torch.cuda.synchronize()
    check_keys(O, 761, 1, res, np.arange(32))
    st = res["stats"]
    # batchInv: 3(B-1) = 93 products per ring for B = 32
    assert st["r3_products"] == 93
    assert st["rq_products"] == 93 + 32           # + H = g * fbar for each key
    assert st["root_inversions"] == 2


def test_cfg1_latency_config(O):
    # configs[0] in bench.py's latency-tuned launch configuration: B = 1, ring streams
    res = S.batch_keygen(761, 32, 1, batch_size=1, flags=S.OPT_RING_STREAMS, debug=True)
    torch.cuda.synchronize()
    check_keys(O, 761, 1, res, np.arange(32))


@pytest.mark.parametrize("B", [1, 2, 8, 32, 128, 512])
def test_batch_size_invariance_ragged(O, B):
    n = 300                                       # ragged: not a multiple of B for B >= 8
    res = S.batch_keygen(761, n, 7, batch_size=B, debug=True, stats=True)
    torch.cuda.synchronize()
    check_keys(O, 761, 7, res, np.arange(n))
    full, rem = divmod(n, B)
    prods = full * 3 * (B - 1) + (3 * (rem - 1) if rem else 0)
    assert res["stats"]["r3_products"] == prods


@pytest.mark.parametrize("impl", ["jump", "jump_shared_sm", "step"])
def test_keygen_root_impls(O, impl):
    # keygen with each root-inversion implementation forced (the automatic policy runs per-step
    # roots inside keygen): ragged trees, both rings' roots on their own streams, and configs[0]
    m = {"jump": S.ROOT_JUMP, "jump_shared_sm": S.ROOT_JUMP | S.ROOT_SHARED_SM, "step": S.ROOT_STEP}[impl]
    try:
        S.set_root_impl(m)
        res = S.batch_keygen(761, 300, 7, batch_size=8, debug=True, flags=S.OPT_RING_STREAMS)
        lat = S.batch_keygen(761, 32, 1, batch_size=1, flags=S.OPT_RING_STREAMS, debug=True)
        torch.cuda.synchronize()
    finally:
        S.set_root_impl(S.ROOT_AUTO)
    check_keys(O, 761, 7, res, np.arange(300))
    check_keys(O, 761, 1, lat, np.arange(32))


def test_graph_mode_configs0(O):
    # SNTRUP_OPT_GRAPH: first call of a shape runs and captures, later calls replay with the seed
    # and first key index patched in; the stream's workspace release drops the graph (rebuilt)
    P = S.params(761)
    s = torch.cuda.Stream()
    pk = torch.empty((32, P["pk_bytes"]), dtype=torch.uint8, device="cuda")
    sk = torch.empty((32, P["sk_bytes"]), dtype=torch.uint8, device="cuda")
    fl = S.OPT_RING_STREAMS | S.OPT_GRAPH
    for seed, first in ((1, 0), (1, 0), (9, 0), (9, 1000), (3, 77)):
        S.batch_keygen(761, 32, seed, batch_size=1, first_key_index=first, pk_out=pk, sk_out=sk, flags=fl,
                       stream=s)
        s.synchronize()
        ref = oracle_keys(O, 761, seed, np.arange(first, first + 32))
        assert np.array_equal(pk.cpu().numpy(), ref["pk"]) and np.array_equal(sk.cpu().numpy(), ref["sk"]), (seed, first)
    S.release_stream_workspace(s)
    S.batch_keygen(761, 32, 5, batch_size=1, pk_out=pk, sk_out=sk, flags=fl, stream=s)
    s.synchronize()
    ref = oracle_keys(O, 761, 5, np.arange(32))
    assert np.array_equal(pk.cpu().numpy(), ref["pk"]) and np.array_equal(sk.cpu().numpy(), ref["sk"])


def test_graph_mode_trees_and_repair(O):
    # a graph with product trees, several chunks and the repair kernel (653 draws non-invertible
    # g often enough with the small test off), replayed with new seeds
    P = S.params(653)
    s = torch.cuda.Stream()
    n = 300
    pk = torch.empty((n, P["pk_bytes"]), dtype=torch.uint8, device="cuda")
    sk = torch.empty((n, P["sk_bytes"]), dtype=torch.uint8, device="cuda")
    fl = S.OPT_RING_STREAMS | S.OPT_GRAPH | S.OPT_NO_SMALL_CHECK
    for seed, first in ((4, 0), (4, 0), (6, 300), (8, 12345)):
        S.batch_keygen(653, n, seed, batch_size=16, chunk_keys=128, first_key_index=first, pk_out=pk, sk_out=sk,
                       flags=fl, stream=s)
        s.synchronize()
        ref = oracle_keys(O, 653, seed, np.arange(first, first + n))
        assert np.array_equal(pk.cpu().numpy(), ref["pk"]) and np.array_equal(sk.cpu().numpy(), ref["sk"]), (seed, first)


def test_graph_cache_is_bounded(O):
    # a graph is cached per call shape including the output pointers: more distinct output buffers
    # than the cache holds (32) evict the least recently used graphs; evicted shapes are rebuilt
    # and every call stays exact
    P = S.params(761)
    s = torch.cuda.Stream()
    fl = S.OPT_RING_STREAMS | S.OPT_GRAPH
    bufs = [(torch.empty((8, P["pk_bytes"]), dtype=torch.uint8, device="cuda"),
             torch.empty((8, P["sk_bytes"]), dtype=torch.uint8, device="cuda")) for _ in range(36)]
    ref = {seed: oracle_keys(O, 761, seed, np.arange(8)) for seed in (1, 2)}
    for seed in (1, 2):                          # second pass: the first buffers were evicted
        for pk, sk in bufs:
            S.batch_keygen(761, 8, seed, batch_size=1, pk_out=pk, sk_out=sk, flags=fl, stream=s)
        s.synchronize()
        for pk, sk in bufs:
            assert np.array_equal(pk.cpu().numpy(), ref[seed]["pk"])
            assert np.array_equal(sk.cpu().numpy(), ref[seed]["sk"])
    S.release_stream_workspace(s)


def test_attempts_only_output(O):
    # attempts=True: only the per-key number of g draws (bench.py's rejection totals)
    res = S.batch_keygen(653, 400, 4, batch_size=16, attempts=True)
    torch.cuda.synchronize()
    assert set(res) == {"pk", "sk", "attempts"}
    ref = oracle_keys(O, 653, 4, np.arange(400))
    assert np.array_equal(res["attempts"].cpu().numpy(), ref["attempts"])
    assert int(res["attempts"].sum()) > 400      # 653 rejects ~3.7% of the draws


def test_graph_mode_rejects_synchronous_host_outputs():
    # graph replay with host outputs is the asynchronous serving mode only: without OPT_ASYNC or a
    # done event (or on the default stream) the call is refused
    P = S.params(761)
    s = torch.cuda.Stream()
    pk = torch.empty((32, P["pk_bytes"]), dtype=torch.uint8).pin_memory()
    sk = torch.empty((32, P["sk_bytes"]), dtype=torch.uint8).pin_memory()
    with pytest.raises((S.SntrupError, ValueError)):
        S.batch_keygen(761, 32, 1, pk_out=pk, sk_out=sk, flags=S.OPT_GRAPH | S.OPT_HOST_OUTPUT, stream=s)
    with pytest.raises((S.SntrupError, ValueError)):
        S.batch_keygen(761, 32, 1, pk_out=pk, sk_out=sk, stream=s,
                       flags=S.OPT_GRAPH | S.OPT_HOST_OUTPUT | S.OPT_ASYNC)          # no done_event
    with pytest.raises((S.SntrupError, ValueError)):
        S.batch_keygen(761, 32, 1, pk_out=pk, sk_out=sk, done_event=S.Event(),
                       flags=S.OPT_GRAPH | S.OPT_HOST_OUTPUT | S.OPT_ASYNC)          # default stream


@pytest.mark.parametrize("n,B,chunk", [(600, 16, 128), (40000, 512, 16384)])
def test_graph_host_output_serving_loop(O, n, B, chunk):
    # SNTRUP_OPT_GRAPH | SNTRUP_OPT_HOST_OUTPUT | SNTRUP_OPT_ASYNC: graph replay into two device
    # output sets, D2H copies on a copy stream, done event after the last byte.  Back-to-back
    # calls with different seeds / first indices into two alternating pinned buffer sets (the
    # serving loop of bench.py's e2e): each call's bytes equal the plain device-output call's, and
    # the oracle's on a sample; a plain host-output call in between (other staging layout) and a
    # workspace release do not disturb it.
    P = S.params(761)
    s = torch.cuda.Stream()
    fl = S.OPT_RING_STREAMS | S.OPT_GRAPH | S.OPT_HOST_OUTPUT | S.OPT_ASYNC
    pk = [torch.empty((n, P["pk_bytes"]), dtype=torch.uint8).pin_memory() for _ in range(2)]
    sk = [torch.empty((n, P["sk_bytes"]), dtype=torch.uint8).pin_memory() for _ in range(2)]
    evs = [S.Event(), S.Event()]
    calls = [(31, 0), (32, 5), (31, 0), (33, n), (34, 7), (31, 0)]
    got = []
    for k, (seed, first) in enumerate(calls):
        if k >= 2:
            evs[k % 2].synchronize()
            got.append((pk[k % 2].clone(), sk[k % 2].clone()))
        if k == 3:                                  # a plain host-output call on the same stream
            S.batch_keygen(761, 64, 9, batch_size=16, stream=s, flags=S.OPT_HOST_OUTPUT)
        if k == 4:
            evs[(k - 1) % 2].synchronize()
            S.release_stream_workspace(s)           # drops the graphs and the staging
        S.batch_keygen(761, n, seed, first_key_index=first, batch_size=B, chunk_keys=chunk, pk_out=pk[k % 2],
                       sk_out=sk[k % 2], flags=fl, stream=s, done_event=evs[k % 2])
    for k in (len(calls) - 2, len(calls) - 1):
        evs[k % 2].synchronize()
        got.append((pk[k % 2].clone(), sk[k % 2].clone()))
    S.async_error(s)                                # raises if a lane hit the g retry bound
    idx = np.unique(np.concatenate([np.arange(0, n, 97), np.arange(n - 4, n)]))
    for (seed, first), (gpk, gsk) in zip(calls, got):
        ref = S.batch_keygen(761, n, seed, first_key_index=first, batch_size=B, chunk_keys=chunk,
                             flags=S.OPT_RING_STREAMS)
        torch.cuda.synchronize()
        assert torch.equal(gpk, ref["pk"].cpu()) and torch.equal(gsk, ref["sk"].cpu()), (seed, first)
        r = oracle_keys(O, 761, seed, first + idx)
        assert np.array_equal(gpk.numpy()[idx], r["pk"]) and np.array_equal(gsk.numpy()[idx], r["sk"])
    S.release_stream_workspace(s)


def test_chunking_and_first_index(O):
    n, first = 200, 1000
    res = S.batch_keygen(761, n, 3, batch_size=16, chunk_keys=48, first_key_index=first, debug=True)
    torch.cuda.synchronize()
    check_keys(O, 761, 3, res, np.arange(first, first + n), offset=first)


@pytest.mark.parametrize("param,seed", [(653, 4), (761, 2), (857, 4), (953, 4), (1013, 4), (1277, 5)])
def test_param_sets(O, param, seed, mul_impl):
    n = 160                                       # covers 653/1277 keys with two g draws
    res = S.batch_keygen(param, n, seed, batch_size=32, debug=True)
    torch.cuda.synchronize()
    check_keys(O, param, seed, res, np.arange(n))


@pytest.mark.parametrize("param,seed", [(653, 4), (1277, 5), (1013, 4)])
def test_repair_path_without_small_check(O, param, seed):
    # Disable the small-factor test: every non-invertible g reaches the product tree, fails the
    # root divstep, and the tree's keys are repaired per key.  Output must be unchanged.
    n = 160
    res = S.batch_keygen(param, n, seed, batch_size=16, debug=True, stats=True,
                         flags=S.OPT_NO_SMALL_CHECK)
    torch.cuda.synchronize()
    check_keys(O, param, seed, res, np.arange(n))
    assert res["stats"]["keys_repaired"] > 0


@pytest.mark.parametrize("flags", [0, S.OPT_FORCE_SMALL_CHECK, S.OPT_NO_SMALL_CHECK, S.OPT_RING_STREAMS,
                                   S.OPT_RING_STREAMS | S.OPT_NO_SMALL_CHECK])
def test_small_check_policies_761(O, flags):
    # the sampler's small-factor test is skipped by default for 761 (3^-19 per draw); forcing it
    # or disabling it must not change a byte
    n = 300
    res = S.batch_keygen(761, n, 17, batch_size=64, debug=True, flags=flags)
    torch.cuda.synchronize()
    check_keys(O, 761, 17, res, np.arange(n))


@pytest.mark.parametrize("flags", [0, S.OPT_RING_STREAMS, S.OPT_LANES4, S.OPT_LANES4 | S.OPT_RING_STREAMS])
def test_host_output(O, flags):
    # host outputs through the staging buffers / copy streams, 1, 2 and 4 lanes (4 chunks of 32
    # keys -> every lane reuses its staging buffer)
    P = S.params(761)
    n = 100 if not flags else 260
    pk = torch.empty((n, P["pk_bytes"]), dtype=torch.uint8).pin_memory()
    sk = torch.empty((n, P["sk_bytes"]), dtype=torch.uint8).pin_memory()
    S.batch_keygen(761, n, 11, pk_out=pk, sk_out=sk, flags=S.OPT_HOST_OUTPUT | flags, chunk_keys=32)
    ref = oracle_keys(O, 761, 11, np.arange(n))
    assert np.array_equal(pk.numpy(), ref["pk"]) and np.array_equal(sk.numpy(), ref["sk"])


@pytest.mark.parametrize("B,chunk,flags", [(64, 2048, 0), (1024, 32768, S.OPT_RING_STREAMS),
                                            (1024, 32768, S.OPT_RING_STREAMS | S.OPT_LANE_PRIORITY),
                                            (1024, 40960, S.OPT_RING_STREAMS | S.OPT_STAGGER | S.OPT_LANE_PRIORITY),
                                            (1024, 24576, S.OPT_RING_STREAMS | S.OPT_STAGGER | S.OPT_LANES4),
                                            (512, 16384, S.OPT_LANES4 | S.OPT_LANE_PRIORITY)])
def test_host_output_grouped_tail(O, B, chunk, flags):
    # host outputs with enough trees per chunk for the grouped tail (bottom down-sweep levels, h and
    # the pk encode per group of subtrees): byte-identical to the device-output call, and to the
    # oracle on a sample (first/last keys of every chunk, every 61st key)
    P = S.params(761)
    n = 65536 if B >= 512 else 4096
    pk = torch.empty((n, P["pk_bytes"]), dtype=torch.uint8).pin_memory()
    sk = torch.empty((n, P["sk_bytes"]), dtype=torch.uint8).pin_memory()
    S.batch_keygen(761, n, 23, batch_size=B, pk_out=pk, sk_out=sk, flags=S.OPT_HOST_OUTPUT | flags,
                   chunk_keys=chunk)
    ref = S.batch_keygen(761, n, 23, batch_size=B, chunk_keys=chunk)
    torch.cuda.synchronize()
    assert torch.equal(pk, ref["pk"].cpu()) and torch.equal(sk, ref["sk"].cpu())
    idx = np.unique(np.concatenate([np.arange(0, n, 61)] +
                                   [np.arange(c, min(c + 4, n)) for c in range(0, n, chunk)] +
                                   [np.arange(max(c - 4, 0), c) for c in range(chunk, n + 1, chunk)]))
    r = oracle_keys(O, 761, 23, idx)
    assert np.array_equal(pk.numpy()[idx], r["pk"]) and np.array_equal(sk.numpy()[idx], r["sk"])


@pytest.mark.parametrize("top,cap,flags", [(1024, 0, S.OPT_RING_STREAMS), (1024, 4, S.OPT_RING_STREAMS),
                                           (256, 8, S.OPT_RING_STREAMS | S.OPT_STAGGER),
                                           (0, 16, S.OPT_RING_STREAMS),
                                           (1 << 20, 2, S.OPT_RING_STREAMS | S.OPT_LANES4)])
def test_tree_top_scheduling_knob(O, top, cap, flags):
    # sntrup_set_sched: tree tops and roots on high-priority companion streams, ring-product CTAs
    # retiring after `cap` items -- a scheduling change only: byte-identical to the default call
    # (host outputs too), and to the oracle on a sample; (1 << 20: every product launch routed)
    n = 40000
    P = S.params(761)
    ref = S.batch_keygen(761, n, 29, batch_size=512, chunk_keys=16384, flags=flags)
    torch.cuda.synchronize()
    S.set_sched(top, cap)
    try:
        res = S.batch_keygen(761, n, 29, batch_size=512, chunk_keys=16384, flags=flags)
        pk = torch.empty((n, P["pk_bytes"]), dtype=torch.uint8).pin_memory()
        sk = torch.empty((n, P["sk_bytes"]), dtype=torch.uint8).pin_memory()
        S.batch_keygen(761, n, 29, batch_size=512, chunk_keys=16384, pk_out=pk, sk_out=sk,
                       flags=flags | S.OPT_HOST_OUTPUT)
        torch.cuda.synchronize()
    finally:
        S.set_sched(0, 0)
    assert torch.equal(res["pk"], ref["pk"]) and torch.equal(res["sk"], ref["sk"])
    assert torch.equal(pk, ref["pk"].cpu()) and torch.equal(sk, ref["sk"].cpu())
    idx = np.unique(np.concatenate([np.arange(0, n, 211), np.arange(n - 8, n), np.arange(16380, 16390)]))
    check_keys(O, 761, 29, res, idx)


def test_cfg2_full_size_sampled(O):
    # BASELINE configs[1]: 65,536 keys, seed 2, in the launch configuration bench.py times;
    # compared on a sample the oracle computes one by one: first and last trees, every 97th key.
    n = 65536
    for B, chunk, fl in ((32, 0, 0), (128, 0, 0), (2048, 0, 0), (1024, 32768, 0),
                         (512, 65536, S.OPT_RING_STREAMS), (512, 16384, S.OPT_LANES4),
                         (1024, 16384, S.OPT_LANES4 | S.OPT_RING_STREAMS),
                         (1024, 32768, S.OPT_RING_STREAMS)):                # last: bench.py's config
        res = S.batch_keygen(761, n, 2, batch_size=B, chunk_keys=chunk, flags=fl)
        torch.cuda.synchronize()
        idx = np.unique(np.concatenate([np.arange(0, 128), np.arange(n - 128, n), np.arange(0, n, 97)]))
        check_keys(O, 761, 2, res, idx)
        if B == 32:
            first = (res["pk"].clone(), res["sk"].clone())
        else:
            assert torch.equal(first[0], res["pk"]) and torch.equal(first[1], res["sk"])


def _rejection_bound(param, att):
    """Total extra g draws vs the per-draw rejection probability (golden): per key the
    extra draws are geometric with mean P/(1-P) and variance P/(1-P)^2; accept within 6 sigma."""
    import json
    import os
    rates = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "rejection_rates.json")))
    P = rates["p_reject_per_draw"][str(param)]
    n = len(att)
    extra = float((att.astype(np.int64) - 1).sum())
    mean, sd = n * P / (1 - P), (n * P) ** 0.5 / (1 - P)
    assert abs(extra - mean) <= 6 * sd + 1, (param, extra, mean, sd)


@pytest.mark.parametrize("param", [653, 857, 953, 1013])
def test_cfg4_full_size_sampled(O, param):
    # BASELINE configs[3]: 65,536 keys per set, seed 4.  Compared with the oracle on every key
    # that needed more than one g draw, the first and last trees, and every 97th key.
    n = 65536
    res = S.batch_keygen(param, n, 4, batch_size=1024, chunk_keys=32768, flags=S.OPT_RING_STREAMS,
                         debug=True)                       # bench.py's configs[3] launch configuration
    torch.cuda.synchronize()
    att = res["attempts"].cpu().numpy()
    assert att.min() >= 1
    _rejection_bound(param, att)
    rej = np.nonzero(att > 1)[0]
    idx = np.unique(np.concatenate([np.arange(0, 64), np.arange(n - 64, n), np.arange(0, n, 97), rej]))
    check_keys(O, param, 4, res, idx)


def test_cfg5_full_size_sampled(O):
    # BASELINE configs[4]: sntrup1277, 1,048,576 keys, seed 5, 1024 keys per product tree,
    # streamed in 65,536-key chunks.  Sampled: first/last chunk edges, every 509th key, every
    # 32nd key that needed more than one g draw; rejection total vs the per-draw probability.
    n = 1 << 20
    res = S.batch_keygen(1277, n, 5, batch_size=1024, chunk_keys=65536, flags=S.OPT_RING_STREAMS,
                         debug=True)
    torch.cuda.synchronize()
    att = res["attempts"].cpu().numpy()
    assert att.min() >= 1
    _rejection_bound(1277, att)
    rej = np.nonzero(att > 1)[0]
    idx = np.unique(np.concatenate([np.arange(0, 64), np.arange(65536 - 32, 65536 + 32),
                                    np.arange(n - 64, n), np.arange(0, n, 509), rej[::32]]))
    check_keys(O, 1277, 5, res, idx)


# --------------------------------------------------------------------------------- KEM core
@pytest.mark.parametrize("param", PSETS)
def test_kem_core_parity_and_roundtrip(O, param, mul_impl):
    # r from the encapsulation stream domain, c = Round(h r), decap recovers r;
    # every output byte against the oracle (encap_core / decap_core / short_from_words)
    P = S.params(param)
    p, q, w = P["p"], P["q"], P["w"]
    n, seed = 40, 23
    keys = S.batch_keygen(param, n, seed, batch_size=8, debug=True)
    r = S.sample_short_batch(param, n, seed, first_key_index=0)
    c = S.encap_core_batch(param, keys["h"], r)
    r2, ok = S.decap_core_batch(param, keys["f"], keys["ginv"], c)
    # a tampered ciphertext row and an all-zero one
    ct = c.clone()
    ct[1, 5] += 3
    ct[2] = 0
    r3, ok3 = S.decap_core_batch(param, keys["f"], keys["ginv"], ct)
    torch.cuda.synchronize()
    h, f, gi = keys["h"].cpu().numpy(), keys["f"].cpu().numpy(), keys["ginv"].cpu().numpy()
    rr, cc, rr2 = r.cpu().numpy(), c.cpu().numpy(), r2.cpu().numpy()
    for i in range(n):
        ref_r = O.short_from_words(p, w, O.stream_words(seed, i, S.ENC_DOMAIN, p))
        assert np.array_equal(rr[i, :p], ref_r) and not rr[i, p:].any()
        ref_c = O.encap_core(p, q, h[i, :p], ref_r)
        assert np.array_equal(cc[i, :p], ref_c) and not cc[i, p:].any()
        assert ok[i] == 1 and np.array_equal(rr2[i, :p], ref_r) and not rr2[i, p:].any()
    ctn, r3n, ok3n = ct.cpu().numpy(), r3.cpu().numpy(), ok3.cpu().numpy()
    for i in (1, 2):
        ref_ok, ref_r3 = O.decap_core(p, q, w, f[i, :p], gi[i, :p], ctn[i, :p])
        assert bool(ok3n[i]) == ref_ok and np.array_equal(r3n[i, :p], ref_r3)
    assert ok3n[2] == 0


# --------------------------------------------------------------------------------- key pool
def test_key_pool_hands_out_oracle_keys_in_order(O):
    # engNTRU batch_lib analogue: consecutive global key indices from first_key_index,
    # each pair byte-identical to the oracle's; refills happen ahead of the consumer
    import time
    pool = S.KeyPool(761, seed=21, capacity=256, batch_keys=64, batch_size=32, first_key_index=1000)
    got = [pool.take() for _ in range(300)]                  # tight loop: crosses several refills
    st = pool.stats()
    idx = np.array([g[2] for g in got], dtype=np.uint64)
    assert np.array_equal(idx, np.arange(1000, 1300, dtype=np.uint64))
    ref = oracle_keys(O, 761, 21, idx)
    for i, (pk, sk, _) in enumerate(got):
        assert pk == ref["pk"][i].tobytes() and sk == ref["sk"][i].tobytes(), i
    assert st["taken"] == 300 and st["generated"] >= 300 and st["waits"] >= 1
    # a paced consumer (1 ms between takes, like sporadic handshakes) never waits for the GPU:
    # each 64-key refill completes long before the ring's ready half is used up
    w0 = st["waits"]
    for _ in range(200):
        time.sleep(0.001)
        pool.take()
    assert pool.stats()["waits"] == w0
    pool.close()


def test_key_pool_arguments():
    with pytest.raises(S.SntrupError):
        S.KeyPool(761, seed=1, capacity=100, batch_keys=64)      # not a multiple of the batch
    with pytest.raises(S.SntrupError):
        S.KeyPool(700, seed=1, capacity=128, batch_keys=64)      # unknown parameter set


# --------------------------------------------------------------------------------- ring ops
def edge_cases(p, p8, q):
    qh = (q - 1) // 2
    rows = []
    for v in ("zero", "one", "x", "xp1", "max", "min", "alt"):
        r = np.zeros(p8, np.int16)
        if v == "one": r[0] = 1
        if v == "x": r[1] = 1
        if v == "xp1": r[p - 1] = 1
        if v == "max": r[:p] = qh
        if v == "min": r[:p] = -qh
        if v == "alt": r[:p:2] = qh; r[1:p:2] = -qh
        rows.append(r)
    return np.stack(rows)


@pytest.mark.parametrize("param", PSETS)
def test_rq_mul(O, param, mul_impl):
    P = S.params(param)
    p, q, p8 = P["p"], P["q"], P["p8"]
    a = synth.uniform_rq(203, p, q, p8, seed=1)
    b = np.concatenate([synth.uniform_rq(100, p, q, p8, seed=2),
                        synth.ternary(103, p, P["w"], p8, seed=3)])
    e = edge_cases(p, p8, q)
    A = np.concatenate([a, np.repeat(e, len(e), 0)])
    Bm = np.concatenate([b, np.tile(e, (len(e), 1))])
    c = S.rq_mul_batch(param, torch.from_numpy(A).cuda(), torch.from_numpy(Bm).cuda()).cpu().numpy()
    ref = O.mul_many(p, q, A, Bm)
    assert np.array_equal(c, ref)


@pytest.mark.parametrize("param", PSETS)
def test_rq_mul_small(O, param, mul_impl):
    # configs[2] shape: one operand uniform in [-(q-1)/2, (q-1)/2], the other ternary of weight w
    P = S.params(param)
    p, q, p8, p16 = P["p"], P["q"], P["p8"], P["p16"]
    a = synth.uniform_rq(150, p, q, p8, seed=11)
    b = np.concatenate([synth.ternary(100, p, P["w"], p16, seed=12, dtype=np.int8),
                        synth.small(50, p, p16, seed=13)])
    qh = (q - 1) // 2
    a[0, :p] = qh
    a[1, :p] = -qh
    b[0, :p] = 1
    b[1, :p] = -1
    b[2] = 0
    c = S.rq_mul_small_batch(param, torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
    ref = O.mul_many(p, q, a, np.pad(b[:, :p].astype(np.int16), ((0, 0), (0, p8 - p))))
    assert np.array_equal(c, ref)


@pytest.mark.parametrize("param", PSETS)
def test_r3_mul(O, param, mul_impl):
    P = S.params(param)
    p, p16 = P["p"], P["p16"]
    a = synth.small(150, p, p16, seed=4)
    b = synth.small(150, p, p16, seed=5)
    c = S.r3_mul_batch(param, torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
    ref = O.mul_many(p, 3, a.astype(np.int16), b.astype(np.int16))
    assert np.array_equal(c.astype(np.int16), ref)


@pytest.mark.parametrize("param", PSETS)
@pytest.mark.parametrize("B", [1, 4, 32])
def test_rq_recip(O, param, B):
    P = S.params(param)
    p, q, p8 = P["p"], P["q"], P["p8"]
    a = synth.uniform_rq(77, p, q, p8, seed=6)
    a[3] = 0
    a[3, 0] = 1
    out = S.rq_recip_batch(param, torch.from_numpy(a).cuda(), batch_size=B).cpu().numpy()
    for i in range(len(a)):
        ok, inv = O.poly_inv(p, q, a[i, :p])
        assert ok and np.array_equal(out[i, :p], inv) and not out[i, p:].any()


def rq_root_cases(p, q, p8, n, seed):
    """Uniform rows plus the shapes that drive the divstep decisions to their extremes: 1, x^k
    (long runs of g_0 = 0 in the reversed input, delta climbing), 1 + x^(p-1), sparse rows and a
    row of all (q-1)/2."""
    a = synth.uniform_rq(n, p, q, p8, seed=seed)
    rng = np.random.default_rng(seed)
    a[0] = 0; a[0, 0] = 1
    a[1] = 0; a[1, p - 1] = 1
    a[2] = 0; a[2, 1] = -1
    a[3] = 0; a[3, 0] = 1; a[3, p - 1] = 1
    a[4] = 0; a[4, :p] = (q - 1) // 2
    for i in range(5, 12):
        a[i] = 0
        idx = rng.choice(p, size=1 + i % 4, replace=False)
        a[i, idx] = rng.integers(-(q - 1) // 2, (q + 1) // 2, size=len(idx))
        if not a[i].any():
            a[i, 0] = 1
    return a


@pytest.mark.parametrize("param", PSETS)
def test_rq_root_jump_vs_step(O, param):
    # the jump-divstep root (default) and the one-step-per-barrier root against the oracle's
    # Euclid inversion, one chain per row (B = 1)
    P = S.params(param)
    p, q, p8 = P["p"], P["q"], P["p8"]
    a = rq_root_cases(p, q, p8, 40, seed=param)
    outs = {}
    try:
        for impl in (S.ROOT_JUMP, S.ROOT_STEP):
            S.set_root_impl(impl)
            outs[impl] = S.rq_recip_batch(param, torch.from_numpy(a).cuda(), batch_size=1).cpu().numpy()
    finally:
        S.set_root_impl(S.ROOT_AUTO)
    for i in range(len(a)):
        ok, inv = O.poly_inv(p, q, a[i, :p])
        assert ok
        assert np.array_equal(outs[S.ROOT_JUMP][i, :p], inv), i
        assert not outs[S.ROOT_JUMP][i, p:].any()
    assert np.array_equal(outs[S.ROOT_JUMP], outs[S.ROOT_STEP])


@pytest.mark.parametrize("kind,p,q,stride", [(0, 383, 3, 384), (1, 383, 4591, 384), (2, 255, 3, 256),
                                             (3, 257, 3, 272)])
def test_probe_split_products(O, kind, p, q, stride):
    # the split-multiplier probes time real products: p' = 383 (Karatsuba halves), 255 / 257 (the
    # 5-way R/3 split) against the oracle's schoolbook product mod x^p' - x - 1
    n = 300
    if q == 3:
        a = synth.small(n, p, stride, seed=kind + 1)
        b = synth.small(n, p, stride, seed=kind + 2)
    else:
        a = synth.uniform_rq(n, p, q, stride, seed=kind + 1)
        b = synth.uniform_rq(n, p, q, stride, seed=kind + 2)
    c = S.probe_half_mul(kind, torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(),
                         torch.empty((n, stride), dtype=torch.int8 if q == 3 else torch.int16, device="cuda"))
    ref = O.mul_many(p, q, a[:, :p].astype(np.int16), b[:, :p].astype(np.int16))
    assert np.array_equal(c.cpu().numpy()[:, :p].astype(np.int16), ref[:, :p])


def test_rq_recip_zero_reports_index():
    P = S.params(761)
    a = synth.uniform_rq(50, 761, 4591, P["p8"], seed=7)
    a[17] = 0
    a[31] = 0
    with pytest.raises(S.SntrupError) as ei:
        S.rq_recip_batch(761, torch.from_numpy(a).cuda())
    assert ei.value.code == S.SNTRUP_E_NOT_INVERTIBLE and ei.value.bad_index == 17


def crafted_r3(O, p, p16, n, seed):
    """Random small elements plus multiples of x^3-x-1 (p = 653/1277) or of the degree-19 /
    big factors via gcd structure (multiples of g(x) = gcd) and the zero element."""
    g = synth.small(n, p, p16, seed=seed)
    rng = np.random.default_rng(seed)
    g[0] = 0
    if p in (653, 1277):
        cubic = np.array([-1, -1, 0, 1])
        for i in range(1, 6):
            u = rng.integers(-1, 2, size=p - 3)
            m = np.convolve(cubic, u)[:p]
            g[i, :p] = ((m + 1) % 3) - 1
    return g


@pytest.mark.parametrize("param", [653, 761, 1277, 953])
@pytest.mark.parametrize("B", [1, 8, 32])
def test_r3_recip(O, param, B):
    P = S.params(param)
    p, p16 = P["p"], P["p16"]
    g = crafted_r3(O, p, p16, 90, seed=param + B)
    out, ok = S.r3_recip_batch(param, torch.from_numpy(g).cuda(), batch_size=B)
    out, ok = out.cpu().numpy(), ok.cpu().numpy()
    for i in range(len(g)):
        rok, inv = O.poly_inv(p, 3, g[i, :p])
        assert bool(ok[i]) == rok, i
        assert np.array_equal(out[i, :p], inv if rok else np.zeros(p)), i
        assert not out[i, p:].any()


@pytest.mark.parametrize("param", PSETS)
def test_r3_root_jump_vs_step(O, param):
    # R/3 roots one chain per row (B = 1): jump-divsteps (default) and the bitsliced one-step warp
    # against the oracle's Euclid inversion, non-invertible rows included
    P = S.params(param)
    p, p16 = P["p"], P["p16"]
    g = crafted_r3(O, p, p16, 40, seed=param + 7)
    g[7] = 0; g[7, p - 1] = 1                     # x^(p-1): long run of g_0 = 0 in the reversed input
    g[8] = 0; g[8, 0] = -1
    outs = {}
    try:
        for impl in (S.ROOT_JUMP, S.ROOT_STEP):
            S.set_root_impl(impl)
            o, ok = S.r3_recip_batch(param, torch.from_numpy(g).cuda(), batch_size=1)
            outs[impl] = (o.cpu().numpy(), ok.cpu().numpy())
    finally:
        S.set_root_impl(S.ROOT_AUTO)
    out, ok = outs[S.ROOT_JUMP]
    for i in range(len(g)):
        rok, inv = O.poly_inv(p, 3, g[i, :p])
        assert bool(ok[i]) == rok, i
        assert np.array_equal(out[i, :p], inv if rok else np.zeros(p)), i
        assert not out[i, p:].any()
    assert np.array_equal(outs[S.ROOT_JUMP][0], outs[S.ROOT_STEP][0])
    assert np.array_equal(outs[S.ROOT_JUMP][1], outs[S.ROOT_STEP][1])


def test_r3_recip_big_factor_multiple(O):
    # a multiple of the degree-60 factor of x^761-x-1 (not covered by... any small test that
    # skips it) must still be reported non-invertible, and its tree-mates still inverted.
    import sys, os
    sys.path.insert(0, os.path.dirname(__file__))
    import polytools as PT
    comps, rest = PT.ddf_degrees(761, 3, 60)
    P = S.params(761)
    g = synth.small(64, 761, P["p16"], seed=9)
    rng = np.random.default_rng(3)
    for i, fac in ((5, comps[60]), (40, rest)):
        u = rng.integers(0, 3, size=761)
        m = PT.fold_reduce(np.convolve(np.mod(fac, 3), u), 761, 3)
        g[i, :761] = PT.center(m, 3)
    out, ok = S.r3_recip_batch(761, torch.from_numpy(g).cuda(), batch_size=32)
    out, ok = out.cpu().numpy(), ok.cpu().numpy()
    assert not ok[5] and not ok[40]
    for i in range(64):
        rok, inv = O.poly_inv(761, 3, g[i, :761])
        assert bool(ok[i]) == rok and np.array_equal(out[i, :761], inv if rok else np.zeros(761))


@pytest.mark.parametrize("param", PSETS)
def test_rq_encode(O, param):
    P = S.params(param)
    p, q, p8 = P["p"], P["q"], P["p8"]
    h = np.concatenate([synth.uniform_rq(40, p, q, p8, seed=10), edge_cases(p, p8, q)])
    pk = S.rq_encode_batch(param, torch.from_numpy(h).cuda()).cpu().numpy()
    for i in range(len(h)):
        assert pk[i].tobytes() == O.rq_encode(p, q, h[i, :p])


@pytest.mark.parametrize("param", [653, 761, 1277])
def test_full_sk_matches_oracle(O, param):
    # full-size secret keys (reading Z24) of a batch, byte-identical to the oracle's, every row;
    # sizes = App. D pair storage minus pk
    n = 300
    res = S.batch_keygen(param, n, 31, first_key_index=1000, batch_size=64)
    full = S.full_sk_batch(param, 31, res["pk"], res["sk"], first_key_index=1000)
    torch.cuda.synchronize()
    assert full.shape[1] == O.full_sk_bytes(param)
    pk, sk, fu = res["pk"].cpu().numpy(), res["sk"].cpu().numpy(), full.cpu().numpy()
    for i in range(n):
        assert fu[i].tobytes() == O.full_sk(param, 31, 1000 + i, pk[i].tobytes(), sk[i].tobytes()), i


def test_concurrent_host_threads(O):
    # calls from several host threads at once (keygen on one stream, ring products on others) are
    # serialised where they share launcher state and stay exact
    import threading
    P = S.params(761)
    rng = np.random.default_rng(5)
    a = torch.from_numpy(rng.integers(-2295, 2296, (64, P["p8"]), dtype=np.int16)).cuda()
    b = torch.from_numpy(rng.integers(-2295, 2296, (64, P["p8"]), dtype=np.int16)).cuda()
    a[:, 761:] = 0
    b[:, 761:] = 0
    ref_c = O.mul_many(761, 4591, a.cpu().numpy(), b.cpu().numpy())
    out, errs = {}, []

    def keygen():
        try:
            st = torch.cuda.Stream()
            out["k"] = S.batch_keygen(761, 200, 13, batch_size=32, stream=st)
            st.synchronize()
        except Exception as e:          # pragma: no cover
            errs.append(e)

    def mul(i):
        try:
            st = torch.cuda.Stream()
            c = torch.empty_like(a)
            for _ in range(20):
                S.rq_mul_batch(761, a, b, c, stream=st)
            st.synchronize()
            out["c%d" % i] = c
        except Exception as e:          # pragma: no cover
            errs.append(e)

    ts = [threading.Thread(target=keygen)] + [threading.Thread(target=mul, args=(i,)) for i in range(3)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    torch.cuda.synchronize()
    assert not errs, errs
    for i in range(3):
        assert np.array_equal(out["c%d" % i].cpu().numpy(), ref_c)
    check_keys(O, 761, 13, out["k"], np.arange(200))


@pytest.mark.parametrize("n,B,chunk,flags", [(1, 1, 0, 0), (1, 4096, 0, 0), (2, 4096, 0, 0), (3, 2, 0, 0),
                                            (31, 32, 0, 0), (33, 32, 0, 0), (33, 32, 16, 0),
                                            (129, 64, 64, 0), (129, 64, 64, 2 | 16 | 32)])
def test_edge_sizes(O, n, B, chunk, flags):
    # single keys, B larger than n, ragged last trees and chunks (odd counts at every tree level),
    # several lanes with the last lane partly empty
    res = S.batch_keygen(761, n, 41, first_key_index=7, batch_size=B, chunk_keys=chunk, flags=flags,
                         debug=True)
    torch.cuda.synchronize()
    check_keys(O, 761, 41, res, np.arange(7, 7 + n), offset=7)


def test_async_host_output_pipeline(O):
    # asynchronous host-output calls back to back (the next call's compute overlaps the previous
    # call's copies; staging buffers are reused across calls): every call's bytes, read after its
    # completion event, equal the synchronous device-output call's and the oracle's (sample)
    P = S.params(761)
    n = 8192
    bufs = [(torch.empty((n, P["pk_bytes"]), dtype=torch.uint8).pin_memory(),
             torch.empty((n, P["sk_bytes"]), dtype=torch.uint8).pin_memory()) for _ in range(2)]
    evs = [S.Event(), S.Event()]
    fl = S.OPT_HOST_OUTPUT | S.OPT_ASYNC | S.OPT_RING_STREAMS
    seeds = [51, 52, 53, 54]
    got = {}
    for k, sd in enumerate(seeds):
        pk, sk = bufs[k % 2]
        S.batch_keygen(761, n, sd, batch_size=256, chunk_keys=2048, pk_out=pk, sk_out=sk, flags=fl,
                       done_event=evs[k % 2])
        if k >= 1:
            evs[(k - 1) % 2].synchronize()
            got[seeds[k - 1]] = (bufs[(k - 1) % 2][0].clone(), bufs[(k - 1) % 2][1].clone())
    evs[(len(seeds) - 1) % 2].synchronize()
    got[seeds[-1]] = (bufs[(len(seeds) - 1) % 2][0].clone(), bufs[(len(seeds) - 1) % 2][1].clone())
    for sd in seeds:
        ref = S.batch_keygen(761, n, sd, batch_size=256, chunk_keys=2048)
        torch.cuda.synchronize()
        assert torch.equal(got[sd][0], ref["pk"].cpu()) and torch.equal(got[sd][1], ref["sk"].cpu()), sd
    idx = np.arange(0, n, 257)
    r = oracle_keys(O, 761, seeds[0], idx)
    assert np.array_equal(got[seeds[0]][0].numpy()[idx], r["pk"])


def test_kernels_really_launch():
    before = S.kernel_launch_count()
    S.batch_keygen(761, 64, 1)
    torch.cuda.synchronize()
    assert S.kernel_launch_count() > before

#!/usr/bin/env python3
"""bench.py -- sntrup761 batch key generation on B200 (BASELINE.json configs[1]).

One step = one call of the whole hot path (sample, isInvertible, R/3 batchInv, R/q batchInv,
H = g * fbar, encode pk/sk) for 65,536 keys (sntrup761, seed 2).  Prints ONE JSON line (rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch-size B] [--impl ours|reference]

N > 1 is launched by torchrun: rank r generates global keys [r*n, (r+1)*n) (weak scaling, no
collective on the data path); the step time is the max over ranks (device events).
--impl reference times the CPU oracle (oracle/, the test-infrastructure implementation) on the
same metric, on bounded samples.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PARAM = 761
N_KEYS = 65536
SEED = 2
METRIC = "sntrup761 keys/sec per B200 (batched keygen); Rq mults/sec; int-pipe % of peak"
UNIT = "keys/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch-size", type=int, default=0, help="Montgomery batch size B (0 = tuned default)")
    ap.add_argument("--chunk-keys", type=int, default=0, help="keys per internal chunk (0 = tuned default); "
                    "two or more chunks run on two pipelined streams")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-extras", action="store_true", help="skip B sweep / rq_mul / cpu baseline")
    ap.add_argument("--ring-streams", type=int, choices=[0, 1], default=-1,
                    help="R/3 and R/q tree chains on separate streams (default: tuned)")
    ap.add_argument("--lanes", type=int, choices=[0, 2, 4], default=0,
                    help="chunks pipelined concurrently (0 = tuned default)")
    ap.add_argument("--mul-impl", choices=["tc", "schoolbook"], default="tc",
                    help="ring products: tcgen05 int8 Hankel GEMM (default) or int32 schoolbook")
    return ap.parse_args()


DEFAULT_B = 1024
DEFAULT_CHUNK = 32768
DEFAULT_RING_STREAMS = True   # R/3 and R/q chains on two streams (measured best; A/B in DESIGN.md)
DEFAULT_LANES = 2
MUL_IMPL = "tc"          # ring products on the tensor cores (see --mul-impl)
TRAFFIC = {}             # dram bytes per launch of the dominant kernel, from profiles/ (ncu)


# ----------------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "25"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thr = threading.Thread(target=self._read, daemon=True)
            self.thr.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        res = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": len(self.rows)}
        if not self.rows:
            return res
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        res["sm_mhz"] = statistics.median(sm) if sm else None
        res["sm_max_mhz"] = max(mx) if mx else None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for k, name in enumerate(names):
                if r[4 + k].lower().startswith("active"):
                    reasons.add(name)
        res["reasons"] = sorted(reasons)
        return res


# ----------------------------------------------------------------------------------- helpers
def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def tensor_peak_tops(peaks: dict, kind: str):
    """Dense tensor peak for the ring-product kernel kind, for a kernel timed ALONE (the serialised
    pass): the measured bf16 cuBLAS burst figure (MEASURED_PEAKS.json) x the nominal ratio of the
    kind's dtype to bf16 (int8 4.5 / 2.25 PF, fp4 9 / 2.25 PF dense; B200_PROFILING.md)."""
    ratio = 2.0 if kind == "tc_int8" else 4.0
    if "bf16_tflops" in peaks:
        return ratio * peaks["bf16_tflops"], "measured bf16 burst %.1f TF/s (MEASURED_PEAKS.json) x %g (nominal %s/bf16)" % (
            peaks["bf16_tflops"], ratio, "int8" if kind == "tc_int8" else "fp4")
    return ratio * 1650.0, "fallback bf16 1650 TF/s (B200_PROFILING.md) x %g" % ratio


def load_ncu_pipes():
    """Time-weighted pipe utilisation per kernel of the step from the committed ncu capture
    (profiles/ncu_pipes.json, written by scripts/ncu_pipes.py); {} if absent."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_pipes.json")))
        return {"source": "profiles/ncu_pipes.json (" + d.get("_source", "")[:60] + "...)",
                "per_kernel_pct": {k.replace("void ", ""): v["time_weighted"] for k, v in d["kernels"].items()}}
    except Exception:
        return {}


def load_traffic():
    """Per-launch DRAM bytes of the ring-product kernels from the committed ncu capture summary
    (profiles/roofline_traffic.json, written by scripts/ncu_traffic.py); {} if absent."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "roofline_traffic.json")))["per_launch_bytes"]
    except Exception:
        return {}


# Algorithmic integer work per unit of the ALU-bound kernels (SURVEY.md 8(d)
# "Algorithmic work per unit").  Lane-ops the method itself needs, not what our code issues.
def sampler_ops_per_key(p: int, nsort: int) -> float:
    # p SplitMix64 outputs (p/2 per domain, f and one g attempt) x 20 lane-ops (two 64-bit
    # multiplies = 6 IMAD, three 64-bit xor-shifts = 12 SHF/LOP3, the counter add = 2), the
    # 1024- (2048-) entry bitonic network (n/4 log2 n (log2 n + 1) compare-exchanges, 2 ops each:
    # min + max), and 5 ops per coefficient to map words to g and tagged f words
    lg = nsort.bit_length() - 1
    return 20.0 * p + 2.0 * (nsort // 4) * lg * (lg + 1) + 5.0 * p


def divstep_ops_per_root(p: int, ring: str) -> float:
    # 2p - 1 divsteps (C15).  R/q: per coefficient of the four p+1 vectors 4 multiplies, 2 adds,
    # 4 selects and 2 reductions = 12 lane-ops; R/3 bitsliced: ~45 LOP3/SHF word-ops per 32
    # coefficients of the vectors
    if ring == "rq":
        return (2 * p - 1) * 12.0 * (p + 1)
    return (2 * p - 1) * 45.0 * ((p + 1 + 31) // 32)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_keygen_rate(target_s: float = 10.0):
    """The oracle as it stands, all host cores, parallel over keys only, bounded sample."""
    import numpy as np
    from oracle import oracle as O
    threads = os.cpu_count() or 1
    n0 = max(threads * 8, 64)
    t = time.perf_counter()
    O.keygen_many(PARAM, SEED, np.arange(n0), threads=threads)
    dt = time.perf_counter() - t
    n = int(max(n0, min(200000, n0 * target_s / max(dt, 1e-3))))
    t = time.perf_counter()
    O.keygen_many(PARAM, SEED, np.arange(n), threads=threads)
    dt = time.perf_counter() - t
    return n / dt, threads, "keys 0..%d of configs[1] (sntrup761, seed 2), %d host threads, %.1f s" % (
        n - 1, threads, dt)


def oracle_single_thread():
    """The oracle on ONE host thread: keys/s over keys 0..255 of configs[1], and R/q schoolbook
    products/s over the first 4096 pairs of configs[2] (inputs by C12)."""
    import numpy as np
    from oracle import oracle as O
    t = time.perf_counter()
    O.keygen_many(PARAM, SEED, np.arange(256), threads=1)
    keys = 256 / (time.perf_counter() - t)
    p, q, w = O.PARAMS[PARAM]
    A = np.zeros((4096, p), np.int16)
    Bm = np.zeros((4096, p), np.int16)
    for i in range(4096):
        a, b = O.c12_pair(PARAM, 3, i)
        A[i], Bm[i] = a, b
    t = time.perf_counter()
    O.mul_many(p, q, A, Bm, threads=1)
    return keys, 4096 / (time.perf_counter() - t)


def other_configs(S, torch, timed):
    """configs[0]: latency of one 32-key call (launch-bound; synchronous C-ABI call, host
    wall clock around it, and device time); configs[3]: keys/s per parameter set at 65,536 keys
    (the headline's B / chunking); configs[4]: sntrup1277, 2^20 keys, B = 1024, streamed in
    65,536-key chunks."""
    out = {}
    # configs[0]: 761, 32 keys, seed 1, one tree of 32
    P = S.params(761)
    pk = torch.empty((32, P["pk_bytes"]), dtype=torch.uint8, device="cuda")
    sk = torch.empty((32, P["sk_bytes"]), dtype=torch.uint8, device="cuda")
    # latency-tuned: B = 1 (each key's reciprocals by its own root chain -- jump-divsteps -- all 32
    # in parallel: no tree levels on the critical path) with the R/3 and R/q chains on separate
    # streams, replayed as a CUDA graph (SNTRUP_OPT_GRAPH: captured on the first call, seed and
    # first key index patched per call); the same call without the graph and the one-tree B = 32
    # configuration beside it (scripts/latency_sweep.py sweeps B)
    st = torch.cuda.Stream()
    l2flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def lat_of(B, fl):
        with torch.cuda.stream(st):
            call = lambda f2: S.batch_keygen(761, 32, 1, batch_size=B, pk_out=pk, sk_out=sk, flags=f2, stream=st)
            for _ in range(5):
                call(fl)
            torch.cuda.synchronize()
            lat = []
            for _ in range(20):
                t0 = time.perf_counter()
                call(fl)                                           # synchronous call
                lat.append((time.perf_counter() - t0) * 1e6)
            # device time on the call's stream, L2 flushed before each call (not timed)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
            for e0, e1 in ev:
                l2flush.zero_()
                e0.record(st)
                call(fl | S.OPT_ASYNC)
                e1.record(st)
            torch.cuda.synchronize()
            dev_ms = sum(e0.elapsed_time(e1) for e0, e1 in ev) / len(ev)
        return statistics.median(lat), dev_ms * 1e3
    lg, dg = lat_of(1, S.OPT_RING_STREAMS | S.OPT_GRAPH)
    l1, d1 = lat_of(1, S.OPT_RING_STREAMS)
    l32, d32 = lat_of(32, 0)
    out["configs[0]"] = {"workload": "sntrup761, 32 keys, seed 1, B = 1, ring streams, CUDA graph (latency-tuned)",
                         "latency_us_median": lg, "device_us": dg, "keys_per_s": 32 / (lg / 1e6),
                         "without_graph": {"latency_us_median": l1, "device_us": d1},
                         "one_tree_B32": {"latency_us_median": l32, "device_us": d32}}
    # configs[3]: parameter sweep at 65,536 keys, seed 4
    sweep = {}
    for ps in (653, 857, 953, 1013):
        P = S.params(ps)
        n = 65536
        pk = torch.empty((n, P["pk_bytes"]), dtype=torch.uint8, device="cuda")
        sk = torch.empty((n, P["sk_bytes"]), dtype=torch.uint8, device="cuda")
        f = lambda: S.batch_keygen(ps, n, 4, batch_size=DEFAULT_B, chunk_keys=DEFAULT_CHUNK, pk_out=pk,
                                   sk_out=sk, flags=S.OPT_ASYNC | S.OPT_RING_STREAMS)
        f()
        ms = timed(f, 3) / 3
        # the same set at B = 32, and the rejection total (extra g draws) of the
        # 65,536 keys (expected from the factor degrees: 653 ~2521, 857 ~0, 953 ~271, 1013 ~819)
        f32 = lambda: S.batch_keygen(ps, n, 4, batch_size=32, chunk_keys=DEFAULT_CHUNK, pk_out=pk,
                                     sk_out=sk, flags=S.OPT_ASYNC | S.OPT_RING_STREAMS)
        f32()
        ms32 = timed(f32, 2) / 2
        att = S.batch_keygen(ps, n, 4, batch_size=DEFAULT_B, chunk_keys=DEFAULT_CHUNK, pk_out=pk, sk_out=sk,
                             flags=S.OPT_RING_STREAMS, attempts=True)["attempts"]
        sweep[str(ps)] = {"keys_per_s": n / (ms / 1e3), "ms": ms, "keys_per_s_B32": n / (ms32 / 1e3),
                          "rejected_g_draws": int(att.to(torch.int64).sum().item()) - n}
        del pk, sk, att
    out["configs[3]"] = {"workload": "65,536 keys per set, seed 4, B = %d, %d-key chunks on two lanes, "
                                     "ring streams" % (DEFAULT_B, DEFAULT_CHUNK), "by_param_set": sweep}
    # configs[4]: 1277, 2^20 keys, B = 1024, 65,536-key chunks (two pipelined lanes)
    P = S.params(1277)
    n = 1 << 20
    pk = torch.empty((n, P["pk_bytes"]), dtype=torch.uint8, device="cuda")
    sk = torch.empty((n, P["sk_bytes"]), dtype=torch.uint8, device="cuda")
    f = lambda: S.batch_keygen(1277, n, 5, batch_size=1024, chunk_keys=65536, pk_out=pk, sk_out=sk,
                               flags=S.OPT_ASYNC | S.OPT_RING_STREAMS)
    f()
    ms = timed(f, 2) / 2
    att = S.batch_keygen(1277, n, 5, batch_size=1024, chunk_keys=65536, pk_out=pk, sk_out=sk,
                         flags=S.OPT_RING_STREAMS, attempts=True)["attempts"]
    out["configs[4]"] = {"workload": "sntrup1277, 2^20 keys, seed 5, B = 1024, 65,536-key chunks, ring streams",
                         "keys_per_s": n / (ms / 1e3), "ms": ms,
                         "rejected_g_draws": int(att.to(torch.int64).sum().item()) - n,
                         "rejected_g_draws_note": "the oracle's count for these 2^20 keys is 54,600 (tests/golden/oracle_digests/cfg4_1277.json; every key's "
                                                  "attempt count is compared in tests/test_gpu_fullsize.py)"}
    del pk, sk, att
    # KEM core: 65,536 encapsulations (r from the encapsulation stream
    # domain + c = Round(h r)) and decapsulations (r' = ((3f c) mod 3)/g + weight check)
    n = 65536
    keys = S.batch_keygen(761, n, 2, batch_size=1024, debug=True)
    r = torch.empty((n, S.params(761)["p16"]), dtype=torch.int8, device="cuda")
    c = torch.empty_like(keys["h"])
    r2 = torch.empty_like(r)
    okb = torch.empty(n, dtype=torch.uint8, device="cuda")

    def enc():
        S.sample_short_batch(761, n, 2, 0, out=r)
        S.encap_core_batch(761, keys["h"], r, c)

    def dec():
        S.decap_core_batch(761, keys["f"], keys["ginv"], c, r2, okb)

    enc(); dec()
    torch.cuda.synchronize()
    assert bool(okb.all()) and torch.equal(r, r2), "KEM core round trip failed"
    enc_ms = timed(enc, 3) / 3
    dec_ms = timed(dec, 3) / 3
    out["kem_core"] = {"workload": "sntrup761, 65,536 keys of configs[1]: encapsulation core (Short r from "
                                   "the stream + Round(h r)) and decapsulation core (+ weight check)",
                       "encaps_per_s": n / (enc_ms / 1e3), "decaps_per_s": n / (dec_ms / 1e3),
                       "paper_context_cycles": {"enc": 46914, "dec": 56241, "hardware": "Haswell, Table 1 P:864-876"}}
    del keys, r, c, r2, okb
    # full-size secret keys (reading Z24): sk || pk || rho || SHA-512(4 || pk)[:32]
    keys = S.batch_keygen(761, n, 2, batch_size=1024)
    full = S.full_sk_batch(761, 2, keys["pk"], keys["sk"])
    fsk_ms = timed(lambda: S.full_sk_batch(761, 2, keys["pk"], keys["sk"], out=full), 3) / 3
    out["full_sk"] = {"workload": "sntrup761, 65,536 keys of configs[1]: full-size sk rows (%d B: sk || pk || "
                                  "rho || SHA-512(4 || pk)[:32]) from device pk/sk" % full.shape[1],
                      "keys_per_s": n / (fsk_ms / 1e3), "ms": fsk_ms}
    del keys, full
    # key pool (the paper's engNTRU batch_lib provider: "first key 2.5 ms, then
    # 0 ms"): first take (lazy fill), then paced takes served from the pinned ring
    pool = S.KeyPool(761, seed=9, capacity=1 << 15, batch_keys=1 << 13, batch_size=512)
    t0 = time.perf_counter()
    pool.take()
    first_ms = (time.perf_counter() - t0) * 1e3
    lat = []
    for _ in range(2000):
        time.sleep(0.0002)
        t0 = time.perf_counter()
        pool.take()
        lat.append((time.perf_counter() - t0) * 1e6)
    st = pool.stats()
    pool.close()
    lat.sort()
    # the paper's series shape: wall time to obtain K keys from a fresh pool, unpaced
    # (engNTRU batch_lib: (0.08 K + 2.5) ms on Haswell)
    series = {}
    for K in (1, 10, 100, 1000, 10000, 100000):
        pool = S.KeyPool(761, seed=11, capacity=1 << 15, batch_keys=1 << 13, batch_size=512)
        t0 = time.perf_counter()
        for _ in range(K):
            pool.take()
        series[str(K)] = (time.perf_counter() - t0) * 1e3
        pool.close()
    out["key_pool"] = {"workload": "sntrup761 pool: capacity 32768, refill batches of 8192 keys (B = 512), "
                                   "2000 takes paced 0.2 ms apart; series: K unpaced takes from a fresh pool",
                       "first_take_ms": first_ms, "take_us_median": lat[len(lat) // 2],
                       "take_us_p99": lat[int(len(lat) * 0.99)], "waits_after_first": st["waits"] - 1,
                       "ms_for_K_keys": series,
                       "paper_context": "engNTRU batch_lib on Haswell: (0.08 K + 2.5) ms for K keys (P:8616-8700)"}
    return out


# ----------------------------------------------------------------------------------- reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np
    from oracle import oracle as O
    threads = os.cpu_count() or 1
    # each step: a bounded sample of the workload (the oracle would need minutes for 65,536 keys)
    n_step = max(64, threads * 16)
    for i in range(args.warmup):
        O.keygen_many(PARAM, SEED, np.arange(i * n_step, (i + 1) * n_step), threads=threads)
    t = time.perf_counter()
    for i in range(args.steps):
        O.keygen_many(PARAM, SEED, np.arange(i * n_step, (i + 1) * n_step), threads=threads)
    dt = time.perf_counter() - t
    v = n_step * args.steps / dt
    sample = "%d keys per step of configs[1] (sntrup761, seed 2), %d host threads (%s)" % (
        n_step, threads, cpu_model())
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": "configs[1]: sntrup761 batch keygen, seed 2 (oracle sample)",
                       "keys_per_step": n_step},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    # the collective code paths (barrier, max over ranks) also run for one rank when the launcher's
    # rendezvous variables are present and BENCH_FORCE_DIST is set (a 1-GPU check of the N > 1 path)
    use_dist = world > 1 or (os.environ.get("BENCH_FORCE_DIST") == "1" and "MASTER_ADDR" in os.environ)
    if use_dist:
        # (the GPU boxes export NCCL_DEBUG=VERSION: NCCL's one-line version banner precedes the JSON
        # line on stdout; left as the launcher set it)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2106_08759_b200 as S

    global MUL_IMPL
    MUL_IMPL = args.mul_impl
    S.set_mul_impl(S.MUL_TENSOR_CORE if MUL_IMPL == "tc" else S.MUL_SCHOOLBOOK)
    TRAFFIC.update(load_traffic())
    P = S.params(PARAM)
    B = args.batch_size or DEFAULT_B
    n = N_KEYS
    first = rank * n
    stream = torch.cuda.current_stream()
    pk = torch.empty((n, P["pk_bytes"]), dtype=torch.uint8, device="cuda")
    sk = torch.empty((n, P["sk_bytes"]), dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")   # > 126 MB L2

    CHUNK = args.chunk_keys or DEFAULT_CHUNK
    RINGS = DEFAULT_RING_STREAMS if args.ring_streams < 0 else bool(args.ring_streams)
    LANES = args.lanes or DEFAULT_LANES
    FLAGS = S.OPT_ASYNC | (S.OPT_RING_STREAMS if RINGS else 0) | (S.OPT_LANES4 if LANES == 4 else 0)

    def step(batch=B, chunk=None, flags=FLAGS):
        S.batch_keygen(PARAM, n, SEED, first_key_index=first, batch_size=batch, pk_out=pk,
                       sk_out=sk, flags=flags, chunk_keys=CHUNK if chunk is None else chunk)

    def barrier():
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, steps):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps)]
        barrier()
        for e0, e1 in ev:
            flush.zero_()                       # L2 flush between timed iterations (not timed)
            e0.record(stream)
            fn()
            e1.record(stream)
        barrier()
        per_step = [e0.elapsed_time(e1) for e0, e1 in ev]
        timed.last = per_step                       # this rank's per-step device times
        ms = sum(per_step)
        if use_dist:
            t = torch.tensor([ms], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    # integer-pipe peaks of this GPU (the metric's "int-pipe % of peak"; MEASURED_PEAKS.json has
    # none): lane-ops per SM clock per SM of IMAD (FMA pipe) and IADD3 / LOP3 / SHF (ALU pipe)
    int_peaks = {op: S.measure_int_peak(op) for op in S.INT_OPS} if rank == 0 else {}

    # clocks are sampled from the warm-up through the timed, profiled and e2e steps (all under
    # load; the timed region alone can be shorter than nvidia-smi's first sample)
    clk = ClockSampler(local)
    clk.start()
    # settle phase before the W warm-up steps: the first ~30 steps of a fresh process run 1-4%
    # slower (SM clocks ramping from idle, first touches of the workspace; scripts/gpu_warm.sh,
    # profiles/r02s4/warm_ab.log) -- a serving process is past this; disclosed in config.settle
    SETTLE_STEPS = 40
    for _ in range(SETTLE_STEPS):
        step()
    torch.cuda.synchronize()
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    # ---- headline: K timed steps
    launches0 = S.kernel_launch_count()
    ms = timed(step, args.steps)
    launches = S.kernel_launch_count() - launches0
    step_ms = sorted(timed.last)
    value = world * n * args.steps / (ms / 1e3)

    # ---- per-kernel times: the same step SERIALISED (SNTRUP_OPT_SERIAL: one lane, every kernel
    # alone on one stream), so each launch's CUDA-event time is its own; the kernel shares of the
    # step and the roofline's launch durations come from this pass (the overlapped step above
    # hides the latency-bound phases behind the other lane's products)
    serial_flags = S.OPT_ASYNC | S.OPT_SERIAL
    step(flags=serial_flags)
    S.profile_enable(True)
    ms_serial = timed(lambda: step(flags=serial_flags), args.steps)
    prof = S.profile_read(reset=True)
    kinds = S.profile_read_kinds(reset=True)
    S.profile_enable(False)

    # ---- e2e through the C ABI with HOST output buffers (D2H inside the timed region), one fixed
    # configuration: the key-serving loop -- asynchronous host-output calls into two alternating
    # pinned buffer sets; the host waits for step k-1's completion event (all of its pk/sk bytes in
    # host memory) and reads its first key before issuing step k+1, so every step's D2H copy is in
    # the timed region while it overlaps the next step's compute; wall clock over max(50, K) steps
    # including the final drain
    pk_h = torch.empty((n, P["pk_bytes"]), dtype=torch.uint8).pin_memory()
    sk_h = torch.empty((n, P["sk_bytes"]), dtype=torch.uint8).pin_memory()
    pk_h2 = [pk_h, torch.empty_like(pk_h).pin_memory()]
    sk_h2 = [sk_h, torch.empty_like(sk_h).pin_memory()]
    evs = [S.Event(), S.Event()]
    E2E_FLAGS = S.OPT_RING_STREAMS
    serve_stream = torch.cuda.Stream()

    def serve(steps, fl=E2E_FLAGS, chunk=CHUNK, graph=True):
        # graph=True: each call replays the keygen as one CUDA graph on a side stream and copies
        # the whole call's pk/sk afterwards (SNTRUP_OPT_GRAPH | SNTRUP_OPT_HOST_OUTPUT); while the
        # previous call's bytes cross PCIe, ~90 separately enqueued launches each start later
        # (the plain asynchronous call, graph=False: reported beside it)
        for k in range(steps):
            S.batch_keygen(PARAM, n, SEED, first_key_index=first, batch_size=B, pk_out=pk_h2[k % 2],
                           sk_out=sk_h2[k % 2], chunk_keys=chunk, done_event=evs[k % 2],
                           flags=S.OPT_HOST_OUTPUT | S.OPT_ASYNC | fl | (S.OPT_GRAPH if graph else 0),
                           stream=serve_stream if graph else None)
            if k >= 1:
                evs[(k - 1) % 2].synchronize()
                _ = int(pk_h2[(k - 1) % 2][0, 0]) + int(sk_h2[(k - 1) % 2][0, 0])
        evs[(steps - 1) % 2].synchronize()

    # (the last step's 1.8 ms of D2H copies cannot overlap a next step: over 50 steps that drain is
    # 1.4% of the wall clock, over 20 it was 3.5%)
    serve_steps = max(50, args.steps)
    e2e_by_mode = {}
    for graph in (False, True):
        serve(3, graph=graph)
        barrier()
        t0 = time.perf_counter()
        serve(serve_steps, graph=graph)
        dt = time.perf_counter() - t0
        if use_dist:
            t = torch.tensor([dt], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e_by_mode[graph] = world * n * serve_steps / dt
    e2e_value = e2e_by_mode[True]
    # context: one synchronous host-output call per step (copies overlap only within the call)
    def step_host_sync():
        S.batch_keygen(PARAM, n, SEED, first_key_index=first, batch_size=B, pk_out=pk_h, sk_out=sk_h,
                       flags=S.OPT_HOST_OUTPUT | E2E_FLAGS, chunk_keys=CHUNK)
    step_host_sync()
    e2e_sync = world * n * args.steps / (timed(step_host_sync, args.steps) / 1e3)
    # the e2e ceiling set by the host link: one device->pinned-host copy of a step's pk+sk bytes
    d2h_b = n * (P["pk_bytes"] + P["sk_bytes"])
    dbuf = torch.empty(d2h_b, dtype=torch.uint8, device="cuda")
    hbuf = torch.empty(d2h_b, dtype=torch.uint8).pin_memory()
    hbuf.copy_(dbuf, non_blocking=True)
    torch.cuda.synchronize()
    d2h_ms = timed(lambda: hbuf.copy_(dbuf, non_blocking=True), 3) / 3
    d2h_gbs = d2h_b / (d2h_ms / 1e3) / 1e9
    del dbuf, hbuf
    clocks = clk.stop()

    result = {}
    if rank == 0:
        peaks = load_peaks()
        sm_mhz = clocks.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
        n_sm = torch.cuda.get_device_properties(local).multi_processor_count
        tot_serial = sum(v["ms"] for v in prof.values())
        share = {k: v["ms"] / tot_serial for k, v in prof.items() if v["launches"]}
        kshare = {k: v["ms"] / tot_serial for k, v in kinds.items() if v["launches"]}
        # the dominant kernel kind by serialised device time
        kd = max(kinds, key=lambda k: kinds[k]["ms"])
        K = kinds[kd]
        roof = None
        if K["launches"]:
            secs = K["ms"] / 1e3                                   # summed launch durations (serial)
            achieved = K["ops"] / secs / 1e12                      # T ops/s: 2 p^2 per product
            if kd in ("tc_int8", "tc_fp4"):
                peak, src = tensor_peak_tops(peaks, kd)
                smem_peak = 128.0 * n_sm * sm_mhz * 1e6            # B/s: 128 B/clk/SM shared-memory reads
                smem_ach = K["smem_bytes"] / secs
                roof = {"bound": "tensor",
                        "kernel": "ring products, " + ("tc_mul_kernel (tcgen05.mma kind::i8)" if kd == "tc_int8"
                                                        else "tc4_mul_kernel (tcgen05.mma kind::mxf4)"),
                        "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                        "unit_note": "tera-ops/s of the method's work: 2 p^2 per ring product (p^2 "
                                     "multiply-adds), whatever the limb / digit / padding overhead",
                        "frac": achieved / peak, "traffic": TRAFFIC.get(kd),
                        "peak_source": src,
                        "launch_time_source": "CUDA events per launch on its stream, serialised pass "
                                              "(SNTRUP_OPT_SERIAL), %d launches" % K["launches"],
                        "products_per_step": K["products"] / args.steps,
                        "share_of_serial_step": K["ms"] / tot_serial,
                        "by_kind_share_of_serial_step": kshare,
                        "smem_operand_roofline": {
                            "achieved_gbs": smem_ach / 1e9, "peak_gbs": smem_peak / 1e9,
                            "frac": smem_ach / smem_peak,
                            "bytes_per_product": K["smem_bytes"] / max(K["products"], 1),
                            "note": "A and B tile bytes the MMAs fetch from shared memory (geometry x "
                                    "MMAs) / launch time, against 128 B/clk/SM x %d SMs x %.0f MHz "
                                    "(the run's median SM clock): the resource that binds these "
                                    "small-N GEMMs (DESIGN.md 6.1)" % (n_sm, sm_mhz)}}
            else:
                imad = int_peaks.get("IMAD", {}).get("lanes_per_clk_sm", 64.0)
                peak = 2 * imad * n_sm * sm_mhz * 1e6 / 1e12
                roof = {"bound": "alu", "kernel": "ring products, ring_mul_kernel (int32 schoolbook)",
                        "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                        "frac": achieved / peak, "traffic": None,
                        "peak_source": "measured IMAD %.1f lanes/clk/SM x 2 ops x %d SMs x %.0f MHz" % (imad, n_sm, sm_mhz)}
        # integer-pipe fractions of the ALU-bound kernels, from the serialised pass and the
        # measured pipe peaks at the run's clock (DESIGN.md 6.2 op counts)
        # ALU pipe = LOP3's rate; FMA pipe = IMAD's; issue = IADD3's (it dual-issues on both pipes,
        # measuring the 4 x 32 lanes/clk/SM issue limit)
        alu = int_peaks["LOP3"]["lanes_per_clk_sm"] if int_peaks else 64.0
        alu_peak = alu * n_sm * sm_mhz * 1e6
        fma_peak = (int_peaks.get("IMAD", {}).get("lanes_per_clk_sm", 64.0)) * n_sm * sm_mhz * 1e6
        issue_peak = (int_peaks.get("IADD3", {}).get("lanes_per_clk_sm", 128.0)) * n_sm * sm_mhz * 1e6
        nsort = 1024 if PARAM <= 1024 else 2048
        pipes = {}
        if prof["sample"]["launches"]:
            r = prof["sample"]["units"] * sampler_ops_per_key(P["p"], nsort) / (prof["sample"]["ms"] / 1e3)
            pipes["sample_kernel"] = {"achieved_lane_ops_per_s": r, "issue_peak": issue_peak,
                                      "frac_of_issue": r / issue_peak,
                                      "ops_per_key": sampler_ops_per_key(P["p"], nsort),
                                      "note": "algorithmic lane-ops (ALU and FMA work) against the "
                                              "issue limit both pipes share"}
        if prof["r3_mul"]["launches"] or prof["root_inv"]["launches"]:
            nroots = prof["root_inv"]["units"]
            r3 = nroots * divstep_ops_per_root(P["p"], "r3") / max(prof["root_inv"]["ms"] / 1e3, 1e-12)
            pipes["divstep_kernel (R/3 roots)"] = {"achieved_lane_ops_per_s": r3, "frac_of_alu": r3 / alu_peak,
                                                   "roots_per_step": nroots / args.steps,
                                                   "note": "latency-bound: one warp per root, few roots"}
        if prof["rq_inv"]["launches"]:
            nr = prof["rq_inv"]["units"]
            rq = nr * divstep_ops_per_root(P["p"], "rq") / (prof["rq_inv"]["ms"] / 1e3)
            pipes["divstep_cta_kernel (R/q roots)"] = {"achieved_lane_ops_per_s": rq, "frac_of_fma": rq / fma_peak,
                                                       "roots_per_step": nr / args.steps,
                                                       "note": "latency-bound: 8 warps per root on <= 2 x %d roots" % n_sm}
        if prof["encode"]["launches"]:
            keys_e = prof["encode"]["units"]              # device outputs: one encode launch per key range
            byt = keys_e * (2 * P["p8"] + 2 * P["p16"] + P["pk_bytes"] + P["sk_bytes"])
            bw = byt / (prof["encode"]["ms"] / 1e3)
            pipes["encode_kernel"] = {"achieved_gbs": bw / 1e9, "hbm_peak_gbs": peaks.get("hbm_gbs", 6552.0),
                                      "frac_of_hbm": bw / 1e9 / peaks.get("hbm_gbs", 6552.0),
                                      "bytes_per_key": byt / keys_e}
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int8/e2m1 MMA -> s32/f32 (exact integer)",
            "data": "synthetic",
            "config": {"workload": "configs[1]: sntrup761 batch keygen, 65,536 keys per GPU, seed 2",
                       "keys_per_gpu": n, "batch_size": B, "chunk_keys": CHUNK, "ring_streams": RINGS,
                       "lanes": LANES, "param_set": PARAM,
                       "l2": "flushed between timed steps (256 MiB write); working set > L2",
                       "settle": "%d untimed steps before the W warm-up steps (clocks from idle, first touches)" % SETTLE_STEPS,
                       "parallelism": "key ranges per GPU (no collective)"},
            "gpu_launches": launches,
            "clocks": clocks,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": world * n * (P["pk_bytes"] + P["sk_bytes"]),
                    "config": "key-serving loop: asynchronous host-output calls (chunk %d, ring streams), "
                              "each a CUDA-graph replay of the keygen on a side stream followed by the "
                              "D2H copies of its pk/sk (SNTRUP_OPT_GRAPH | SNTRUP_OPT_HOST_OUTPUT), "
                              "into two alternating pinned buffer sets; the host waits for each step's "
                              "completion event and reads its bytes; wall clock over %d steps incl. the "
                              "final drain" % (CHUNK, serve_steps),
                    "plain_async_calls_no_graph": e2e_by_mode[False],
                    "one_synchronous_call_per_step": e2e_sync,
                    "d2h_gbs_measured": d2h_gbs,
                    "d2h_ceiling_keys_per_s": world * d2h_gbs * 1e9 / (P["pk_bytes"] + P["sk_bytes"]),
                    "note": "inputs are (param, n, seed, first key index): no H2D payload"},
            "roofline": roof,
            "int_pipe": {"peaks_lanes_per_clk_sm": {k: v["lanes_per_clk_sm"] for k, v in int_peaks.items()},
                         "source": "sntrup_measure_int_peak microkernels, this run",
                         "kernels": pipes},
            "step_ms_min_median_max": [step_ms[0], step_ms[len(step_ms) // 2], step_ms[-1]],
            "serial_ms_per_step": ms_serial / args.steps,
            "serial_share_by_class": share,
            "serial_ms_per_step_by_class": {k: v["ms"] / args.steps for k, v in prof.items() if v["launches"]},
            "mul_impl": MUL_IMPL,
            "ncu_pipes": load_ncu_pipes(),
        }

    if not args.no_extras and rank == 0:
        # Montgomery batch-size sweep (configs[1])
        sweep = {}
        for b in (32, 128, 512, 1024, 2048):
            step(b)
            sweep[str(b)] = n * 3 / (timed(lambda: step(b), 3) / 1e3)
        result["batch_size_sweep_keys_per_s"] = sweep
        # chunking: one chunk, or 2/4 chunks pipelined on two streams
        csweep = {}
        for ck in (65536, 32768, 16384):
            step(chunk=ck)
            csweep[str(ck)] = n * 3 / (timed(lambda: step(chunk=ck), 3) / 1e3)
        result["chunk_sweep_keys_per_s"] = csweep
        # A/B: the same step under the other ring-product implementations
        ab = {}
        for name, impl in (("tc_int8_m64", S.MUL_TENSOR_CORE_M64),
                           ("tc_int8_big_single", S.MUL_TENSOR_CORE_I8_SINGLE),
                           ("tc_u_fused_level1", S.MUL_TENSOR_CORE_U_FUSED),
                           ("tc_fp4_all_small", S.MUL_TENSOR_CORE_FP4_ALL),
                           ("tc_int8_shared_a", S.MUL_TENSOR_CORE_INT8),
                           ("tc_int8_no_shared_a", S.MUL_TENSOR_CORE_NO_SHARED_A),
                           ("int32_schoolbook", S.MUL_SCHOOLBOOK)):
            S.set_mul_impl(impl)
            step()
            ab[name] = n * 2 / (timed(step, 2) / 1e3)
        S.set_mul_impl(S.MUL_TENSOR_CORE if MUL_IMPL == "tc" else S.MUL_SCHOOLBOOK)
        result["mul_impl_ab_keys_per_s"] = ab
        # R/q multiplication microbenchmark (configs[2]): 2^20 pairs, inputs per SURVEY.md C12 drawn
        # on the GPU by the library's samplers (a uniform from domain 0, b Short(286) from domain 1,
        # seed 3), through the big x small entry point; big x big and the int32 schoolbook beside it
        npairs = 1 << 20
        a = S.sample_uniform_rq_batch(PARAM, npairs, 3, domain=0)
        bt = S.sample_short_batch(PARAM, npairs, 3, domain=1)
        c = torch.empty_like(a)
        S.rq_mul_small_batch(PARAM, a, bt, c)
        rq_ms = timed(lambda: S.rq_mul_small_batch(PARAM, a, bt, c), 3) / 3
        b2 = S.sample_uniform_rq_batch(PARAM, npairs, 3, domain=2)
        S.rq_mul_batch(PARAM, a, b2, c)
        bb_ms = timed(lambda: S.rq_mul_batch(PARAM, a, b2, c), 3) / 3
        S.set_mul_impl(S.MUL_SCHOOLBOOK)
        sb_ms = timed(lambda: S.rq_mul_batch(PARAM, a, b2, c), 2) / 2
        S.set_mul_impl(S.MUL_TENSOR_CORE if MUL_IMPL == "tc" else S.MUL_SCHOOLBOOK)
        result["rq_mul"] = {"value": npairs / (rq_ms / 1e3), "unit": "Rq mults/s",
                            "config": "configs[2]: 2^20 pairs in Z/4591[x]/(x^761-x-1), a uniform (C12, "
                                      "domain 0) x Short w=286 (domain 1), seed 3, rq_mul_small_batch",
                            "ms": rq_ms,
                            # a int16 row + b int8 row read, c int16 row written per pair
                            "hbm_gbs": npairs * (2 * P["p8"] * 2 + P["p16"]) / (rq_ms / 1e3) / 1e9,
                            "big_x_big_path_mults_per_s": npairs / (bb_ms / 1e3),
                            "int32_schoolbook_mults_per_s": npairs / (sb_ms / 1e3)}
        del a, bt, c, b2
        # the other configs' reported quantities; parity for each is in
        # tests/test_gpu_parity.py and tests/test_gpu_fullsize.py
        result["other_configs"] = other_configs(S, torch, timed)
        # CPU baseline: the oracle on this host -- all cores (bounded sample), one thread on 256
        # keys, and R/q schoolbook products (SURVEY.md 8(d) "Oracle timing beside the GPU")
        v, cores, sample = oracle_keygen_rate(10.0)
        v1, rq1 = oracle_single_thread()
        result["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                                  "sample": sample, "cpu_model": cpu_model(),
                                  "single_thread_keys_per_s": v1,
                                  "single_thread_rq_mults_per_s": rq1,
                                  "single_thread_sample": "keys 0..255 of configs[1]; R/q products of "
                                                          "4096 configs[2] pairs (C12)"}
    if rank == 0:
        print(json.dumps(result))
    if use_dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

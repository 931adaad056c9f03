#!/usr/bin/env python3
"""Alternating-round A/B of the root-inversion implementation (sntrup_set_root_impl) on the keygen
step of configs[1] (bench.py's launch configuration, L2 flushed between steps) and on configs[0]
(32 keys, B = 1, ring streams: latency of one synchronous call)."""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2106_08759_b200 as S  # noqa: E402

n = 65536
P = S.params(761)
pk = torch.empty((n, P["pk_bytes"]), dtype=torch.uint8, device="cuda")
sk = torch.empty((n, P["sk_bytes"]), dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
R = S.OPT_RING_STREAMS
impls = {"auto": S.ROOT_AUTO, "jump": S.ROOT_JUMP, "step": S.ROOT_STEP, "jump_shared_sm": S.ROOT_JUMP | S.ROOT_SHARED_SM}
step = {k: [] for k in impls}
lat = {k: [] for k in impls}
dev = {k: [] for k in impls}
for rnd in range(int(os.environ.get("ROUNDS", "8"))):
    for name, impl in impls.items():
        S.set_root_impl(impl)
        f = lambda: S.batch_keygen(761, n, 2, batch_size=1024, chunk_keys=32768, pk_out=pk, sk_out=sk,
                                   flags=S.OPT_ASYNC | R)
        f()
        torch.cuda.synchronize()
        for _ in range(3):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            f()
            e1.record()
            torch.cuda.synchronize()
            step[name].append(e0.elapsed_time(e1))
        g = lambda: S.batch_keygen(761, 32, 1, batch_size=1, flags=R)
        g()
        torch.cuda.synchronize()
        for _ in range(5):
            t0 = time.perf_counter()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g()
            e1.record()
            torch.cuda.synchronize()
            lat[name].append((time.perf_counter() - t0) * 1e6)
            dev[name].append(e0.elapsed_time(e1) * 1e3)
S.set_root_impl(S.ROOT_AUTO)
out = {}
for name in impls:
    ms = statistics.median(step[name])
    out[name] = {"cfg1_step_ms": ms, "cfg1_keys_per_s": n / ms * 1e3,
                 "cfg0_latency_us": statistics.median(lat[name]), "cfg0_device_us": statistics.median(dev[name])}
    print(name, json.dumps(out[name]), flush=True)
print(json.dumps(out))

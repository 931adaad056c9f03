#!/usr/bin/env python3
"""Experiment: capture one configs[0] keygen call (asynchronous, device outputs) into a CUDA graph
with torch.cuda.graph and replay it: device span and synchronous wall time per replay against
the plain call, and the replayed bytes against the plain call's."""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2106_08759_b200 as S  # noqa: E402

P = S.params(761)
pk = torch.empty((32, P["pk_bytes"]), dtype=torch.uint8, device="cuda")
sk = torch.empty((32, P["sk_bytes"]), dtype=torch.uint8, device="cuda")
R = S.OPT_RING_STREAMS
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(5):
        S.batch_keygen(761, 32, 1, batch_size=1, pk_out=pk, sk_out=sk, flags=R | S.OPT_ASYNC, stream=s)
torch.cuda.synchronize()
ref_pk, ref_sk = pk.clone(), sk.clone()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    S.batch_keygen(761, 32, 1, batch_size=1, pk_out=pk, sk_out=sk, flags=R | S.OPT_ASYNC, stream=s)
pk.zero_(); sk.zero_()
g.replay()
torch.cuda.synchronize()
same = bool(torch.equal(pk, ref_pk) and torch.equal(sk, ref_sk))


def measure(fn):
    span, wall = [], []
    for _ in range(30):
        torch.cuda.synchronize()
        time.sleep(0.002)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        torch.cuda.synchronize()
        span.append(e0.elapsed_time(e1) * 1e3)
    for _ in range(30):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        s.synchronize()
        wall.append((time.perf_counter() - t0) * 1e6)
    return statistics.median(span), statistics.median(wall)


def replay_on_s():
    with torch.cuda.stream(s):
        g.replay()


plain = measure(lambda: S.batch_keygen(761, 32, 1, batch_size=1, pk_out=pk, sk_out=sk, flags=R | S.OPT_ASYNC, stream=s))
graph = measure(replay_on_s)
print(json.dumps({"graph_replay_bytes_equal": same, "plain_span_us": plain[0], "plain_wall_us": plain[1],
                  "graph_span_us": graph[0], "graph_wall_us": graph[1]}))

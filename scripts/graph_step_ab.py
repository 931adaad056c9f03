#!/usr/bin/env python3
"""Alternating-round A/B of the configs[1] keygen step (bench configuration: B = 1024, 32,768-key
chunks, ring streams, device outputs, L2 flushed between steps) with and without SNTRUP_OPT_GRAPH,
on one non-default stream; the outputs of the two variants compared byte for byte."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2106_08759_b200 as S  # noqa: E402

n = 65536
P = S.params(761)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
pk = torch.empty((n, P["pk_bytes"]), dtype=torch.uint8, device="cuda")
sk = torch.empty((n, P["sk_bytes"]), dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
base = S.OPT_ASYNC | S.OPT_RING_STREAMS
variants = {"plain": base, "graph": base | S.OPT_GRAPH}
res = {k: [] for k in variants}
outs = {}
for rnd in range(int(os.environ.get("ROUNDS", "6"))):
    for name, fl in variants.items():
        f = lambda: S.batch_keygen(761, n, 2, batch_size=1024, chunk_keys=32768, pk_out=pk, sk_out=sk, flags=fl, stream=st)
        f()
        torch.cuda.synchronize()
        if rnd == 0:
            outs[name] = (pk.clone(), sk.clone())
        for _ in range(3):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            f()
            e1.record(st)
            torch.cuda.synchronize()
            res[name].append(e0.elapsed_time(e1))
same = all(torch.equal(a, b) for a, b in zip(outs["plain"], outs["graph"]))
out = {k: {"median_ms": statistics.median(v), "keys_per_s": n / statistics.median(v) * 1e3} for k, v in res.items()}
out["graph_equals_plain"] = same
print(json.dumps(out))

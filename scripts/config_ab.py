#!/usr/bin/env python3
"""Alternating-round A/B of keygen launch configurations (B, chunk, flags) on configs[1]
(device outputs, L2 flushed between steps): medians, so clock drift hits every variant alike."""
import os
import statistics
import sys

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
ST, L4 = S.OPT_STAGGER, S.OPT_LANES4
cfgs = [(1024, 32768, R), (1024, 32768, R | ST), (1024, 16384, R | ST | L4), (1024, 16384, ST | L4),
        (1024, 24576, R | ST), (1024, 16384, R | L4)]
if len(sys.argv) > 1:      # B:chunk:flags ...
    cfgs = [tuple(int(x) for x in a.split(":")) for a in sys.argv[1:]]
res = {c: [] for c in cfgs}
for rnd in range(6):
    for c in cfgs:
        B, chunk, fl = c
        f = lambda: S.batch_keygen(761, n, 2, batch_size=B, chunk_keys=chunk, pk_out=pk, sk_out=sk, flags=S.OPT_ASYNC | fl)
        f()
        torch.cuda.synchronize()
        for _ in range(3):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            f()
            e1.record()
            torch.cuda.synchronize()
            res[c].append(e0.elapsed_time(e1))
for c in cfgs:
    ms = statistics.median(res[c])
    print("B=%4d chunk=%6d flags=%3d: median %.3f ms  %.2f M keys/s" % (c[0], c[1], c[2], ms, n / ms / 1e3))

#!/usr/bin/env python3
"""A/B of keygen configurations timed as bench.py times its step: 10 back-to-back asynchronous
calls, L2 flushed before each (not timed), per-call CUDA events, the mean; alternating rounds.
Arguments: B:chunk:flags ..."""
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
cfgs = [tuple(int(x) for x in a.split(":")) for a in sys.argv[1:]] or [(1024, 32768, 16), (2048, 32768, 16)]
res = {c: [] for c in cfgs}
for rnd in range(8):
    for c in cfgs:
        B, chunk, fl = c
        f = lambda: S.batch_keygen(761, n, 2, batch_size=B, chunk_keys=chunk, pk_out=pk, sk_out=sk, flags=S.OPT_ASYNC | fl)
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
        for e0, e1 in ev:
            flush.zero_()
            e0.record()
            f()
            e1.record()
        torch.cuda.synchronize()
        res[c].append(sum(e0.elapsed_time(e1) for e0, e1 in ev) / 10)
for c in cfgs:
    ms = statistics.median(res[c])
    print("B=%4d chunk=%6d flags=%3d: median of means %.3f ms  %.2f M keys/s  (min %.3f max %.3f)" % (
        c[0], c[1], c[2], ms, n / ms / 1e3, min(res[c]), max(res[c])))

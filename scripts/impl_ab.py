#!/usr/bin/env python3
"""Alternating A/B of ring-product implementations on the bench step (configs[1], device outputs,
L2 flushed between steps): medians over rounds, so clock drift hits every variant alike.

  python scripts/impl_ab.py [impl ...]      (default: 0 7 6)
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2106_08759_b200 as S  # noqa: E402

impls = [int(x) for x in sys.argv[1:]] or [0, 7, 6]
n = 65536
P = S.params(761)
pk = torch.empty((n, P["pk_bytes"]), dtype=torch.uint8, device="cuda")
sk = torch.empty((n, P["sk_bytes"]), dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
f = lambda: S.batch_keygen(761, n, 2, batch_size=1024, chunk_keys=32768, pk_out=pk, sk_out=sk,
                           flags=S.OPT_ASYNC | S.OPT_RING_STREAMS)
res = {i: [] for i in impls}
for rnd in range(6):
    for i in impls:
        S.set_mul_impl(i)
        f(); f()
        torch.cuda.synchronize()
        for _ in range(3):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            f()
            e1.record()
            torch.cuda.synchronize()
            res[i].append(e0.elapsed_time(e1))
S.set_mul_impl(0)
for i in impls:
    ms = statistics.median(res[i])
    print("impl %d: median %.3f ms  %.2f M keys/s  (min %.3f)" % (i, ms, n / ms / 1e3, min(res[i])))

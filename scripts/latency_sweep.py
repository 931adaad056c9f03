#!/usr/bin/env python3
"""configs[0] latency (32 sntrup761 keys, seed 1) over the Montgomery batch size B: wall clock of
the synchronous C-ABI call and device time."""
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
for B in (1, 2, 4, 8, 16, 32):
    for fl, tag in ((0, ""), (S.OPT_RING_STREAMS, "+rings")):
        f = lambda: S.batch_keygen(761, 32, 1, batch_size=B, pk_out=pk, sk_out=sk, flags=fl)
        for _ in range(5):
            f()
        torch.cuda.synchronize()
        lat = []
        for _ in range(30):
            t0 = time.perf_counter()
            f()
            lat.append((time.perf_counter() - t0) * 1e6)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g = lambda: S.batch_keygen(761, 32, 1, batch_size=B, pk_out=pk, sk_out=sk, flags=fl | S.OPT_ASYNC)
        e0.record()
        for _ in range(20):
            g()
        e1.record()
        torch.cuda.synchronize()
        print("B=%2d%-7s wall median %6.1f us  device %6.1f us" % (B, tag, statistics.median(lat), e0.elapsed_time(e1) * 1e3 / 20))

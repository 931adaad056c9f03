#!/usr/bin/env python3
"""Host-side cost of one keygen call (enqueue) vs its device time, configs[1] shape."""
import os
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
pkh = torch.empty((n, P["pk_bytes"]), dtype=torch.uint8).pin_memory()
skh = torch.empty((n, P["sk_bytes"]), dtype=torch.uint8).pin_memory()
R = S.OPT_RING_STREAMS
for name, kw in (("device async", dict(pk_out=pk, sk_out=sk, flags=S.OPT_ASYNC | R)),
                 ("host out", dict(pk_out=pkh, sk_out=skh, flags=S.OPT_HOST_OUTPUT | R))):
    for _ in range(3):
        S.batch_keygen(761, n, 2, batch_size=1024, chunk_keys=32768, **kw)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        S.batch_keygen(761, n, 2, batch_size=1024, chunk_keys=32768, **kw)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        ts.append((t1 - t0, t2 - t0))
    c0 = S.kernel_launch_count()
    S.batch_keygen(761, n, 2, batch_size=1024, chunk_keys=32768, **kw)
    torch.cuda.synchronize()
    print("%-14s call returns after %.3f ms, device done after %.3f ms (medians); %d launches" % (
        name, sorted(t[0] for t in ts)[2] * 1e3, sorted(t[1] for t in ts)[2] * 1e3, S.kernel_launch_count() - c0))

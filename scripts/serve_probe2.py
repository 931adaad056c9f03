#!/usr/bin/env python3
"""Serving loop diagnostic: device time of each asynchronous host-output call on the caller's
stream (its lanes join it; copies are off-stream) and the gaps between consecutive calls."""
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
pk = [torch.empty((n, P["pk_bytes"]), dtype=torch.uint8).pin_memory() for _ in range(2)]
sk = [torch.empty((n, P["sk_bytes"]), dtype=torch.uint8).pin_memory() for _ in range(2)]
dpk = torch.empty((n, P["pk_bytes"]), dtype=torch.uint8, device="cuda")
dsk = torch.empty((n, P["sk_bytes"]), dtype=torch.uint8, device="cuda")
evs = [S.Event() for _ in range(2)]


def serve(steps, host=True):
    te = []
    for k in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if host:
            S.batch_keygen(761, n, 2, batch_size=1024, pk_out=pk[k % 2], sk_out=sk[k % 2],
                           flags=S.OPT_HOST_OUTPUT | S.OPT_ASYNC | S.OPT_RING_STREAMS,
                           chunk_keys=32768, done_event=evs[k % 2])
        else:
            S.batch_keygen(761, n, 2, batch_size=1024, pk_out=dpk, sk_out=dsk,
                           flags=S.OPT_ASYNC | S.OPT_RING_STREAMS, chunk_keys=32768)
        e1.record()
        te.append((e0, e1))
        if host and k >= 1:
            evs[(k - 1) % 2].synchronize()
    if host:
        evs[(steps - 1) % 2].synchronize()
    torch.cuda.synchronize()
    return te


for host in (False, True, False, True):
    serve(3, host)
    t0 = time.perf_counter()
    te = serve(30, host)
    wall = time.perf_counter() - t0
    calls = [a.elapsed_time(b) for a, b in te]
    gaps = [te[i][1].elapsed_time(te[i + 1][0]) for i in range(len(te) - 1)]
    span = te[0][0].elapsed_time(te[-1][1])
    print("host_out %d: call device time median %.3f ms (min %.3f max %.3f); gap between calls median %.3f ms max %.3f; "
          "first start to last end %.2f ms = %.3f per call; wall %.2f ms -> %.2f M keys/s" % (
              host, statistics.median(calls), min(calls), max(calls), statistics.median(gaps), max(gaps),
              span, span / 30, wall * 1e3, n * 30 / wall / 1e6), flush=True)

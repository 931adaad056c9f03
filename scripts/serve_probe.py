#!/usr/bin/env python3
"""Key-serving loop (asynchronous host-output calls, bench.py's e2e configuration): keys/s over the
number of steps (the final drain's share), the run-ahead depth (buffer sets), and the host's
enqueue time per call."""
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
NB = 3
pk = [torch.empty((n, P["pk_bytes"]), dtype=torch.uint8).pin_memory() for _ in range(NB)]
sk = [torch.empty((n, P["sk_bytes"]), dtype=torch.uint8).pin_memory() for _ in range(NB)]
evs = [S.Event() for _ in range(NB)]


def serve(steps, depth, fl=S.OPT_RING_STREAMS, chunk=32768, graph=False):
    enq = []
    nb = depth + 1
    for k in range(steps):
        t = time.perf_counter()
        S.batch_keygen(761, n, 2, batch_size=1024, pk_out=pk[k % nb], sk_out=sk[k % nb],
                       flags=S.OPT_HOST_OUTPUT | S.OPT_ASYNC | fl | (S.OPT_GRAPH if graph else 0),
                       chunk_keys=chunk, done_event=evs[k % nb])
        enq.append(time.perf_counter() - t)
        if k >= depth:
            evs[(k - depth) % nb].synchronize()
            _ = int(pk[(k - depth) % nb][0, 0]) + int(sk[(k - depth) % nb][0, 0])
    for j in range(max(steps - depth, 0), steps):
        evs[j % nb].synchronize()
    return enq


for depth in (1, 2):
    for steps in (20, 60):
        for graph in (False,):
            serve(3, depth, graph=graph)
            torch.cuda.synchronize()
            rs = []
            for _ in range(3):
                t0 = time.perf_counter()
                enq = serve(steps, depth, graph=graph)
                rs.append(n * steps / (time.perf_counter() - t0))
            print("depth %d steps %3d graph %d: %.2f M keys/s (median of 3; %s)  host enqueue median %.3f ms max %.3f" % (
                depth, steps, graph, statistics.median(rs) / 1e6, " ".join("%.2f" % (r / 1e6) for r in rs),
                statistics.median(enq) * 1e3, max(enq) * 1e3), flush=True)

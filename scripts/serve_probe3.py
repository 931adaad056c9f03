#!/usr/bin/env python3
"""Does PCIe D2H traffic stretch the keygen call's launch chains?  Device-output keygen calls
(plain enqueue vs CUDA-graph replay) on a side stream while a copy stream moves the previous
step's 100.9 MB to pinned host memory."""
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
dpk = [torch.empty((n, P["pk_bytes"]), dtype=torch.uint8, device="cuda") for _ in range(2)]
dsk = [torch.empty((n, P["sk_bytes"]), dtype=torch.uint8, device="cuda") for _ in range(2)]
hpk = [torch.empty((n, P["pk_bytes"]), dtype=torch.uint8).pin_memory() for _ in range(2)]
hsk = [torch.empty((n, P["sk_bytes"]), dtype=torch.uint8).pin_memory() for _ in range(2)]
cs = torch.cuda.Stream()
ws = torch.cuda.Stream()


def loop(steps, graph, copies):
    te = []
    done = [None, None]
    with torch.cuda.stream(ws):
        for k in range(steps):
            b = k % 2
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if done[b] is not None:
                ws.wait_event(done[b])          # the device buffers' previous copies are done
            e0.record(ws)
            S.batch_keygen(761, n, 2, batch_size=1024, pk_out=dpk[b], sk_out=dsk[b], stream=ws,
                           flags=S.OPT_ASYNC | S.OPT_RING_STREAMS | (S.OPT_GRAPH if graph else 0), chunk_keys=32768)
            e1.record(ws)
            te.append((e0, e1))
            if copies:
                cs.wait_event(e1)
                with torch.cuda.stream(cs):
                    hpk[b].copy_(dpk[b], non_blocking=True)
                    hsk[b].copy_(dsk[b], non_blocking=True)
                    done[b] = torch.cuda.Event()
                    done[b].record(cs)
                if k >= 1 and done[1 - b] is not None:
                    done[1 - b].synchronize()
    torch.cuda.synchronize()
    return te


for graph in (False, True):
    for copies in (False, True):
        loop(3, graph, copies)
        t0 = time.perf_counter()
        te = loop(30, graph, copies)
        wall = time.perf_counter() - t0
        calls = [a.elapsed_time(b) for a, b in te]
        print("graph %d copies %d: call device time median %.3f ms (min %.3f max %.3f); wall %.2f ms -> %.2f M keys/s" % (
            graph, copies, statistics.median(calls), min(calls), max(calls), wall * 1e3, n * 30 / wall / 1e6), flush=True)

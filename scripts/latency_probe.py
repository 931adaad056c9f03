#!/usr/bin/env python3
"""configs[0] (32 sntrup761 keys, B = 1, ring streams): where the synchronous call's time goes --
host enqueue time of an asynchronous call, device span of one isolated call (events on the
caller's stream around it, device idle before), wall clock of the synchronous call, and the
kernels launched per call."""
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
extra = int(os.environ.get("FLAGS", "0"))
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
f = lambda fl: S.batch_keygen(761, 32, 1, batch_size=1, pk_out=pk, sk_out=sk, flags=R | extra | fl, stream=st)
for _ in range(10):
    f(0)
torch.cuda.synchronize()
enq, span, wall = [], [], []
k0 = S.kernel_launch_count()
for _ in range(30):
    torch.cuda.synchronize()
    time.sleep(0.002)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    f(S.OPT_ASYNC)
    enq.append((time.perf_counter() - t0) * 1e6)
    e1.record()
    torch.cuda.synchronize()
    span.append(e0.elapsed_time(e1) * 1e3)
launches = (S.kernel_launch_count() - k0) / 30
for _ in range(30):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f(0)
    wall.append((time.perf_counter() - t0) * 1e6)
r = {"enqueue_us": statistics.median(enq), "device_span_us": statistics.median(span),
     "sync_call_wall_us": statistics.median(wall), "kernels_per_call": launches, "flags": extra}
print(json.dumps(r))

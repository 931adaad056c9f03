#!/usr/bin/env python3
"""Alternating-round A/B of the tree-top scheduling knob (sntrup_set_sched) on configs[1]
(device outputs, L2 flushed between steps).  Arguments: top:cap:flags ... (flags: 16 = ring
streams, + 128 = stagger).  Every variant's pk/sk are compared with the default's."""
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
cfgs = [tuple(int(x) for x in a.split(":")) for a in sys.argv[1:]] or [(0, 0, 16), (1024, 4, 16), (1024, 4, 144)]
res = {c: [] for c in cfgs}
ref = None
for rnd in range(5):
    for c in cfgs:
        top, cap, fl = c
        S.set_sched(top, cap)
        f = lambda: S.batch_keygen(761, n, 2, batch_size=1024, chunk_keys=32768, pk_out=pk, sk_out=sk, flags=S.OPT_ASYNC | fl)
        pk.zero_(); sk.zero_()
        f()
        torch.cuda.synchronize()
        if rnd == 0:
            if ref is None:
                ref = (pk.clone(), sk.clone())
            else:
                assert torch.equal(pk, ref[0]) and torch.equal(sk, ref[1]), ("output differs", c)
        for _ in range(3):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            f()
            e1.record()
            torch.cuda.synchronize()
            res[c].append(e0.elapsed_time(e1))
S.set_sched(0, 0)
for c in cfgs:
    ms = statistics.median(res[c])
    print("top=%5d cap=%3d flags=%3d: median %.3f ms  %.2f M keys/s  (min %.3f)" % (c[0], c[1], c[2], ms, n / ms / 1e3, min(res[c])))

#!/usr/bin/env python3
"""Latency of the root inversions alone: r3_recip_batch / rq_recip_batch on 32 rows with B = 1
(one divstep chain per row, all in parallel), device time per call."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2106_08759_b200 as S  # noqa: E402
from inputs import synth  # noqa: E402

P = S.params(761)
g = torch.from_numpy(synth.small(32, 761, P["p16"], seed=4)).cuda()
a = torch.from_numpy(synth.uniform_rq(32, 761, 4591, P["p8"], seed=1)).cuda()
tests = [("r3_recip B=1", None, lambda: S.r3_recip_batch(761, g, batch_size=1))]
for nt in (128, 256, 512, 768):
    tests.append(("rq_recip B=1 (%d threads/root)" % nt, nt, lambda: S.rq_recip_batch(761, a, batch_size=1)))
ref = S.rq_recip_batch(761, a, batch_size=1).clone()
for name, nt, f in tests:
    if nt:
        S._lib.sntrup_set_divstep_threads(nt)
        assert torch.equal(f(), ref)
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    print("%s: %.1f us per call" % (name, e0.elapsed_time(e1) * 100))
S._lib.sntrup_set_divstep_threads(256)

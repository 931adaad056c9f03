#!/usr/bin/env python3
"""e2e (host outputs) keys/s over chunk sizes and lane options, configs[1] shape."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2106_08759_b200 as S  # noqa: E402

n = 65536
P = S.params(761)
pk = torch.empty((n, P["pk_bytes"]), dtype=torch.uint8).pin_memory()
sk = torch.empty((n, P["sk_bytes"]), dtype=torch.uint8).pin_memory()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
R, PR, L4, ST = S.OPT_RING_STREAMS, S.OPT_LANE_PRIORITY, S.OPT_LANES4, S.OPT_STAGGER
for B in (1024,):
    for chunk in (49152, 40960, 32768, 24576, 20480, 16384):
        for fl, tag in ((R, "rings"), (R | ST, "rings+stagger"), (R | ST | PR, "rings+stagger+prio"),
                        (ST | L4, "stagger+lanes4"), (R | ST | L4, "rings+stagger+lanes4")):
            if (fl & L4) and chunk > 24576:
                continue
            f = lambda: S.batch_keygen(761, n, 2, batch_size=B, chunk_keys=chunk, pk_out=pk, sk_out=sk,
                                       flags=S.OPT_HOST_OUTPUT | fl)
            f()
            ts = []
            for _ in range(4):
                flush.zero_()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                f()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ts.sort()
            ms = ts[1]
            print("B=%4d chunk=%6d %-18s %7.3f ms  %6.2f M keys/s" % (B, chunk, tag, ms, n / ms / 1e3), flush=True)

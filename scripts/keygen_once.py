#!/usr/bin/env python3
"""One timed keygen call for a parameter set (for ncu launch lists of non-default workloads).

  python scripts/keygen_once.py <param> <n> [B] [chunk]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2106_08759_b200 as S  # noqa: E402

ps, n = int(sys.argv[1]), int(sys.argv[2])
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
chunk = int(sys.argv[4]) if len(sys.argv) > 4 else 32768
P = S.params(ps)
pk = torch.empty((n, P["pk_bytes"]), dtype=torch.uint8, device="cuda")
sk = torch.empty((n, P["sk_bytes"]), dtype=torch.uint8, device="cuda")
f = lambda: S.batch_keygen(ps, n, 5, batch_size=B, chunk_keys=chunk, pk_out=pk, sk_out=sk,
                           flags=S.OPT_ASYNC | S.OPT_RING_STREAMS)
f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
f()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print("param %d n %d B %d chunk %d: %.3f ms, %.2f M keys/s" % (ps, n, B, chunk, ms, n / ms / 1e3))

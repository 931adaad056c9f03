#!/usr/bin/env python3
"""One configs[0] keygen call (32 sntrup761 keys, seed 1, B = 1, ring streams) after warm-up, for ncu."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2106_08759_b200 as S  # noqa: E402

P = S.params(761)
pk = torch.empty((32, P["pk_bytes"]), dtype=torch.uint8, device="cuda")
sk = torch.empty((32, P["sk_bytes"]), dtype=torch.uint8, device="cuda")
for _ in range(3):
    S.batch_keygen(761, 32, 1, batch_size=1, pk_out=pk, sk_out=sk, flags=S.OPT_RING_STREAMS)
torch.cuda.synchronize()

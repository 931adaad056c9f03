#!/usr/bin/env python3
"""Per-item phase timing of the shared-memory fp4 ring-product kernel (trace build,
SNTRUP_WS_TRACE): thread 0's clock between the loop's barriers, averaged over CTAs and items, for
R/3 products at p = 761 (r3_mul_batch: one product per item) and at p' = 255 (probe kind 2).

  SNTRUP_GPU_LIB=paper_2106_08759_b200/libsntrup_gpu_trace.so python scripts/tc4_phase_trace.py
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2106_08759_b200 as S  # noqa: E402
from inputs import synth  # noqa: E402

PH = ["stage(!ES)+loop", "barrier 1 (staging done)", "build A/B + barrier 2 + MMA issue",
      "prefetch of the item after next", "MMA wait (thread 0)", "barrier 3", "epilogue", "stage next item"]


def run(fn):
    L = S._lib
    L.sntrup_ws_trace_read.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
    buf = (ctypes.c_uint64 * (160 * 16))()
    fn()
    torch.cuda.synchronize()
    assert L.sntrup_ws_trace_read(1, buf, 160 * 16) > 0, "not a trace build"
    fn()
    torch.cuda.synchronize()
    L.sntrup_ws_trace_read(0, buf, 160 * 16)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(160, 16).astype(np.float64)
    items = a[:, 0].sum()
    per = a[:, 8:16].sum(0) / max(items, 1)
    return {PH[i]: round(per[i], 1) for i in range(8)} | {"cycles_per_item_per_cta": round(per.sum(), 1),
                                                           "items": int(items)}


n = 1 << 18
P = S.params(761)
g = torch.from_numpy(synth.small(n, 761, P["p16"], seed=4)).cuda()
h = torch.from_numpy(synth.small(n, 761, P["p16"], seed=5)).cuda()
c = torch.empty_like(g)
r761 = run(lambda: S.r3_mul_batch(761, g, h, c))
g5 = torch.from_numpy(synth.small(n, 255, 256, seed=8)).cuda()
h5 = torch.from_numpy(synth.small(n, 255, 256, seed=9)).cuda()
c5 = torch.empty_like(g5)
r255 = run(lambda: S.probe_half_mul(2, g5, h5, c5))
print(json.dumps({"r3_761": r761, "r3_255": r255}, indent=1))

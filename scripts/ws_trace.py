#!/usr/bin/env python3
"""Role timing of the warp-specialised ring-product kernels (trace build, SNTRUP_WS_TRACE):
per role, the share of its loop time spent waiting on each hand-off.

  SNTRUP_GPU_LIB=paper_2106_08759_b200/libsntrup_gpu_trace.so python scripts/ws_trace.py [--n N]
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2106_08759_b200 as S  # noqa: E402
from inputs import synth  # noqa: E402

NAMES = {0: "prod wait hfull", 1: "prod wait aempty", 2: "prod total",
         3: "load wait raw", 4: "load wait hempty", 5: "load wait bempty", 6: "load total",
         7: "epi wait accfull", 8: "epi total",
         9: "mma wait bfull", 10: "mma wait accempty", 11: "mma wait afull", 12: "mma total",
         13: "prod LDS+SHF", 14: "prod st+wait::st"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 18)
    ap.add_argument("--which", default="r3")
    a = ap.parse_args()
    L = S._lib
    L.sntrup_ws_trace_read.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
    buf = (ctypes.c_uint64 * (160 * 16))()
    assert L.sntrup_ws_trace_read(1, buf, 160 * 16) > 0, "not a trace build"
    P = S.params(761)
    n = a.n
    g = torch.from_numpy(synth.small(n, 761, P["p16"], seed=4)).cuda()
    h = torch.from_numpy(synth.small(n, 761, P["p16"], seed=5)).cuda()
    c3 = torch.empty_like(g)
    S.set_mul_impl(11)
    S.r3_mul_batch(761, g, h, c3)
    torch.cuda.synchronize()
    L.sntrup_ws_trace_read(1, buf, 160 * 16)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    S.r3_mul_batch(761, g, h, c3)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    L.sntrup_ws_trace_read(0, buf, 160 * 16)
    t = np.array(buf[:], dtype=np.float64).reshape(160, 16)[:148]
    per = t.sum(0) / 148
    items = n / 148
    print("r3 products %d: %.3f ms, %.1f M/s; per SM %.0f items" % (n, ms, n / ms / 1e3, items))
    for k, nm in NAMES.items():
        # each counter sums over the role's warps (lane 0 of each): divide by warps per role
        wr = 4 if (k < 9 or k >= 13) else 1
        print("%-20s %10.0f cycles/item per warp" % (nm, per[k] / wr / items))
    S.set_mul_impl(0)


if __name__ == "__main__":
    main()

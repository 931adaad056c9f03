#!/usr/bin/env python3
"""Keygen step time over (chunk keys, lanes, ring streams, B) for configs[1] (65,536 sntrup761 keys),
device outputs, CUDA-event timed with an L2 flush between steps.  Exploration helper.

  python scripts/step_sweep.py [--n 65536] [--steps 5]
"""
import argparse
import itertools
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2106_08759_b200 as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=65536)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--param", type=int, default=761)
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    P = S.params(args.param)
    n = args.n
    pk = torch.empty((n, P["pk_bytes"]), dtype=torch.uint8, device="cuda")
    sk = torch.empty((n, P["sk_bytes"]), dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    grid = [(B, c, l, r, 0) for B, c, l, r in itertools.product((512, 1024), (65536, 32768, 16384, 8192), (2, 4), (0, 1))
            if not (l == 4 and c > 16384)]
    if args.quick:
        grid = [(1024, 32768, 2, 1, 0), (1024, 32768, 2, 1, 1), (1024, 16384, 4, 0, 0), (1024, 16384, 4, 0, 1),
                (1024, 16384, 2, 1, 1), (512, 32768, 2, 0, 0), (1024, 32768, 2, 0, 1)]
    for B, chunk, lanes, rings, prio in grid:
        fl = S.OPT_ASYNC | (S.OPT_RING_STREAMS if rings else 0) | (S.OPT_LANES4 if lanes == 4 else 0) | \
            (S.OPT_LANE_PRIORITY if prio else 0)
        f = lambda: S.batch_keygen(args.param, n, 2, batch_size=B, pk_out=pk, sk_out=sk, flags=fl, chunk_keys=chunk)
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        tot = 0.0
        for _ in range(args.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            f()
            e1.record(st)
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        ms = tot / args.steps
        print("B=%5d chunk=%6d lanes=%d rings=%d prio=%d  %7.3f ms  %6.2f M keys/s" % (B, chunk, lanes, rings, prio, ms, n / ms / 1e3),
              flush=True)


if __name__ == "__main__":
    main()

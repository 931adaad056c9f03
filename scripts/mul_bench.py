#!/usr/bin/env python3
"""Microbenchmark of the ring-product kernels through the C ABI (rq_mul_batch / r3_mul_batch):
both implementations, CUDA-event timed, inputs resident.  Used for A/B evidence and ncu runs.

  python scripts/mul_bench.py [--param 761] [--n 262144] [--iters 5] [--impl both|tc|school]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2106_08759_b200 as S  # noqa: E402
from inputs import synth  # noqa: E402


def timeit(fn, iters):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--param", type=int, default=761)
    ap.add_argument("--n", type=int, default=1 << 18)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--impl", default="both")
    ap.add_argument("--which", default="rq,rqt,r3")
    args = ap.parse_args()
    P = S.params(args.param)
    p, q = P["p"], P["q"]
    n = args.n
    a = torch.from_numpy(synth.uniform_rq(n, p, q, P["p8"], seed=1)).cuda()
    b = torch.from_numpy(synth.uniform_rq(n, p, q, P["p8"], seed=2)).cuda()
    t = torch.from_numpy(synth.ternary_fast(n, p, P["w"], P["p8"], seed=3)).cuda()
    g = torch.from_numpy(synth.small(n, p, P["p16"], seed=4)).cuda()
    h = torch.from_numpy(synth.small(n, p, P["p16"], seed=5)).cuda()
    c = torch.empty_like(a)
    c3 = torch.empty_like(g)
    impls = {"tc": [S.MUL_TENSOR_CORE], "school": [S.MUL_SCHOOLBOOK]}.get(
        args.impl, [S.MUL_TENSOR_CORE, S.MUL_SCHOOLBOOK])
    if args.impl.replace(",", "").isdigit():
        impls = [int(x) for x in args.impl.split(",")]
    for impl in impls:
        S.set_mul_impl(impl)
        name = {S.MUL_TENSOR_CORE: "tc", S.MUL_SCHOOLBOOK: "schoolbook"}.get(impl, "impl%d" % impl)
        w = args.which.split(",")
        if "rq" in w:
            ms = timeit(lambda: S.rq_mul_batch(args.param, a, b, c), args.iters)
            print("%-10s rq big x big   %8.3f ms  %10.3f M mults/s  %8.1f ns/product" % (name, ms, n / ms / 1e3, ms * 1e6 / n))
        if "rqt" in w:
            ms = timeit(lambda: S.rq_mul_batch(args.param, a, t, c), args.iters)
            print("%-10s rq x ternary   %8.3f ms  %10.3f M mults/s  (rq_mul_batch treats both as big)" % (name, ms, n / ms / 1e3))
        if "rqs" in w:        # big x small entry point (configs[2]'s path); t8 = the ternary rows as int8
            t8 = t[:, :P["p16"]].to(torch.int8).contiguous() if P["p16"] <= t.shape[1] else torch.nn.functional.pad(t, (0, P["p16"] - t.shape[1])).to(torch.int8).contiguous()
            ms = timeit(lambda: S.rq_mul_small_batch(args.param, a, t8, c), args.iters)
            print("%-10s rq big x small %8.3f ms  %10.3f M mults/s" % (name, ms, n / ms / 1e3))
        if "r3" in w:
            ms = timeit(lambda: S.r3_mul_batch(args.param, g, h, c3), args.iters)
            print("%-10s r3             %8.3f ms  %10.3f M mults/s  %8.1f ns/product" % (name, ms, n / ms / 1e3, ms * 1e6 / n))
    S.set_mul_impl(S.MUL_TENSOR_CORE)


if __name__ == "__main__":
    main()

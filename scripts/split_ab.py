#!/usr/bin/env python3
"""A/B for the paper's splitting multipliers (Karatsuba P:4400-5110):
one 761 ring product vs the three 383-coefficient sub-products a one-level Karatsuba split needs,
through the same tensor-core kernels (sntrup_probe_half_mul), CUDA-event timed, 2^20 products.
The split's pre-additions and recombination/fold (elementwise, HBM-bound) are not included, so the
Karatsuba column is a lower bound on its cost."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2106_08759_b200 as S  # noqa: E402
from inputs import synth  # noqa: E402


def timeit(fn, iters=5):
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
    n = 1 << 20
    P = S.params(761)
    out = {}
    g = torch.from_numpy(synth.small(n, 761, P["p16"], seed=4)).cuda()
    h = torch.from_numpy(synth.small(n, 761, P["p16"], seed=5)).cuda()
    c3 = torch.empty_like(g)
    g2 = torch.from_numpy(synth.small(n, 383, 384, seed=6)).cuda()
    h2 = torch.from_numpy(synth.small(n, 383, 384, seed=7)).cuda()
    c2 = torch.empty_like(g2)
    t761 = timeit(lambda: S.r3_mul_batch(761, g, h, c3))
    t383 = timeit(lambda: S.probe_half_mul(0, g2, h2, c2))
    out["r3_fp4"] = {"ms_761_product": t761, "ms_383_product": t383,
                     "karatsuba_lower_bound_ms": 3 * t383, "ratio_karatsuba_over_direct": 3 * t383 / t761}
    # the paper's 5-way R/3 multiplier: 4 sub-products of <= 254 coefficients (run
    # at p' = 255) and H(x) of 256 (p' = 257)
    g5 = torch.from_numpy(synth.small(n, 255, 256, seed=8)).cuda()
    h5 = torch.from_numpy(synth.small(n, 255, 256, seed=9)).cuda()
    c5 = torch.empty_like(g5)
    g7 = torch.from_numpy(synth.small(n, 257, 272, seed=10)).cuda()
    h7 = torch.from_numpy(synth.small(n, 257, 272, seed=11)).cuda()
    c7 = torch.empty_like(g7)
    t255 = timeit(lambda: S.probe_half_mul(2, g5, h5, c5))
    t257 = timeit(lambda: S.probe_half_mul(3, g7, h7, c7))
    out["r3_fp4_5way"] = {"ms_761_product": t761, "ms_255_product": t255, "ms_257_product": t257,
                          "five_way_lower_bound_ms": 4 * t255 + t257,
                          "ratio_five_way_over_direct": (4 * t255 + t257) / t761}
    del g, h, c3, g2, h2, c2, g5, h5, c5, g7, h7, c7
    a = torch.from_numpy(synth.uniform_rq(n, 761, 4591, P["p8"], seed=1)).cuda()
    b = torch.from_numpy(synth.uniform_rq(n, 761, 4591, P["p8"], seed=2)).cuda()
    c = torch.empty_like(a)
    a2 = torch.from_numpy(synth.uniform_rq(n, 383, 4591, 384, seed=3)).cuda()
    b2 = torch.from_numpy(synth.uniform_rq(n, 383, 4591, 384, seed=4)).cuda()
    c2 = torch.empty_like(a2)
    t761 = timeit(lambda: S.rq_mul_batch(761, a, b, c))
    t383 = timeit(lambda: S.probe_half_mul(1, a2, b2, c2))
    out["rq_int8_big_x_big"] = {"ms_761_product": t761, "ms_383_product": t383,
                                "karatsuba_lower_bound_ms": 3 * t383, "ratio_karatsuba_over_direct": 3 * t383 / t761}
    out["note"] = ("2^20 products each; one-level Karatsuba = 3 sub-products of 383 coefficients; the 5-way "
                   "R/3 split = 4 of <= 254 (run at 255) + 1 of 256 (run at 257); elementwise pre-adds, "
                   "interpolation and the x^2-1 divisions not counted")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

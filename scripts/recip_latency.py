#!/usr/bin/env python3
"""Latency of the root inversions alone: r3_recip_batch / rq_recip_batch on 32 rows with B = 1
(one inversion chain per row, all in parallel), device time per call, per parameter set; the R/q
root by jump-divsteps (default) and by one divstep per barrier (sntrup_set_root_impl(1)).  Each
variant's output is compared with the other's before timing."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2106_08759_b200 as S  # noqa: E402
from inputs import synth  # noqa: E402


def timed(f, reps=10):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000.0 / reps


res = {}
for ps in [int(x) for x in (sys.argv[1:] or ["653", "761", "857", "953", "1013", "1277"])]:
    P = S.params(ps)
    g = torch.from_numpy(synth.small(32, P["p"], P["p16"], seed=4)).cuda()
    a = torch.from_numpy(synth.uniform_rq(32, P["p"], P["q"], P["p8"], seed=1)).cuda()
    r = {}
    o3 = {}
    for name, impl in (("jump", S.ROOT_JUMP), ("step", S.ROOT_STEP)):
        S.set_root_impl(impl)
        o3[name] = [x.clone() for x in S.r3_recip_batch(ps, g, batch_size=1)]
        r["r3_recip_B1_us_" + name] = timed(lambda: S.r3_recip_batch(ps, g, batch_size=1))
    r["r3_jump_equals_step"] = all(bool(torch.equal(x, y)) for x, y in zip(o3["jump"], o3["step"]))
    outs = {}
    for name, impl in (("jump", S.ROOT_JUMP), ("step", S.ROOT_STEP)):
        S.set_root_impl(impl)
        outs[name] = S.rq_recip_batch(ps, a, batch_size=1).clone()
        r["rq_recip_B1_us_" + name] = timed(lambda: S.rq_recip_batch(ps, a, batch_size=1))
    S.set_root_impl(S.ROOT_AUTO)
    r["rq_jump_equals_step"] = bool(torch.equal(outs["jump"], outs["step"]))
    res[ps] = r
    print(ps, json.dumps(r), flush=True)
print(json.dumps(res))

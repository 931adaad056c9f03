#!/usr/bin/env python3
"""Small invocations of every entry point for compute-sanitizer runs (config-1 sized)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2106_08759_b200 as S  # noqa: E402
from inputs import synth  # noqa: E402

for impl in (S.MUL_TENSOR_CORE, S.MUL_TENSOR_CORE_INT8, S.MUL_TENSOR_CORE_FP4_ALL, S.MUL_TENSOR_CORE_M64):
    S.set_mul_impl(impl)
    S.batch_keygen(761, 32, 1, batch_size=32, debug=True)                      # configs[0]
    for ps in (953, 1277):                                                     # no fix row / big smem
        S.batch_keygen(ps, 64, 2, batch_size=16, chunk_keys=32, debug=True, flags=S.OPT_RING_STREAMS)
    r = S.batch_keygen(761, 64, 3, batch_size=16, chunk_keys=16, debug=True, flags=S.OPT_LANES4)
    S.full_sk_batch(761, 3, r["pk"], r["sk"])
    rr = S.sample_short_batch(761, 64, 3)
    c = S.encap_core_batch(761, r["h"], rr)
    S.decap_core_batch(761, r["f"], r["ginv"], c)
    S.batch_keygen(653, 96, 4, batch_size=16, chunk_keys=48, debug=True,       # 2 lanes, repair
                   flags=S.OPT_NO_SMALL_CHECK)
    P = S.params(761)
    a = torch.from_numpy(synth.uniform_rq(8, 761, 4591, P["p8"], seed=1)).cuda()
    b = torch.from_numpy(synth.uniform_rq(8, 761, 4591, P["p8"], seed=2)).cuda()
    S.rq_mul_batch(761, a, b)
    S.rq_mul_small_batch(761, a, torch.from_numpy(synth.small(8, 761, P["p16"], seed=3)).cuda())
    S.rq_recip_batch(761, a, batch_size=4)
    g = torch.from_numpy(synth.small(8, 761, P["p16"], seed=4)).cuda()
    S.r3_recip_batch(761, g, batch_size=4)
    S.r3_mul_batch(761, g, g)
torch.cuda.synchronize()
print("sanitize_small ok")

#!/usr/bin/env python3
"""One rq_recip_batch / r3_recip_batch call on 32 rows with B = 1 (for ncu): argv = param set,
root impl (0 jump, 1 step), ring ('q' or '3')."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2106_08759_b200 as S  # noqa: E402
from inputs import synth  # noqa: E402

ps = int(sys.argv[1]) if len(sys.argv) > 1 else 761
impl = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ring = sys.argv[3] if len(sys.argv) > 3 else "q"
P = S.params(ps)
S.set_root_impl(impl)
if ring == "q":
    a = torch.from_numpy(synth.uniform_rq(32, P["p"], P["q"], P["p8"], seed=1)).cuda()
    for _ in range(2):
        S.rq_recip_batch(ps, a, batch_size=1)
else:
    g = torch.from_numpy(synth.small(32, P["p"], P["p16"], seed=4)).cuda()
    for _ in range(2):
        S.r3_recip_batch(ps, g, batch_size=1)
torch.cuda.synchronize()

#!/usr/bin/env python3
"""Per-jump phase timing of the jump-divstep decision warp (root 0), from the trace build
(SNTRUP_GPU_LIB=.../libsntrup_gpu_jt.so): decide, wait for the f, g application of the previous
jump, publish U, prep of the next window."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2106_08759_b200 as S  # noqa: E402
from inputs import synth  # noqa: E402

P = S.params(761)
a = torch.from_numpy(synth.uniform_rq(32, 761, 4591, P["p8"], seed=1)).cuda()
for _ in range(3):
    S.rq_recip_batch(761, a, batch_size=1)
torch.cuda.synchronize()
buf = np.zeros(1024, dtype=np.int64)
S._lib.sntrup_debug_jump_trace(buf.ctypes.data_as(ctypes.c_void_p), 1024)
t = buf.reshape(128, 8)[:50]
dec = t[:, 1] - t[:, 0]
wait = t[:, 2] - t[:, 1]
pub_prep = t[:, 3] - t[:, 2]
per = np.diff(t[:, 0])
print("cycles per jump: decide %.0f  wait(f,g applied) %.0f  publish+prep %.0f  total %.0f (median %.0f)" % (
    dec.mean(), wait.mean(), pub_prep.mean(), per.mean(), np.median(per)))
print("publish to CTA 1: %.0f  f,g apply (warp 1): %.0f  apply start after bar.arrive(1)->prep end: %.0f" % (
    (t[:, 4] - t[:, 1]).mean(), (t[:, 6] - t[:, 5]).mean(), (t[:, 3] - t[:, 5]).mean()))
print("decide per jump:", dec[:8], "... wait:", wait[:8], "... pub+prep:", pub_prep[:8])
t0 = t[0, 0]
for k in range(6):
    print(k, [int(x - t0) for x in t[k]])

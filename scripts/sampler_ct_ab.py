#!/usr/bin/env python3
"""Sampler time per key with the small-factor test forced on (653, 1013, 1277, 65,536 keys), from
the library's per-class CUDA-event profile; run once per library build (SNTRUP_GPU_LIB) to A/B
the constant-time residue test against the old data-dependent one."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2106_08759_b200 as S  # noqa: E402

for ps in (653, 1013, 1277):
    n = 65536
    f = lambda: S.batch_keygen(ps, n, 4, batch_size=1024, chunk_keys=32768,
                               flags=S.OPT_FORCE_SMALL_CHECK | S.OPT_SERIAL)
    f()
    torch.cuda.synchronize()
    S.profile_enable(True)
    for _ in range(3):
        f()
    prof = S.profile_read(reset=True)
    S.profile_enable(False)
    print("%s %d: sampler %.3f ms per 65,536 keys (%.1f ns/key)" % (os.path.basename(S.library_path()), ps,
          prof["sample"]["ms"] / 3, prof["sample"]["ms"] / 3 / n * 1e6))

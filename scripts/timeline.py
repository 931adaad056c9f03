#!/usr/bin/env python3
"""Timeline of one bench step (configs[1], overlapped lanes) from the library's per-launch events
(SNTRUP_TIMELINE): per stream, when each launch became runnable and when it finished.  Shows how
long the latency-bound launches of one lane (tree tops, roots) queue behind the other lane's
persistent bulk kernels.

  python scripts/timeline.py [out.csv] [B] [chunk]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/timeline.csv"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
chunk = int(sys.argv[3]) if len(sys.argv) > 3 else 32768
extra = int(sys.argv[4]) if len(sys.argv) > 4 else 0
if os.path.exists(out):
    os.remove(out)
os.environ["SNTRUP_TIMELINE"] = out
import torch  # noqa: E402

import paper_2106_08759_b200 as S  # noqa: E402

n = 65536
P = S.params(761)
pk = torch.empty((n, P["pk_bytes"]), dtype=torch.uint8, device="cuda")
sk = torch.empty((n, P["sk_bytes"]), dtype=torch.uint8, device="cuda")
f = lambda: S.batch_keygen(761, n, 2, batch_size=B, chunk_keys=chunk, pk_out=pk, sk_out=sk,
                           flags=S.OPT_ASYNC | S.OPT_RING_STREAMS | extra)
for _ in range(3):
    f()
torch.cuda.synchronize()
S.profile_enable(True)
f()
torch.cuda.synchronize()
S.profile_read(True)
S.profile_enable(False)
rows = [l.strip().split(",") for l in open(out) if not l.startswith("#")]
names = S.PROFILE_CLASSES
streams = {}
for r in rows:
    streams.setdefault(r[3], []).append(r)
t_end = max(float(r[5]) for r in rows)
print("step: %.3f ms, %d launches on %d streams" % (t_end, len(rows), len(streams)))
for sid, rs in streams.items():
    busy = sum(float(r[5]) - float(r[4]) for r in rs)
    print("stream %s: %d launches, first %.3f last %.3f, sum(end-start) %.3f ms" % (
        sid, len(rs), float(rs[0][4]), float(rs[-1][5]), busy))
    for r in rs:
        print("   %-8s kind %2s units %8s  runnable %.3f  done %.3f  (%.1f us)" % (
            names[int(r[0])], r[1], r[2], float(r[4]), float(r[5]), 1e3 * (float(r[5]) - float(r[4]))))

"""Write the full-size parity digests under tests/golden/oracle_digests/ -- calls ONLY oracle/.

For every key of BASELINE.json configs[1] (sntrup761, 65,536 keys, seed 2), configs[3]
(653/857/953/1013, 65,536 keys each, seed 4) and configs[4] (sntrup1277, 2^20 keys, seed 5), and
for every pair of configs[2] (2^20 R/q products, inputs per SURVEY.md C12, seed 3), the oracle
computes the plain definition one key / pair at a time (oracle/sntrup_oracle.c).  The outputs are
too large to commit, so the file stores, per group of consecutive keys (pairs):
  keygen:  sha256(pk rows || sk rows) and sha256(attempts as uint8) of the group, plus the
           number of extra g draws (rejections) per group;
  rq_mul:  sha256 of the group's a, b and c rows (int16 / int8, p coefficients, little endian).
tests/test_gpu_parity.py recomputes the same digests from the CUDA path's outputs at the bench's
launch configuration and compares group by group.  Resumable: groups already present are kept.

  python scripts/gen_oracle_digests.py [--only NAME ...] [--threads T]
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "oracle_digests")

KEYGEN_JOBS = {   # name: (param, seed, n_keys, keys per group)      BASELINE.json configs[...]
    "cfg1_761": (761, 2, 65536, 1024),      # configs[1]
    "cfg3_653": (653, 4, 65536, 1024),      # configs[3]
    "cfg3_857": (857, 4, 65536, 1024),
    "cfg3_953": (953, 4, 65536, 1024),
    "cfg3_1013": (1013, 4, 65536, 1024),
    "cfg4_1277": (1277, 5, 1 << 20, 8192),  # configs[4]
}
RQ_JOBS = {"cfg2_761": (761, 3, 1 << 20, 16384)}   # configs[2]: pairs (a from domain 0, b from 1)


def _load(path):
    if os.path.exists(path):
        return json.load(open(path))
    return None


def _save(path, d):
    tmp = path + ".tmp"
    with open(tmp, "w") as fh:
        json.dump(d, fh, indent=0)
    os.replace(tmp, path)


def run_keygen(name, threads):
    param, seed, n, G = KEYGEN_JOBS[name]
    path = os.path.join(OUT, name + ".json")
    d = _load(path) or dict(kind="keygen", param=param, seed=seed, n_keys=n, group=G,
                            pk_bytes=O.pk_bytes(param), sk_bytes=O.sk_bytes(param),
                            digest="sha256(pk[g*G:(g+1)*G] rows || sk[...] rows)",
                            attempts_digest="sha256(uint8 attempts of the group)",
                            groups=[])
    t0 = time.time()
    for g in range(len(d["groups"]), n // G):
        r = O.keygen_many(param, seed, np.arange(g * G, (g + 1) * G), threads=threads)
        att = r["attempts"].astype(np.uint8)
        d["groups"].append(dict(
            kv=hashlib.sha256(r["pk"].tobytes() + r["sk"].tobytes()).hexdigest(),
            att=hashlib.sha256(att.tobytes()).hexdigest(),
            rej=int(r["attempts"].sum()) - G))
        _save(path, d)
        print("%s group %d/%d  %.0f s" % (name, g + 1, n // G, time.time() - t0), flush=True)


def run_rq(name, threads):
    param, seed, n, G = RQ_JOBS[name]
    p, q, w = O.PARAMS[param]
    path = os.path.join(OUT, name + ".json")
    d = _load(path) or dict(kind="rq_mul", param=param, seed=seed, n_pairs=n, group=G,
                            inputs="C12: K_i = SM(seed, i); a from domain 0 (uniform), "
                                   "b from domain 1 (Short, weight w)",
                            digest="sha256 of the group's rows, p coefficients each "
                                   "(a, c int16 LE; b int8)",
                            groups=[])
    t0 = time.time()
    for g in range(len(d["groups"]), n // G):
        A = np.zeros((G, p), np.int16); B = np.zeros((G, p), np.int8)
        for j in range(G):
            A[j], B[j] = O.c12_pair(param, seed, g * G + j)
        C = O.mul_many(p, q, A, B.astype(np.int16), threads=threads)
        d["groups"].append(dict(a=hashlib.sha256(A.tobytes()).hexdigest(),
                                b=hashlib.sha256(B.tobytes()).hexdigest(),
                                c=hashlib.sha256(C.tobytes()).hexdigest()))
        _save(path, d)
        print("%s group %d/%d  %.0f s" % (name, g + 1, n // G, time.time() - t0), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*", default=None)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    names = a.only or (list(KEYGEN_JOBS)[:1] + list(RQ_JOBS) + list(KEYGEN_JOBS)[1:])
    for name in names:
        (run_rq if name in RQ_JOBS else run_keygen)(name, a.threads)


if __name__ == "__main__":
    main()

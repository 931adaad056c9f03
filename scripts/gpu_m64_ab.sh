cd $GRAFT_REPO_ROOT
python scripts/impl_ab.py 0 5 2>&1 | tail -2
python - <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_2106_08759_b200 as S
from inputs import synth
P = S.params(761)
n = 1 << 18
a = torch.from_numpy(synth.uniform_rq(n, 761, 4591, P["p8"], seed=1)).cuda()
b = torch.from_numpy(synth.uniform_rq(n, 761, 4591, P["p8"], seed=2)).cuda()
c = torch.empty_like(a)
for impl in (0, 5, 0, 5):
    S.set_mul_impl(impl)
    S.rq_mul_batch(761, a, b, c); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): S.rq_mul_batch(761, a, b, c)
    e1.record(); torch.cuda.synchronize()
    print("impl", impl, "big x big %.1f M/s" % (n * 5 / e0.elapsed_time(e1) / 1e3))
S.set_mul_impl(0)
PY

cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "tc_pipe" 2>&1 | tail -2
python - <<'PY'
import sys; sys.path.insert(0,'.')
import torch, paper_2106_08759_b200 as S
from inputs import synth
P=S.params(761); n=1<<18
a=torch.from_numpy(synth.uniform_rq(n,761,4591,P["p8"],seed=1)).cuda(); b=torch.from_numpy(synth.uniform_rq(n,761,4591,P["p8"],seed=2)).cuda()
c=torch.empty_like(a)
for impl in (0,8,0,8):
    S.set_mul_impl(impl); S.rq_mul_batch(761,a,b,c); torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): S.rq_mul_batch(761,a,b,c)
    e1.record(); torch.cuda.synchronize()
    print("impl",impl,"big x big ZIP %.1f M/s" % (n*5/e0.elapsed_time(e1)/1e3))
PY
python scripts/impl_ab.py 0 8

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat > /tmp/pipe_one.py <<'PY'
import sys; sys.path.insert(0,'.')
import torch, paper_2106_08759_b200 as S
from inputs import synth
P=S.params(761); n=1<<16
a=torch.from_numpy(synth.uniform_rq(n,761,4591,P["p8"],seed=1)).cuda(); b=torch.from_numpy(synth.uniform_rq(n,761,4591,P["p8"],seed=2)).cuda()
c=torch.empty_like(a)
S.set_mul_impl(int(sys.argv[1])); S.rq_mul_batch(761,a,b,c); torch.cuda.synchronize()
PY
python /tmp/pipe_one.py 8 && ncu -f --set full --clock-control none -k regex:tc_mul_kernel -c 1 -o /tmp/prof_pipe python /tmp/pipe_one.py 8 > gpurun_out/ncu_pipe.log 2>&1
ncu -i /tmp/prof_pipe.ncu-rep --page details --csv > gpurun_out/details_pipe.csv 2>&1
ncu -i /tmp/prof_pipe.ncu-rep --page raw --csv > gpurun_out/raw_pipe.csv 2>&1

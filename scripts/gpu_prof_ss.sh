# ncu full captures of the SS fp4 R/3 kernel at p = 761 and p' = 383 (one launch each)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat > /tmp/ss_two.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2106_08759_b200 as S
from inputs import synth
n = 1 << 18
P = S.params(761)
g = torch.from_numpy(synth.small(n, 761, P["p16"], seed=4)).cuda()
h = torch.from_numpy(synth.small(n, 761, P["p16"], seed=5)).cuda()
S.r3_mul_batch(761, g, h)
g2 = torch.from_numpy(synth.small(n, 383, 384, seed=6)).cuda()
h2 = torch.from_numpy(synth.small(n, 383, 384, seed=7)).cuda()
c2 = torch.empty_like(g2)
S.probe_half_mul(0, g2, h2, c2)
torch.cuda.synchronize()
PY
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:tc4_mul_kernel -c 2 -o /tmp/prof_ss python /tmp/ss_two.py > gpurun_out/ncu_ss.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/prof_ss.ncu-rep --page raw --csv > gpurun_out/raw_ss.csv 2>&1
cp /tmp/prof_ss.ncu-rep gpurun_out/

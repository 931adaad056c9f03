import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_08759_b200 as S
from inputs import synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
P = S.params(761)
g = torch.from_numpy(synth.small(n, 761, P["p16"], seed=4)).cuda()
h = torch.from_numpy(synth.small(n, 761, P["p16"], seed=5)).cuda()
S.set_mul_impl(11)
c = S.r3_mul_batch(761, g, h)
torch.cuda.synchronize()
S.set_mul_impl(0)
c0 = S.r3_mul_batch(761, g, h)
torch.cuda.synchronize()
print("n", n, "equal", torch.equal(c, c0))

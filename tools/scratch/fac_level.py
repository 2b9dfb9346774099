import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2309_11488_b200 as P
from paper_2309_11488_b200 import _device as D
from paper_2309_11488_b200.bridge import plan_device
from paper_2309_11488_b200.ilu0 import factor_device
a = P.generate(P.GeneratorSpec(100, 100, 100, seed=0)).a
bsr = D.DevBSR.upload(a)
plan = plan_device(P.Backend.LEVEL_SCHEDULED, bsr.pat)
for _ in range(3):
    f = factor_device(a, plan, bsr)
torch.cuda.synchronize()

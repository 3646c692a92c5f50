import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2312_12771_b200 import workloads as W
from paper_2312_12771_b200.hom import Homogenizer
torch.cuda.set_device(0)
nel = int(sys.argv[1])
h = Homogenizer.from_workload(W.config2(nel=nel, r=4))
C = h.condense()
u, info = h.macro_solve(C)
torch.cuda.synchronize()
print("nel", nel, "it", info.iterations)

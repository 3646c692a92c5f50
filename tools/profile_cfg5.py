"""Minimal driver for ncu: config 5 Newton iterations at a mid-load state (the bench's step)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_12771_b200 import workloads as W  # noqa: E402
from paper_2312_12771_b200.hom import Homogenizer  # noqa: E402

wl = W.config5()
h = Homogenizer.from_workload(wl)
u, _ = h.newton(1, tol=1e-9)
F = h.macro_kinematics(u)
for _ in range(2):
    h.condense(F)
torch.cuda.synchronize()
print("ok")

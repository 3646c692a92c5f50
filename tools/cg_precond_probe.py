"""Macro solve time, two-level vs node-block Jacobi PCG, on 2-D (config 2 type) and 3-D (config 4 type)
macro meshes of growing size (small RVEs: only the macro solve matters).  usage: python tools/cg_precond_probe.py"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_12771_b200 import workloads as W  # noqa: E402
from paper_2312_12771_b200.hom import Homogenizer  # noqa: E402

torch.cuda.set_device(0)
cases = [(3, n) for n in (4, 6, 8, 10, 13, 16)] + [(2, n) for n in (16, 24, 32, 45, 64)]
for dim, nel in cases:
    for pc in ("two_level", "jacobi"):
        wl = W.config4(nel=nel, r=2) if dim == 3 else W.config2(nel=nel, r=4)
        h = Homogenizer.from_workload(wl, macro_precond=pc)
        C = h.condense()
        for _ in range(2):
            u, info = h.macro_solve(C)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            u, info = h.macro_solve(C)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 5 * 1e3
        print(f"dim {dim} nel {nel} dofs {wl.n_dof} {pc:9s} it {info.iterations:4d} solve {dt:.3f} ms", flush=True)
        h.close()

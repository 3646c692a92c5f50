"""Small invocations of every device path (an all-paths smoke run; compute-sanitizer -- memcheck / racecheck / synccheck /
initcheck -- is closed on this GPU pool): linear dense + tile-sparse (2-D, 3-D), constant basis, finite strain (kind 1, 2),
1-D, the grid-wide PCG, SpMV, RVE sharding."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_12771_b200 import workloads as W  # noqa: E402
from paper_2312_12771_b200.hom import Homogenizer  # noqa: E402

torch.cuda.set_device(0)
for wl, kw in [(W.config1(), {}), (W.config2(nel=4, r=8), {"tile_sparse": True}), (W.config4(nel=2, r=4), {}),
               (W.config3(nel=2, r=6), {"macro_basis": "constant"}), (W.bench1d(3), {})]:
    h = Homogenizer.from_workload(wl, **kw)
    C, u, w, info = h.solve_linear()
    y = h.macro_spmv(u)
    torch.cuda.synchronize()
    h.close()
# RVE sharding: a local range condenses / recovers only its rows (C of the rest from a full context)
wl = W.config2(nel=4, r=8)
full = Homogenizer.from_workload(wl)
C, u, w, info = full.solve_linear()
h = Homogenizer.from_workload(wl, rve_range=(8, 24))
h.condense(None, C)
h.recover(u, w)
torch.cuda.synchronize()
h.close()
full.close()
for wl in (W.config5(nel=2, r=6, n_steps=1), W.cook(nel=2, r=6, n_steps=1)):
    h = Homogenizer.from_workload(wl, tile_sparse=True)
    h.newton(1, tol=1e-9, micro_tol=float("inf"), force_load=wl.kind == "mr")
    torch.cuda.synchronize()
    h.close()
wl = W.config2(nel=128, r=2)  # grid-wide PCG path
h = Homogenizer.from_workload(wl)
h.solve_linear()
torch.cuda.synchronize()
print("paths ok")

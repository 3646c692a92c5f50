HOM_CG_VERBOSE=1 python tools/cg_scaling_probe.py 181 2>&1 | grep -v slices
HOM_CG_FORCE_GRID=1 HOM_CG_VERBOSE=1 python tools/cg_scaling_probe.py 32 64 2>&1 | grep -v slices
python - <<'PY'
import os, numpy as np
os.environ["HOM_CG_FORCE_GRID"] = "1"
import oracle
from paper_2312_12771_b200 import workloads as W
from paper_2312_12771_b200.hom import Homogenizer
for nel in (32, 64):
    wl = W.config2(nel=nel, r=4)
    h = Homogenizer.from_workload(wl)
    C, u, w, info = h.solve_linear()
    o = oracle.macro_solve(2, nel, C.cpu().numpy(), wl.dir_dof, wl.dir_val, body=wl.body)
    uu = u.cpu().numpy()
    print("grid path nel", nel, "it", info.iterations, "rel err vs direct", np.linalg.norm(uu - o) / np.linalg.norm(o))
PY

import json, sys, torch
sys.path.insert(0, ".")
import bench
from paper_2312_12771_b200 import workloads as W
torch.cuda.set_device(0)
lam, mu = 0.3 / (1.3 * 0.4), 1.0 / 2.6
C = torch.tensor([[[lam + 2 * mu, lam, 0.0], [lam, lam + 2 * mu, 0.0], [0.0, 0.0, mu]]], dtype=torch.float64, device="cuda")
print(json.dumps(bench.spmv_scaled(C, int(sys.argv[1]) if len(sys.argv) > 1 else 2048)))

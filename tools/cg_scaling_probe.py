import sys, time, torch
sys.path.insert(0, "/root/repo")
from paper_2312_12771_b200 import workloads as W
from paper_2312_12771_b200.hom import Homogenizer
torch.cuda.set_device(0)
for nel in [int(a) for a in sys.argv[1:]] or (32, 45, 64, 91):
    wl = W.config2(nel=nel, r=4)  # small RVEs: only the macro solve matters here
    h = Homogenizer.from_workload(wl)
    C = h.condense()
    for _ in range(2): u, info = h.macro_solve(C)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(5): u, info = h.macro_solve(C)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 5 * 1e3
    print(f"nel {nel} dofs {wl.n_dof} cg it {info.iterations} solve {dt:.2f} ms ({dt*1e3/max(info.iterations,1):.2f} us/it)", flush=True)
    print("   slices", h._ctx_info() if hasattr(h, "_ctx_info") else "", flush=True)
    h.close()

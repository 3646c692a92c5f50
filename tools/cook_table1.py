"""Cook's membrane (§4.2) on the GPU: Newton iterations per load step of the
generalized (null-space) and the classical (staggered) scheme for n_l in {2, 12, 22, 32, 42}
(Table 1) and the residual histories of load steps 1 and 22 at n_l = 22 (Table 2).

  python tools/cook_table1.py [--nl 2 12 22 32 42] [--json out.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2312_12771_b200 import workloads as W  # noqa: E402
from paper_2312_12771_b200.hom import Homogenizer  # noqa: E402


def run(n_l, scheme, tile_sparse=True, nel=20, r=30, predictor=True):
    wl = W.cook(nel=nel, r=r, n_steps=n_l)
    h = Homogenizer.from_workload(wl, tile_sparse=tile_sparse, check_info=True)
    t0 = time.perf_counter()
    if scheme == "generalized":
        _, hist = h.newton(n_l, tol=1e-9, micro_tol=float("inf"), max_iter=30, force_load=True,
                           raise_on_fail=False)
        ok = len(hist) == n_l and hist[-1][-1][0] <= 1e-9
        iters = [len(s) - 1 for s in hist]
        hist_out = [[x[0] for x in s] for s in hist]
    else:
        _, hist, ok = h.newton_classical(n_l, tol=1e-9, micro_tol=1e-13, max_iter=30, max_inner=30,
                                         predictor=predictor)
        iters = [len(s) - 1 for s in hist]
        hist_out = [[(x[0], x[1]) for x in s] for s in hist]
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    h.close()
    return {"n_l": n_l, "scheme": scheme, "converged": bool(ok), "iterations_per_step": iters,
            "failed_at_step": None if ok else len(hist), "seconds": dt, "history": hist_out}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--nl", type=int, nargs="*", default=[2, 12, 22, 32, 42])
    ap.add_argument("--json", default=None)
    ap.add_argument("--dense", action="store_true")
    ap.add_argument("--no-predictor", action="store_true", help="classical variant without the eq:reduction update")
    ap.add_argument("--schemes", nargs="*", default=["generalized", "classical"])
    a = ap.parse_args()
    torch.cuda.set_device(0)
    res = []
    for scheme in a.schemes:
        for n_l in a.nl:
            r = run(n_l, scheme, tile_sparse=not a.dense, predictor=not a.no_predictor)
            res.append(r)
            its = r["iterations_per_step"]
            print(f"{scheme:11s} n_l={n_l:2d} converged={r['converged']!s:5s} iterations/step "
                  f"min {min(its)} max {max(its)} (first {its[:3]}) failed_at_step={r['failed_at_step']} "
                  f"{r['seconds']:.1f} s", flush=True)
            if n_l == 22:
                for k in (0, -1):
                    if len(r["history"]) > (k if k >= 0 else len(r["history"]) + k):
                        hs = r["history"][k]
                        if scheme == "generalized":
                            print(f"   step {k % n_l + 1} ||R_macro||: " + ", ".join(f"{x:.2e}" for x in hs))
                        else:
                            print(f"   step {k % n_l + 1} ||R_macro|| (inner max ||r_f||): " +
                                  "; ".join(f"{x[0]:.2e} ({', '.join(f'{y:.1e}' for y in x[1])})" for x in hs))
    if a.json:
        with open(a.json, "w") as f:
            json.dump(res, f)

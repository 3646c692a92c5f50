"""Measured GPU-vs-oracle errors for the five configs (relative Frobenius norms), dense and
tile-sparse factorisation; writes one line per case.  Test infrastructure (uses oracle/).

  python tools/parity_report.py > profiles/r01/parity_r01.txt
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402
from paper_2312_12771_b200 import workloads as W  # noqa: E402
from paper_2312_12771_b200.hom import Homogenizer  # noqa: E402


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0))


def linear(name, wl, sample=None):
    for ts in (False, True):
        t0 = time.perf_counter()
        h = Homogenizer.from_workload(wl, tile_sparse=ts)
        C, u, w, info = h.solve_linear()
        C, u, w = C.cpu().numpy(), u.cpu().numpy(), w.cpu().numpy()
        if sample is None:
            o = oracle.solve_linear(wl)
            eC = rel(C, o["C_eff"])
            eu = rel(u, o["u"])
            ew = rel(w, oracle.recover_linear(o["W"], o["eps"]))
        else:
            o = oracle.solve_linear(wl, rve_ids=sample)
            eC = rel(C[sample], o["C_eff_subset"])
            ud = oracle.macro_solve(wl.dim, wl.nel, C, wl.dir_dof, wl.dir_val, body=wl.body)
            eu = rel(u, ud)
            eps = oracle.macro_kin(wl.dim, wl.nel, u)
            ew = rel(w[sample], oracle.recover_linear(o["W_subset"], eps[sample]))
        print(f"{name:28s} {'tile-sparse' if ts else 'dense':11s} B={wl.n_rve:6d} C_eff {eC:.2e}  u {eu:.2e}  "
              f"w {ew:.2e}  CG {info.iterations:4d} it rel.res {info.rel_residual:.1e}  "
              f"({'sampled ' + str(len(sample)) + ' RVEs' if sample is not None else 'all RVEs'}; "
              f"{time.perf_counter() - t0:.1f} s)", flush=True)
        h.close()


def finite_per_state(name, wl):
    import torch
    steps = oracle.newton_nh(wl, steps=1)
    u, w = steps[-1]["u"], steps[-1]["w"]
    rng = np.random.default_rng(1)
    w = w + 1e-3 * rng.standard_normal(w.shape)
    w[:, :2] = 0.0
    G = oracle.macro_kin(2, wl.nel, u, kind=1) + np.array([1.0, 0, 0, 1.0])
    c = oracle.condense_batch_nh(wl.r, wl.phase, wl.mat, G, w)
    for ts in (False, True):
        h = Homogenizer.from_workload(wl, tile_sparse=ts)
        h.set_fluctuations(torch.tensor(w, device="cuda"))
        F = h.macro_kinematics(torch.tensor(u, device="cuda"))
        A, Pe, Pa = h.condense(F)
        print(f"{name:28s} {'tile-sparse' if ts else 'dense':11s} B={wl.n_rve:6d} A_eff {rel(A.cpu().numpy(), c['A_eff']):.2e}  "
              f"P_eff {rel(Pe.cpu().numpy(), c['P_eff']):.2e}  <P> {rel(Pa.cpu().numpy(), c['P_avg']):.2e}  "
              f"(non-equilibrium state after load step 1 + 1e-3 noise on w)", flush=True)
        h.close()


if __name__ == "__main__":
    import torch
    torch.cuda.set_device(0)
    print(f"# GPU vs oracle, relative Frobenius errors (north_star: C_eff <= 1e-10, u <= 1e-8); "
          f"{torch.cuda.get_device_name(0)}")
    linear("cfg1 laminate (full)", W.config1())
    linear("cfg2 disc (full)", W.config2())
    rng = np.random.default_rng(0)
    wl3 = W.config3()
    linear("cfg3 random (full, sampled)", wl3, np.sort(np.unique(np.concatenate(
        [rng.choice(wl3.n_rve, 254, replace=False), [0, wl3.n_rve - 1]]))))
    linear("cfg4 sphere (full)", W.config4())
    finite_per_state("cfg5 neo-hooke (full)", W.config5())

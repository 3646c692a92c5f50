"""Measured GPU-vs-oracle errors for the five configs at full size (relative Frobenius norm over
the batch AND the largest per-RVE relative error), dense and tile-sparse factorisation; every value
is compared with the oracle's OWN answer (its C_eff, its direct macro solve, its Newton run).
Test infrastructure (uses oracle/).

  python tools/parity_report.py > profiles/r02/parity_r02.txt
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


def rel_max(a, b):
    a = np.asarray(a).reshape(len(a), -1)
    b = np.asarray(b).reshape(len(b), -1)
    nb = np.linalg.norm(b, axis=1)
    return float(np.max(np.linalg.norm(a - b, axis=1) / np.where(nb > 0, nb, 1.0)))


def linear(name, wl):
    t0 = time.perf_counter()
    o = oracle.solve_linear(wl)
    w_o = oracle.recover_linear(o["W"], o["eps"])
    t_o = time.perf_counter() - t0
    for ts in (False, True):
        t0 = time.perf_counter()
        h = Homogenizer.from_workload(wl, tile_sparse=ts)
        C, u, w, info = h.solve_linear()
        C, u, w = C.cpu().numpy(), u.cpu().numpy(), w.cpu().numpy()
        print(f"{name:22s} {'tile-sparse' if ts else 'dense':11s} B={wl.n_rve:6d} "
              f"C_eff {rel(C, o['C_eff']):.2e} (per-RVE max {rel_max(C, o['C_eff']):.2e})  "
              f"u {rel(u, o['u']):.2e}  w {rel(w, w_o):.2e} (per-RVE max {rel_max(w, w_o):.2e})  "
              f"CG {info.iterations:4d} it rel.res {info.rel_residual:.1e}  (all RVEs vs the oracle's own "
              f"C_eff/u/w; GPU {time.perf_counter() - t0:.1f} s, oracle {t_o:.1f} s)", flush=True)
        h.close()


def finite_newton(name, wl):
    import torch
    t0 = time.perf_counter()
    o = oracle.newton_nh(wl, tol=1e-11)
    t_o = time.perf_counter() - t0
    for ts in (False, True):
        h = Homogenizer.from_workload(wl, tile_sparse=ts)
        us = {}
        _, hist = h.newton(wl.n_steps, tol=1e-11, on_step=lambda k, u: us.__setitem__(k, u.cpu().numpy()))
        eu = [rel(us[k], o[k - 1]["u"]) for k in range(1, wl.n_steps + 1)]
        w = h.get_fluctuations().cpu().numpy()
        its = "".join(str(len(s) - 1) for s in hist)
        its_o = "".join(str(len(s["history"]) - 1) for s in o)
        print(f"{name:22s} {'tile-sparse' if ts else 'dense':11s} B={wl.n_rve:6d} {wl.n_steps} load steps, "
              f"Newton tol 1e-11: u per step max {max(eu):.2e} (steps: {', '.join(f'{e:.1e}' for e in eu)})  "
              f"final w {rel(w, o[-1]['w']):.2e} (per-RVE max {rel_max(w, o[-1]['w']):.2e})  "
              f"iterations/step GPU {its} oracle {its_o}  (oracle {t_o:.1f} s)", flush=True)
        h.close()
    # one non-equilibrium state, condensation alone
    steps = o[:1]
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
        A, Pe, Pa = A.cpu().numpy(), Pe.cpu().numpy(), Pa.cpu().numpy()
        print(f"{name:22s} {'tile-sparse' if ts else 'dense':11s} B={wl.n_rve:6d} per state: "
              f"A_eff {rel(A, c['A_eff']):.2e} (per-RVE max {rel_max(A, c['A_eff']):.2e})  "
              f"P_eff {rel(Pe, c['P_eff']):.2e} (per-RVE max {rel_max(Pe, c['P_eff']):.2e})  "
              f"<P> {rel(Pa, c['P_avg']):.2e}  (state after load step 1 + 1e-3 noise on w)", flush=True)
        h.close()


if __name__ == "__main__":
    import torch
    torch.cuda.set_device(0)
    print(f"# GPU vs oracle at full size (north_star: C_eff <= 1e-10, u <= 1e-8); relative Frobenius error over "
          f"the batch and the largest per-RVE relative error; {torch.cuda.get_device_name(0)}, oracle on "
          f"{oracle.default_threads()} host threads")
    linear("cfg1 laminate", W.config1())
    linear("cfg2 disc", W.config2())
    linear("cfg3 random", W.config3())
    linear("cfg4 sphere", W.config4())
    finite_newton("cfg5 neo-hooke", W.config5())

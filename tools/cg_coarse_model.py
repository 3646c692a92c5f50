"""Numpy model (CPU, oracle-built macro matrix) of the macro PCG iteration count with the
block-Jacobi preconditioner of k_macro_cg_cluster2 and with an additive two-level variant
(aggregates of na x na macro nodes, translations (+ rotation) per aggregate as coarse space).
Run: PYTHONPATH=. python tools/cg_coarse_model.py [nel]"""
import numpy as np, oracle, sys
from paper_2312_12771_b200 import workloads as W
nel = int(sys.argv[1]) if len(sys.argv) > 1 else 32
wl = W.config2(nel=32, r=16)

o = oracle.solve_linear(W.config2(nel=2, r=16))
C = np.tile(o["C_eff"][0], (nel * nel * 4, 1, 1))
wl = W.config2(nel=nel, r=16)
n = wl.n_dof
R0 = oracle.macro_residual(2, nel, np.zeros((nel*nel*4, 3)), wl.body)
K = np.zeros((n, n))
for j in range(n):
    e = np.zeros(n); e[j] = 1.0
    eps = oracle.macro_kin(2, nel, e)
    K[:, j] = oracle.macro_residual(2, nel, np.einsum("bij,bj->bi", C, eps), wl.body) - R0
free = np.ones(n, bool); free[wl.dir_dof] = False
b = -R0.copy(); b[~free] = 0
Kf = K.copy(); Kf[~free, :] = 0; Kf[:, ~free] = 0; Kf[~free, ~free] = 1
# block Jacobi
Minv = np.zeros((n, n))
for nd in range(n // 2):
    s = slice(2*nd, 2*nd+2)
    B = Kf[s, s].copy()
    Minv[s, s] = np.linalg.inv(B)
nn1 = nel + 1
def coarse(na, modes):
    xs = np.arange(n // 2) % nn1; ys = np.arange(n // 2) // nn1
    ax = np.minimum(xs * na // nn1, na - 1); ay = np.minimum(ys * na // nn1, na - 1)
    agg = ay * na + ax
    P = np.zeros((n, na * na * modes))
    for nd in range(n // 2):
        a = agg[nd]
        P[2*nd, a*modes] = 1; P[2*nd+1, a*modes+1] = 1
        if modes == 3:
            x, y = xs[nd] / nel, ys[nd] / nel
            P[2*nd, a*modes+2] = -y; P[2*nd+1, a*modes+2] = x
    P[~free, :] = 0
    keep = np.abs(P).sum(0) > 0
    return P[:, keep]
def pcg(Mfun, tol=1e-13):
    x = np.zeros(n); r = b.copy(); z = Mfun(r); p = z.copy(); rz = r @ z; bn = np.linalg.norm(b)
    for it in range(1, 5000):
        q = Kf @ p; a = rz / (p @ q); x += a * p; r -= a * q
        if np.linalg.norm(r) <= tol * bn: return it
        z = Mfun(r); rz2 = r @ z; p = z + rz2 / rz * p; rz = rz2
    return -1
print("n", n, "block-Jacobi:", pcg(lambda r: Minv @ r))
for na in (4, 6, 8):
    for modes in (2, 3):
        P = coarse(na, modes); Ac = P.T @ Kf @ P; Aci = np.linalg.inv(Ac)
        print(f"agg {na}x{na} modes {modes} nc {P.shape[1]}:", pcg(lambda r: Minv @ r + P @ (Aci @ (P.T @ r))))

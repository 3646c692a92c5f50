"""ctypes binding of oracle/hom_oracle.c plus plain numpy drivers.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Every function here is a
thin marshalling layer or a textbook driver (Dirichlet bookkeeping, the
Newton / load-step loop of PAPER.md P:325-342 and P:613-617).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hom_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

ORC_OK, ORC_ERR_ARG, ORC_ERR_NOT_SPD, ORC_ERR_JACOBIAN, ORC_ERR_OOM = 0, 1, 3, 4, 8


class OracleError(RuntimeError):
    def __init__(self, code, what, rve=-1):
        super().__init__(f"oracle {what} failed with code {code} (rve {rve})")
        self.code, self.rve = code, rve


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C99, -O2, pthreads)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-o", _LIB, _SRC,
                               "-lm", "-lpthread"])
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            I = ctypes.c_int
            D = ctypes.c_double
            L.orc_linear_C.argtypes = [I, D, D, P]
            L.orc_nh_material.argtypes = [P, D, D, P, P, P]
            L.orc_mr_material.argtypes = [P, D, D, D, P, P, P]
            L.orc_rve_condense_linear.argtypes = [I, I, D, I, P, P, P]
            L.orc_rve_condense_nh.argtypes = [I, D, I, P, P, P, P, P, P, P, P, P, P]
            L.orc_condense_batch_linear.argtypes = [I, I, I, I, P, I, I, P, P, P, I, P]
            L.orc_condense_batch_linear_axes.argtypes = [I, I, P, I, I, P, I, I, P, P, P, I, P]
            L.orc_rve_condense_linear_axes.argtypes = [I, I, P, I, P, P, P]
            L.orc_condense_batch_nh.argtypes = [I, D, I, I, I, P, I, I, P, P, P, P, P, P, P, P, P, I, P]
            L.orc_macro_kin.argtypes = [I, I, D, I, P, P]
            L.orc_macro_residual.argtypes = [I, I, D, I, P, P, P]
            L.orc_macro_solve.argtypes = [I, I, D, I, P, P, P, I, P, P]
            L.orc_mesh_macro_kin.argtypes = [I, I, I, P, P, I, P, P]
            L.orc_macro_kin_const.argtypes = [I, I, D, P, P]
            L.orc_macro_solve_const.argtypes = [I, I, D, P, P, P, I, P, P]
            L.orc_mesh_macro_residual.argtypes = [I, I, I, P, P, I, P, P, P, P]
            L.orc_mesh_macro_solve.argtypes = [I, I, I, P, P, I, P, P, P, P, I, P, P]
            L.orc_dense_spd_solve.argtypes = [I, P, P]
            _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def m_of(dim: int, kind: int = 0) -> int:
    if kind == 1:
        return dim * dim
    return {1: 1, 2: 3, 3: 6}[dim]


def default_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)))


# --------------------------------------------------------------------------
# material points
# --------------------------------------------------------------------------
def linear_C(dim: int, E: float, nu: float) -> np.ndarray:
    m = m_of(dim)
    C = np.zeros((m, m))
    lib().orc_linear_C(dim, E, nu, _p(C))
    return C


def nh_material(F, alpha: float, kappa: float, beta: float = 0.0):
    """Return (psi, P[4], A[4,4]) of the Cook energy; beta = 0 is config 5 (R11)."""
    F = _f64(np.asarray(F).reshape(4))
    P = np.zeros(4)
    A = np.zeros((4, 4))
    psi = ctypes.c_double(0.0)
    rc = lib().orc_mr_material(_p(F), alpha, beta, kappa, ctypes.byref(psi), _p(P), _p(A))
    if rc:
        raise OracleError(rc, "nh_material")
    return psi.value, P, A


# --------------------------------------------------------------------------
# RVE condensation
# --------------------------------------------------------------------------
def rve_condense_linear(dim: int, r: int, Cq, mode: int = 0, L: float = 1.0, want_W: bool = False):
    """C_eff (and W = -X^T, [m][dim r^dim]) of one RVE with per-(element,qp) tangent Cq."""
    m = m_of(dim)
    nel, nq = r ** dim, 2 ** dim
    Cq = _f64(np.broadcast_to(np.asarray(Cq, dtype=np.float64), (nel, nq, m, m)))
    C = np.zeros((m, m))
    W = np.zeros((m, dim * nel)) if want_W else None
    rc = lib().orc_rve_condense_linear(dim, r, L, mode, _p(Cq), _p(C), _p(W))
    if rc:
        raise OracleError(rc, "rve_condense_linear")
    return (C, W) if want_W else C


def condense_batch_linear(dim: int, r: int, phase, mat, n_rve: int | None = None,
                          want_W: bool = False, nthreads: int | None = None, axes=None):
    """Batched linear condensation.  phase [n_rve|1][r^dim] u8, mat [n_rve|1][n_phase][2] (E, nu);
    axes [dim][r+1]: node coordinates of a tensor-product (graded) RVE grid (None = uniform [0,1]^dim)."""
    phase = np.ascontiguousarray(phase, dtype=np.uint8)
    mat = _f64(mat)
    nel = r ** dim
    phase = phase.reshape(-1, nel)
    n_phase = mat.shape[-2]
    mat = mat.reshape(-1, n_phase, 2)
    if n_rve is None:
        n_rve = max(phase.shape[0], mat.shape[0])
    m = m_of(dim)
    C = np.zeros((n_rve, m, m))
    W = np.zeros((n_rve, m, dim * nel)) if want_W else None
    bad = ctypes.c_int(-1)
    if axes is not None:
        ax = _f64(np.asarray(axes, dtype=np.float64).reshape(dim, r + 1))
        rc = lib().orc_condense_batch_linear_axes(dim, r, _p(ax), n_rve, int(phase.shape[0] > 1), _p(phase),
                                                  int(mat.shape[0] > 1), n_phase, _p(mat), _p(C), _p(W),
                                                  nthreads or default_threads(), ctypes.byref(bad))
    else:
        rc = lib().orc_condense_batch_linear(dim, r, n_rve, int(phase.shape[0] > 1), _p(phase),
                                             int(mat.shape[0] > 1), n_phase, _p(mat), _p(C), _p(W),
                                             nthreads or default_threads(), ctypes.byref(bad))
    if rc:
        raise OracleError(rc, "condense_batch_linear", bad.value)
    return (C, W) if want_W else C


def condense_batch_nh(r: int, phase, mat, Fbar, w=None, nthreads: int | None = None, L: float = 1.0):
    """Batched finite-strain condensation (2-D, RVE [0,L]^2).  mat [..][n_phase][2] (alpha, kappa) or
    [..][n_phase][3] (alpha, beta, kappa).  Returns dict of A_eff, P_eff, P_avg, Z, W, rf_norm."""
    phase = np.ascontiguousarray(phase, dtype=np.uint8).reshape(-1, r * r)
    mat = _f64(mat)
    n_phase, ms = mat.shape[-2], mat.shape[-1]
    mat = mat.reshape(-1, n_phase, ms)
    Fbar = _f64(np.asarray(Fbar).reshape(-1, 4))
    n_rve = Fbar.shape[0]
    npad = 2 * r * r
    w = None if w is None else _f64(np.asarray(w).reshape(n_rve, npad))
    out = {
        "A_eff": np.zeros((n_rve, 4, 4)), "P_eff": np.zeros((n_rve, 4)), "P_avg": np.zeros((n_rve, 4)),
        "Z": np.zeros((n_rve, npad)), "W": np.zeros((n_rve, 4, npad)), "rf_norm": np.zeros(n_rve),
    }
    bad = ctypes.c_int(-1)
    rc = lib().orc_condense_batch_nh(r, L, ms, n_rve, int(phase.shape[0] > 1), _p(phase), int(mat.shape[0] > 1),
                                     n_phase, _p(mat), _p(Fbar), _p(w), _p(out["A_eff"]),
                                     _p(out["P_eff"]), _p(out["P_avg"]), _p(out["Z"]), _p(out["W"]),
                                     _p(out["rf_norm"]), nthreads or default_threads(), ctypes.byref(bad))
    if rc:
        raise OracleError(rc, "condense_batch_nh", bad.value)
    return out


# --------------------------------------------------------------------------
# macro problem
# --------------------------------------------------------------------------
def _mesh(mesh):
    xc, conn = mesh
    return _f64(xc), np.ascontiguousarray(conn, dtype=np.int32)


def macro_kin(dim: int, nel: int, u, kind: int = 0, Lm: float = 1.0, mesh=None) -> np.ndarray:
    """Kinematics at every macro qp; mesh = (coords, conn) for a non-structured macro mesh."""
    m = m_of(dim, kind)
    u = _f64(u)
    if mesh is not None:
        xc, conn = _mesh(mesh)
        out = np.zeros((conn.shape[0] * 2 ** dim, m))
        lib().orc_mesh_macro_kin(dim, xc.shape[0], conn.shape[0], _p(xc), _p(conn), kind, _p(u), _p(out))
        return out
    out = np.zeros((nel ** dim * 2 ** dim, m))
    lib().orc_macro_kin(dim, nel, Lm, kind, _p(u), _p(out))
    return out


def macro_residual(dim: int, nel: int, S=None, body=None, kind: int = 0, Lm: float = 1.0, mesh=None,
                   fext=None) -> np.ndarray:
    """R = sum eta B^T S - f_body - f_ext over all DOFs."""
    if mesh is not None:
        xc, conn = _mesh(mesh)
        R = np.zeros(xc.shape[0] * dim)
        lib().orc_mesh_macro_residual(dim, xc.shape[0], conn.shape[0], _p(xc), _p(conn), kind, _p(_f64(S)),
                                      _p(_f64(body)), _p(_f64(fext)), _p(R))
        return R
    R = np.zeros((nel + 1) ** dim * dim)
    lib().orc_macro_residual(dim, nel, Lm, kind, _p(_f64(S)), _p(_f64(body)), _p(R))
    if fext is not None:
        R -= fext
    return R


def macro_solve(dim: int, nel: int, D, dir_dof, x_dir, S=None, body=None, kind: int = 0,
                Lm: float = 1.0, mesh=None, fext=None) -> np.ndarray:
    """Direct solve of K_FF x_F = -R_F - K_FD x_D (see hom_oracle.c orc_macro_solve)."""
    dir_dof = np.ascontiguousarray(dir_dof, dtype=np.int32)
    if mesh is not None:
        xc, conn = _mesh(mesh)
        x = np.zeros(xc.shape[0] * dim)
        x[dir_dof] = x_dir
        rc = lib().orc_mesh_macro_solve(dim, xc.shape[0], conn.shape[0], _p(xc), _p(conn), kind, _p(_f64(D)),
                                        _p(_f64(S)), _p(_f64(body)), _p(_f64(fext)), len(dir_dof), _p(dir_dof),
                                        _p(x))
        if rc:
            raise OracleError(rc, "mesh_macro_solve")
        return x
    ndof = (nel + 1) ** dim * dim
    x = np.zeros(ndof)
    x[dir_dof] = x_dir
    if fext is not None:
        raise ValueError("fext needs mesh=")
    rc = lib().orc_macro_solve(dim, nel, Lm, kind, _p(_f64(D)), _p(_f64(S)), _p(_f64(body)),
                               len(dir_dof), _p(dir_dof), _p(x))
    if rc:
        raise OracleError(rc, "macro_solve")
    return x


def dense_spd_solve(A, b) -> np.ndarray:
    A = _f64(A)
    x = _f64(np.array(b, dtype=np.float64, copy=True))
    rc = lib().orc_dense_spd_solve(A.shape[0], _p(A), _p(x))
    if rc:
        raise OracleError(rc, "dense_spd_solve")
    return x


# --------------------------------------------------------------------------
# whole-workload drivers (use the seeded arrays from paper_2312_12771_b200.workloads)
# --------------------------------------------------------------------------
def solve_linear(wl, rve_ids=None, nthreads: int | None = None):
    """Linear configs: condense every RVE (or the given subset), direct macro solve, recovery.

    RVEs whose phase and material rows are shared (per_rve = 0) are condensed once
    -- the oracle is allowed to, the GPU path is not.
    Returns dict(C_eff [B][m][m], u [n_dof], eps [B][m], W [B or subset][m][N_pad]).
    """
    dim, r = wl.dim, wl.r
    axes = getattr(wl, "rve_axes", None)
    shared = wl.phase.shape[0] == 1 and wl.mat.shape[0] == 1
    if shared:
        C1, W1 = condense_batch_linear(dim, r, wl.phase, wl.mat, 1, want_W=True, nthreads=nthreads, axes=axes)
        C = np.broadcast_to(C1, (wl.n_rve,) + C1.shape[1:]).copy()
        Wsel = W1[0]
    else:
        ids = np.arange(wl.n_rve) if rve_ids is None else np.asarray(rve_ids)
        ph = wl.phase[ids] if wl.phase.shape[0] > 1 else wl.phase
        mt = wl.mat[ids] if wl.mat.shape[0] > 1 else wl.mat
        Csub, Wsel = condense_batch_linear(dim, r, ph, mt, len(ids), want_W=True, nthreads=nthreads, axes=axes)
        if rve_ids is None:
            C = Csub
        else:
            return {"C_eff_subset": Csub, "W_subset": Wsel, "ids": ids}
    u = macro_solve(dim, wl.nel, C, wl.dir_dof, wl.dir_val, body=wl.body)
    eps = macro_kin(dim, wl.nel, u)
    return {"C_eff": C, "u": u, "eps": eps, "W": Wsel}


def C_avg_linear(dim: int, r: int, phase, mat) -> np.ndarray:
    """<C> = |Omega|^-1 sum_e |e| C(phase_e) (plain definition, uniform RVE grid) per RVE row."""
    phase = np.asarray(phase).reshape(-1, r ** dim)
    mat = np.asarray(mat, dtype=np.float64)
    mat = mat.reshape(-1, mat.shape[-2], 2)
    n = max(phase.shape[0], mat.shape[0])
    out = np.zeros((n, m_of(dim), m_of(dim)))
    for b in range(n):
        ph = phase[b if phase.shape[0] > 1 else 0]
        mt = mat[b if mat.shape[0] > 1 else 0]
        for p in np.unique(ph):
            out[b] += np.count_nonzero(ph == p) / ph.size * linear_C(dim, mt[p, 0], mt[p, 1])
    return out


def solve_linear_constant(wl, nthreads: int | None = None):
    """Piecewise-constant macro fluctuation basis (eq:constSolution1/2), small strain:
    one RVE per macro element (phase/material rows of element e = those of its first Gauss point
    RVE), C_eff and <C> per element, direct macro solve with
    K_e = int B^T <C> B - |B_e|^-1 Bbar^T (<C> - C_eff) Bbar, recovery w_e = W_e eps_bar_e.
    Returns dict(C_eff [E][m][m], C_avg [E][m][m], u, eps_bar [E][m], w [E][N_pad])."""
    dim, r, nq = wl.dim, wl.r, wl.n_qp
    ne = wl.nel ** dim
    ph = wl.phase[::nq] if wl.phase.shape[0] > 1 else wl.phase
    mt = wl.mat[::nq] if wl.mat.shape[0] > 1 else wl.mat
    C, W = condense_batch_linear(dim, r, ph, mt, ne if (ph.shape[0] > 1 or mt.shape[0] > 1) else 1,
                                 want_W=True, nthreads=nthreads)
    Ca = C_avg_linear(dim, r, ph, mt)
    if C.shape[0] == 1:
        C, W, Ca = (np.broadcast_to(a, (ne,) + a.shape[1:]).copy() for a in (C, W, Ca))
    x = np.zeros(wl.n_dof)
    dd = np.ascontiguousarray(wl.dir_dof, dtype=np.int32)
    x[dd] = wl.dir_val
    rc = lib().orc_macro_solve_const(dim, wl.nel, 1.0, _p(_f64(Ca)), _p(_f64(C)), _p(_f64(wl.body)), len(dd),
                                     _p(dd), _p(x))
    if rc:
        raise OracleError(rc, "macro_solve_const")
    eps = np.zeros((ne, m_of(dim)))
    lib().orc_macro_kin_const(dim, wl.nel, 1.0, _p(x), _p(eps))
    return {"C_eff": C, "C_avg": Ca, "u": x, "eps_bar": eps, "w": recover_linear(W, eps)}


def recover_linear(W, eps):
    """w_b = sum_j eps_bj W_j  (= -X_b eps_b, eq:reduction P:388-390)."""
    if W.ndim == 2:
        return eps @ W
    return np.einsum("bj,bjn->bn", eps, W)


def _fs(wl):
    """Finite-strain workload plumbing: (mesh or None, external nodal force or None, RVE size)."""
    mesh = None if getattr(wl, "macro_coords", None) is None else wl.macro_mesh()
    return mesh, getattr(wl, "nodal_force", None), getattr(wl, "rve_size", 1.0)


def newton_step_nh(wl, u, w, x_dir, nthreads: int | None = None, load_factor: float = 1.0):
    """One monolithic Newton step at state (u, w) (eq:solution2 P:420-423).

    Returns (du, dw, info) with info = dict(R_norm, rf_max, cond) at the *current* state.
    """
    dim, nel, r = 2, wl.nel, wl.r
    mesh, fn, L = _fs(wl)
    fext = None if fn is None else load_factor * fn
    G = macro_kin(dim, nel, u, kind=1, mesh=mesh)
    Fbar = G + np.array([1.0, 0.0, 0.0, 1.0])
    c = condense_batch_nh(r, wl.phase, wl.mat, Fbar, w, nthreads=nthreads, L=L)
    R = macro_residual(dim, nel, c["P_avg"], wl.body, kind=1, mesh=mesh, fext=fext)
    free = np.ones(len(u), bool)
    free[wl.dir_dof] = False
    # R_micro per RVE = r_f / |Omega| (eq:constSolution2 with the Dirac shifting property, P:248-250,
    # P:305-315; R21), |Omega| = L^2
    info = {"R_norm": float(np.linalg.norm(R[free])), "rf_max": float(c["rf_norm"].max()) / L ** 2, "cond": c}
    du = macro_solve(dim, nel, c["A_eff"], wl.dir_dof, x_dir, S=c["P_eff"], body=wl.body, kind=1, mesh=mesh,
                     fext=fext)
    dF = macro_kin(dim, nel, du, kind=1, mesh=mesh)
    dw = c["Z"] + np.einsum("bj,bjn->bn", dF, c["W"])
    return du, dw, info


def newton_nh(wl, tol: float = 1e-11, max_iter: int = 25, steps=None, nthreads: int | None = None,
              micro_tol=None, divergence: float = 1e10):
    """Finite strain: monolithic Newton with null-space (Schur) reduction and load stepping.

    Per iteration (CS-paper-1): condense at (u, w); check
    ||R_macro|| (with <P>) and max_b ||r_f,b|| against tol (reading R3; micro_tol=inf checks the
    macro residual only); solve the condensed system (eq:solution2); dw = z + W dF.
    Load steps: the Dirichlet increment in the first iteration of each step (config 5),
    or the external load factor k/n_steps when the workload has nodal forces (Cook).
    Returns a list of per-step dicts with u, w and the residual history.
    """
    n_rve, r = wl.n_rve, wl.r
    force = getattr(wl, "nodal_force", None) is not None
    mtol = tol if micro_tol is None else micro_tol
    u = np.zeros(wl.n_dof)
    w = np.zeros((n_rve, 2 * r * r))
    out = []
    n_steps = wl.n_steps if steps is None else steps
    for k in range(1, n_steps + 1):
        hist, converged = [], False
        for it in range(max_iter + 1):
            x_dir = wl.dir_val / wl.n_steps if (it == 0 and not force) else np.zeros(len(wl.dir_dof))
            try:
                du, dw, info = newton_step_nh(wl, u, w, x_dir, nthreads=nthreads,
                                              load_factor=k / wl.n_steps if force else 1.0)
            except OracleError as e:
                if e.code != 4:
                    raise
                hist.append((float("inf"), float("inf")))
                break
            hist.append((info["R_norm"], info["rf_max"]))
            if it > 0 and info["R_norm"] <= tol and info["rf_max"] <= mtol:
                converged = True
                break
            if not (info["R_norm"] <= divergence) or it == max_iter:
                break
            u, w = u + du, w + dw
        out.append({"step": k, "u": u.copy(), "w": w.copy(), "history": hist, "converged": converged})
        if not converged:
            break
    return out


def newton_classical(wl, tol: float = 1e-9, micro_tol: float = 1e-13, max_iter: int = 25, max_inner: int = 30,
                     steps=None, nthreads: int | None = None, divergence: float = 1e10):
    """Classical staggered FE^2: per macro iteration, equilibrate every RVE at the
    fixed macro deformation (inner Newton w <- w + z, z = -K_ff^-1 r_f, until max ||r_f|| <
    micro_tol), then solve [K - D L^-1 E] dq = -R_macro (eq:solution1, R_macro with <P>), update q
    and w += W dF (eq:reduction) and restart until ||R_macro|| < tol.  Load factor k/n_steps on the
    external nodal forces.  Returns a list of per-step dicts (history: (||R_macro||, inner list))."""
    dim, nel, r = 2, wl.nel, wl.r
    mesh, fn, L = _fs(wl)
    u = np.zeros(wl.n_dof)
    w = np.zeros((wl.n_rve, 2 * r * r))
    free = np.ones(wl.n_dof, bool)
    free[wl.dir_dof] = False
    out = []
    n_steps = wl.n_steps if steps is None else steps
    for k in range(1, n_steps + 1):
        fext = None if fn is None else (k / wl.n_steps) * fn
        hist, converged = [], False
        for it in range(max_iter + 1):
            Fbar = macro_kin(dim, nel, u, kind=1, mesh=mesh) + np.array([1.0, 0.0, 0.0, 1.0])
            inner = []
            try:
                for _ in range(max_inner + 1):
                    c = condense_batch_nh(r, wl.phase, wl.mat, Fbar, w, nthreads=nthreads, L=L)
                    rf = float(c["rf_norm"].max()) / L ** 2  # max_b ||R_micro,b|| (R21)
                    inner.append(rf)
                    if rf < micro_tol or not (rf <= divergence):
                        break
                    w = w + c["Z"]
            except OracleError as e:
                if e.code != 4:
                    raise
                hist.append((float("inf"), inner))
                break
            R = macro_residual(dim, nel, c["P_avg"], wl.body, kind=1, mesh=mesh, fext=fext)
            rn = float(np.linalg.norm(R[free]))
            hist.append((rn, inner))
            if not inner[-1] < micro_tol:  # inner loop exhausted max_inner
                break
            if it > 0 and rn <= tol:
                converged = True
                break
            if not (rn <= divergence) or it == max_iter:
                break
            du = macro_solve(dim, nel, c["A_eff"], wl.dir_dof, np.zeros(len(wl.dir_dof)), S=c["P_avg"],
                             body=wl.body, kind=1, mesh=mesh, fext=fext)
            dF = macro_kin(dim, nel, du, kind=1, mesh=mesh)
            u = u + du
            w = w + c["Z"] + np.einsum("bj,bjn->bn", dF, c["W"])
        out.append({"step": k, "u": u.copy(), "w": w.copy(), "history": hist, "converged": converged})
        if not converged:
            break
    return out

"""Thin Python binding of libhom.so (include/hom.h) -- argument marshalling only.

Every step of the hot path runs inside libhom.so's sm_100a kernels; PyTorch is
used here only to own device memory and to hand the current CUDA stream to the
library.  There is no CPU fallback: if libhom.so cannot be loaded, or no CUDA
device is present, the calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import build as _build

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhom.so")

HOM_OK = 0
STATUS = {0: "HOM_OK", 1: "HOM_ERR_INVALID_ARG", 2: "HOM_ERR_MESH", 3: "HOM_ERR_NOT_SPD",
          4: "HOM_ERR_JACOBIAN", 5: "HOM_ERR_CG_NOT_CONVERGED", 6: "HOM_ERR_CG_BREAKDOWN",
          7: "HOM_ERR_CUDA", 8: "HOM_ERR_OOM"}

# every symbol include/hom.h declares (checked by tests/test_abi.py)
EXPORTS = ["hom_setup", "hom_get_sizes", "hom_get_work", "hom_debug_rve_kff", "hom_set_load_factor", "hom_macro_assemble", "hom_macro_spmv", "hom_macro_kinematics", "hom_condense", "hom_macro_solve",
           "hom_macro_residual_norm", "hom_recover_fluctuations", "hom_newton_update", "hom_macro_update", "hom_set_fluctuations",
           "hom_get_fluctuations", "hom_micro_residual_max", "hom_set_phases", "hom_get_element_cavg",
           "hom_set_element_cavg", "hom_launch_count",
           "hom_profile_enable", "hom_profile_read", "hom_last_error", "hom_destroy"]
PROF_CLASSES = ["rve_assemble", "condense", "macro_assemble", "cg", "recover", "other"]


class MacroMesh(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("n_nodes", ctypes.c_int32), ("n_elems", ctypes.c_int32),
                ("nodes_per_elem", ctypes.c_int32), ("coords", ctypes.c_void_p), ("conn", ctypes.c_void_p),
                ("n_dirichlet", ctypes.c_int32), ("dirichlet_dof", ctypes.c_void_p),
                ("dirichlet_value", ctypes.c_void_p), ("body_force", ctypes.c_void_p),
                ("nodal_force", ctypes.c_void_p)]


class RveMesh(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("n_nodes", ctypes.c_int32), ("n_elems", ctypes.c_int32),
                ("nodes_per_elem", ctypes.c_int32), ("coords", ctypes.c_void_p), ("conn", ctypes.c_void_p)]


class PhaseField(ctypes.Structure):
    _fields_ = [("per_rve", ctypes.c_int32), ("phase", ctypes.c_void_p)]


class Materials(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("n_phases", ctypes.c_int32), ("per_rve", ctypes.c_int32),
                ("params", ctypes.c_void_p)]


class Options(ctypes.Structure):
    _fields_ = [("finite_strain", ctypes.c_int32), ("cg_rtol", ctypes.c_double), ("cg_max_iter", ctypes.c_int32),
                ("rve_chunk", ctypes.c_int32), ("check_info", ctypes.c_int32), ("mem_budget_gb", ctypes.c_double),
                ("tile_sparse", ctypes.c_int32), ("rve_begin", ctypes.c_int32), ("rve_count", ctypes.c_int32),
                ("macro_basis", ctypes.c_int32), ("rve_ordering", ctypes.c_int32), ("macro_precond", ctypes.c_int32)]


class Sizes(ctypes.Structure):
    _fields_ = [("n_rve", ctypes.c_int32), ("m", ctypes.c_int32), ("n_pad", ctypes.c_int32),
                ("n_tiles", ctypes.c_int32), ("n_macro_dof", ctypes.c_int32), ("n_macro_free", ctypes.c_int32),
                ("macro_nnz", ctypes.c_int32), ("rve_chunk", ctypes.c_int32), ("rve_volume", ctypes.c_double),
                ("rve_begin", ctypes.c_int32), ("rve_count", ctypes.c_int32)]


class Work(ctypes.Structure):
    _fields_ = [("a_tiles", ctypes.c_int32), ("g_tiles", ctypes.c_int32), ("diag_tiles", ctypes.c_int32),
                ("syrk_tiles", ctypes.c_int32), ("gemm_tiles", ctypes.c_int32), ("trsm_tiles", ctypes.c_int32),
                ("flop_dense", ctypes.c_double), ("flop_executed", ctypes.c_double)]


class SolveInfo(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("rel_residual", ctypes.c_double), ("rhs_norm", ctypes.c_double)]


class ErrorInfo(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("rve", ctypes.c_int32), ("row", ctypes.c_int32),
                ("cuda_error", ctypes.c_int32), ("message", ctypes.c_char * 256)]


class HomError(RuntimeError):
    def __init__(self, code, info: ErrorInfo | None = None, where=""):
        msg = f"{where}: {STATUS.get(code, code)}"
        if info is not None:
            msg += f" (rve {info.rve}, row {info.row}): {info.message.decode(errors='replace')}"
        super().__init__(msg)
        self.code = code
        self.rve = info.rve if info is not None else -1
        self.row = info.row if info is not None else -1


_lib = None


def lib(build_if_missing: bool = True):
    """Load libhom.so (building it in-tree with nvcc if missing).  Raises if it cannot be loaded."""
    global _lib
    if _lib is None:
        if build_if_missing:
            _build.build()
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libhom.so not found at {LIB_PATH}; run paper_2312_12771_b200/build.py")
        L = ctypes.CDLL(LIB_PATH)
        P, I, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
        L.hom_setup.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(MacroMesh), ctypes.POINTER(RveMesh),
                                ctypes.POINTER(PhaseField), ctypes.POINTER(Materials), ctypes.POINTER(Options), P]
        L.hom_get_sizes.argtypes = [P, ctypes.POINTER(Sizes)]
        L.hom_get_work.argtypes = [P, ctypes.POINTER(Work)]
        L.hom_macro_kinematics.argtypes = [P, P, P, P]
        L.hom_condense.argtypes = [P, P, P, P, P, P]
        L.hom_macro_solve.argtypes = [P, P, P, D, P, ctypes.POINTER(SolveInfo), P]
        L.hom_macro_residual_norm.argtypes = [P, P, ctypes.POINTER(ctypes.c_double), P]
        L.hom_macro_assemble.argtypes = [P, P, P]
        L.hom_set_load_factor.argtypes = [P, D]
        L.hom_macro_spmv.argtypes = [P, P, P, P]
        L.hom_debug_rve_kff.argtypes = [P, I, P, P]
        L.hom_recover_fluctuations.argtypes = [P, P, P, P]
        L.hom_newton_update.argtypes = [P, P, P, P]
        L.hom_macro_update.argtypes = [P, P, P, P]
        L.hom_set_fluctuations.argtypes = [P, P, P]
        L.hom_get_fluctuations.argtypes = [P, P, P]
        L.hom_micro_residual_max.argtypes = [P, ctypes.POINTER(ctypes.c_double), P]
        L.hom_set_phases.argtypes = [P, P, P, P]
        L.hom_get_element_cavg.argtypes = [P, P, P]
        L.hom_set_element_cavg.argtypes = [P, P, P]
        L.hom_profile_enable.argtypes = [P, I]
        L.hom_profile_read.argtypes = [P, P, P]
        L.hom_launch_count.argtypes = [P]
        L.hom_launch_count.restype = ctypes.c_int64
        L.hom_last_error.argtypes = [P, ctypes.POINTER(ErrorInfo)]
        L.hom_destroy.argtypes = [P]
        L.hom_destroy.restype = None
        for name in EXPORTS:
            getattr(L, name)
        _lib = L
    return _lib


def _np_ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class Homogenizer:
    """One context (hom_ctx) on the current CUDA device.

    Tensors passed in and out are torch float64 CUDA tensors; the library only
    sees their raw device pointers and the current stream.
    """

    def __init__(self, macro_coords, macro_conn, dirichlet_dof, dirichlet_value, body_force,
                 rve_coords, rve_conn, phase, materials, kind="linear", cg_rtol=1e-13, cg_max_iter=20000,
                 rve_chunk=0, check_info=True, mem_budget_gb=0.0, tile_sparse=False, rve_range=None,
                 nodal_force=None, macro_basis="dirac", rve_ordering="folded", macro_precond="auto"):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("Homogenizer needs a CUDA device (no CPU fallback)")
        self.torch = torch
        L = lib()
        dim = macro_coords.shape[1]
        self._keep = []

        def arr(x, dt):
            a = np.ascontiguousarray(x, dtype=dt)
            self._keep.append(a)
            return a

        mc, mconn = arr(macro_coords, np.float64), arr(macro_conn, np.int32)
        dd, dv = arr(dirichlet_dof, np.int32), arr(dirichlet_value, np.float64)
        bf = None if body_force is None else arr(body_force, np.float64)
        nf = None if nodal_force is None else arr(nodal_force, np.float64)
        rc_, rconn = arr(rve_coords, np.float64), arr(rve_conn, np.int32)
        ph = arr(phase, np.uint8)
        mt = arr(materials, np.float64)
        if macro_basis not in ("dirac", "constant"):
            raise ValueError("macro_basis must be 'dirac' (one RVE per Gauss point) or 'constant' (per element)")
        n_rve = mconn.shape[0] * (2 ** dim if macro_basis == "dirac" else 1)
        per_rve_phase = int(ph.ndim == 2 and ph.shape[0] > 1)
        per_rve_mat = int(mt.ndim == 3 and mt.shape[0] > 1)
        if per_rve_phase and ph.shape[0] != n_rve:
            raise ValueError("phase must be [n_rve][n_rve_elems] or [n_rve_elems]")
        if per_rve_mat and mt.shape[0] != n_rve:
            raise ValueError("materials must be [n_rve][n_phase][2] or [n_phase][2]")
        n_phase = mt.shape[-2]
        self.macro = MacroMesh(dim, mc.shape[0], mconn.shape[0], mconn.shape[1], _np_ptr(mc), _np_ptr(mconn),
                               len(dd), _np_ptr(dd), _np_ptr(dv), _np_ptr(bf), _np_ptr(nf))
        self.rve = RveMesh(dim, rc_.shape[0], rconn.shape[0], rconn.shape[1], _np_ptr(rc_), _np_ptr(rconn))
        self.phase = PhaseField(per_rve_phase, _np_ptr(ph))
        kinds = {"linear": 0, "nh": 1, "mr": 2}  # mr: the paper's Cook energy with beta
        self.mat = Materials(kinds[kind], n_phase, per_rve_mat, _np_ptr(mt))
        rb, rn = (0, 0) if rve_range is None else (int(rve_range[0]), int(rve_range[1]) - int(rve_range[0]))
        self.opt = Options(int(kind != "linear"), cg_rtol, cg_max_iter, rve_chunk, int(check_info), mem_budget_gb,
                           int(tile_sparse), rb, rn, int(macro_basis == "constant"),
                           {"folded": 0, "natural": 1}[rve_ordering], {"auto": 0, "jacobi": 1, "two_level": 2}[macro_precond])
        self.finite = kind != "linear"
        h = ctypes.c_void_p()
        rc = L.hom_setup(ctypes.byref(h), ctypes.byref(self.macro), ctypes.byref(self.rve),
                         ctypes.byref(self.phase), ctypes.byref(self.mat), ctypes.byref(self.opt), self._stream())
        self.h = h
        if rc != HOM_OK:
            err = self.last_error()
            L.hom_destroy(h)
            self.h = None
            raise HomError(rc, err, "hom_setup")
        s = Sizes()
        L.hom_get_sizes(h, ctypes.byref(s))
        self.sizes = s
        w = Work()
        L.hom_get_work(h, ctypes.byref(w))
        self.work = w
        self.n_rve, self.m, self.n_pad = s.n_rve, s.m, s.n_pad
        self.n_dof = s.n_macro_dof
        self.dim = dim

    @classmethod
    def from_workload(cls, wl, **kw):
        """Context for a workload; with macro_basis="constant" the RVE of element e takes the phase
        and material rows of the element's first Gauss-point RVE."""
        mc, mconn = wl.macro_mesh()
        rc_, rconn = wl.rve_mesh()
        step = wl.n_qp if kw.get("macro_basis", "dirac") == "constant" else 1
        phase = wl.phase[::step] if wl.phase.shape[0] > 1 else wl.phase[0]
        mat = wl.mat[::step] if wl.mat.shape[0] > 1 else wl.mat[0]
        nodal = getattr(wl, "nodal_force", None)
        return cls(mc, mconn, wl.dir_dof, wl.dir_val, wl.body, rc_, rconn, phase, mat, kind=wl.kind,
                   nodal_force=nodal, **kw)

    # ------------------------------------------------------------------ helpers
    def _stream(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream().cuda_stream)

    def _ptr(self, t):
        if t is None:
            return None
        if not (t.is_cuda and t.dtype == self.torch.float64 and t.is_contiguous()):
            raise ValueError("expected a contiguous float64 CUDA tensor")
        return ctypes.c_void_p(t.data_ptr())

    def _check(self, rc, where):
        if rc != HOM_OK:
            raise HomError(rc, self.last_error(), where)

    def empty(self, *shape):
        return self.torch.empty(*shape, dtype=self.torch.float64, device="cuda")

    def last_error(self) -> ErrorInfo:
        e = ErrorInfo()
        if self.h:
            lib().hom_last_error(self.h, ctypes.byref(e))
        return e

    # ------------------------------------------------------------------ API
    def macro_kinematics(self, u, out=None):
        out = self.empty(self.n_rve, self.m) if out is None else out
        self._check(lib().hom_macro_kinematics(self.h, self._ptr(u), self._ptr(out), self._stream()),
                    "hom_macro_kinematics")
        return out

    def condense(self, kin=None, C_eff=None, P_eff=None, P_avg=None):
        C_eff = self.empty(self.n_rve, self.m, self.m) if C_eff is None else C_eff
        if self.finite:
            P_eff = self.empty(self.n_rve, self.m) if P_eff is None else P_eff
            P_avg = self.empty(self.n_rve, self.m) if P_avg is None else P_avg
        self._check(lib().hom_condense(self.h, self._ptr(kin), self._ptr(C_eff), self._ptr(P_eff),
                                       self._ptr(P_avg), self._stream()), "hom_condense")
        return (C_eff, P_eff, P_avg) if self.finite else C_eff

    def macro_solve(self, D, S=None, scale=1.0, x=None):
        x = self.empty(self.n_dof) if x is None else x
        info = SolveInfo()
        self._check(lib().hom_macro_solve(self.h, self._ptr(D), self._ptr(S), float(scale), self._ptr(x),
                                          ctypes.byref(info), self._stream()), "hom_macro_solve")
        return x, info

    def set_load_factor(self, lf):
        self._check(lib().hom_set_load_factor(self.h, float(lf)), "hom_set_load_factor")

    def macro_assemble(self, D):
        self._check(lib().hom_macro_assemble(self.h, self._ptr(D), self._stream()), "hom_macro_assemble")

    def debug_rve_kff(self, rve):
        """K1 output of one RVE as a dense [N_pad][N_pad] tensor in the natural layout (verification)."""
        out = self.empty(self.n_pad, self.n_pad)
        self._check(lib().hom_debug_rve_kff(self.h, int(rve), self._ptr(out), self._stream()), "hom_debug_rve_kff")
        return out

    def macro_spmv(self, x, y=None):
        y = self.empty(self.n_dof) if y is None else y
        self._check(lib().hom_macro_spmv(self.h, self._ptr(x), self._ptr(y), self._stream()), "hom_macro_spmv")
        return y

    def macro_residual_norm(self, S):
        v = ctypes.c_double()
        self._check(lib().hom_macro_residual_norm(self.h, self._ptr(S), ctypes.byref(v), self._stream()),
                    "hom_macro_residual_norm")
        return v.value

    def recover(self, x, w=None):
        if not self.finite and w is None:
            w = self.empty(self.n_rve, self.n_pad)
        self._check(lib().hom_recover_fluctuations(self.h, self._ptr(x), self._ptr(w), self._stream()),
                    "hom_recover_fluctuations")
        return w

    def newton_update(self, u, du):
        self._check(lib().hom_newton_update(self.h, self._ptr(u), self._ptr(du), self._stream()),
                    "hom_newton_update")

    def macro_update(self, u, du):
        self._check(lib().hom_macro_update(self.h, self._ptr(u), self._ptr(du), self._stream()), "hom_macro_update")

    def set_fluctuations(self, w):
        self._check(lib().hom_set_fluctuations(self.h, self._ptr(w), self._stream()), "hom_set_fluctuations")

    def get_fluctuations(self, w=None):
        w = self.empty(self.n_rve, self.n_pad) if w is None else w
        self._check(lib().hom_get_fluctuations(self.h, self._ptr(w), self._stream()), "hom_get_fluctuations")
        return w

    def micro_residual_max(self):
        v = ctypes.c_double()
        self._check(lib().hom_micro_residual_max(self.h, ctypes.byref(v), self._stream()), "hom_micro_residual_max")
        return v.value

    def set_phases(self, phase=None, params=None):
        """Copy a new phase field / material table from HOST memory (numpy or pinned torch CPU tensors)."""
        def hp(x):
            if x is None:
                return None
            if hasattr(x, "data_ptr"):
                return ctypes.c_void_p(x.data_ptr())
            return x.ctypes.data_as(ctypes.c_void_p)
        self._check(lib().hom_set_phases(self.h, hp(phase), hp(params), self._stream()), "hom_set_phases")

    def get_element_cavg(self, out=None):
        """Constant basis: the local rows of the per-element <C> [B][m][m] (other rows untouched)."""
        out = self.empty(self.n_rve, self.m, self.m) if out is None else out
        self._check(lib().hom_get_element_cavg(self.h, self._ptr(out), self._stream()), "hom_get_element_cavg")
        return out

    def set_element_cavg(self, cavg):
        self._check(lib().hom_set_element_cavg(self.h, self._ptr(cavg), self._stream()), "hom_set_element_cavg")

    def profile(self, enable=True):
        self._check(lib().hom_profile_enable(self.h, int(enable)), "hom_profile_enable")

    def profile_read(self):
        ms = (ctypes.c_double * 6)()
        n = (ctypes.c_int64 * 6)()
        self._check(lib().hom_profile_read(self.h, ms, n), "hom_profile_read")
        return {k: (ms[i], n[i]) for i, k in enumerate(PROF_CLASSES)}

    def launch_count(self) -> int:
        return int(lib().hom_launch_count(self.h))

    def close(self):
        if getattr(self, "h", None):
            lib().hom_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ drivers
    def solve_linear(self):
        """Linear step: condense -> macro CG -> recovery.  Returns (C_eff, u, w, info)."""
        C = self.condense()
        u, info = self.macro_solve(C)
        w = self.recover(u)
        return C, u, w, info

    def newton(self, n_steps, tol=1e-11, max_iter=25, history=None, force_load=False, micro_tol=None,
               divergence=1e10, raise_on_fail=True, on_step=None):
        """Finite-strain load stepping with the monolithic null-space Newton (generalized scheme,
        P:325-342).

        Per iteration: F = I + grad u; condense -> (A_eff, P_eff, <P>); check ||R_macro|| (with <P>)
        and max ||r_f|| / |Omega| (reading R3; micro_tol=None uses tol, micro_tol=inf checks the macro
        residual only, as the paper's Cook study); solve the condensed system for du
        (eq:solution2); update u and w.  Load steps: the Dirichlet values (default) or,
        with force_load, the external load factor k/n_steps (T_k = k T / n_l).  Failure:
        ||R_macro|| > divergence, a micro J <= 0, or max_iter.  Returns u (device) and the
        per-step residual histories [(||R_macro||, max ||r_f||), ...]; on_step(k, u) is called after
        every converged load step k (u on the device)."""
        u = self.torch.zeros(self.n_dof, dtype=self.torch.float64, device="cuda")
        du = self.empty(self.n_dof)
        mtol = tol if micro_tol is None else micro_tol
        hist_all = []
        for k in range(1, n_steps + 1):
            if force_load:
                self.set_load_factor(k / n_steps)
            hist = []
            converged = False
            for it in range(max_iter + 1):
                F = self.macro_kinematics(u)
                try:
                    A, Pe, Pa = self.condense(F)
                except HomError as e:
                    if e.code != 4:
                        raise
                    hist.append((float("inf"), float("inf")))
                    break
                rn = self.macro_residual_norm(Pa)
                rf = self.micro_residual_max()
                hist.append((rn, rf))
                if it > 0 and rn <= tol and rf <= mtol:
                    converged = True
                    break
                if not (rn <= divergence) or it == max_iter:
                    break
                scale = (1.0 / n_steps) if (it == 0 and not force_load) else 0.0
                self.macro_solve(A, Pe, scale=scale, x=du)
                self.newton_update(u, du)
            hist_all.append(hist)
            if history is not None:
                history.append(hist)
            if on_step is not None and converged:
                on_step(k, u)
            if not converged:
                if raise_on_fail:
                    raise HomError(5, None, f"Newton did not converge in load step {k}: {hist[-1]}")
                return u, hist_all
        return u, hist_all

    def newton_classical(self, n_steps, tol=1e-9, micro_tol=1e-13, max_iter=25, max_inner=30, divergence=1e10,
                         force_load=True, predictor=True):
        """Classical staggered FE^2 scheme for comparison with the generalized one:
        every macro iteration first equilibrates all RVEs at the fixed macro deformation
        (batched inner Newton on R_micro: w <- w - K_ff^-1 r_f until max ||r_f|| / |Omega| < micro_tol,
        the paper's 1e-13; R_micro normalisation: DESIGN.md R21),
        then solves [K - D L^-1 E] dq = -R_macro (eq:solution1, no -D L^-1 R_micro term),
        updates q and w with eq:reduction (dw = -L^-1 E dq) and restarts until
        ||R_macro|| < tol; failure if ||R_macro|| > divergence, J <= 0 or no convergence.
        Returns (u, histories [(||R_macro||, [inner max ||r_f||, ...]), ...] per step, ok)."""
        u = self.torch.zeros(self.n_dof, dtype=self.torch.float64, device="cuda")
        du = self.empty(self.n_dof)
        zero = self.torch.zeros(self.n_dof, dtype=self.torch.float64, device="cuda")
        hist_all = []
        for k in range(1, n_steps + 1):
            if force_load:
                self.set_load_factor(k / n_steps)
            hist = []
            converged = False
            for it in range(max_iter + 1):
                F = self.macro_kinematics(u)
                inner = []
                try:
                    for _ in range(max_inner + 1):
                        A, Pe, Pa = self.condense(F)
                        rf = self.micro_residual_max()
                        inner.append(rf)
                        if rf < micro_tol or not (rf <= divergence):
                            break
                        self.newton_update(u, zero)  # w -= K_ff^-1 r_f at fixed F
                except HomError as e:
                    if e.code != 4:
                        raise
                    hist.append((float("inf"), inner))
                    break
                rn = self.macro_residual_norm(Pa)
                hist.append((rn, inner))
                if not inner[-1] < micro_tol:
                    break
                if it > 0 and rn <= tol:
                    converged = True
                    break
                if not (rn <= divergence) or it == max_iter:
                    break
                self.macro_solve(A, Pa, scale=0.0, x=du)
                if predictor:
                    self.newton_update(u, du)  # q += dq; w += -L^-1 E dq (r_f ~ 0 after the inner loop)
                else:  # variant without the eq:reduction predictor: q += dq only
                    self.macro_update(u, du)
            hist_all.append(hist)
            if not converged:
                return u, hist_all, False
        return u, hist_all, True

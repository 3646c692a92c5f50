"""CPU checks of the C-ABI boundary: libhom.so builds for sm_100a, loads, exports
every symbol include/hom.h declares, and rejects bad meshes before touching the GPU."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2312_12771_b200 import hom
from paper_2312_12771_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_declares_exactly_the_exported_api():
    src = open(os.path.join(ROOT, "include", "hom.h")).read()
    declared = set(re.findall(r"^\s*(?:int|void|int64_t)\s+(hom_\w+)\s*\(", src, re.M))
    assert declared == set(hom.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    L = hom.lib()
    for name in hom.EXPORTS:
        assert getattr(L, name) is not None
    out = subprocess.run(["nm", "-D", hom.LIB_PATH], capture_output=True, text=True).stdout
    for name in hom.EXPORTS:
        assert re.search(rf"\bT {name}\b", out), name


def test_library_is_sm100a_with_dmma():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", hom.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert "DMMA" in out  # FP64 tensor-core path of the condensation kernel


def _setup_raw(wl, coords=None, dirichlet_dof=None):
    mc, mconn = wl.macro_mesh()
    rc_, rconn = wl.rve_mesh()
    if coords is not None:
        rc_ = coords
    dd = np.ascontiguousarray(wl.dir_dof if dirichlet_dof is None else dirichlet_dof, np.int32)
    dv = np.zeros(len(dd))
    ph = np.ascontiguousarray(wl.phase[0])
    mt = np.ascontiguousarray(wl.mat[0])
    keep = [mc, mconn, rc_, rconn, dd, dv, ph, mt]
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    macro = hom.MacroMesh(2, mc.shape[0], mconn.shape[0], 4, p(mc), p(mconn), len(dd), p(dd), p(dv), None)
    rve = hom.RveMesh(2, rc_.shape[0], rconn.shape[0], 4, p(rc_), p(rconn))
    phase = hom.PhaseField(0, p(ph))
    mat = hom.Materials(0, mt.shape[0], 0, p(mt))
    opt = hom.Options(0, 1e-13, 100, 0, 1, 0.0)
    h = ctypes.c_void_p()
    rc = hom.lib().hom_setup(ctypes.byref(h), macro, rve, phase, mat, opt, None)
    err = hom.ErrorInfo()
    hom.lib().hom_last_error(h, ctypes.byref(err))
    hom.lib().hom_destroy(h)
    del keep
    return rc, err


def test_unmatched_periodic_faces_rejected():
    wl = W.config1(nel=2, r=4)
    rc_, _ = wl.rve_mesh()
    bad = rc_.copy()
    bad[4, 1] += 0.05  # node (4, 0) on the right face no longer matches (0, 0)
    rc, err = _setup_raw(wl, coords=bad)
    assert rc == 2, err.message  # HOM_ERR_MESH


def test_dirichlet_dof_out_of_range_rejected():
    wl = W.config1(nel=2, r=4)
    rc, err = _setup_raw(wl, dirichlet_dof=np.array([10 ** 6], np.int32))
    assert rc == 1, err.message  # HOM_ERR_INVALID_ARG


def test_no_cpu_fallback_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(RuntimeError):
        hom.Homogenizer.from_workload(W.config1())

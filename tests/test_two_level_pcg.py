"""Two-level macro preconditioner (coarse.cu) on the GPU.

The coarse space changes only the PCG iteration count, never the solution of
K_M u = -R (eq:linSys): u is held to the oracle's direct solve at the
north_star tolerance (1e-8) with and without it, the iteration counts must drop
to the numpy model's range (tools/cg_coarse_model.py), and the result is
bitwise reproducible run to run (fixed summation order in A_c, its inverse and
the per-iteration restriction).
"""
import numpy as np
import pytest

import oracle
from paper_2312_12771_b200 import workloads as W

pytestmark = pytest.mark.gpu

TOL_U = 1e-8


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def solve(wl, coarse=True):
    from paper_2312_12771_b200.hom import Homogenizer
    h = Homogenizer.from_workload(wl, macro_precond="two_level" if coarse else "jacobi")
    C, u, w, info = h.solve_linear()
    out = (C.cpu().numpy(), u.cpu().numpy(), info)
    h.close()
    return out


def test_config2_two_level_iterations_and_parity(torch_cuda):
    wl = W.config2()
    C1, u1, i1 = solve(wl, coarse=False)
    C2, u2, i2 = solve(wl, coarse=True)
    o = oracle.macro_solve(2, wl.nel, C2, wl.dir_dof, wl.dir_val, body=wl.body)
    assert rel(u1, o) <= TOL_U and rel(u2, o) <= TOL_U, (rel(u1, o), rel(u2, o))
    assert i2.rel_residual <= 1e-13
    # numpy model: 244 one-level, 83 two-level (8x8 aggregates, translations + rotation)
    assert i1.iterations >= 200 and i2.iterations <= 110, (i1.iterations, i2.iterations)
    _, u3, i3 = solve(wl, coarse=True)
    assert i3.iterations == i2.iterations and np.array_equal(u3, u2)  # bitwise reproducible


def test_config3_macro_two_level_under_400_iterations(torch_cuda):
    """Config 3's macro problem (nel 64, a random C_eff per Gauss point from E in [1, 100]) with
    the RVEs at r = 8 (same macro matrix structure and contrast, fast oracle)."""
    wl = W.config3(r=8)
    C1, u1, i1 = solve(wl, coarse=False)
    C2, u2, i2 = solve(wl, coarse=True)
    o = oracle.solve_linear(wl)
    assert rel(C2, o["C_eff"]) <= 1e-10
    assert rel(u1, o["u"]) <= TOL_U and rel(u2, o["u"]) <= TOL_U, (rel(u1, o["u"]), rel(u2, o["u"]))
    assert i1.iterations >= 600 and i2.iterations < 400, (i1.iterations, i2.iterations)


def test_config4_3d_two_level_parity(torch_cuda):
    """3-D: 6 rigid-body modes per aggregate (3 x 3 x 3 boxes)."""
    wl = W.config4()
    C1, u1, i1 = solve(wl, coarse=False)
    C2, u2, i2 = solve(wl, coarse=True)
    o = oracle.macro_solve(3, wl.nel, C2, wl.dir_dof, wl.dir_val, body=wl.body)
    assert rel(u1, o) <= TOL_U and rel(u2, o) <= TOL_U, (rel(u1, o), rel(u2, o))
    assert i2.iterations < i1.iterations, (i1.iterations, i2.iterations)


def test_mapped_mesh_two_level_parity(torch_cuda):
    """Cook's trapezoid (mapped macro mesh) at nel 24: aggregates are boxes of the
    bounding box, so some are partly empty; one small-strain solve with the phase pattern of the
    Cook workload and the Neo-Hookean reference tangent replaced by a linear material."""
    ck = W.cook(nel=24, r=8, n_steps=1)
    mc, conn = ck.macro_mesh()
    wl = W.config2(nel=24, r=8)
    wl.macro_coords = mc
    wl.body = np.array([0.0, -1.0])
    C1, u1, i1 = solve(wl, coarse=False)
    C2, u2, i2 = solve(wl, coarse=True)
    o = oracle.macro_solve(2, 24, C2, wl.dir_dof, wl.dir_val, body=wl.body, mesh=(mc, conn))
    assert rel(u1, o) <= TOL_U and rel(u2, o) <= TOL_U, (rel(u1, o), rel(u2, o))
    assert i2.iterations < i1.iterations, (i1.iterations, i2.iterations)


def test_fully_constrained_aggregates_drop_their_modes(torch_cuda):
    """The leftmost node columns (both components) are prescribed: the aggregates of that strip have
    no free DOF, their rows of A_c are zero and the sweep drops those modes (pivot <= 1e-10 of the
    original diagonal); a roller strip (x components only) leaves a rank-deficient mode pattern in
    the next aggregates.  u must still match the direct solve and the coarse space must still pay."""
    wl = W.config2(nel=32, r=8)
    nn = wl.nel + 1
    nodes = np.arange(nn * nn)
    ix = nodes % nn
    clamp = nodes[ix <= 5]
    roll = nodes[(ix >= 6) & (ix <= 9)]
    dof = np.concatenate([2 * clamp, 2 * clamp + 1, 2 * roll]).astype(np.int32)
    wl.dir_dof = np.sort(dof)
    wl.dir_val = np.zeros(len(dof))
    C1, u1, i1 = solve(wl, coarse=False)
    C2, u2, i2 = solve(wl, coarse=True)
    o = oracle.macro_solve(2, wl.nel, C2, wl.dir_dof, wl.dir_val, body=wl.body)
    assert rel(u1, o) <= TOL_U and rel(u2, o) <= TOL_U, (rel(u1, o), rel(u2, o))
    assert i2.iterations < i1.iterations, (i1.iterations, i2.iterations)


@pytest.mark.parametrize("precond", ["two_level", "jacobi"])
@pytest.mark.parametrize("cfg", [2, 4])
def test_persistent_grid_pcg_matches_direct_solve(torch_cuda, precond, cfg, monkeypatch):
    """The cooperative one-CTA-per-SM PCG (meshes beyond one cluster; forced here on the config-2 and the
    3-D config-4 meshes) gives the direct solve's u and the cluster kernel's iteration count with the
    two-level form."""
    from paper_2312_12771_b200.hom import Homogenizer
    wl = W.config2(nel=32, r=8) if cfg == 2 else W.config4(r=4)
    h = Homogenizer.from_workload(wl, macro_precond=precond)
    C = h.condense()
    u_c, i_c = h.macro_solve(C)
    u_c = u_c.cpu().numpy()
    monkeypatch.setenv("HOM_CG_FORCE_GRID", "1")
    u_g, i_g = h.macro_solve(C)
    u_g = u_g.cpu().numpy()
    monkeypatch.delenv("HOM_CG_FORCE_GRID")
    o = oracle.macro_solve(wl.dim, wl.nel, C.cpu().numpy(), wl.dir_dof, wl.dir_val, body=wl.body)
    h.close()
    assert rel(u_g, o) <= TOL_U and rel(u_c, o) <= TOL_U, (rel(u_g, o), rel(u_c, o))
    assert i_g.rel_residual <= 1e-13
    if precond == "two_level":
        assert abs(i_g.iterations - i_c.iterations) <= 3, (i_g.iterations, i_c.iterations)

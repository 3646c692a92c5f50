"""The RVE-sharded driver (paper_2312_12771_b200/dist.py) on a real GPU with the NCCL backend.
Only one GPU is available, so the process group has world size 1: this exercises the device
path end to end (context with an RVE range, padded all-gather over NCCL, replicated macro CG,
local recovery, the finite-strain iteration with its MAX all-reduce) against the
single-context path, bit for bit.  The partition / exchange logic for world size 2 is covered
on CPU by tests/test_dist_gloo.py."""
import os
import socket

import numpy as np
import pytest

from paper_2312_12771_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def nccl_group():
    import torch
    import torch.distributed as dist
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


def test_sharded_linear_solve_nccl_equals_single_context(nccl_group):
    import torch
    from paper_2312_12771_b200.dist import ShardedHomogenizer
    from paper_2312_12771_b200.hom import Homogenizer
    wl = W.config3(nel=3, r=10, seed=29)
    sh = ShardedHomogenizer(wl)
    C, u, w, info = sh.solve_linear()
    torch.cuda.synchronize()
    h = Homogenizer.from_workload(wl)
    C1, u1, w1, info1 = h.solve_linear()
    assert info.iterations == info1.iterations
    assert torch.equal(C, C1) and torch.equal(u, u1) and torch.equal(w, w1)


def test_sharded_newton_iteration_nccl_equals_single_context(nccl_group):
    import torch
    from paper_2312_12771_b200.dist import ShardedHomogenizer
    from paper_2312_12771_b200.hom import Homogenizer
    wl = W.config5(nel=2, n_steps=2)
    out = []
    for sharded in (True, False):
        h = ShardedHomogenizer(wl) if sharded else Homogenizer.from_workload(wl)
        hh = h.h if sharded else h
        B, m = hh.n_rve, hh.m
        u = hh.empty(hh.n_dof).zero_()
        F, A, Pe, Pa, du = hh.empty(B, m), hh.empty(B, m, m), hh.empty(B, m), hh.empty(B, m), hh.empty(hh.n_dof)
        if sharded:
            rn, rf, _ = h.newton_iteration(u, F, A, Pe, Pa, du, scale=1.0 / wl.n_steps)
        else:
            hh.macro_kinematics(u, F)
            hh.condense(F, A, Pe, Pa)
            rn = hh.macro_residual_norm(Pa)
            rf = hh.micro_residual_max()
            hh.macro_solve(A, Pe, scale=1.0 / wl.n_steps, x=du)
            hh.newton_update(u, du)
        torch.cuda.synchronize()
        out.append((rn, rf, A.cpu().numpy(), u.cpu().numpy()))
    (rn0, rf0, A0, u0), (rn1, rf1, A1, u1) = out
    assert rn0 == rn1 and rf0 == rf1
    assert np.array_equal(A0, A1) and np.array_equal(u0, u1)

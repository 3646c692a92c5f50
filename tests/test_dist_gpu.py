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


def test_sharded_constant_basis_nccl_equals_single_context(nccl_group):
    import torch
    from paper_2312_12771_b200.dist import ShardedHomogenizer
    from paper_2312_12771_b200.hom import Homogenizer
    wl = W.config3(nel=3, r=8, seed=37)
    C, u, w, _ = ShardedHomogenizer(wl, macro_basis="constant").solve_linear()
    C1, u1, w1, _ = Homogenizer.from_workload(wl, macro_basis="constant").solve_linear()
    torch.cuda.synchronize()
    assert torch.equal(C, C1) and torch.equal(u, u1) and torch.equal(w, w1)


def _nccl_world2_worker(rank, port, out_dir):
    import torch
    import torch.distributed as dist

    from paper_2312_12771_b200.dist import ShardedHomogenizer
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=2,
                            device_id=torch.device("cuda", rank))
    wl = W.config3(nel=3, r=10, seed=29)
    C, u, w, info = ShardedHomogenizer(wl).solve_linear()
    torch.cuda.synchronize()
    lo, hi = ShardedHomogenizer(wl).parts[rank]
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), C=C.cpu().numpy(), u=u.cpu().numpy(),
             w=w[lo:hi].cpu().numpy(), lo=lo, hi=hi)
    dist.destroy_process_group()


def test_sharded_linear_solve_nccl_world2():
    """World size 2 over NCCL on two GPUs (skipped on a one-GPU box): every rank ends with the
    single-context C_eff and u bit for bit, and its own rows of w."""
    import tempfile

    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    from paper_2312_12771_b200.hom import Homogenizer
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_nccl_world2_worker, args=(_free_port(), d), nprocs=2, join=True)
        res = [np.load(os.path.join(d, f"r{r}.npz")) for r in range(2)]
    torch.cuda.set_device(0)
    C1, u1, w1, _ = Homogenizer.from_workload(W.config3(nel=3, r=10, seed=29)).solve_linear()
    for r in res:
        assert np.array_equal(r["C"], C1.cpu().numpy()) and np.array_equal(r["u"], u1.cpu().numpy())
        assert np.array_equal(r["w"], w1.cpu().numpy()[int(r["lo"]):int(r["hi"])])

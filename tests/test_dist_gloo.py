"""Host-side logic of the RVE-sharded multi-GPU path (paper_2312_12771_b200/dist.py)
on CPU: world size 2 over gloo, with the CPU oracle standing in for the per-rank condensation and
the macro solve (only the partition, the collective and the orchestration are under test here;
the GPU kernels are covered by tests/test_gpu_parity.py)."""
import os
import socket
import tempfile

import numpy as np
import pytest

from paper_2312_12771_b200 import workloads as W
from paper_2312_12771_b200.dist import rve_partition


@pytest.mark.parametrize("n_elems,n_qp,world", [(16, 4, 1), (16, 4, 2), (9, 4, 2), (512, 8, 3), (3, 4, 8)])
def test_rve_partition_is_element_aligned_balanced_cover(n_elems, n_qp, world):
    parts = rve_partition(n_elems, n_qp, world)
    assert len(parts) == world
    assert parts[0][0] == 0 and parts[-1][1] == n_elems * n_qp
    for (a, b), (c, d) in zip(parts, parts[1:]):
        assert b == c
    sizes = [(b - a) for a, b in parts]
    assert all(s % n_qp == 0 for s in sizes)
    assert max(sizes) - min(sizes) <= n_qp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2312_12771_b200.dist import allgather_rows, sharded_linear_solve
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl = W.config3(nel=3, r=6, seed=21)  # 9 macro elements -> uneven 5/4 split
    parts = rve_partition(wl.nel ** wl.dim, wl.n_qp, world)
    lo, hi = parts[rank]
    m = wl.m

    def condense_local():
        C = torch.full((wl.n_rve, m, m), float("nan"), dtype=torch.float64)
        Cl, Wl = oracle.condense_batch_linear(wl.dim, wl.r, wl.phase[lo:hi], wl.mat[lo:hi], hi - lo, want_W=True,
                                              nthreads=1)
        C[lo:hi] = torch.from_numpy(Cl)
        condense_local.W = Wl
        return C

    def solve(C):
        assert not torch.isnan(C).any()  # every row arrived through the exchange
        return oracle.macro_solve(wl.dim, wl.nel, C.numpy(), wl.dir_dof, wl.dir_val, body=wl.body)

    def recover(u):
        eps = oracle.macro_kin(wl.dim, wl.nel, u)[lo:hi]
        return oracle.recover_linear(condense_local.W, eps)

    C, u, w = sharded_linear_solve(condense_local, lambda C: allgather_rows(C, parts, rank), solve, recover)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), C=C.numpy(), u=u, w=w, lo=lo, hi=hi)
    dist.destroy_process_group()


def test_sharded_linear_solve_world2_matches_single_process():
    import torch.multiprocessing as mp

    import oracle
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        res = [np.load(os.path.join(d, f"r{r}.npz")) for r in range(2)]
    wl = W.config3(nel=3, r=6, seed=21)
    o = oracle.solve_linear(wl)
    w_o = oracle.recover_linear(o["W"], o["eps"])
    for r in res:
        # per-RVE work is independent of the partition: the exchanged tangents and the
        # replicated macro solution equal the single-process oracle bit for bit
        assert np.array_equal(r["C"], o["C_eff"])
        assert np.array_equal(r["u"], o["u"])
        assert np.array_equal(r["w"], w_o[int(r["lo"]):int(r["hi"])])
    assert int(res[0]["hi"]) == int(res[1]["lo"])


def _packed_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    from paper_2312_12771_b200.dist import allgather_packed
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    parts = rve_partition(9, 4, world)  # uneven 5/4 element split
    B = 36
    lo, hi = parts[rank]
    A = torch.full((B, 4, 4), float("nan"), dtype=torch.float64)
    P = torch.full((B, 4), float("nan"), dtype=torch.float64)
    b = torch.arange(B, dtype=torch.float64)
    A[lo:hi] = b[lo:hi, None, None] * 100 + torch.arange(16, dtype=torch.float64).reshape(4, 4)
    P[lo:hi] = -b[lo:hi, None] - torch.arange(4, dtype=torch.float64) / 10
    sc = allgather_packed([A, P], parts, rank, scalars=(float(rank + 1) * 1.5, -rank))
    np.savez(os.path.join(out_dir, f"p{rank}.npz"), A=A.numpy(), P=P.numpy(), sc=np.array(sc))
    dist.destroy_process_group()


def test_allgather_packed_world2_one_collective_for_all_tensors_and_scalars():
    """The packed exchange (one all-gather per Newton iteration: A_eff, P_eff, <P> and each rank's
    max ||R_micro||) delivers every row of every tensor and every rank's scalars to every rank."""
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_packed_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        res = [np.load(os.path.join(d, f"p{r}.npz")) for r in range(2)]
    b = np.arange(36, dtype=np.float64)
    A = b[:, None, None] * 100 + np.arange(16).reshape(4, 4)
    P = -b[:, None] - np.arange(4) / 10
    for r in res:
        assert np.array_equal(r["A"], A) and np.array_equal(r["P"], P)
        assert r["sc"].tolist() == [[1.5, 0.0], [3.0, -1.0]]

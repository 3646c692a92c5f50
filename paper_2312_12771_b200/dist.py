"""RVE-sharded multi-GPU driver.

The micro problems are independent: the micro-micro block L of the monolithic system is
block-diagonal over the RVEs, so the batch shards across GPUs with no
communication inside the condensation.  The one real exchange step is the macro Schur
system eq:solution2, which couples every RVE through its condensed tangent:

  1. macro elements are split into contiguous ranges, one per rank, so all 2^dim Gauss-point
     RVEs of an element live on the same rank (``rve_partition``);
  2. each rank condenses its RVEs (``hom_condense`` with ``rve_range``);
  3. ONE all-gather of the condensed tangents C_eff (and P_eff, <P> in finite strain) over
     NCCL (NVLink / NVSwitch) -- ``allgather_rows``;
  4. every rank solves the small macro problem redundantly (identical inputs, deterministic
     kernels -> identical u on every rank), and
  5. recovers the fluctuations of its own RVEs.

Only argument marshalling and the collective live here; all arithmetic runs in libhom.so.
The orchestration (``sharded_linear_solve``) takes its compute steps as callables so that the
host-side logic is exercised by world-size-2 gloo tests on CPU (tests/test_dist_gloo.py).
"""
from __future__ import annotations

from typing import Callable, List, Sequence, Tuple


def rve_partition(n_elems: int, n_qp: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous, balanced split of the macro elements over `world` ranks, returned as
    RVE ranges [b_lo, b_hi) (RVE b = e * n_qp + q)."""
    if world <= 0 or n_elems < 0:
        raise ValueError("world must be positive")
    base, extra = divmod(n_elems, world)
    out, e0 = [], 0
    for r in range(world):
        ne = base + (1 if r < extra else 0)
        out.append((e0 * n_qp, (e0 + ne) * n_qp))
        e0 += ne
    return out


def allgather_rows(full, parts: Sequence[Tuple[int, int]], rank: int, group=None):
    """All-gather the rows [b_lo, b_hi) each rank owns into every rank's `full` (a torch tensor,
    first dimension = RVE).  Ranks may own different row counts: every rank contributes a slab
    padded to the largest part (equal-size collectives), the padding is dropped on receipt."""
    import torch
    import torch.distributed as dist
    rows = max(hi - lo for lo, hi in parts)
    lo, hi = parts[rank]
    send = torch.zeros((rows,) + tuple(full.shape[1:]), dtype=full.dtype, device=full.device)
    send[: hi - lo] = full[lo:hi]
    recv = [torch.empty_like(send) for _ in parts]
    dist.all_gather(recv, send, group=group)
    for (l, h), r in zip(parts, recv):
        full[l:h] = r[: h - l]
    return full


def sharded_linear_solve(condense_local: Callable, exchange: Callable, macro_solve: Callable,
                         recover_local: Callable):
    """Small-strain path on one rank: local condensation -> exchange of C_eff -> replicated
    macro solve -> local recovery.  Returns (C_eff (all rows after the exchange), u, w)."""
    C = condense_local()
    C = exchange(C)
    u = macro_solve(C)
    w = recover_local(u)
    return C, u, w


class ShardedHomogenizer:
    """One libhom context per rank, condensing only that rank's RVE range of one macro problem.

    Needs an initialised torch.distributed process group (NCCL on GPUs) and the current CUDA
    device set to this rank's GPU."""

    def __init__(self, wl, group=None, **kw):
        import torch.distributed as dist

        from .hom import Homogenizer
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        n_elems = wl.nel ** wl.dim
        per_elem = 1 if kw.get("macro_basis", "dirac") == "constant" else wl.n_qp
        self.parts = rve_partition(n_elems, per_elem, self.world)
        self.b_lo, self.b_hi = self.parts[self.rank]
        self.h = Homogenizer.from_workload(wl, rve_range=(self.b_lo, self.b_hi), **kw)
        self.n_rve, self.m, self.n_pad, self.n_dof = self.h.n_rve, self.h.m, self.h.n_pad, self.h.n_dof

    @property
    def n_local(self) -> int:
        return self.b_hi - self.b_lo

    def exchange(self, full):
        return allgather_rows(full, self.parts, self.rank, self.group)

    def solve_linear(self, C=None, u=None, w=None):
        h = self.h
        C = h.empty(self.n_rve, self.m, self.m) if C is None else C
        u = h.empty(self.n_dof) if u is None else u
        w = h.empty(self.n_rve, self.n_pad) if w is None else w
        info = {}

        def solve(Cf):
            x, inf = h.macro_solve(Cf, None, 1.0, u)
            info["cg"] = inf
            return x

        C, u, w = sharded_linear_solve(lambda: h.condense(None, C), self.exchange, solve, lambda x: h.recover(x, w))
        return C, u, w, info["cg"]

    def newton_iteration(self, u, F, A, Pe, Pa, du, scale=0.0):
        """One monolithic Newton iteration of the finite-strain path (eq:solution2,
        P:424-427) on this rank: local condensation, exchange of A_eff / P_eff / <P>, replicated
        residual check and macro solve, local fluctuation update.  Returns (||R_macro||,
        max_b ||r_f,b|| over all ranks, CG info)."""
        import torch
        import torch.distributed as dist
        h = self.h
        h.macro_kinematics(u, F)
        h.condense(F, A, Pe, Pa)
        for t in (A, Pe, Pa):
            self.exchange(t)
        rn = h.macro_residual_norm(Pa)
        rf = torch.tensor([h.micro_residual_max()], dtype=torch.float64, device=A.device)
        dist.all_reduce(rf, op=dist.ReduceOp.MAX, group=self.group)
        _, info = h.macro_solve(A, Pe, scale=scale, x=du)
        h.newton_update(u, du)
        return rn, float(rf.item()), info

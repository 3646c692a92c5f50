"""RVE-sharded multi-GPU driver.

The micro problems are independent: the micro-micro block L of the monolithic system is
block-diagonal over the RVEs, so the batch shards across GPUs with no
communication inside the condensation.  The one real exchange step is the macro Schur
system eq:solution2, which couples every RVE through its condensed tangent:

  1. macro elements are split into contiguous ranges, one per rank, so all 2^dim Gauss-point
     RVEs of an element live on the same rank (``rve_partition``);
  2. each rank condenses its RVEs (``hom_condense`` with ``rve_range``);
  3. ONE all-gather per solve / Newton iteration over NCCL (NVLink / NVSwitch): the condensed
     tangents C_eff (plus <C>_e with the constant macro basis; A_eff, P_eff, <P> and the rank's
     max ||R_micro|| in finite strain) packed into one slab per rank -- ``allgather_packed``;
  4. every rank solves the small macro problem redundantly (identical inputs, deterministic
     kernels -> identical u on every rank), and
  5. recovers the fluctuations of its own RVEs.

Only argument marshalling and the collective live here; all arithmetic runs in libhom.so.
The orchestration (``sharded_linear_solve``) takes its compute steps as callables so that the
host-side logic is exercised by world-size-2 gloo tests on CPU (tests/test_dist_gloo.py).
"""
from __future__ import annotations

import math
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


def allgather_packed(tensors, parts: Sequence[Tuple[int, int]], rank: int, group=None, scalars=()):
    """ONE all-gather for several per-RVE tensors (first dimension = RVE, all on one device) plus a
    few per-rank scalars: each rank packs its rows [b_lo, b_hi) of every tensor side by side into
    one [rows_max + 1][K] slab (the extra row carries the scalars), the slabs are all-gathered in
    a single collective, and every rank unpacks all rows into its tensors.  Returns the list of
    per-rank scalar tuples (rank order)."""
    import torch
    import torch.distributed as dist
    rows = max(hi - lo for lo, hi in parts)
    lo, hi = parts[rank]
    widths = [math.prod(t.shape[1:]) for t in tensors]
    K = max(sum(widths), len(scalars), 1)
    ref = tensors[0]
    send = torch.zeros((rows + 1, K), dtype=torch.float64, device=ref.device)
    c0 = 0
    for t, wd in zip(tensors, widths):
        send[: hi - lo, c0:c0 + wd] = t[lo:hi].reshape(hi - lo, wd)
        c0 += wd
    if scalars:
        send[rows, : len(scalars)] = torch.tensor([float(x) for x in scalars], dtype=torch.float64)
    recv = [torch.empty_like(send) for _ in parts]
    dist.all_gather(recv, send, group=group)
    out = []
    for (l, h), r in zip(parts, recv):
        c0 = 0
        for t, wd in zip(tensors, widths):
            t[l:h] = r[: h - l, c0:c0 + wd].reshape((h - l,) + tuple(t.shape[1:]))
            c0 += wd
        out.append(tuple(r[rows, : len(scalars)].tolist()))
    return out


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
        self.macro_basis = kw.get("macro_basis", "dirac")
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
        constant = self.macro_basis == "constant"
        Ca = h.empty(self.n_rve, self.m, self.m) if constant else None

        def exchange(Cf):
            # constant basis: the macro stiffness also needs <C>_e of every element (hom_get/set_element_cavg)
            if constant:
                h.get_element_cavg(Ca)
            allgather_packed([Cf, Ca] if constant else [Cf], self.parts, self.rank, self.group)
            if constant:
                h.set_element_cavg(Ca)
            return Cf

        def solve(Cf):
            x, inf = h.macro_solve(Cf, None, 1.0, u)
            info["cg"] = inf
            return x

        C, u, w = sharded_linear_solve(lambda: h.condense(None, C), exchange, solve, lambda x: h.recover(x, w))
        return C, u, w, info["cg"]

    def newton_iteration(self, u, F, A, Pe, Pa, du, scale=0.0):
        """One monolithic Newton iteration of the finite-strain path (eq:solution2,
        P:424-427) on this rank: local condensation, exchange of A_eff / P_eff / <P>, replicated
        residual check and macro solve, local fluctuation update.  Returns (||R_macro||,
        max_b ||r_f,b|| / |Omega| over all ranks, CG info)."""
        h = self.h
        h.macro_kinematics(u, F)
        h.condense(F, A, Pe, Pa)
        # one collective per Newton iteration: A_eff, P_eff, <P> rows and this rank's max ||R_micro||
        rf_local = h.micro_residual_max()
        per_rank = allgather_packed([A, Pe, Pa], self.parts, self.rank, self.group, scalars=(rf_local,))
        rf = max(x[0] for x in per_rank)
        rn = h.macro_residual_norm(Pa)
        _, info = h.macro_solve(A, Pe, scale=scale, x=du)
        h.newton_update(u, du)
        return rn, rf, info

"""Brute-force monolithic two-scale solver for tiny instances (test code, numpy only).

Assembles the FULL uncondensed system of PAPER.md eq:discreteSystem_global
 with the blocks K, D, E, L of eq:discreteSys_K/D/L,
using the Dirac macro basis (one RVE per macro Gauss point), and
solves it densely.  It has its own shape functions, periodic map and material
laws and shares nothing with oracle/hom_oracle.c, so agreement with the
oracle's condensed path (check (e) of BASELINE.json north_star) pins the
condensation, the unit-strain route and the macro solve at once.
"""
from __future__ import annotations

import itertools

import numpy as np

G = 1.0 / np.sqrt(3.0)


def _ref_nodes(dim):
    if dim == 2:
        return np.array([[-1, -1], [1, -1], [1, 1], [-1, 1]], float)
    quad = [[-1, -1], [1, -1], [1, 1], [-1, 1]]
    return np.array([[x, y, z] for z in (-1, 1) for x, y in quad], float)


def _qps(dim):
    # x fastest
    return [np.array(p[::-1]) * G for p in itertools.product([-1, 1], repeat=dim)]


def _grads(dim, h, xi):
    """Physical gradients of the multilinear shape functions on an axis-aligned box with edge
    lengths h (a scalar: cube)."""
    h = np.broadcast_to(np.asarray(h, dtype=float), (dim,))
    sn = _ref_nodes(dim)
    out = np.zeros((len(sn), dim))
    for a, s in enumerate(sn):
        for k in range(dim):
            v = s[k] / 2.0
            for l in range(dim):
                if l != k:
                    v *= (1 + s[l] * xi[l]) / 2.0
            out[a, k] = v * 2.0 / h[k]
    return out


def _shape(dim, xi):
    sn = _ref_nodes(dim)
    return np.array([np.prod([(1 + s[k] * xi[k]) / 2.0 for k in range(dim)]) for s in sn])


def _elem_nodes(dim, n, e):
    idx = []
    t = e
    for _ in range(dim):
        idx.append(t % n)
        t //= n
    offs = ((_ref_nodes(dim) + 1) / 2).astype(int)
    return [sum((idx[k] + o[k]) * (n + 1) ** k for k in range(dim)) for o in offs], idx


def _grad_op(dim, g):
    """Displacement gradient operator: rows (i,J) row-major, cols (a,c)."""
    nen = g.shape[0]
    B = np.zeros((dim * dim, nen * dim))
    for a in range(nen):
        for i in range(dim):
            for J in range(dim):
                B[i * dim + J, a * dim + i] = g[a, J]
    return B


def iso_tangent_full(dim, E, nu):
    """Fourth-order isotropic tangent lambda d_ij d_kl + mu (d_ik d_jl + d_il d_jk), (ij),(kl) row-major."""
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    d = np.eye(dim)
    C = (lam * np.einsum("ij,kl->ijkl", d, d) + mu * (np.einsum("ik,jl->ijkl", d, d)
                                                      + np.einsum("il,jk->ijkl", d, d)))
    return C.reshape(dim * dim, dim * dim)


def nh_response(F, alpha, kappa):
    """P and A of Psi = alpha(F:F-2) + kappa/2 (J-1)^2 - 2 alpha ln J (2-D), by direct differentiation."""
    F = F.reshape(2, 2)
    J = np.linalg.det(F)
    H = np.array([[F[1, 1], -F[1, 0]], [-F[0, 1], F[0, 0]]])  # dJ/dF
    s = kappa * (J - 1) - 2 * alpha / J
    P = 2 * alpha * F + s * H
    t = kappa + 2 * alpha / J ** 2
    dH = np.zeros((2, 2, 2, 2))
    dH[0, 0, 1, 1] = 1
    dH[0, 1, 1, 0] = -1
    dH[1, 0, 0, 1] = -1
    dH[1, 1, 0, 0] = 1
    A = 2 * alpha * np.einsum("ik,jl->ijkl", np.eye(2), np.eye(2)) + t * np.einsum("ij,kl->ijkl", H, H) + s * dH
    return P.reshape(4), A.reshape(4, 4), J


def periodic_dofs(dim, r):
    """Map full RVE node -> free DOF index (or -1) with the corner class fixed."""
    nn = (r + 1) ** dim
    m = {}
    cnt = 0
    dofmap = -np.ones((nn, dim), int)
    indep = np.zeros(nn, int)
    for node in range(nn):
        t, ijk = node, []
        for _ in range(dim):
            ijk.append(t % (r + 1))
            t //= (r + 1)
        p = sum((ijk[k] % r) * r ** k for k in range(dim))
        indep[node] = p
        if p == 0:
            continue
        if p not in m:
            m[p] = cnt
            cnt += 1
        dofmap[node] = [m[p] * dim + c for c in range(dim)]
    return dofmap, cnt * dim, indep


class Monolithic:
    """Tiny two-scale problem: macro grid nel^dim on [0,1]^dim, RVE r^dim on [0,1]^dim.

    basis "dirac": one fluctuation field per macro Gauss point (eq:fluctVaria_dirac);
    basis "constant": one per macro element, shared by its Gauss points (eq:constSolution1/2,
    P:294-315) -- the micro equations are then integrated over the whole element."""

    def __init__(self, dim, nel, r, tangent_of, dir_dof, body=None, basis="dirac", rve_axes=None):
        """tangent_of(b, e) -> full-gradient tangent (dim^2 x dim^2) for linear problems
        (b = fluctuation field index: Gauss point or element)."""
        self.dim, self.nel, self.r = dim, nel, r
        self.rve_axes = rve_axes  # [dim][r+1] node coordinates of a tensor-product RVE grid (None: uniform)
        self.tangent_of = tangent_of
        self.dir_dof = np.asarray(dir_dof)
        self.body = body
        self.basis = basis
        self.nq = 2 ** dim
        self.ndof_M = (nel + 1) ** dim * dim
        self.dofmap, self.nf, self.indep = periodic_dofs(dim, r)
        self.n_rve = nel ** dim * (self.nq if basis == "dirac" else 1)
        self.N = self.ndof_M + self.n_rve * self.nf

    def _macro_ops(self):
        dim, nel = self.dim, self.nel
        for e in range(nel ** dim):
            nodes, _ = _elem_nodes(dim, nel, e)
            dofs = [n * dim + c for n in nodes for c in range(dim)]
            for q, xi in enumerate(_qps(dim)):
                g = _grads(dim, 1.0 / nel, xi)
                yield e * self.nq + q, dofs, _grad_op(dim, g), _shape(dim, xi), (1.0 / nel) ** dim / 2 ** dim * 1.0

    def _micro_ops(self):
        dim, r = self.dim, self.r
        for e in range(r ** dim):
            nodes, idx = _elem_nodes(dim, r, e)
            fd = np.concatenate([self.dofmap[n] for n in nodes])
            if self.rve_axes is None:
                h = np.full(dim, 1.0 / r)
            else:
                h = np.array([self.rve_axes[k][idx[k] + 1] - self.rve_axes[k][idx[k]] for k in range(dim)])
            for xi in _qps(dim):
                g = _grads(dim, h, xi)
                yield e, fd, _grad_op(dim, g), np.prod(h) / 2 ** dim

    def assemble(self, u=None, w=None, material=None):
        """Hessian and gradient of the two-scale energy (linear: quadratic energy).

        For nonlinear problems pass material(b, e, Ftilde) -> (P, A) and the state (u, w).
        Weights: macro eta_k j_k = (h^d/2^d)*2^d... (unit Gauss weights times det J).
        """
        dim = self.dim
        N = self.N
        Kg = np.zeros((N, N))
        Rg = np.zeros(N)
        vol = 1.0  # |Omega| of the unit cell
        for b, mdofs, Bm, Nm, _ in self._macro_ops():
            wM = (1.0 / self.nel) ** dim  # Gauss weight 1 x det J = (h/2)^d * 2^d / 2^d ... see below
            wM = (0.5 / self.nel) ** dim
            grad_u = Bm @ u[mdofs] if u is not None else np.zeros(dim * dim)
            if self.basis == "constant":
                b = b // self.nq  # the element's single fluctuation field
            off = self.ndof_M + b * self.nf
            for e, fd, Bf, wm in self._micro_ops():  # wm = det J (unit Gauss weights) of the micro element
                free = fd >= 0
                cols = np.concatenate([np.asarray(mdofs), off + fd[free]])
                Bfull = np.concatenate([Bm, Bf[:, free]], axis=1)
                if material is None:
                    A = self.tangent_of(b, e)
                    P = None
                else:
                    wl = np.zeros(Bf.shape[1])
                    if w is not None:
                        wl[free] = w[b][fd[free]]
                    F = np.eye(dim).reshape(-1) + grad_u + Bf @ wl
                    P, A = material(b, e, F)
                    Rg[cols] += wM * wm / vol * (Bfull.T @ P)
                Kg[np.ix_(cols, cols)] += wM * wm / vol * (Bfull.T @ A @ Bfull)
            if self.body is not None:
                for a in range(len(Nm)):
                    for c in range(dim):
                        Rg[mdofs[a * dim + c]] -= wM * Nm[a] * self.body[c]
        return Kg, Rg

    def solve_linear(self, u_dir):
        """Minimise the quadratic two-scale energy with Dirichlet values u_dir at dir_dof."""
        K, R = self.assemble(u=np.zeros(self.ndof_M))
        x = np.zeros(self.N)
        x[self.dir_dof] = u_dir
        free = np.ones(self.N, bool)
        free[self.dir_dof] = False
        rhs = -R[free] - K[np.ix_(free, self.dir_dof)] @ x[self.dir_dof]
        x[free] = np.linalg.solve(K[np.ix_(free, free)], rhs)
        return self.split(x)

    def newton_step(self, u, w, material, du_dir):
        K, R = self.assemble(u=u, w=w, material=material)
        dx = np.zeros(self.N)
        dx[self.dir_dof] = du_dir
        free = np.ones(self.N, bool)
        free[self.dir_dof] = False
        rhs = -R[free] - K[np.ix_(free, self.dir_dof)] @ dx[self.dir_dof]
        dx[free] = np.linalg.solve(K[np.ix_(free, free)], rhs)
        return self.split(dx)

    def split(self, x):
        u = x[: self.ndof_M]
        w = x[self.ndof_M:].reshape(self.n_rve, self.nf)
        return u, w

    def to_indep_layout(self, w):
        """Free-DOF fluctuations -> [n_rve][dim r^dim] independent-node layout (pad = 0)."""
        dim, r = self.dim, self.r
        out = np.zeros((w.shape[0], dim * r ** dim))
        for node in range((r + 1) ** dim):
            p = self.indep[node]
            for c in range(dim):
                d = self.dofmap[node, c]
                if d >= 0:
                    out[:, p * dim + c] = w[:, d]
        return out

    def from_indep_layout(self, W):
        out = np.zeros((W.shape[0], self.nf))
        for node in range((self.r + 1) ** self.dim):
            p = self.indep[node]
            for c in range(self.dim):
                d = self.dofmap[node, c]
                if d >= 0:
                    out[:, d] = W[:, p * self.dim + c]
        return out

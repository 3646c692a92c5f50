"""Seeded synthetic workloads for the five BASELINE.json configs.

This module holds input generation only -- meshes, phase fields, material
tables, boundary data -- and none of the method's arithmetic.  It is the one
module shared by the oracle-side tests and the GPU path.

Conventions:
  * macro and RVE domains are [0,1]^d with uniform grids, nodes lexicographic
    (x fastest), Q1 counter-clockwise / hex8 bottom-then-top local order;
  * RVE b = e * 2^d + q (one RVE per macro Gauss point, Dirac basis P:246-292);
  * phases are per RVE element, assigned by element centroid;
  * config 3 draws u_s(i, j) = top 53 bits of splitmix64(seed ^ (s << 56) ^
    (i << 24) ^ j) / 2^53, seed 12771.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

SEED = 12771
_M64 = (1 << 64) - 1


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 finaliser on uint64 (wrapping arithmetic)."""
    z = (x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15))
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def uniform(seed: int, s: int, i, j) -> np.ndarray:
    """Counter-based U[0,1) draw u_s(i, j)."""
    i = np.asarray(i, dtype=np.uint64)
    j = np.asarray(j, dtype=np.uint64)
    key = np.uint64(seed) ^ (np.uint64(s) << np.uint64(56)) ^ (i << np.uint64(24)) ^ j
    with np.errstate(over="ignore"):
        z = splitmix64(key)
    return (z >> np.uint64(11)).astype(np.float64) / float(1 << 53)


# --------------------------------------------------------------------------
# structured meshes
# --------------------------------------------------------------------------
def local_offsets(dim: int) -> np.ndarray:
    """Integer offsets of the local nodes (CCW in 2-D, bottom then top face in 3-D)."""
    if dim == 1:
        return np.array([[0], [1]])
    quad = np.array([[0, 0], [1, 0], [1, 1], [0, 1]])
    if dim == 2:
        return quad
    return np.array([[x, y, z] for z in (0, 1) for x, y in quad])


def grid_mesh(dim: int, n: int, L: float = 1.0):
    """Uniform grid of [0,L]^dim with n cells per direction -> (coords, conn)."""
    idx = np.indices([n + 1] * dim).reshape(dim, -1)[::-1].T  # columns x, y, z; x fastest
    coords = idx * (L / n)
    off = local_offsets(dim)
    cells = np.indices([n] * dim).reshape(dim, -1)[::-1].T  # columns: x, y, z with x fastest
    strides = np.array([(n + 1) ** k for k in range(dim)])
    conn = ((cells[:, None, :] + off[None, :, :]) * strides).sum(-1).astype(np.int32)
    return np.ascontiguousarray(coords, dtype=np.float64), np.ascontiguousarray(conn)


def centroids(dim: int, n: int) -> np.ndarray:
    cells = np.indices([n] * dim).reshape(dim, -1)[::-1].T
    return (cells + 0.5) / n


def boundary_nodes(dim: int, n: int) -> np.ndarray:
    idx = np.indices([n + 1] * dim).reshape(dim, -1)[::-1].T
    return np.nonzero(((idx == 0) | (idx == n)).any(1))[0]


def face_nodes(dim: int, n: int, axis: int, value: int) -> np.ndarray:
    idx = np.indices([n + 1] * dim).reshape(dim, -1)[::-1].T
    return np.nonzero(idx[:, axis] == value)[0]


# --------------------------------------------------------------------------
# workloads
# --------------------------------------------------------------------------
@dataclasses.dataclass
class Workload:
    name: str
    dim: int
    nel: int               # macro cells per direction
    r: int                 # RVE cells per direction
    kind: str              # "linear" (E, nu), "nh" (alpha, kappa) or "mr" (alpha, beta, kappa)
    phase: np.ndarray      # [n_rve | 1][r^dim] uint8
    mat: np.ndarray        # [n_rve | 1][n_phase][2] float64
    dir_dof: np.ndarray    # int32 Dirichlet DOFs (node*dim + comp)
    dir_val: np.ndarray    # float64 prescribed values (total load)
    body: np.ndarray | None
    n_steps: int = 1
    description: str = ""
    macro_coords: np.ndarray | None = None   # mapped (non-rectangular) macro grid; None = [0,1]^dim
    nodal_force: np.ndarray | None = None    # [n_dof] external nodal forces (surface tractions)
    rve_size: float = 1.0
    rve_origin: float = 0.0
    rve_axes: np.ndarray | None = None     # [dim][r+1] node coordinates of a graded tensor-product RVE grid

    @property
    def n_qp(self) -> int:
        return 2 ** self.dim

    @property
    def n_rve(self) -> int:
        return self.nel ** self.dim * self.n_qp

    @property
    def n_dof(self) -> int:
        return (self.nel + 1) ** self.dim * self.dim

    @property
    def n_pad(self) -> int:
        return self.dim * self.r ** self.dim

    @property
    def n_f(self) -> int:
        return self.n_pad - self.dim

    @property
    def m(self) -> int:
        if self.kind in ("nh", "mr"):
            return self.dim * self.dim
        return {1: 1, 2: 3, 3: 6}[self.dim]

    def macro_mesh(self):
        coords, conn = grid_mesh(self.dim, self.nel)
        return (coords if self.macro_coords is None else self.macro_coords), conn

    def rve_mesh(self):
        coords, conn = grid_mesh(self.dim, self.r, self.rve_size)
        if self.rve_axes is not None:  # graded tensor-product grid: node index -> axis coordinate
            idx = np.rint(coords * (self.r / self.rve_size)).astype(np.int64)
            coords = np.stack([self.rve_axes[d][idx[:, d]] for d in range(self.dim)], -1)
            return np.ascontiguousarray(coords), conn
        return np.ascontiguousarray(coords + self.rve_origin), conn

    def flop_per_rve(self) -> float:
        """Dense condensation flops counted on n_f: n^3/3 + 2 n^2 m + n m^2."""
        n, m = self.n_f, self.m + (1 if self.kind == "nh" else 0)
        return n ** 3 / 3.0 + 2.0 * n * n * m + n * m * m


def _affine_dirichlet(dim, nel, strain11):
    nodes = boundary_nodes(dim, nel)
    coords, _ = grid_mesh(dim, nel)
    dofs, vals = [], []
    for n in nodes:
        for c in range(dim):
            dofs.append(n * dim + c)
            vals.append(strain11 * coords[n, 0] if c == 0 else 0.0)
    return np.array(dofs, np.int32), np.array(vals)


def _clamped_left(dim, nel):
    nodes = face_nodes(dim, nel, 0, 0)
    dofs = np.array([n * dim + c for n in nodes for c in range(dim)], np.int32)
    return dofs, np.zeros(len(dofs))


def _inclusion_phase(dim, r, vf):
    rad = math.sqrt(vf / math.pi) if dim == 2 else (3.0 * vf / (4.0 * math.pi)) ** (1.0 / 3.0)
    c = centroids(dim, r)
    return (np.linalg.norm(c - 0.5, axis=1) < rad).astype(np.uint8)[None, :]


def config1(nel: int = 4, r: int = 8) -> Workload:
    c = centroids(2, r)
    phase = (c[:, 0] >= 0.5).astype(np.uint8)[None, :]
    mat = np.array([[[1.0, 0.3], [10.0, 0.3]]])
    d, v = _affine_dirichlet(2, nel, 1e-3)
    return Workload("cfg1_laminate", 2, nel, r, "linear", phase, mat, d, v, None,
                    description="2-D laminate, affine eps_xx = 1e-3 on the boundary")


def config2(nel: int = 32, r: int = 16) -> Workload:
    phase = _inclusion_phase(2, r, 0.3)
    mat = np.array([[[1.0, 0.3], [10.0, 0.3]]])
    d, v = _clamped_left(2, nel)
    return Workload("cfg2_disc", 2, nel, r, "linear", phase, mat, d, v, np.array([0.0, -1.0]),
                    description="2-D centred disc vf 0.3, E ratio 10, clamped left edge, body force (0,-1)")


def config3(nel: int = 64, r: int = 32, seed: int = SEED) -> Workload:
    n_rve = nel * nel * 4
    nelr = r * r
    b = np.arange(n_rve, dtype=np.uint64)[:, None]
    e = np.arange(nelr, dtype=np.uint64)[None, :]
    phase = (uniform(seed, 0, b, e) < 0.4).astype(np.uint8)
    p = np.arange(2, dtype=np.uint64)[None, :]
    E = 10.0 ** (2.0 * uniform(seed, 1, b, p))
    nu = 0.2 + 0.2 * uniform(seed, 2, b, p)
    mat = np.stack([E, nu], axis=-1)
    d, v = _clamped_left(2, nel)
    return Workload("cfg3_random", 2, nel, r, "linear", phase, mat, d, v, np.array([0.0, -1.0]),
                    description="2-D Bernoulli(0.4) phases, E log-uniform [1,100], nu U[0.2,0.4] per phase per RVE")


def config4(nel: int = 8, r: int = 8) -> Workload:
    phase = _inclusion_phase(3, r, 0.2)
    mat = np.array([[[1.0, 0.3], [20.0, 0.3]]])
    d, v = _affine_dirichlet(3, nel, 1e-3)
    return Workload("cfg4_sphere", 3, nel, r, "linear", phase, mat, d, v, None,
                    description="3-D centred sphere vf 0.2, E ratio 20, affine uniaxial strain 1e-3")


def config5(nel: int = 32, r: int = 16, n_steps: int = 10, stretch: float = 0.1) -> Workload:
    phase = _inclusion_phase(2, r, 0.3)
    mat = np.array([[[0.5, 2.0], [5.0, 20.0]]])  # (alpha, kappa): mu = 2 alpha, lambda = kappa
    dl, vl = _clamped_left(2, nel)
    right = face_nodes(2, nel, 0, nel)
    dr = np.array([n * 2 for n in right], np.int32)
    d = np.concatenate([dl, dr])
    v = np.concatenate([vl, np.full(len(dr), stretch)])
    return Workload("cfg5_neohooke", 2, nel, r, "nh", phase, mat, d, v, None, n_steps=n_steps,
                    description="2-D finite-strain Neo-Hookean disc, right edge stretched to 1.1 in 10 steps")


COOK_CORNERS = np.array([[0.0, 0.0], [480.0, 440.0], [480.0, 600.0], [0.0, 440.0]])  # P1..P4
COOK_TRACTION = np.array([-5.0, 10.0])  # on the right edge Gamma^sigma_r (eq:load)
COOK_MATERIALS = np.array([[27.0, 18.0, 60.0], [13.5, 6.5, 30.0]])  # (alpha, beta, kappa)


def cook(nel: int = 20, r: int = 30, n_steps: int = 22) -> Workload:
    """Cook's membrane of PAPER.md §4.2: the trapezoid P1 (0,0), P2 (480,440),
    P3 (480,600), P4 (0,440) meshed with nel x nel bilinear Q1 (the image of the uniform grid
    under the bilinear map of the corners), left edge X1 = 0 fixed, traction T = (-5, 10) on the
    right edge as consistent nodal forces (exact for the constant traction and linear edge
    shape functions), one periodic RVE (-3,3)^2 with r x r Q1 per macro Gauss point (Dirac
    basis), a centred cross of width 2 of material 2 (by element centroid) in material 1, the
    paper's energy with beta (kind "mr"), T_k = k T / n_steps."""
    coords, conn = grid_mesh(2, nel)
    xi, eta = coords[:, 0], coords[:, 1]
    P = COOK_CORNERS
    X = (np.outer((1 - xi) * (1 - eta), P[0]) + np.outer(xi * (1 - eta), P[1]) + np.outer(xi * eta, P[2]) +
         np.outer((1 - xi) * eta, P[3]))
    left = face_nodes(2, nel, 0, 0)
    d = np.array([2 * n + c for n in left for c in (0, 1)], np.int32)
    f = np.zeros((nel + 1) ** 2 * 2)
    right = face_nodes(2, nel, 0, nel)  # ordered by eta
    ys = X[right, 1]
    seg = np.diff(ys)
    wgt = np.zeros(len(right))
    wgt[:-1] += seg / 2
    wgt[1:] += seg / 2
    for n, wv in zip(right, wgt):
        f[2 * n:2 * n + 2] += wv * COOK_TRACTION
    c = (centroids(2, r) - 0.5) * 6.0  # element centroids in (-3,3)^2
    phase = ((np.abs(c[:, 0]) < 1.0) | (np.abs(c[:, 1]) < 1.0)).astype(np.uint8)[None]
    return Workload("cook", 2, nel, r, "mr", phase, COOK_MATERIALS[None].copy(), d, np.zeros(len(d)), None,
                    n_steps=n_steps, description=f"Cook's membrane, {nel}x{nel} macro Q1, RVE {r}x{r} cross, "
                                                 f"{n_steps} load steps",
                    macro_coords=np.ascontiguousarray(X), nodal_force=f, rve_size=6.0, rve_origin=-3.0)


def bench1d(k: int) -> Workload:
    """The paper's 1-D analytical benchmark (§5.1), Dirac basis [delta,1]:
    B_0 = (0,1000) with 2^k P1 macro elements (2 Gauss points), RVE (0,1) with 2^k P1 elements,
    lambda(X~) = 20 / cos(2 pi X~/3 - pi/3), Psi~ = lambda (F~^2 - 1) -> tangent 2 lambda (R14),
    body load B = 1, phi(0) = 0, phi(1000) = 37575 sqrt(3) / (2 pi); the unknown is the position
    phi (linear problem).  For P1 elements only the element average of the tangent enters, so each
    RVE element carries its own "phase" with E = 2 * (2-point Gauss average of lambda), nu = 0
    (1-D C = lambda_Lame + 2 mu = E); 2^k <= 255."""
    n = 2 ** k
    if n > 255:
        raise ValueError("bench1d: one phase per RVE element, 2^k <= 255")
    g = 1.0 / np.sqrt(3.0)
    xc = (np.arange(n)[:, None] + 0.5 + 0.5 * np.array([-g, g])[None, :]) / n
    lam = 20.0 / np.cos(2 * np.pi * xc / 3 - np.pi / 3)
    mat = np.stack([2.0 * lam.mean(1), np.zeros(n)], -1)[None]
    coords, _ = grid_mesh(1, n, 1000.0)
    phi1000 = 37575.0 * np.sqrt(3.0) / (2.0 * np.pi)  # P:459 (R14)
    return Workload(f"bench1d_k{k}", 1, n, n, "linear", np.arange(n, dtype=np.uint8)[None], mat,
                    np.array([0, n], np.int32), np.array([0.0, phi1000]), np.array([1.0]),
                    description=f"paper 1-D benchmark, 2^{k} elements per scale", macro_coords=coords)


def graded_axes(r: int, dim: int, a: float = 0.6) -> np.ndarray:
    """Graded node coordinates per axis on [0,1]: x(s) = s - a sin(2 pi s) / (2 pi), s = k / r
    (monotone for a < 1, element widths from (1 - a)/r at the faces to (1 + a)/r in the middle,
    symmetric about 1/2; the periodic faces stay at 0 and 1)."""
    s = np.arange(r + 1) / r
    x = s - a * np.sin(2 * np.pi * s) / (2 * np.pi)
    x[0], x[-1] = 0.0, 1.0
    return np.tile(x, (dim, 1))


def graded(dim: int = 2, nel: int = 4, r: int = 16, seed: int = SEED, a: float = 0.6) -> Workload:
    """A graded periodic RVE (the K1 path for meshes with many distinct element geometries, DESIGN.md
    §5.3): config 3's inputs (per-RVE random phases and moduli, body force, clamped left edge) in 2-D,
    config 4's (affine uniaxial strain, all boundary nodes) in 3-D, on a tensor-product RVE grid with
    the element widths of graded_axes."""
    wl = config3(nel=nel, r=r, seed=seed) if dim == 2 else config4(nel=nel, r=r)
    if dim == 3:  # per-RVE random phases / moduli in 3-D as well
        n = wl.n_rve
        e = np.arange(r ** 3)
        b = np.arange(n)[:, None]
        wl.phase = (uniform(seed, 0, b, e[None, :]) < 0.4).astype(np.uint8)
        u1 = uniform(seed, 1, b, np.arange(2)[None, :])
        u2 = uniform(seed, 2, b, np.arange(2)[None, :])
        wl.mat = np.stack([10.0 ** (2 * u1), 0.2 + 0.2 * u2], -1)
    wl.rve_axes = graded_axes(r, dim, a)
    wl.name = f"graded{dim}d"
    wl.description = f"{dim}-D graded periodic RVE {r}^{dim} (x = s - {a} sin(2 pi s)/(2 pi)), per-RVE random phases"
    return wl


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}


def make(cfg: int, **kw) -> Workload:
    return CONFIGS[cfg](**kw)

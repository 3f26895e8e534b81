"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no basis functions, no quadrature,
no Jacobians, no contractions): only the structured hexahedral meshes, the
connectivity tables and the seeded random material / DOF arrays that both the
oracle (oracle/) and the CUDA path (paper_2107_04121_b200/) consume.  It imports
neither of them.

Recipe (the paper's own 1D-bar mesh, PAPER.md
P:1091-1100, is replaced by the BASELINE.json configs' perturbed N^3 grids):
  * unit-cube structured grid of nx*ny*nz hexahedra, h = 1/n per axis;
  * vertices lexicographic (x fastest); elements lexicographic (ex fastest);
  * element vertex v = a + 2b + 4c (x fastest, not VTK order);
  * order-p nodes on the (p nx + 1)(p ny + 1)(p nz + 1) lattice, element-local
    node (i,j,k) of element (ex,ey,ez) = global node
    (p ex + i) + Mx ((p ey + j) + My (p ez + k));
  * rng = numpy.random.default_rng(210704121 + config_index), draws in order:
      1. displacements U(-0.15 h, 0.15 h) of shape (n_vertices, 3), then
         multiplied by the interior-vertex mask (boundary vertices stay put);
      2. materials: per-qp arrays [E][n_q] U[1,2] (kappa, then rho), or
         per-element Lame lambda then mu [E] U[0.5, 2];
      3. the DOF / state vector [n_nodes][D].
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

SEED_BASE = 210704121

# form identifiers (same numbering as include/feb200.h fe_form and the oracle)
DIFFUSION = 0
MASS = 1
VECTOR_MASS = 2
MASS_DIFFUSION = 3
ELASTICITY = 4
CONVECTIVE = 5
WEIGHTED_DOT = 6    # Tab. 2 'ij,i,j': M per qp [E][n_q][3][3]
DIVERGENCE = 7      # Tab. 2 'i.i': linear form, no material
FORM_NAMES = {DIFFUSION: "diffusion", MASS: "mass", VECTOR_MASS: "vector_mass",
              MASS_DIFFUSION: "mass_diffusion", ELASTICITY: "elasticity",
              CONVECTIVE: "convective", WEIGHTED_DOT: "weighted_dot",
              DIVERGENCE: "divergence"}
FORM_NCOMP = {DIFFUSION: 1, MASS: 1, VECTOR_MASS: 3, MASS_DIFFUSION: 1,
              ELASTICITY: 3, CONVECTIVE: 3, WEIGHTED_DOT: 3, DIVERGENCE: 3}

# material kinds (include/feb200.h fe_material_kind)
MAT_PER_QP = 0
MAT_PER_ELEM = 1
MAT_FULL_D = 2


@dataclass
class Problem:
    """One seeded FE problem: mesh + material + DOF vector (host numpy arrays)."""
    name: str
    form: int
    p: int
    q1d: int
    shape: tuple                      # (nx, ny, nz) cells per axis
    coords: np.ndarray                # [V][3] float64
    conn: np.ndarray                  # [E][8] int32
    dof_conn: np.ndarray              # [E][n_b] int32
    n_nodes: int
    mat_kind: int
    mat_a: Optional[np.ndarray]       # kappa | rho | rho (mass+diff) | lambda
    mat_b: Optional[np.ndarray]       # None  | None | kappa           | mu
    u: np.ndarray                     # [n_nodes][D] float64 (DOF or state vector)
    meta: dict = field(default_factory=dict)

    @property
    def n_elems(self) -> int:
        return int(self.conn.shape[0])

    @property
    def nb(self) -> int:
        return (self.p + 1) ** 3

    @property
    def nq(self) -> int:
        return self.q1d ** 3

    @property
    def ncomp(self) -> int:
        return FORM_NCOMP[self.form]

    @property
    def ndof(self) -> int:
        return self.ncomp * self.nb


def grid_vertices(nx: int, ny: int, nz: int) -> np.ndarray:
    """Unperturbed vertices of the unit-cube grid, lexicographic, x fastest."""
    x = np.linspace(0.0, 1.0, nx + 1)
    y = np.linspace(0.0, 1.0, ny + 1)
    z = np.linspace(0.0, 1.0, nz + 1)
    Z, Y, X = np.meshgrid(z, y, x, indexing="ij")
    return np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)


def interior_mask(nx: int, ny: int, nz: int) -> np.ndarray:
    iz, iy, ix = np.meshgrid(np.arange(nz + 1), np.arange(ny + 1), np.arange(nx + 1), indexing="ij")
    m = (ix > 0) & (ix < nx) & (iy > 0) & (iy < ny) & (iz > 0) & (iz < nz)
    return m.ravel()


def hex_connectivity(nx: int, ny: int, nz: int) -> np.ndarray:
    """conn[E][8] int32, element vertex v = a + 2b + 4c (x fastest)."""
    ez, ey, ex = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    ex, ey, ez = ex.ravel(), ey.ravel(), ez.ravel()
    conn = np.empty((ex.size, 8), dtype=np.int64)
    for c in range(2):
        for b in range(2):
            for a in range(2):
                conn[:, a + 2 * b + 4 * c] = (ex + a) + (nx + 1) * ((ey + b) + (ny + 1) * (ez + c))
    return conn.astype(np.int32)


def lattice_dof_conn(nx: int, ny: int, nz: int, p: int) -> tuple[np.ndarray, int]:
    """dof_conn[E][(p+1)^3] int32 on the order-p node lattice and the node count."""
    Mx, My, Mz = p * nx + 1, p * ny + 1, p * nz + 1
    ez, ey, ex = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    ex, ey, ez = ex.ravel(), ey.ravel(), ez.ravel()
    n1 = p + 1
    dc = np.empty((ex.size, n1 ** 3), dtype=np.int64)
    for k in range(n1):
        for j in range(n1):
            for i in range(n1):
                dc[:, i + n1 * (j + n1 * k)] = (p * ex + i) + Mx * ((p * ey + j) + My * (p * ez + k))
    n_nodes = Mx * My * Mz
    assert n_nodes < 2 ** 31
    return dc.astype(np.int32), n_nodes


def make_problem(form: int, p: int, shape, seed: int, *, q1d: Optional[int] = None,
                 perturb: float = 0.15, mat_kind: Optional[int] = None,
                 u_range: Optional[tuple] = None, name: str = "custom") -> Problem:
    """Build a seeded problem on an nx*ny*nz perturbed grid of the unit cube."""
    nx, ny, nz = shape
    q1d = p + 1 if q1d is None else q1d
    nq = q1d ** 3
    rng = np.random.default_rng(seed)
    V = (nx + 1) * (ny + 1) * (nz + 1)
    h = np.array([1.0 / nx, 1.0 / ny, 1.0 / nz])
    coords = grid_vertices(nx, ny, nz)
    disp = rng.uniform(-perturb, perturb, size=(V, 3)) * h[None, :]  # draw 1
    coords = coords + disp * interior_mask(nx, ny, nz)[:, None]
    conn = hex_connectivity(nx, ny, nz)
    E = conn.shape[0]
    dof_conn, n_nodes = lattice_dof_conn(nx, ny, nz, p)
    D = FORM_NCOMP[form]
    # draw 2: materials
    mat_b = None
    if form in (DIFFUSION, MASS, VECTOR_MASS):
        mk = MAT_PER_QP
        mat_a = rng.uniform(1.0, 2.0, size=(E, nq))
    elif form == MASS_DIFFUSION:
        mk = MAT_PER_QP
        kappa = rng.uniform(1.0, 2.0, size=(E, nq))
        rho = rng.uniform(1.0, 2.0, size=(E, nq))
        mat_a, mat_b = rho, kappa
    elif form == ELASTICITY:
        mk = MAT_PER_ELEM if mat_kind is None else mat_kind
        if mk == MAT_PER_ELEM:
            mat_a = rng.uniform(0.5, 2.0, size=E)
            mat_b = rng.uniform(0.5, 2.0, size=E)
        elif mk == MAT_PER_QP:
            mat_a = rng.uniform(0.5, 2.0, size=(E, nq))
            mat_b = rng.uniform(0.5, 2.0, size=(E, nq))
        else:  # FULL_D: random symmetric positive definite 6x6 per qp
            Araw = rng.uniform(-1.0, 1.0, size=(E, nq, 6, 6))
            mat_a = np.einsum("eqik,eqjk->eqij", Araw, Araw) + 6.0 * np.eye(6)
            mat_b = None
    elif form == WEIGHTED_DOT:  # a general (non-symmetric) 3 x 3 weight per qp, U[-1, 1] + 2 I
        mk = MAT_PER_QP
        mat_a = rng.uniform(-1.0, 1.0, size=(E, nq, 3, 3)) + 2.0 * np.eye(3)
    else:  # CONVECTIVE, DIVERGENCE: no material
        mk = MAT_PER_QP
        mat_a = None
    # draw 3: DOF / state vector
    if u_range is None:
        u_range = (-1e-3, 1e-3) if form == ELASTICITY else (-1.0, 1.0)
    u = rng.uniform(u_range[0], u_range[1], size=(n_nodes, D))
    return Problem(name=name, form=form, p=p, q1d=q1d, shape=(nx, ny, nz), coords=coords,
                   conn=conn, dof_conn=dof_conn, n_nodes=n_nodes, mat_kind=mk,
                   mat_a=None if mat_a is None else np.ascontiguousarray(mat_a),
                   mat_b=None if mat_b is None else np.ascontiguousarray(mat_b),
                   u=np.ascontiguousarray(u))


@dataclass
class MixedProblem:
    """Velocity-pressure pair for the Stokes coupling forms (Tab. 2): `vel` is a
    vector problem of order pv (its u is the velocity DOF vector [n_nodes][3]); the pressure
    space has order pp on the same cells (lattice numbering), nodal values `pres` [n_p]."""
    vel: Problem
    pp: int
    p_dof_conn: np.ndarray            # [E][(pp+1)^3] int32
    n_p_nodes: int
    pres: np.ndarray                  # [n_p] float64

    @property
    def nbp(self) -> int:
        return (self.pp + 1) ** 3


def make_mixed_problem(pv: int, pp: int, shape, seed: int, *, perturb: float = 0.15) -> MixedProblem:
    """Q_pv x Q_pp pair on the perturbed grid of make_problem (draws 1 and 3 as there), plus
    draw 4: pressure values U[-1, 1] from a second generator seeded seed + 1."""
    vel = make_problem(DIVERGENCE, pv, shape, seed, perturb=perturb, name="mixed")
    pdc, n_p = lattice_dof_conn(*shape, pp)
    pres = np.random.default_rng(seed + 1).uniform(-1.0, 1.0, size=n_p)
    return MixedProblem(vel=vel, pp=pp, p_dof_conn=pdc, n_p_nodes=n_p, pres=pres)


# BASELINE.json configs (index k -> seed 210704121 + k)
CONFIGS = {
    "C1": dict(index=0, form=DIFFUSION, p=1, N=4,
               desc="Q1 scalar Laplace matrices, 4^3 perturbed unit cube, 2^3 Gauss, kappa/qp U[1,2]"),
    "C2": dict(index=1, form=DIFFUSION, p=2, N=64,
               desc="Q2 scalar diffusion, 64^3, 3^3 Gauss, kappa/qp U[1,2]; matrix + residual, u U[-1,1]"),
    "C3": dict(index=2, form=ELASTICITY, p=2, N=48,
               desc="Q2 vector isotropic elasticity, 48^3, lambda,mu/elem U[0.5,2]; matrix + residual, u U[-1e-3,1e-3]"),
    "C4": dict(index=3, form=MASS_DIFFUSION, p=4, N=40,
               desc="Q4 scalar mass+Laplace residual, 40^3, 5^3 Gauss, rho,kappa/qp U[1,2], u U[-1,1]; fp64 and fp32"),
    "C5": dict(index=4, form=CONVECTIVE, p=2, N=128,
               desc="Q2 vector convective residual, 128^3, velocity U[-1,1]; tangent matrices on the 64^3 corner"),
}


def make_config(name: str, N: Optional[int] = None) -> Problem:
    """The BASELINE.json config `name` (C1..C5); N overrides the grid size for small tests."""
    c = CONFIGS[name]
    n = c["N"] if N is None else N
    prob = make_problem(c["form"], c["p"], (n, n, n), SEED_BASE + c["index"], name=name)
    prob.meta["desc"] = c["desc"]
    return prob


def corner_subproblem(prob: Problem, n_sub: int) -> Problem:
    """Restriction to the elements with ex, ey, ez < n_sub (C5t, reading 18).

    Keeps the full vertex / node numbering and state vector; only selects elements."""
    nx, ny, nz = prob.shape
    E = prob.n_elems
    idx = np.arange(E)
    ex, ey, ez = idx % nx, (idx // nx) % ny, idx // (nx * ny)
    sel = (ex < n_sub) & (ey < n_sub) & (ez < n_sub)
    sub = Problem(name=prob.name + "t", form=prob.form, p=prob.p, q1d=prob.q1d,
                  shape=(n_sub, n_sub, n_sub), coords=prob.coords,
                  conn=np.ascontiguousarray(prob.conn[sel]),
                  dof_conn=np.ascontiguousarray(prob.dof_conn[sel]), n_nodes=prob.n_nodes,
                  mat_kind=prob.mat_kind,
                  mat_a=None if prob.mat_a is None else np.ascontiguousarray(prob.mat_a[sel]),
                  mat_b=None if prob.mat_b is None else np.ascontiguousarray(prob.mat_b[sel]),
                  u=prob.u)
    sub.meta["parent_shape"] = prob.shape
    return sub


def slab_partition(shape, p: int, n_parts: int, rank: int):
    """Contiguous z-slab of rank `rank` of n_parts (DESIGN.md multi-GPU).

    Returns (elem_begin, elem_end, node_begin, node_end): the rank's element range
    and the contiguous global node range [node_begin, node_end) of the node planes
    p*z0 .. p*z1 inclusive (both interface planes included)."""
    nx, ny, nz = shape
    if nz % n_parts != 0:
        raise ValueError(f"nz={nz} not divisible by {n_parts} ranks")
    z0 = nz * rank // n_parts
    z1 = nz * (rank + 1) // n_parts
    plane = (p * nx + 1) * (p * ny + 1)
    return z0 * nx * ny, z1 * nx * ny, p * z0 * plane, (p * z1 + 1) * plane

"""Pins of the CPU oracle (oracle/) against what the paper and FE theory fix.

CPU only (-m "not gpu").  Each test names the pin of DESIGN.md "Oracle pins":
P1-P3 closed forms (exact rationals computed here with fractions, independently
of the oracle), P4-P10 invariants, P11 the second einsum oracle on the paper's
own strings (tests/einsum_oracle.py), plus the paper's printed shapes
(tests/golden/paper_einsum_examples.txt).
"""
from __future__ import annotations

import os
from fractions import Fraction

import numpy as np
import pytest

import einsum_oracle as eo
import fe_inputs as fi
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- exact 1D
def _poly_mul(a, b):
    out = [Fraction(0)] * (len(a) + len(b) - 1)
    for i, x in enumerate(a):
        for j, y in enumerate(b):
            out[i + j] += x * y
    return out


def _poly_deriv(a):
    return [a[i] * i for i in range(1, len(a))] or [Fraction(0)]


def _poly_int01(a):
    return sum(c / (i + 1) for i, c in enumerate(a))


def _lagrange_exact(p):
    nodes = [Fraction(i, p) for i in range(p + 1)]
    polys = []
    for i in range(p + 1):
        P = [Fraction(1)]
        for j in range(p + 1):
            if j != i:
                P = _poly_mul(P, [-nodes[j] / (nodes[i] - nodes[j]), 1 / (nodes[i] - nodes[j])])
        polys.append(P)
    return polys


def exact_1d(p):
    """M1 = int phi_i phi_j, S1 = int phi_i' phi_j', C1 = int phi_i' phi_j on [0,1]."""
    L = _lagrange_exact(p)
    dL = [_poly_deriv(P) for P in L]
    n = p + 1
    M = [[_poly_int01(_poly_mul(L[i], L[j])) for j in range(n)] for i in range(n)]
    S = [[_poly_int01(_poly_mul(dL[i], dL[j])) for j in range(n)] for i in range(n)]
    C = [[_poly_int01(_poly_mul(dL[i], L[j])) for j in range(n)] for i in range(n)]
    return M, S, C


def _kron3(Az, Ay, Ax):
    """Exact Kronecker product with x fastest: index k = i + n(j + n l)."""
    nz, ny, nx = len(Az), len(Ay), len(Ax)
    N = nx * ny * nz
    out = [[None] * N for _ in range(N)]
    for l in range(nz):
        for j in range(ny):
            for i in range(nx):
                r = i + nx * (j + ny * l)
                for l2 in range(nz):
                    for j2 in range(ny):
                        for i2 in range(nx):
                            c = i2 + nx * (j2 + ny * l2)
                            out[r][c] = Az[l][l2] * Ay[j][j2] * Ax[i][i2]
    return out


def _to_np(A):
    return np.array([[float(x) for x in row] for row in A])


def exact_box_matrices(p, hx, hy, hz):
    """Exact Q_p stiffness and mass on an axis-aligned box (pin P2)."""
    M, S, _ = exact_1d(p)
    vol = Fraction(hx) * Fraction(hy) * Fraction(hz)
    Mx = [[m for m in row] for row in M]
    Kx = _kron3(M, M, S)
    Ky = _kron3(M, S, M)
    Kz = _kron3(S, M, M)
    Mm = _kron3(M, M, M)
    n = len(Mm)
    hx, hy, hz = Fraction(hx), Fraction(hy), Fraction(hz)
    K = [[vol * (Kx[r][c] / hx ** 2 + Ky[r][c] / hy ** 2 + Kz[r][c] / hz ** 2) for c in range(n)]
         for r in range(n)]
    Mass = [[vol * Mm[r][c] for c in range(n)] for r in range(n)]
    del Mx
    return K, Mass


def exact_elasticity_unit(p, lam, mu):
    """Exact isotropic elasticity on the unit cube (pin P3):
    K_(a,k),(b,l) = lam int d_a phi_k d_b phi_l + mu (delta_ab int grad phi_k . grad phi_l
                    + int d_b phi_k d_a phi_l)."""
    M, S, C = exact_1d(p)
    CT = [list(r) for r in zip(*C)]

    def factor(a, b, d):
        # 1D factor along axis d of int (d==a ? phi' : phi)_k (d==b ? phi' : phi)_l
        if d == a and d == b:
            return S
        if d == a:
            return C       # int phi_k' phi_l
        if d == b:
            return CT      # int phi_k phi_l'
        return M

    def Dab(a, b):
        return _kron3(factor(a, b, 2), factor(a, b, 1), factor(a, b, 0))

    nb = (p + 1) ** 3
    G = {(a, b): Dab(a, b) for a in range(3) for b in range(3)}
    K = np.zeros((3 * nb, 3 * nb))
    lam, mu = Fraction(lam), Fraction(mu)
    for a in range(3):
        for b in range(3):
            for k in range(nb):
                for l in range(nb):
                    v = lam * G[(a, b)][k][l] + mu * G[(b, a)][k][l]
                    if a == b:
                        v += mu * sum(G[(d, d)][k][l] for d in range(3))
                    K[a * nb + k, b * nb + l] = float(v)
    return K


def _golden_kv(fname):
    out = {}
    for line in open(os.path.join(GOLDEN, fname)):
        line = line.split("#")[0].strip()
        if "=" in line:
            k, v = line.split("=", 1)
            out[k.strip()] = [Fraction(x) for x in v.split()]
    return out


def unit_cube():
    return fi.grid_vertices(1, 1, 1), fi.hex_connectivity(1, 1, 1)


def box(hx, hy, hz, origin=(0.0, 0.0, 0.0)):
    c = fi.grid_vertices(1, 1, 1) * np.array([hx, hy, hz]) + np.array(origin)
    return c, fi.hex_connectivity(1, 1, 1)


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


# ---------------------------------------------------------------- tables
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 8, 12])
def test_gauss_legendre_matches_library(n):
    """Oracle Gauss rule == numpy leggauss mapped to [0,1] (textbook rule)."""
    x, w = oracle.gauss_legendre(n)
    t, wt = np.polynomial.legendre.leggauss(n)
    np.testing.assert_allclose(x, (t + 1) / 2, rtol=0, atol=1e-15)
    np.testing.assert_allclose(w, wt / 2, rtol=0, atol=1e-15)
    assert abs(w.sum() - 1.0) < 1e-15
    # exactness: int_0^1 x^k = 1/(k+1) for k <= 2n-1
    for k in range(2 * n):
        assert abs((w * x ** k).sum() - 1.0 / (k + 1)) < 1e-14


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
def test_lagrange_1d_properties(p):
    """Kronecker-delta at nodes, partition of unity, derivatives sum to 0,
    derivative matches the exact polynomial."""
    L = _lagrange_exact(p)
    for i in range(p + 1):
        phi, _ = oracle.lagrange_1d(p, i / p)
        np.testing.assert_allclose(phi, np.eye(p + 1)[i], atol=1e-14)
    for t in np.linspace(-0.2, 1.3, 11):
        phi, dphi = oracle.lagrange_1d(p, t)
        assert abs(phi.sum() - 1) < 1e-13 and abs(dphi.sum()) < 1e-12
        exact_d = [float(sum(c * Fraction(t) ** (k - 1) * k for k, c in enumerate(P) if k > 0))
                   for P in L]
        np.testing.assert_allclose(dphi, exact_d, rtol=1e-12, atol=1e-12)


def test_tables_match_independent_construction():
    """Tensorised Phi / grad Phi equal the numpy-polynomial construction."""
    for p, q in [(1, 2), (2, 3), (4, 5), (2, 2)]:
        xi, w, Phi, dPhi = oracle.tables(p, q)
        X, W, bf, bfg = eo.tables(p, q)
        np.testing.assert_allclose(xi, X, atol=1e-15)
        np.testing.assert_allclose(w, W, atol=1e-16)
        np.testing.assert_allclose(Phi, bf, atol=1e-13)
        np.testing.assert_allclose(dPhi, bfg, atol=1e-12)


# ---------------------------------------------------------------- P1 / P2 / P3
def test_P1_q1_unit_cube_golden():
    g = _golden_kv("q1_unit_cube.txt")
    c, conn = unit_cube()
    K = oracle.eval_matrix(fi.DIFFUSION, 1, 2, c, conn, None, 0, np.ones((1, 8)))[0]
    M = oracle.eval_matrix(fi.MASS, 1, 2, c, conn, None, 0, np.ones((1, 8)))[0]
    np.testing.assert_allclose(M[0], [float(x) for x in g["mass_row0"]], rtol=1e-14, atol=1e-17)
    np.testing.assert_allclose(K[0], [float(x) for x in g["stiffness_row0"]], rtol=1e-14,
                               atol=1e-15)
    assert abs(M.sum() - float(g["mass_sum"][0])) < 1e-14
    # the golden rationals agree with the exact 1D-factor construction
    Ke, Me = exact_box_matrices(1, 1, 1, 1)
    assert [Fraction(x) for x in Me[0]] == g["mass_row0"]
    assert [Fraction(x) for x in Ke[0]] == g["stiffness_row0"]


@pytest.mark.parametrize("p", [1, 2, 3, 4])
@pytest.mark.parametrize("dims", [(1, 1, 1), (Fraction(1, 2), Fraction(1, 3), Fraction(2, 5))])
def test_P2_box_closed_form(p, dims):
    Ke, Me = exact_box_matrices(p, *dims)
    c, conn = box(*[float(d) for d in dims], origin=(0.3, -0.2, 1.1))
    nb = (p + 1) ** 3
    dc, _ = fi.lattice_dof_conn(1, 1, 1, p)
    K = oracle.eval_matrix(fi.DIFFUSION, p, p + 1, c, conn, dc, 0, np.ones((1, (p + 1) ** 3)))[0]
    M = oracle.eval_matrix(fi.MASS, p, p + 1, c, conn, dc, 0, np.ones((1, (p + 1) ** 3)))[0]
    assert K.shape == (nb, nb)
    assert rel(K, _to_np(Ke)) < 1e-14
    assert rel(M, _to_np(Me)) < 1e-14


def test_P2_golden_diagonals():
    g = _golden_kv("q1_unit_cube.txt")
    for p, kk, mk in [(2, "q2_K00", "q2_M00"), (4, "q4_K00", "q4_M00")]:
        Ke, Me = exact_box_matrices(p, 1, 1, 1)
        assert Ke[0][0] == g[kk][0] and Me[0][0] == g[mk][0]
        c, conn = unit_cube()
        dc, _ = fi.lattice_dof_conn(1, 1, 1, p)
        nq = (p + 1) ** 3
        K = oracle.eval_matrix(fi.DIFFUSION, p, p + 1, c, conn, dc, 0, np.ones((1, nq)))[0]
        M = oracle.eval_matrix(fi.MASS, p, p + 1, c, conn, dc, 0, np.ones((1, nq)))[0]
        assert abs(K[0, 0] / float(g[kk][0]) - 1) < 1e-14
        assert abs(M[0, 0] / float(g[mk][0]) - 1) < 1e-14


@pytest.mark.parametrize("p", [1, 2])
def test_P3_elasticity_closed_form(p):
    c, conn = unit_cube()
    dc, _ = fi.lattice_dof_conn(1, 1, 1, p)
    lam, mu = 1.25, 0.75
    K = oracle.eval_matrix(fi.ELASTICITY, p, p + 1, c, conn, dc, fi.MAT_PER_ELEM,
                           np.array([lam]), np.array([mu]))[0]
    Kx = exact_elasticity_unit(p, Fraction(5, 4), Fraction(3, 4))
    assert rel(K, Kx) < 1e-14
    if p == 1:
        g = _golden_kv("q1_unit_cube.txt")
        K1 = oracle.eval_matrix(fi.ELASTICITY, 1, 2, c, conn, None, fi.MAT_PER_ELEM,
                                np.array([1.0]), np.array([1.0]))[0]
        assert abs(K1[0, 0] - float(g["el_K_x0x0"][0])) < 1e-15
        assert abs(K1[0, 8] - float(g["el_K_x0y0"][0])) < 1e-15


def test_P3_full_D_equals_isotropic():
    pr = fi.make_problem(fi.ELASTICITY, 2, (2, 1, 1), 3)
    Dfull = np.broadcast_to(np.stack([np.stack([oracle.isotropic_D(a, b)] * pr.nq)
                                      for a, b in zip(pr.mat_a, pr.mat_b)]), (2, pr.nq, 6, 6))
    K1 = oracle.problem_matrix(pr)
    K2 = oracle.eval_matrix(fi.ELASTICITY, 2, 3, pr.coords, pr.conn, pr.dof_conn, fi.MAT_FULL_D,
                            np.ascontiguousarray(Dfull))
    assert rel(K2, K1) < 1e-15


# ---------------------------------------------------------------- P4 .. P10
def node_coords(prob):
    """Physical coordinates of the order-p lattice nodes: trilinear image of
    the reference nodes (i/p, j/p, k/p) of each element (reading 4)."""
    p = prob.p
    X = np.zeros((prob.n_nodes, 3))
    t = np.arange(p + 1) / p
    for l in range(p + 1):
        for j in range(p + 1):
            for i in range(p + 1):
                k = i + (p + 1) * (j + (p + 1) * l)
                xi = (t[i], t[j], t[l])
                w = np.array([(xi[0] if a else 1 - xi[0]) * (xi[1] if b else 1 - xi[1]) *
                              (xi[2] if cc else 1 - xi[2])
                              for cc in (0, 1) for b in (0, 1) for a in (0, 1)])
                X[prob.dof_conn[:, k]] = np.einsum("v,evi->ei", w, prob.coords[prob.conn])
    return X


@pytest.mark.parametrize("p", [1, 2, 4])
def test_P4_volume(p):
    pr = fi.make_problem(fi.MASS, p, (3, 3, 2), 11)
    M = oracle.eval_matrix(fi.MASS, p, p + 1, pr.coords, pr.conn, pr.dof_conn, 0,
                           np.ones((pr.n_elems, pr.nq)))
    assert abs(M.sum() - 1.0) < 1e-13
    detw, _ = oracle.geometry(p + 1, pr.coords, pr.conn)
    np.testing.assert_allclose(M.sum(axis=(1, 2)), detw.sum(axis=1), rtol=1e-13)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_P5_patch_test(p):
    pr = fi.make_problem(fi.DIFFUSION, p, (3, 3, 3), 5)
    X = node_coords(pr)
    u = X @ np.array([0.3, -1.1, 0.7]) + 0.25
    kappa = np.full((pr.n_elems, pr.nq), 1.7)
    r = oracle.eval_residual(fi.DIFFUSION, p, p + 1, pr.coords, pr.conn, pr.dof_conn, u[:, None],
                             0, kappa)
    R = oracle.assemble(r, pr.dof_conn, pr.n_nodes, 1)
    M = p * 3 + 1
    idx = np.arange(pr.n_nodes)
    ix, iy, iz = idx % M, (idx // M) % M, idx // (M * M)
    interior = (ix > 0) & (ix < M - 1) & (iy > 0) & (iy < M - 1) & (iz > 0) & (iz < M - 1)
    assert np.abs(R[interior]).max() <= 1e-13 * np.abs(R).max()
    assert np.abs(R[~interior]).max() > 1e-3


@pytest.mark.parametrize("p", [1, 2])
def test_P6_rigid_modes(p):
    pr = fi.make_problem(fi.ELASTICITY, p, (2, 2, 1), 9)
    X = node_coords(pr)
    K = oracle.problem_matrix(pr)
    nb = pr.nb
    for e in range(pr.n_elems):
        xe = X[pr.dof_conn[e]]
        modes = []
        for a in range(3):
            m = np.zeros((3, nb))
            m[a] = 1.0
            modes.append(m)
        for w in np.eye(3):
            modes.append(np.cross(w, xe).T)
        for m in modes:
            v = m.reshape(-1)
            assert np.linalg.norm(K[e] @ v) <= 1e-13 * np.linalg.norm(K[e]) * np.linalg.norm(v)
    # a one-sided Psg (6 ones) would not annihilate rotations: K must be rank 3*nb-6
    s = np.linalg.svd(K[0], compute_uv=False)
    assert (s < 1e-12 * s[0]).sum() == 6


@pytest.mark.parametrize("form,p", [(fi.DIFFUSION, 1), (fi.DIFFUSION, 2), (fi.MASS, 2),
                                    (fi.ELASTICITY, 2), (fi.VECTOR_MASS, 1),
                                    (fi.MASS_DIFFUSION, 2)])
def test_P7_symmetry_rowsums(form, p):
    pr = fi.make_problem(form, p, (2, 2, 2), 13)
    K = oracle.problem_matrix(pr)
    assert rel(K, K.transpose(0, 2, 1)) < 1e-14
    if form == fi.DIFFUSION:
        assert np.abs(K.sum(axis=2)).max() < 1e-13 * np.abs(K).max()


def test_P7_vector_mass_blocks():
    """Vector mass = D copies of the scalar mass block."""
    pr = fi.make_problem(fi.VECTOR_MASS, 2, (2, 1, 2), 21)
    Kv = oracle.problem_matrix(pr)
    Ms = oracle.eval_matrix(fi.MASS, 2, 3, pr.coords, pr.conn, pr.dof_conn, 0, pr.mat_a)
    nb = pr.nb
    for r in range(3):
        for s in range(3):
            blk = Kv[:, r * nb:(r + 1) * nb, s * nb:(s + 1) * nb]
            if r == s:
                assert rel(blk, Ms) < 1e-15
            else:
                assert np.abs(blk).max() == 0.0


def test_P7_mass_diffusion_constant():
    pr = fi.make_problem(fi.MASS_DIFFUSION, 2, (2, 2, 2), 4)
    rho = np.ones_like(pr.mat_a)
    r = oracle.eval_residual(fi.MASS_DIFFUSION, 2, 3, pr.coords, pr.conn, pr.dof_conn,
                             np.ones((pr.n_nodes, 1)), 0, rho, pr.mat_b)
    assert abs(r.sum() - 1.0) < 1e-13


@pytest.mark.parametrize("form,p", [(fi.DIFFUSION, 1), (fi.DIFFUSION, 2), (fi.MASS, 2),
                                    (fi.VECTOR_MASS, 2), (fi.MASS_DIFFUSION, 2),
                                    (fi.ELASTICITY, 1), (fi.ELASTICITY, 2)])
def test_P8_linear_consistency(form, p):
    """r_e = K_e u_e for the linear forms (Alg. 1 vs Alg. 2)."""
    pr = fi.make_problem(form, p, (3, 2, 2), 17)
    K = oracle.problem_matrix(pr)
    r = oracle.problem_residual(pr)
    ue = pr.u[pr.dof_conn].transpose(0, 2, 1).reshape(pr.n_elems, -1)
    Ku = np.einsum("eij,ej->ei", K, ue)
    assert rel(r, Ku) < 1e-13


@pytest.mark.parametrize("p", [1, 2])
def test_P8_convective_identities(p):
    """Quadratic residual: K(u) u = 2 r(u); (r(u+d) - r(u-d))/2 = K(u) d exactly."""
    pr = fi.make_problem(fi.CONVECTIVE, p, (2, 2, 2), 23)
    K = oracle.problem_matrix(pr)
    r = oracle.problem_residual(pr)
    ue = pr.u[pr.dof_conn].transpose(0, 2, 1).reshape(pr.n_elems, -1)
    assert rel(np.einsum("eij,ej->ei", K, ue), 2 * r) < 1e-13
    rng = np.random.default_rng(1)
    d = rng.uniform(-0.3, 0.3, size=pr.u.shape)
    args = (fi.CONVECTIVE, p, p + 1, pr.coords, pr.conn, pr.dof_conn)
    rp = oracle.eval_residual(*args, pr.u + d)
    rm = oracle.eval_residual(*args, pr.u - d)
    de = d[pr.dof_conn].transpose(0, 2, 1).reshape(pr.n_elems, -1)
    assert rel((rp - rm) / 2, np.einsum("eij,ej->ei", K, de)) < 1e-13


def test_P9_scaling_rotation():
    pr = fi.make_problem(fi.DIFFUSION, 2, (1, 1, 1), 2, perturb=0.0)
    rng = np.random.default_rng(5)
    c = pr.coords + rng.uniform(-0.1, 0.1, size=pr.coords.shape)
    one = np.ones((1, 27))
    args = (2, 3)
    K = oracle.eval_matrix(fi.DIFFUSION, *args, c, pr.conn, pr.dof_conn, 0, one)
    M = oracle.eval_matrix(fi.MASS, *args, c, pr.conn, pr.dof_conn, 0, one)
    s = 2.5
    Ks = oracle.eval_matrix(fi.DIFFUSION, *args, c * s, pr.conn, pr.dof_conn, 0, one)
    Ms = oracle.eval_matrix(fi.MASS, *args, c * s, pr.conn, pr.dof_conn, 0, one)
    assert rel(Ks, s * K) < 1e-14 and rel(Ms, s ** 3 * M) < 1e-14
    th = 0.7
    R = np.array([[np.cos(th), -np.sin(th), 0], [np.sin(th), np.cos(th), 0], [0, 0, 1.0]])
    R = R @ np.array([[1, 0, 0], [0, np.cos(0.3), -np.sin(0.3)], [0, np.sin(0.3), np.cos(0.3)]])
    Kr = oracle.eval_matrix(fi.DIFFUSION, *args, c @ R.T, pr.conn, pr.dof_conn, 0, one)
    assert rel(Kr, K) < 1e-14


def test_P10_zero_and_constant():
    for form in (fi.DIFFUSION, fi.ELASTICITY, fi.CONVECTIVE, fi.MASS_DIFFUSION):
        pr = fi.make_problem(form, 2, (2, 1, 1), 8)
        r = oracle.eval_residual(form, 2, 3, pr.coords, pr.conn, pr.dof_conn,
                                 np.zeros_like(pr.u), pr.mat_kind, pr.mat_a, pr.mat_b)
        assert np.abs(r).max() == 0.0
    pr = fi.make_problem(fi.DIFFUSION, 2, (2, 2, 1), 8)
    r = oracle.eval_residual(fi.DIFFUSION, 2, 3, pr.coords, pr.conn, pr.dof_conn,
                             np.full_like(pr.u, 3.0), 0, pr.mat_a)
    assert np.abs(r).max() < 1e-14
    # constant velocity: the reaction block (term 2 of Eq. fe4) vanishes
    pr = fi.make_problem(fi.CONVECTIVE, 2, (2, 1, 1), 8)
    u = np.tile([0.3, -0.2, 0.5], (pr.n_nodes, 1))
    K = oracle.eval_matrix(fi.CONVECTIVE, 2, 3, pr.coords, pr.conn, pr.dof_conn, 0, None, None, u)
    nb = pr.nb
    for a in range(3):
        for b in range(3):
            if a != b:
                assert np.abs(K[:, a * nb:(a + 1) * nb, b * nb:(b + 1) * nb]).max() < 1e-15


def test_degenerate_element_reported():
    pr = fi.make_problem(fi.DIFFUSION, 1, (3, 1, 1), 1)
    c = pr.coords.copy()
    conn = pr.conn.copy()
    conn[1] = conn[1][[1, 0, 3, 2, 5, 4, 7, 6]]     # mirror element 1 -> det J < 0
    with pytest.raises(oracle.OracleError) as ei:
        oracle.eval_matrix(fi.DIFFUSION, 1, 2, c, conn, None, 0, pr.mat_a)
    assert ei.value.status == oracle.ERR_DEGENERATE and ei.value.element == 1
    with pytest.raises(oracle.OracleError) as ei:
        oracle.geometry(2, c, conn)
    assert ei.value.element == 1


# ---------------------------------------------------------------- P11
@pytest.mark.parametrize("form,p,kind", [(0, 1, 0), (0, 2, 0), (0, 4, 0), (1, 2, 0), (2, 1, 0),
                                         (2, 2, 0), (3, 2, 0), (3, 4, 0), (4, 1, 1), (4, 2, 1),
                                         (4, 2, 0), (4, 2, 2), (5, 1, 0), (5, 2, 0)])
def test_P11_second_oracle(form, p, kind):
    pr = fi.make_problem(form, p, (3, 2, 2), 100 + form, mat_kind=kind if form == 4 else None)
    K = oracle.problem_matrix(pr)
    K2 = eo.matrix(form, pr.coords, pr.conn, p, pr.q1d, pr.dof_conn, pr.mat_a, pr.mat_b,
                   pr.mat_kind, pr.u)
    assert rel(K, K2) < 1e-13
    r = oracle.problem_residual(pr)
    r2 = eo.residual(form, pr.coords, pr.conn, p, pr.q1d, pr.dof_conn, pr.u, pr.mat_a, pr.mat_b,
                     pr.mat_kind)
    assert rel(r, r2) < 1e-13


def test_P11_C1_in_full():
    pr = fi.make_config("C1")
    K = oracle.problem_matrix(pr)
    K2 = eo.matrix(0, pr.coords, pr.conn, 1, 2, None, pr.mat_a)
    assert K.shape == (64, 8, 8)
    assert rel(K, K2) < 1e-13


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_P11_config_subsets(name):
    """Seeded <= 64-element subsets of the BASELINE configs (small N, same recipe)."""
    pr = fi.make_config(name, N=4)
    rng = np.random.default_rng(0)
    sel = np.sort(rng.choice(pr.n_elems, size=16, replace=False))
    sub = fi.Problem(name, pr.form, pr.p, pr.q1d, pr.shape, pr.coords, pr.conn[sel],
                     pr.dof_conn[sel], pr.n_nodes, pr.mat_kind,
                     None if pr.mat_a is None else pr.mat_a[sel],
                     None if pr.mat_b is None else pr.mat_b[sel], pr.u)
    r = oracle.problem_residual(sub)
    r2 = eo.residual(sub.form, sub.coords, sub.conn, sub.p, sub.q1d, sub.dof_conn, sub.u,
                     sub.mat_a, sub.mat_b, sub.mat_kind)
    assert rel(r, r2) < 1e-13
    if name != "C4":
        K = oracle.problem_matrix(sub)
        K2 = eo.matrix(sub.form, sub.coords, sub.conn, sub.p, sub.q1d, sub.dof_conn, sub.mat_a,
                       sub.mat_b, sub.mat_kind, sub.u)
        assert rel(K, K2) < 1e-13


def _parse_examples():
    rows = []
    for line in open(os.path.join(GOLDEN, "paper_einsum_examples.txt")):
        if line.startswith("#") or not line.strip():
            continue
        name, cite, expr, p, nc, out, ops = [x.strip() for x in line.split("|")]
        shapes = {kv.split("=")[0]: tuple(int(x) for x in kv.split("=")[1].split(","))
                  for kv in ops.split()}
        rows.append((name, cite, expr, int(p), int(nc), tuple(int(x) for x in out.split(",")),
                     shapes))
    return rows


@pytest.mark.parametrize("row", _parse_examples(), ids=lambda r: r[0])
def test_paper_worked_examples(row):
    """The paper's printed einsum strings and sizes (Sec. 5.3) on a 1D bar of 1024
    hexahedra: operand shapes are the printed ones and the result equals
    the oracle."""
    name, cite, expr, p, nc, out_shape, shapes = row
    c = fi.grid_vertices(1, 1, nc)
    conn = fi.hex_connectivity(1, 1, nc)
    dc, n_nodes = fi.lattice_dof_conn(1, 1, nc, p)
    q1d = p + 1
    det, bf, bfg = eo.operands(c, conn, p, q1d)
    rng = np.random.default_rng(2)
    ops = {"cq": det, "qd": bf, "qe": bf, "ir": np.eye(3), "is": np.eye(3),
           "cqjd": bfg, "cqje": bfg, "cqlf": bfg, "rjI": eo.psg(), "slK": eo.psg()}
    if "cqIK" in shapes:
        lam = rng.uniform(0.5, 2, nc)
        mu = rng.uniform(0.5, 2, nc)
        ops["cqIK"] = np.ascontiguousarray(
            np.broadcast_to(eo.iso_D(lam, mu)[:, None], (nc, q1d ** 3, 6, 6)))
    u = rng.uniform(-1, 1, size=(n_nodes, 3))
    ops["cie"] = u[dc].transpose(0, 2, 1)
    names = expr.split("->")[0].split(",")
    for nm in names:
        assert ops[nm].shape == shapes[nm], (nm, ops[nm].shape, shapes[nm])
    res = np.einsum(expr, *[ops[nm] for nm in names], optimize=True)
    assert res.shape == out_shape
    if name == "laplace_matrix":
        K = oracle.eval_matrix(fi.DIFFUSION, p, q1d, c, conn, dc, 0, np.ones((nc, q1d ** 3)))
    elif name == "dot_matrix":
        K = oracle.eval_matrix(fi.VECTOR_MASS, p, q1d, c, conn, dc, 0, np.ones((nc, q1d ** 3)))
    elif name == "dot_residual":
        K = oracle.eval_residual(fi.VECTOR_MASS, p, q1d, c, conn, dc, u, 0,
                                 np.ones((nc, q1d ** 3)))
    else:
        K = oracle.eval_matrix(fi.ELASTICITY, p, q1d, c, conn, dc, fi.MAT_PER_ELEM, lam, mu)
    assert rel(K.reshape(res.shape), res) < 1e-13


# ---------------------------------------------------------------- eval mode (N3)
def test_eval_mode_closed_forms():
    """'eval' mode pinned by closed forms on perturbed meshes:
    int kappa |grad(a.x + b)|^2 = kappa |a|^2 vol, int rho 1 = rho vol, and the definition
    u^T K u = sum_e u_e . r_e(u) for the bilinear forms."""
    pr = fi.make_problem(fi.DIFFUSION, 2, (3, 2, 2), 19)
    X = node_coords(pr)
    a = np.array([0.4, -1.3, 0.8])
    u = (X @ a + 0.7)[:, None]
    kap = np.full((pr.n_elems, pr.nq), 1.5)
    v = oracle.eval_scalar(fi.DIFFUSION, 2, 3, pr.coords, pr.conn, pr.dof_conn, u, 0, kap)
    assert abs(v - 1.5 * a @ a) < 1e-13
    rho = np.full((pr.n_elems, pr.nq), 2.5)
    v = oracle.eval_scalar(fi.MASS, 2, 3, pr.coords, pr.conn, pr.dof_conn, np.ones_like(u), 0, rho)
    assert abs(v - 2.5) < 1e-13


@pytest.mark.parametrize("form,p", [(fi.DIFFUSION, 2), (fi.MASS_DIFFUSION, 2), (fi.ELASTICITY, 2),
                                    (fi.VECTOR_MASS, 1), (fi.CONVECTIVE, 2)])
def test_eval_mode_equals_u_dot_r(form, p):
    pr = fi.make_problem(form, p, (2, 3, 2), 29)
    v = oracle.problem_eval_scalar(pr)
    r = oracle.problem_residual(pr)
    ue = pr.u[pr.dof_conn].transpose(0, 2, 1).reshape(pr.n_elems, -1)
    ref = float(np.sum(r * ue))
    assert abs(v - ref) <= 1e-13 * max(abs(ref), 1e-300)


# ---------------------------------------------------------------- N3: remaining Tab. 2 forms
@pytest.mark.parametrize("p", [1, 2])
def test_N3_weighted_dot_closed_form(p):
    """'ij,i,j' with a constant M on an axis-aligned box: K_ab = M_ab * (scalar mass
    matrix), whose entries are the exact rationals rho h^3 M1 x M1 x M1 (P2)."""
    dims = (Fraction(1, 2), Fraction(1, 3), Fraction(2, 5))
    _, Me = exact_box_matrices(p, *dims)
    Ms = _to_np(Me)
    c, conn = box(*[float(d) for d in dims], origin=(0.1, 0.2, -0.3))
    dc, _ = fi.lattice_dof_conn(1, 1, 1, p)
    nq, nb = (p + 1) ** 3, (p + 1) ** 3
    Mw = np.array([[1.5, -0.25, 0.5], [0.75, 2.0, -1.0], [0.125, 0.5, 1.25]])
    K = oracle.eval_matrix(fi.WEIGHTED_DOT, p, p + 1, c, conn, dc, 0,
                           np.broadcast_to(Mw, (1, nq, 3, 3)).copy())[0]
    for a in range(3):
        for b in range(3):
            assert rel(K[a * nb:(a + 1) * nb, b * nb:(b + 1) * nb], Mw[a, b] * Ms) < 1e-14


def test_N3_weighted_dot_reduces_to_vector_mass():
    """M = rho I per qp gives the vector mass form 'i,i' exactly."""
    pr = fi.make_problem(fi.VECTOR_MASS, 2, (2, 2, 1), 21)
    Mw = pr.mat_a[:, :, None, None] * np.eye(3)[None, None]
    K1 = oracle.problem_matrix(pr)
    K2 = oracle.eval_matrix(fi.WEIGHTED_DOT, 2, 3, pr.coords, pr.conn, pr.dof_conn, 0,
                            np.ascontiguousarray(Mw))
    assert rel(K2, K1) < 1e-15
    r1 = oracle.problem_residual(pr)
    r2 = oracle.eval_residual(fi.WEIGHTED_DOT, 2, 3, pr.coords, pr.conn, pr.dof_conn, pr.u, 0,
                              np.ascontiguousarray(Mw))
    assert rel(r2, r1) < 1e-15


@pytest.mark.parametrize("p", [1, 2])
def test_N3_weighted_dot_linear_consistency(p):
    """r_e = K_e u_e (P8) and eval = u . r (eval mode) for a non-symmetric M per qp."""
    pr = fi.make_problem(fi.WEIGHTED_DOT, p, (2, 3, 2), 23)
    K = oracle.problem_matrix(pr)
    r = oracle.problem_residual(pr)
    ue = np.stack([pr.u[pr.dof_conn][:, :, a] for a in range(3)], axis=1).reshape(pr.n_elems, -1)
    assert rel(np.einsum("eij,ej->ei", K, ue), r) < 1e-14
    assert abs(oracle.problem_eval_scalar(pr) - float((ue * r).sum())) < 1e-13 * abs((ue * r).sum())
    # non-symmetric weight -> K_ab != K_ba^T in general, but K^T is the form with M^T
    Mt = np.ascontiguousarray(np.swapaxes(pr.mat_a, 2, 3))
    Kt = oracle.eval_matrix(fi.WEIGHTED_DOT, p, p + 1, pr.coords, pr.conn, pr.dof_conn, 0, Mt)
    assert rel(Kt, np.swapaxes(K, 1, 2)) < 1e-15


@pytest.mark.parametrize("p", [1, 2, 3])
def test_N3_divergence(p):
    """'i.i': r[(a,k)] = int dphi_k/dx_a.  Partition of unity: sum_k r = 0 per cell
    and component; eval with u = x (node coordinates, exact in Q_p on trilinear cells) gives
    int div x = 3 * volume = 3 on the unit cube."""
    pr = fi.make_problem(fi.DIVERGENCE, p, (2, 2, 3), 31)
    r = oracle.problem_residual(pr).reshape(pr.n_elems, 3, -1)
    assert np.abs(r.sum(axis=2)).max() < 1e-14
    X = node_coords(pr)
    v = oracle.eval_scalar(fi.DIVERGENCE, p, p + 1, pr.coords, pr.conn, pr.dof_conn, X)
    assert abs(v - 3.0) < 1e-13
    # residual mode does not depend on u
    r2 = oracle.eval_residual(fi.DIVERGENCE, p, p + 1, pr.coords, pr.conn, pr.dof_conn,
                              np.zeros_like(pr.u)).reshape(pr.n_elems, 3, -1)
    assert np.array_equal(r, r2)
    with pytest.raises(oracle.OracleError):  # no trial variable: no matrix mode
        oracle.eval_matrix(fi.DIVERGENCE, p, p + 1, pr.coords, pr.conn, pr.dof_conn)


@pytest.mark.parametrize("p", [1, 2])
def test_N3_cauchy_stress(p):
    """'IK,s(k:l)->K', eval only: an affine displacement u = A x + b is exact in
    Q_p on trilinear cells, so sigma = D eps(A) at every qp; a rigid motion gives sigma = 0."""
    pr = fi.make_problem(fi.ELASTICITY, p, (2, 2, 2), 41)
    X = node_coords(pr)
    A = np.array([[0.3, -0.2, 0.1], [0.05, -0.4, 0.25], [0.2, 0.15, 0.6]])
    u = X @ A.T + np.array([0.1, -0.3, 0.2])
    sig = oracle.eval_stress(p, p + 1, pr.coords, pr.conn, pr.dof_conn, u, pr.mat_kind,
                             pr.mat_a, pr.mat_b)
    eps = np.array([A[0, 0], A[1, 1], A[2, 2], A[0, 1] + A[1, 0], A[0, 2] + A[2, 0],
                    A[1, 2] + A[2, 1]])
    for e in range(pr.n_elems):
        ref = oracle.isotropic_D(pr.mat_a[e], pr.mat_b[e]) @ eps
        assert np.abs(sig[e] - ref[None, :]).max() < 1e-13 * np.abs(ref).max()
    W = np.array([[0.0, -0.3, 0.2], [0.3, 0.0, -0.1], [-0.2, 0.1, 0.0]])  # skew: rotation
    sig0 = oracle.eval_stress(p, p + 1, pr.coords, pr.conn, pr.dof_conn, X @ W.T + 1.0,
                              pr.mat_kind, pr.mat_a, pr.mat_b)
    scale = max(np.abs(oracle.isotropic_D(a, b)).max() for a, b in zip(pr.mat_a, pr.mat_b))
    assert np.abs(sig0).max() < 1e-13 * scale * np.abs(W).max()  # zero up to rounding


# ---------------------------------------------------------------- N3: Stokes coupling pair
def _exact_1d_mixed(pv, pp):
    """Mv[i][j] = int phi_i psi_j, Cv[i][j] = int phi_i' psi_j on [0,1]; phi of order pv, psi
    of order pp (exact rationals)."""
    Lv, Lp = _lagrange_exact(pv), _lagrange_exact(pp)
    dLv = [_poly_deriv(P) for P in Lv]
    Mv = [[_poly_int01(_poly_mul(Lv[i], Lp[j])) for j in range(pp + 1)] for i in range(pv + 1)]
    Cv = [[_poly_int01(_poly_mul(dLv[i], Lp[j])) for j in range(pp + 1)] for i in range(pv + 1)]
    return Mv, Cv


def _node_coords_order(prob, p, dof_conn, n_nodes):
    """Physical coordinates of an order-p node lattice (trilinear images, reading 4)."""
    X = np.zeros((n_nodes, 3))
    t = np.arange(p + 1) / p
    for l in range(p + 1):
        for j in range(p + 1):
            for i in range(p + 1):
                k = i + (p + 1) * (j + (p + 1) * l)
                w = np.array([(t[i] if a else 1 - t[i]) * (t[j] if b else 1 - t[j]) *
                              (t[l] if cc else 1 - t[l])
                              for cc in (0, 1) for b in (0, 1) for a in (0, 1)])
                X[dof_conn[:, k]] = np.einsum("v,evi->ei", w, prob.coords[prob.conn])
    return X


@pytest.mark.parametrize("pv,pp", [(1, 1), (2, 1), (3, 2), (2, 2)])
def test_N3_stokes_coupling_box_closed_form(pv, pp):
    """'i.i,0' on an axis-aligned box: B[(a,k), l] = vol * prod_d F_d[k_d][l_d] / h_a
    with F_d = Cv (int phi' psi) along d == a and Mv (int phi psi) otherwise, exact rationals;
    the transposed coupling is C[l, (a,k)] with the same entries."""
    dims = (Fraction(1, 2), Fraction(1, 3), Fraction(2, 5))
    vol = dims[0] * dims[1] * dims[2]
    Mv, Cv = _exact_1d_mixed(pv, pp)
    nv, npp = pv + 1, pp + 1
    nbv, nbp = nv ** 3, npp ** 3
    ref = np.zeros((3 * nbv, nbp))
    for a in range(3):
        for kz in range(nv):
            for ky in range(nv):
                for kx in range(nv):
                    k = kx + nv * (ky + nv * kz)
                    for lz in range(npp):
                        for ly in range(npp):
                            for lx in range(npp):
                                l = lx + npp * (ly + npp * lz)
                                f = [(Cv if a == d else Mv)[kk][ll]
                                     for d, (kk, ll) in enumerate(((kx, lx), (ky, ly), (kz, lz)))]
                                ref[a * nbv + k, l] = float(vol * f[0] * f[1] * f[2] / dims[a])
    c, conn = box(*[float(d) for d in dims], origin=(0.1, 0.2, -0.3))
    B = oracle.coupling_matrix(pv, pp, pv + 1, c, conn)[0]
    assert rel(B, ref) < 1e-14
    C = oracle.coupling_matrix(pv, pp, pv + 1, c, conn, transposed=True)[0]
    assert rel(C, ref.T) < 1e-14


@pytest.mark.parametrize("pv,pp", [(2, 1), (1, 1), (3, 2)])
def test_N3_stokes_coupling_consistency(pv, pp):
    """On a perturbed grid: r_v(p) = B p_e and r_q(u) = C u_e (Alg. 1 = Alg. 2 applied, P8);
    C = B^T; eval = p_e . r_q(u) = u_e . r_v(p); constant pressure p = 1 gives the divergence
    form 'i.i' residual exactly."""
    mp = fi.make_mixed_problem(pv, pp, (3, 2, 2), 51)
    v = mp.vel
    q1d = pv + 1
    args = (pv, pp, q1d, v.coords, v.conn)
    B = oracle.coupling_matrix(*args)
    C = oracle.coupling_matrix(*args, transposed=True)
    assert rel(C, np.swapaxes(B, 1, 2)) < 1e-15
    pe = mp.pres[mp.p_dof_conn]
    ue = np.stack([v.u[v.dof_conn][:, :, a] for a in range(3)], axis=1).reshape(v.n_elems, -1)
    rv = oracle.coupling_residual(*args, v.dof_conn, mp.p_dof_conn, p=mp.pres)
    rq = oracle.coupling_residual(*args, v.dof_conn, mp.p_dof_conn, u=v.u, transposed=True)
    assert rel(rv, np.einsum("eij,ej->ei", B, pe)) < 1e-14
    assert rel(rq, np.einsum("eij,ej->ei", C, ue)) < 1e-14
    ev = oracle.coupling_eval(*args, v.dof_conn, mp.p_dof_conn, v.u, mp.pres)
    assert abs(ev - float((pe * rq).sum())) < 1e-13 * max(abs(ev), 1.0)
    assert abs(ev - float((ue * rv).sum())) < 1e-13 * max(abs(ev), 1.0)
    r1 = oracle.coupling_residual(*args, v.dof_conn, mp.p_dof_conn, p=np.ones(mp.n_p_nodes))
    rd = oracle.eval_residual(fi.DIVERGENCE, pv, q1d, v.coords, v.conn, v.dof_conn, v.u)
    assert rel(r1, rd) < 1e-14


@pytest.mark.parametrize("pv,pp", [(2, 1), (1, 1), (3, 2)])
def test_N3_stokes_coupling_linear_fields(pv, pp):
    """u = x and p = x_0 + 2 x_1 - x_2 are exact in Q_pv / Q_pp on trilinear cells, so
    eval = int p div x = 3 int (x_0 + 2 x_1 - x_2) = 3 (1/2 + 1 - 1/2) = 3 on the unit cube;
    with p = 1: int div x = 3."""
    mp = fi.make_mixed_problem(pv, pp, (2, 3, 2), 57)
    v = mp.vel
    X = _node_coords_order(v, pv, v.dof_conn, v.n_nodes)
    Xp = _node_coords_order(v, pp, mp.p_dof_conn, mp.n_p_nodes)
    pl = Xp[:, 0] + 2 * Xp[:, 1] - Xp[:, 2]
    args = (pv, pp, pv + 1, v.coords, v.conn, v.dof_conn, mp.p_dof_conn)
    assert abs(oracle.coupling_eval(*args, X, pl) - 3.0) < 1e-13
    assert abs(oracle.coupling_eval(*args, X, np.ones(mp.n_p_nodes)) - 3.0) < 1e-13


# ---------------------------------------------------------------- geometry output layout
def _corners01():
    """Reference corners of [0,1]^3 in the lexicographic vertex order v = a + 2b + 4c."""
    return np.array([[a, b, c] for c in (0, 1) for b in (0, 1) for a in (0, 1)], dtype=float)


def _trilinear(xv, xi):
    """x(xi) of the trilinear map with vertex coordinates xv[8][3] (reading 4)."""
    w = np.array([(xi[0] if a else 1 - xi[0]) * (xi[1] if b else 1 - xi[1]) *
                  (xi[2] if c else 1 - xi[2]) for c in (0, 1) for b in (0, 1) for a in (0, 1)])
    return w @ xv


@pytest.mark.parametrize("q1d", [2, 3, 5])
def test_geometry_affine_closed_form(q1d):
    """Affine cell x = A xi + b: J = A at every qp, so the stored J^-1 is A^-1 (row-major,
    J_ij = dx_i/dxi_j) and detw = w_q det A.  A is non-symmetric, so a transposed
    J^-1 store, a permuted qp order or a dropped weight fails."""
    A = np.array([[0.9, 0.2, -0.1], [0.05, 1.3, 0.3], [-0.2, 0.1, 0.7]])
    b = np.array([0.1, -0.4, 2.0])
    coords = _corners01() @ A.T + b
    conn = np.arange(8, dtype=np.int32)[None]
    detw, Jinv = oracle.geometry(q1d, coords, conn)
    t, w = np.polynomial.legendre.leggauss(q1d)
    w = w / 2.0
    W = np.einsum("c,b,a->cba", w, w, w).ravel()          # q = a + q1d (b + q1d c)
    Ainv = np.linalg.inv(A)
    assert np.abs(Jinv[0] - Ainv[None]).max() <= 1e-14 * np.abs(Ainv).max()
    np.testing.assert_allclose(detw[0], W * np.linalg.det(A), rtol=1e-14)


def test_geometry_jinv_perturbed():
    """Perturbed cells: J from exact central differences of the trilinear map (linear in each
    xi_j separately, so the difference quotient is exact up to rounding) times the oracle's
    J^-1 is the identity at every qp; J^-1 also equals numpy.linalg.inv of the einsum oracle's
    Jacobian (tests/einsum_oracle.py) in the same [E][q][3][3] layout."""
    pr = fi.make_problem(fi.DIFFUSION, 2, (3, 2, 2), 31)
    q1d = 3
    detw, Jinv = oracle.geometry(q1d, pr.coords, pr.conn)
    t, w = np.polynomial.legendre.leggauss(q1d)
    x = (t + 1) / 2
    qps = [(x[a], x[b], x[c]) for c in range(q1d) for b in range(q1d) for a in range(q1d)]
    h = 0.25
    for e in range(pr.n_elems):
        xv = pr.coords[pr.conn[e]]
        for q, xi in enumerate(qps):
            J = np.zeros((3, 3))
            for j in range(3):
                d = np.zeros(3)
                d[j] = h
                J[:, j] = (_trilinear(xv, np.add(xi, d)) - _trilinear(xv, np.subtract(xi, d))) / (2 * h)
            assert np.abs(J @ Jinv[e, q] - np.eye(3)).max() <= 1e-13
            assert abs(detw[e, q] - np.linalg.det(J) * w[q % 3] * w[(q // 3) % 3] * w[q // 9] / 8) \
                <= 1e-14 * abs(detw[e, q])
    det2, Jinv2 = eo.mapping(pr.coords, pr.conn, q1d)
    assert rel(Jinv, Jinv2) < 1e-14
    assert rel(detw, det2) < 1e-14


# ---------------------------------------------------------------- D = 3 gather / scatter
@pytest.mark.parametrize("p", [1, 2])
def test_P5_vector_patch_test(p):
    """Vector patch test (the D = 3 analogue of P5, gather/scatter through the connectivity,
    P:1093-1095): u = A x + b at the nodes with constant lambda, mu gives a constant stress, so
    the assembled elasticity residual int sigma : grad v vanishes at every interior node of a
    perturbed mesh (div sigma = 0, and the integrand sigma : cof(J)^T grad phi is integrated
    exactly by q1d = p + 1).  Global vector node-major interleaved [n_nodes][3] (reading 9): a
    component-major scatter or gather puts boundary values on interior rows and fails."""
    pr = fi.make_problem(fi.ELASTICITY, p, (3, 3, 3), 41)
    X = node_coords(pr)
    A = np.array([[0.3, -0.7, 0.2], [0.5, 0.1, -0.4], [-0.6, 0.8, 0.25]])
    u = X @ A.T + np.array([0.2, -0.1, 0.4])
    lam = np.full(pr.n_elems, 1.3)
    mu = np.full(pr.n_elems, 0.8)
    r = oracle.eval_residual(fi.ELASTICITY, p, p + 1, pr.coords, pr.conn, pr.dof_conn, u,
                             fi.MAT_PER_ELEM, lam, mu)
    R = oracle.assemble(r, pr.dof_conn, pr.n_nodes, 3).reshape(pr.n_nodes, 3)
    M = 3 * p + 1
    idx = np.arange(pr.n_nodes)
    ix, iy, iz = idx % M, (idx // M) % M, idx // (M * M)
    interior = (ix > 0) & (ix < M - 1) & (iy > 0) & (iy < M - 1) & (iz > 0) & (iz < M - 1)
    assert np.abs(R[interior]).max() <= 1e-13 * np.abs(R).max()
    assert (np.abs(R[~interior]).max(axis=0) > 1e-3).all()
    # the per-component boundary tractions balance: sum over all nodes of R[:, a] = 0
    assert np.abs(R.sum(axis=0)).max() <= 1e-13 * np.abs(R).max()


def test_vector_assembly_component_sums():
    """Vector mass with rho = 1 and u = c (constant vector): sum_nodes R[:, a] = c_a vol (= c_a
    on the unit cube), per component, through the interleaved scatter (reading 9)."""
    pr = fi.make_problem(fi.VECTOR_MASS, 2, (3, 2, 2), 43)
    c = np.array([1.0, -2.0, 3.5])
    u = np.tile(c, (pr.n_nodes, 1))
    r = oracle.eval_residual(fi.VECTOR_MASS, 2, 3, pr.coords, pr.conn, pr.dof_conn, u, 0,
                             np.ones((pr.n_elems, pr.nq)))
    R = oracle.assemble(r, pr.dof_conn, pr.n_nodes, 3).reshape(pr.n_nodes, 3)
    np.testing.assert_allclose(R.sum(axis=0), c, rtol=1e-13)
    # and each node's three entries are c times the same lumped mass
    lumped = R[:, 0] / c[0]
    np.testing.assert_allclose(R, lumped[:, None] * c[None], rtol=1e-12, atol=1e-16)


@pytest.mark.parametrize("p", [1, 2])
def test_N3_cauchy_stress_integral(p):
    """Cauchy stress in 'eval' mode, "returning the integral value": for an affine
    u and constant lambda, mu, sigma is the constant D eps(A), so int_e sigma = D eps(A) vol(e)
    with vol(e) from the mass-matrix pin (P4), and the cells sum to D eps(A) on the unit cube."""
    pr = fi.make_problem(fi.ELASTICITY, p, (3, 2, 2), 45)
    X = node_coords(pr)
    A = np.array([[0.3, -0.2, 0.1], [0.05, -0.4, 0.25], [0.2, 0.15, 0.6]])
    u = X @ A.T + np.array([0.1, -0.3, 0.2])
    lam = np.full(pr.n_elems, 1.1)
    mu = np.full(pr.n_elems, 0.7)
    si = oracle.eval_stress_integral(p, p + 1, pr.coords, pr.conn, pr.dof_conn, u,
                                     fi.MAT_PER_ELEM, lam, mu)
    eps = np.array([A[0, 0], A[1, 1], A[2, 2], A[0, 1] + A[1, 0], A[0, 2] + A[2, 0],
                    A[1, 2] + A[2, 1]])
    ref = oracle.isotropic_D(1.1, 0.7) @ eps
    M = oracle.eval_matrix(fi.MASS, p, p + 1, pr.coords, pr.conn, pr.dof_conn, 0,
                           np.ones((pr.n_elems, pr.nq)))
    vol = M.sum(axis=(1, 2))
    np.testing.assert_allclose(si, vol[:, None] * ref[None, :], rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(si.sum(axis=0), ref, rtol=1e-13)
    # with random materials: the integral is the quadrature sum of the per-qp oracle stress
    # weighted by detw (two oracle entry points, same definition, different loops)
    pr2 = fi.make_problem(fi.ELASTICITY, p, (2, 2, 2), 46, mat_kind=fi.MAT_PER_QP)
    si2 = oracle.eval_stress_integral(p, p + 1, pr2.coords, pr2.conn, pr2.dof_conn, pr2.u,
                                      pr2.mat_kind, pr2.mat_a, pr2.mat_b, 2, 7)
    sq = oracle.eval_stress(p, p + 1, pr2.coords, pr2.conn, pr2.dof_conn, pr2.u, pr2.mat_kind,
                            pr2.mat_a, pr2.mat_b, 2, 7)
    detw, _ = oracle.geometry(p + 1, pr2.coords, pr2.conn)
    np.testing.assert_allclose(si2, np.einsum("eq,eqi->ei", detw[2:7], sq), rtol=1e-12, atol=1e-18)

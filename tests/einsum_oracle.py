"""Second, independent oracle (pin P11): numpy.einsum on the paper's own einsum strings.

Test infrastructure.  Operands are built here from scratch, independently of
oracle/fe_oracle.c and of the CUDA path:
  * Gauss-Legendre points from numpy.polynomial.legendre.leggauss (on [-1,1],
    mapped to [0,1]);
  * Lagrange polynomials from numpy.polynomial.Polynomial.fromroots;
  * Jacobians by einsum over the 8 vertices, inverse and determinant by
    numpy.linalg.inv / numpy.linalg.det.
The contractions are the transpiled strings printed in PAPER.md Sec. 5.3:
  weak Laplacian matrix   'cq,cqjd,cqje->cde'
  vector dot matrix       'cq,qd,ir,qe,is->crdse'
  vector dot residual     'cq,qd,ir,qe,cie->crd'
  linear elasticity       'cq,cqje,rjI,cqIK,cqlf,slK->cresf'
and, for the convective form, the strings that follow from Eq. fe3 / fe4
 by the same rule (drop one DOF factor per derivative).
Material values per qp are folded into the 'cq' det operand.
"""
from __future__ import annotations

import numpy as np
from numpy.polynomial import Polynomial


def gauss01(n):
    t, w = np.polynomial.legendre.leggauss(n)
    return (t + 1.0) / 2.0, w / 2.0


def lagrange_polys(p):
    nodes = np.arange(p + 1) / p
    polys = []
    for i in range(p + 1):
        others = np.delete(nodes, i)
        P = Polynomial.fromroots(others)
        polys.append(P / P(nodes[i]))
    return polys


def tables(p, q1d):
    """bf[q][d], bfg_ref[q][l][d] with x-fastest lexicographic q and d."""
    x, w = gauss01(q1d)
    polys = lagrange_polys(p)
    v1 = np.array([[P(t) for P in polys] for t in x])            # [q1d][p+1]
    d1 = np.array([[P.deriv()(t) for P in polys] for t in x])
    # index order (c,b,a) for qp and (l,j,i) for nodes, flattened x fastest
    # q = (qz, qy, qx), d = (kz, ky, kx), flattened x fastest
    bf = np.einsum("zc,yb,xa->zyxcba", v1, v1, v1).reshape(q1d ** 3, (p + 1) ** 3)
    gx = np.einsum("zc,yb,xa->zyxcba", v1, v1, d1).reshape(q1d ** 3, (p + 1) ** 3)
    gy = np.einsum("zc,yb,xa->zyxcba", v1, d1, v1).reshape(q1d ** 3, (p + 1) ** 3)
    gz = np.einsum("zc,yb,xa->zyxcba", d1, v1, v1).reshape(q1d ** 3, (p + 1) ** 3)
    bfg = np.stack([gx, gy, gz], axis=1)
    W = np.einsum("z,y,x->zyx", w, w, w).ravel()
    X = np.stack(np.meshgrid(x, x, x, indexing="ij")[::-1], axis=-1).reshape(-1, 3)
    return X, W, bf, bfg


def mapping(coords, conn, q1d):
    """det (incl. weights) [c][q] and physical gradients of the trilinear map."""
    X, W, _, g1 = tables(1, q1d)           # trilinear basis gradients [q][3][8]
    xv = coords[conn]                       # [c][8][3]
    J = np.einsum("cvi,qjv->cqij", xv, g1)  # J_ij = dx_i/dxi_j
    det = np.linalg.det(J)
    Jinv = np.linalg.inv(J)
    return det * W[None, :], Jinv


def operands(coords, conn, p, q1d):
    det, Jinv = mapping(coords, conn, q1d)
    _, _, bf, bfg_ref = tables(p, q1d)
    # physical: bfg[c,q,j,d] = sum_l bfg_ref[q,l,d] Jinv[c,q,l,j]
    bfg = np.einsum("qld,cqlj->cqjd", bfg_ref, Jinv)
    return det, bf, bfg


def psg():
    P = np.zeros((3, 3, 6))
    P[0, 0, 0] = P[1, 1, 1] = P[2, 2, 2] = 1.0
    P[0, 1, 3] = P[1, 0, 3] = 1.0
    P[0, 2, 4] = P[2, 0, 4] = 1.0
    P[1, 2, 5] = P[2, 1, 5] = 1.0
    return P


def iso_D(lam, mu):
    """[..., 6, 6] isotropic Voigt matrix (engineering shears)."""
    lam = np.asarray(lam)[..., None, None]
    mu = np.asarray(mu)[..., None, None]
    L = np.zeros((6, 6))
    L[:3, :3] = 1.0
    M = np.diag([2.0, 2, 2, 1, 1, 1])
    return lam * L + mu * M


def matrix(form, coords, conn, p, q1d, dof_conn=None, mat_a=None, mat_b=None, mat_kind=0,
           u_state=None):
    det, bf, bfg = operands(coords, conn, p, q1d)
    nb = bf.shape[1]
    c = det.shape[0]
    I3 = np.eye(3)
    if form == 0:
        return np.einsum("cq,cqjd,cqje->cde", det * mat_a, bfg, bfg)
    if form == 1:
        return np.einsum("cq,qd,qe->cde", det * mat_a, bf, bf)
    if form == 2:
        K = np.einsum("cq,qd,ir,qe,is->crdse", det * mat_a, bf, I3, bf, I3)
        return K.reshape(c, 3 * nb, 3 * nb)
    if form == 3:
        return (np.einsum("cq,qd,qe->cde", det * mat_a, bf, bf)
                + np.einsum("cq,cqjd,cqje->cde", det * mat_b, bfg, bfg))
    if form == 4:
        if mat_kind == 1:
            D = np.broadcast_to(iso_D(mat_a, mat_b)[:, None], (c, det.shape[1], 6, 6))
        elif mat_kind == 0:
            D = iso_D(mat_a, mat_b)
        else:
            D = mat_a
        P = psg()
        K = np.einsum("cq,cqje,rjI,cqIK,cqlf,slK->cresf", det, bfg, P, D, bfg, P, optimize=True)
        return K.reshape(c, 3 * nb, 3 * nb)
    if form == 5:
        ue = u_state[dof_conn].transpose(0, 2, 1)   # [c][i][m]
        t1 = np.einsum("cq,qk,ab,cqjl,cjm,qm->cakbl", det, bf, I3, bfg, ue, bf, optimize=True)
        t2 = np.einsum("cq,qk,cal,cqbl,qm->cakbm", det, bf, ue, bfg, bf, optimize=True)
        return (t1 + t2).reshape(c, 3 * nb, 3 * nb)
    raise ValueError(form)


def residual(form, coords, conn, p, q1d, dof_conn, u, mat_a=None, mat_b=None, mat_kind=0):
    det, bf, bfg = operands(coords, conn, p, q1d)
    c = det.shape[0]
    ue = u[dof_conn].transpose(0, 2, 1)             # u.dofs 'cie' [c][D][nb]
    if form == 0:
        return np.einsum("cq,cqjd,cqje,ce->cd", det * mat_a, bfg, bfg, ue[:, 0])
    if form == 1:
        return np.einsum("cq,qd,qe,ce->cd", det * mat_a, bf, bf, ue[:, 0])
    if form == 2:
        I3 = np.eye(3)
        return np.einsum("cq,qd,ir,qe,cie->crd", det * mat_a, bf, I3, bf, ue).reshape(c, -1)
    if form == 3:
        return (np.einsum("cq,qd,qe,ce->cd", det * mat_a, bf, bf, ue[:, 0])
                + np.einsum("cq,cqjd,cqje,ce->cd", det * mat_b, bfg, bfg, ue[:, 0]))
    if form == 4:
        if mat_kind == 1:
            D = np.broadcast_to(iso_D(mat_a, mat_b)[:, None], (c, det.shape[1], 6, 6))
        elif mat_kind == 0:
            D = iso_D(mat_a, mat_b)
        else:
            D = mat_a
        P = psg()
        return np.einsum("cq,cqje,rjI,cqIK,cqlf,slK,csf->cre", det, bfg, P, D, bfg, P, ue,
                         optimize=True).reshape(c, -1)
    if form == 5:
        return np.einsum("cq,qk,cal,cqjl,cjm,qm->cak", det, bf, ue, bfg, ue, bf,
                         optimize=True).reshape(c, -1)
    raise ValueError(form)

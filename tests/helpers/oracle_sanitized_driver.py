"""Run every oracle entry point on small problems; executed by tests/test_oracle_sanitized.py in
a subprocess with ORACLE_SANITIZE=1 and libasan / libubsan preloaded.  Prints 'done <n>'."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import fe_inputs as fi  # noqa: E402
import oracle  # noqa: E402

assert oracle.build().endswith("liboracle_san.so")
n = 0
for nq in range(1, 8):
    x, w = oracle.gauss_legendre(nq)
    assert abs(w.sum() - 1.0) < 1e-13      # reference cell [0, 1]
for p in (1, 2, 3, 4):
    oracle.lagrange_1d(p, 0.3)
    oracle.tables(p, p + 1)
oracle.isotropic_D(1.0, 2.0)
shape = (3, 2, 2)
for form in range(8):
    for p in (1, 2, 3, 4):
        kinds = [None]
        if form == fi.ELASTICITY:
            kinds = [fi.MAT_PER_QP, fi.MAT_PER_ELEM, fi.MAT_FULL_D]
        for kind in kinds:
            pr = fi.make_problem(form, p, shape, 900 + 10 * form + p, mat_kind=kind)
            if form != fi.DIVERGENCE:
                K = oracle.problem_matrix(pr)
                assert np.isfinite(K).all()
            r = oracle.problem_residual(pr)
            assert np.isfinite(r).all()
            oracle.problem_residual(pr, 1, pr.n_elems - 1)
            oracle.problem_assembled_residual(pr)
            if form != fi.DIVERGENCE:
                oracle.problem_eval_scalar(pr)
            if form == fi.ELASTICITY:
                oracle.problem_stress(pr)
                oracle.eval_stress_integral(p, p + 1, pr.coords, pr.conn, pr.dof_conn, pr.u,
                                            pr.mat_kind, pr.mat_a, pr.mat_b)
            oracle.geometry(p + 1, pr.coords, pr.conn)
            n += 1
for pv, pp in ((1, 1), (2, 1), (2, 2), (3, 2), (4, 3)):
    mp = fi.make_mixed_problem(pv, pp, shape, 950 + 10 * pv + pp)
    v = mp.vel
    a = (pv, pp, pv + 1, v.coords, v.conn)
    for tr in (False, True):
        oracle.coupling_matrix(*a, transposed=tr)
        oracle.coupling_matrix(*a, transposed=tr, elem_begin=1, elem_end=v.n_elems - 1)
    oracle.coupling_residual(*a, v.dof_conn, mp.p_dof_conn, p=mp.pres)
    oracle.coupling_residual(*a, v.dof_conn, mp.p_dof_conn, u=v.u, transposed=True)
    oracle.coupling_eval(*a, v.dof_conn, mp.p_dof_conn, v.u, mp.pres)
    n += 1
# the degenerate-cell error path
pr = fi.make_problem(fi.DIFFUSION, 1, shape, 7)
conn = pr.conn.copy()
conn[1] = conn[1][[1, 0, 3, 2, 5, 4, 7, 6]]
try:
    oracle.eval_matrix(fi.DIFFUSION, 1, 2, pr.coords, conn, None, pr.mat_kind, pr.mat_a, pr.mat_b)
except Exception:  # noqa: BLE001 - the status is what the pins check; here only memory safety
    pass
print("done", n)

"""Guard-band checks of every C-ABI call that writes device memory.

compute-sanitizer is not available on the GPU pool, so the out-of-bounds checks are built into
the tests: every output is a view into the middle of a larger buffer filled with a fixed NaN
bit pattern, every input (u, material arrays) sits between NaN guard bands, and an element
sub-range [lo, hi) with odd bounds is evaluated.  After each call

* the guard bands of the outputs are bitwise intact (no write outside [lo, hi) / the view),
* the view equals the oracle's rows lo..hi (tolerances of test_gpu_parity.py): a kernel that
  used an input it fetched from outside the arrays (the kernels fetch 16-B-aligned enclosing
  ranges) would carry the guard NaN into its result.

The offsets of the views are chosen so that both the 16-B-aligned (bulk-store, vector) and the
8-B-aligned (fallback) code paths run, with the grid capped to 2 CTAs (several batches per CTA
and a ragged tail) and uncapped.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import fe_inputs as fi
import oracle
from test_gpu_parity import TOL32, TOL64, _dense_global, fe, gpu_mesh, rel

pytestmark = pytest.mark.gpu

SENT = 0x7FF8DEADBEEF1234          # a quiet NaN with a payload no kernel produces
SENT32 = 0x7FC0BEEF
GUARD = 257                        # guard-band length in values on each side


class Banded:
    """A view of `shape` starting `off` values into a sentinel-filled flat buffer."""

    def __init__(self, shape, off, dtype=torch.float64, fill=None):
        n = int(np.prod(shape))
        it = torch.int64 if dtype == torch.float64 else torch.int32
        self.bits = torch.full((off + n + GUARD,), SENT if dtype == torch.float64 else SENT32,
                               dtype=it, device="cuda")
        self.flat = self.bits.view(dtype)
        self.off, self.n = off, n
        self.view = self.flat[off:off + n].view(shape)
        if fill is not None:
            self.view.copy_(fill)
        self.sent = SENT if dtype == torch.float64 else SENT32

    def intact(self):
        lo = self.bits[:self.off]
        hi = self.bits[self.off + self.n:]
        return bool((lo == self.sent).all()) and bool((hi == self.sent).all())

    def rows_untouched(self, a, b):
        """rows [a, b) of the view (first axis) still hold the sentinel"""
        it = self.bits.dtype
        return bool((self.view[a:b].contiguous().view(it) == self.sent).all())


def banded_input(a, off, dtype=torch.float64):
    if a is None:
        return None
    t = torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)
    return Banded(t.shape, off, dtype, fill=t).view


CASES = [(f, p) for f in (0, 1, 2, 3, 4, 5) for p in (1, 2)] + [(0, 3), (3, 4), (2, 3), (5, 4)]


@pytest.mark.parametrize("cap", [0, 2])
@pytest.mark.parametrize("off", [GUARD - 1, GUARD])      # 16-B aligned / 8-B aligned views
@pytest.mark.parametrize("form,p", CASES)
def test_residual_guard_bands(form, p, off, cap, fe_opts):
    fe_opts(max_ctas=cap)
    pr = fi.make_problem(form, p, (5, 3, 4), 21000 + 7 * form + p)
    mesh = gpu_mesh(pr)
    E, nd = pr.n_elems, pr.ncomp * pr.nb
    lo, hi = 3, E - 2
    mat = (pr.mat_kind, banded_input(pr.mat_a, off), banded_input(pr.mat_b, off))
    u = banded_input(pr.u, off)
    re = Banded((hi - lo, nd), off)
    rg = Banded((pr.n_nodes, pr.ncomp), off)
    rg.view.zero_()
    mesh.residual(form, u, *mat, elem_begin=lo, elem_end=hi, r_elem=re.view, r_global=rg.view)
    torch.cuda.synchronize()
    assert re.intact() and rg.intact()
    r_ref = oracle.problem_residual(pr)
    assert rel(re.view.cpu().numpy(), r_ref[lo:hi]) <= TOL64
    R_ref = oracle.assemble(r_ref[lo:hi], pr.dof_conn[lo:hi], pr.n_nodes, pr.ncomp)
    assert rel(rg.view.cpu().numpy().ravel(), R_ref) <= TOL64
    # fe_assemble_vector on its own (r_elem holds the rows of the range [lo, hi))
    ra = Banded((pr.n_nodes, pr.ncomp), off)
    ra.view.zero_()
    rin = banded_input(r_ref[lo:hi], off)
    mesh.assemble(rin, pr.ncomp, r_global=ra.view, elem_begin=lo, elem_end=hi)
    torch.cuda.synchronize()
    assert ra.intact()
    assert rel(ra.view.cpu().numpy().ravel(), R_ref) <= TOL64


@pytest.mark.parametrize("off", [GUARD - 1, GUARD])
@pytest.mark.parametrize("form,p", [(3, 4), (0, 2), (1, 2), (0, 1)])
def test_residual_fp32_guard_bands(form, p, off):
    pr = fi.make_problem(form, p, (5, 3, 4), 22000 + form)
    mesh = gpu_mesh(pr)
    E, nd = pr.n_elems, pr.ncomp * pr.nb
    lo, hi = 3, E - 2
    f32 = torch.float32
    mat = (pr.mat_kind, banded_input(pr.mat_a, off, f32), banded_input(pr.mat_b, off, f32))
    re = Banded((hi - lo, nd), off, f32)
    rg = Banded((pr.n_nodes, pr.ncomp), off, f32)
    rg.view.zero_()
    mesh.residual(form, banded_input(pr.u, off, f32), *mat, elem_begin=lo, elem_end=hi,
                  r_elem=re.view, r_global=rg.view)
    torch.cuda.synchronize()
    assert re.intact() and rg.intact()
    r_ref = oracle.problem_residual(pr)
    assert rel(re.view.cpu().numpy(), r_ref[lo:hi]) <= TOL32
    R_ref = oracle.assemble(r_ref[lo:hi], pr.dof_conn[lo:hi], pr.n_nodes, pr.ncomp)
    assert rel(rg.view.cpu().numpy().ravel(), R_ref) <= TOL32


MATRIX_CASES = [(f, p) for f in (0, 1, 2, 3, 4, 5) for p in (1, 2)] + [(0, 3), (3, 3), (2, 3)]


@pytest.mark.parametrize("cap", [0, 2])
@pytest.mark.parametrize("off", [GUARD - 1, GUARD])
@pytest.mark.parametrize("form,p", MATRIX_CASES)
def test_matrix_guard_bands(form, p, off, cap, fe_opts):
    fe_opts(max_ctas=cap)
    pr = fi.make_problem(form, p, (5, 3, 4), 23000 + 7 * form + p)
    mesh = gpu_mesh(pr)
    E, nd = pr.n_elems, pr.ncomp * pr.nb
    lo, hi = 3, E - 2
    mat = (pr.mat_kind, banded_input(pr.mat_a, off), banded_input(pr.mat_b, off))
    su = banded_input(pr.u, off) if form == fi.CONVECTIVE else None
    # the whole-mesh K buffer: rows outside [lo, hi) must stay untouched as well
    K = Banded((E, nd, nd), off)
    mesh.element_matrices(form, *mat, su, elem_begin=lo, elem_end=hi, out=K.view[lo:hi])
    torch.cuda.synchronize()
    assert K.intact()
    assert K.rows_untouched(0, lo) and K.rows_untouched(hi, E)
    Kref = oracle.problem_matrix(pr)
    assert rel(K.view[lo:hi].cpu().numpy(), Kref[lo:hi]) <= TOL64


@pytest.mark.parametrize("off", [GUARD - 1, GUARD])
@pytest.mark.parametrize("form,p", [(0, 1), (0, 2), (1, 2), (3, 2)])
def test_matrix_fp32_guard_bands(form, p, off):
    pr = fi.make_problem(form, p, (5, 3, 4), 24000 + form)
    mesh = gpu_mesh(pr)
    E, nd = pr.n_elems, pr.ncomp * pr.nb
    lo, hi = 3, E - 2
    f32 = torch.float32
    mat = (pr.mat_kind, banded_input(pr.mat_a, off, f32), banded_input(pr.mat_b, off, f32))
    K = Banded((E, nd, nd), off, f32)
    mesh.element_matrices(form, *mat, None, elem_begin=lo, elem_end=hi, out=K.view[lo:hi])
    torch.cuda.synchronize()
    assert K.intact() and K.rows_untouched(0, lo) and K.rows_untouched(hi, E)
    assert rel(K.view[lo:hi].cpu().numpy(), oracle.problem_matrix(pr)[lo:hi]) <= TOL32


@pytest.mark.parametrize("cap", [0, 2])
@pytest.mark.parametrize("off", [GUARD - 1, GUARD])
@pytest.mark.parametrize("form,p", [(0, 1), (0, 2), (1, 2), (3, 2)])
def test_fused_matrix_residual_guard_bands(form, p, off, cap, fe_opts):
    fe_opts(max_ctas=cap)
    pr = fi.make_problem(form, p, (5, 3, 4), 25000 + form)
    mesh = gpu_mesh(pr)
    E, nd = pr.n_elems, pr.nb
    lo, hi = 3, E - 2
    mat = (pr.mat_kind, banded_input(pr.mat_a, off), banded_input(pr.mat_b, off))
    K = Banded((hi - lo, nd, nd), off)
    re = Banded((hi - lo, nd), off)
    rg = Banded((pr.n_nodes, 1), off)
    rg.view.zero_()
    mesh.matrix_residual(form, banded_input(pr.u, off), *mat, elem_begin=lo, elem_end=hi,
                         K=K.view, r_elem=re.view, r_global=rg.view)
    torch.cuda.synchronize()
    assert K.intact() and re.intact() and rg.intact()
    assert rel(K.view.cpu().numpy(), oracle.problem_matrix(pr)[lo:hi]) <= TOL64
    r_ref = oracle.problem_residual(pr)
    assert rel(re.view.cpu().numpy(), r_ref[lo:hi]) <= TOL64
    R_ref = oracle.assemble(r_ref[lo:hi], pr.dof_conn[lo:hi], pr.n_nodes, 1)
    assert rel(rg.view.cpu().numpy().ravel(), R_ref) <= TOL64


@pytest.mark.parametrize("off", [GUARD - 1, GUARD])
@pytest.mark.parametrize("p", [1, 2, 4])
def test_geometry_stress_guard_bands(p, off):
    m = fe()
    pr = fi.make_problem(fi.ELASTICITY, p, (4, 3, 2), 26000 + p)
    mesh = gpu_mesh(pr)
    E, nq = pr.n_elems, (p + 1) ** 3
    detw, jinv = Banded((E, nq), off), Banded((E, nq, 3, 3), off)
    m.fe_geometry(mesh.handle, detw.view, jinv.view)
    torch.cuda.synchronize()
    assert detw.intact() and jinv.intact()
    detw_ref, jinv_ref = oracle.geometry(p + 1, pr.coords, pr.conn)
    assert rel(detw.view.cpu().numpy(), detw_ref) <= TOL64
    assert rel(jinv.view.cpu().numpy(), jinv_ref) <= TOL64
    if p > 2:
        return
    lo, hi = 3, E - 2
    mat = (pr.mat_kind, banded_input(pr.mat_a, off), banded_input(pr.mat_b, off))
    u = banded_input(pr.u, off)
    sig, sint = Banded((hi - lo, nq, 6), off), Banded((hi - lo, 6), off)
    m.fe_eval_stress(mesh.handle, *mat, u, lo, hi, sig.view)
    m.fe_eval_stress_integral(mesh.handle, *mat, u, lo, hi, sint.view)
    torch.cuda.synchronize()
    assert sig.intact() and sint.intact()
    assert rel(sig.view.cpu().numpy(), oracle.problem_stress(pr)[lo:hi]) <= TOL64
    ref_i = oracle.eval_stress_integral(p, p + 1, pr.coords, pr.conn, pr.dof_conn, pr.u,
                                        pr.mat_kind, pr.mat_a, pr.mat_b)
    assert rel(sint.view.cpu().numpy(), ref_i[lo:hi]) <= TOL64


@pytest.mark.parametrize("impl", ["atomic", "gather"])
@pytest.mark.parametrize("off", [GUARD - 1, GUARD])
@pytest.mark.parametrize("form,p", [(0, 1), (0, 2), (2, 1), (2, 2)])
def test_csr_guard_bands(form, p, off, impl, fe_opts):
    import scipy.sparse as sp
    fe_opts(csr_impl=impl)
    m = fe()
    pr = fi.make_problem(form, p, (3, 2, 3), 27000 + form)
    mesh = gpu_mesh(pr)
    Kref = oracle.problem_matrix(pr)
    K = banded_input(Kref, off)
    csr = m.CSR(mesh, pr.ncomp)
    vals = Banded((csr.nnz,), off)
    vals.view.zero_()
    csr.assemble(K, values=vals.view)
    torch.cuda.synchronize()
    assert vals.intact()
    rp, ci = csr.arrays()
    A = sp.csr_matrix((vals.view.cpu().numpy(), ci, rp), shape=(csr.n_rows, csr.n_rows)).toarray()
    Aref = _dense_global(pr, Kref)
    assert rel(A, Aref) <= TOL64
    csr.close()


# ---- the non-default implementations, the remaining forms and material kinds ----------------

@pytest.mark.parametrize("off", [GUARD - 1, GUARD])
@pytest.mark.parametrize("impl", ["sf1", "dense"])
@pytest.mark.parametrize("form,p", [(0, 1), (0, 2), (3, 2), (4, 1), (4, 2), (5, 2), (2, 2), (4, 3)])
def test_matrix_impl_guard_bands(form, p, impl, off, fe_opts):
    fe_opts(matrix_impl=impl, max_ctas=2)
    pr = fi.make_problem(form, p, (5, 3, 4), 28000 + 7 * form + p)
    mesh = gpu_mesh(pr)
    E, nd = pr.n_elems, pr.ncomp * pr.nb
    lo, hi = 3, E - 2
    mat = (pr.mat_kind, banded_input(pr.mat_a, off), banded_input(pr.mat_b, off))
    su = banded_input(pr.u, off) if form == fi.CONVECTIVE else None
    K = Banded((E, nd, nd), off)
    mesh.element_matrices(form, *mat, su, elem_begin=lo, elem_end=hi, out=K.view[lo:hi])
    torch.cuda.synchronize()
    assert K.intact() and K.rows_untouched(0, lo) and K.rows_untouched(hi, E)
    assert rel(K.view[lo:hi].cpu().numpy(), oracle.problem_matrix(pr)[lo:hi]) <= TOL64


@pytest.mark.parametrize("off", [GUARD - 1, GUARD])
@pytest.mark.parametrize("impl", ["sf", "dense"])
@pytest.mark.parametrize("form,p", [(0, 1), (0, 2), (3, 2), (4, 2), (5, 2), (3, 4), (4, 3),
                                    (fi.WEIGHTED_DOT, 2), (fi.DIVERGENCE, 2), (fi.WEIGHTED_DOT, 4)])
def test_residual_impl_guard_bands(form, p, impl, off, fe_opts):
    fe_opts(residual_impl=impl, max_ctas=2)
    pr = fi.make_problem(form, p, (5, 3, 4), 29000 + 7 * form + p)
    mesh = gpu_mesh(pr)
    E, nd = pr.n_elems, pr.ncomp * pr.nb
    lo, hi = 3, E - 2
    mat = (pr.mat_kind, banded_input(pr.mat_a, off), banded_input(pr.mat_b, off))
    re = Banded((hi - lo, nd), off)
    rg = Banded((pr.n_nodes, pr.ncomp), off)
    rg.view.zero_()
    mesh.residual(form, banded_input(pr.u, off), *mat, elem_begin=lo, elem_end=hi,
                  r_elem=re.view, r_global=rg.view)
    torch.cuda.synchronize()
    assert re.intact() and rg.intact()
    r_ref = oracle.problem_residual(pr)
    assert rel(re.view.cpu().numpy(), r_ref[lo:hi]) <= TOL64
    R_ref = oracle.assemble(r_ref[lo:hi], pr.dof_conn[lo:hi], pr.n_nodes, pr.ncomp)
    assert rel(rg.view.cpu().numpy().ravel(), R_ref) <= TOL64


@pytest.mark.parametrize("cap", [0, 2])
@pytest.mark.parametrize("off", [GUARD - 1, GUARD])
@pytest.mark.parametrize("kind", [fi.MAT_PER_QP, fi.MAT_PER_ELEM, fi.MAT_FULL_D])
@pytest.mark.parametrize("p", [1, 2])
def test_elasticity_kinds_guard_bands(p, kind, off, cap, fe_opts):
    """Every material layout of the elasticity form (lambda, mu per qp / per cell, D[6][6] per
    qp), matrix and residual mode, plus the weighted dot 'ij,i,j' matrix."""
    fe_opts(max_ctas=cap)
    pr = fi.make_problem(fi.ELASTICITY, p, (5, 3, 4), 30000 + 10 * p + kind, mat_kind=kind)
    mesh = gpu_mesh(pr)
    E, nd = pr.n_elems, 3 * pr.nb
    lo, hi = 3, E - 2
    mat = (kind, banded_input(pr.mat_a, off), banded_input(pr.mat_b, off))
    K = Banded((E, nd, nd), off)
    mesh.element_matrices(fi.ELASTICITY, *mat, None, elem_begin=lo, elem_end=hi, out=K.view[lo:hi])
    re = Banded((hi - lo, nd), off)
    mesh.residual(fi.ELASTICITY, banded_input(pr.u, off), *mat, elem_begin=lo, elem_end=hi,
                  r_elem=re.view, want_global=False)
    torch.cuda.synchronize()
    assert K.intact() and K.rows_untouched(0, lo) and K.rows_untouched(hi, E) and re.intact()
    assert rel(K.view[lo:hi].cpu().numpy(), oracle.problem_matrix(pr)[lo:hi]) <= TOL64
    assert rel(re.view.cpu().numpy(), oracle.problem_residual(pr)[lo:hi]) <= TOL64
    wd = fi.make_problem(fi.WEIGHTED_DOT, p, (5, 3, 4), 31000 + p)
    mesh2 = gpu_mesh(wd)
    K2 = Banded((E, nd, nd), off)
    mesh2.element_matrices(fi.WEIGHTED_DOT, wd.mat_kind, banded_input(wd.mat_a, off), None, None,
                           elem_begin=lo, elem_end=hi, out=K2.view[lo:hi])
    torch.cuda.synchronize()
    assert K2.intact() and K2.rows_untouched(0, lo) and K2.rows_untouched(hi, E)
    assert rel(K2.view[lo:hi].cpu().numpy(), oracle.problem_matrix(wd)[lo:hi]) <= TOL64


@pytest.mark.parametrize("off", [GUARD - 1, GUARD])
@pytest.mark.parametrize("pv,pp", [(2, 1), (1, 1), (3, 2)])
def test_stokes_coupling_guard_bands(pv, pp, off):
    m = fe()
    shape = (5, 3, 4) if pv <= 2 else (3, 2, 3)
    mp = fi.make_mixed_problem(pv, pp, shape, 32000 + 10 * pv + pp)
    v = mp.vel
    mesh = gpu_mesh(v)
    pf = m.PressureField(mesh, pp, torch.from_numpy(mp.p_dof_conn), n_nodes=mp.n_p_nodes)
    E = v.n_elems
    lo, hi = 3, E - 2
    args = (pv, pp, pv + 1, v.coords, v.conn)
    for tr in (False, True):
        shape_k = (pf.nb, 3 * mesh.nb) if tr else (3 * mesh.nb, pf.nb)
        B = Banded((E,) + shape_k, off)
        pf.coupling_matrices(transposed=tr, elem_begin=lo, elem_end=hi, out=B.view[lo:hi])
        torch.cuda.synchronize()
        assert B.intact() and B.rows_untouched(0, lo) and B.rows_untouched(hi, E)
        ref = oracle.coupling_matrix(*args, transposed=tr)
        assert rel(B.view[lo:hi].cpu().numpy(), ref[lo:hi]) <= TOL64
    # r_v = B p (velocity-shaped) and r_q = C u (pressure-shaped), element rows + fused scatter
    rv_ref = oracle.coupling_residual(*args, v.dof_conn, mp.p_dof_conn, p=mp.pres)
    rq_ref = oracle.coupling_residual(*args, v.dof_conn, mp.p_dof_conn, u=v.u, transposed=True)
    for tr, x, ref, conn, nn, D in ((False, mp.pres, rv_ref, v.dof_conn, v.n_nodes, 3),
                                    (True, v.u, rq_ref, mp.p_dof_conn, mp.n_p_nodes, 1)):
        re = Banded((hi - lo, ref.shape[1]), off)
        rg = Banded((nn, 3) if not tr else (nn,), off)
        rg.view.zero_()
        pf.coupling_residual(banded_input(x, off), transposed=tr, elem_begin=lo, elem_end=hi,
                             r_elem=re.view, r_global=rg.view)
        torch.cuda.synchronize()
        assert re.intact() and rg.intact()
        assert rel(re.view.cpu().numpy(), ref[lo:hi]) <= TOL64
        assert rel(rg.view.cpu().numpy().ravel(),
                   oracle.assemble(ref[lo:hi], conn[lo:hi], nn, D)) <= TOL64
    pf.close()


@pytest.mark.parametrize("off", [GUARD - 1, GUARD])
def test_eval_scalar_guard_bands(off):
    """Eval mode adds into one fp64 value: its neighbours stay untouched."""
    m = fe()
    for form, p in ((fi.DIFFUSION, 2), (fi.ELASTICITY, 2), (fi.MASS_DIFFUSION, 4), (fi.CONVECTIVE, 2)):
        pr = fi.make_problem(form, p, (4, 3, 3), 33000 + form)
        mesh = gpu_mesh(pr)
        val = Banded((1,), off)
        val.view.zero_()
        lo, hi = 3, pr.n_elems - 2
        m.fe_eval_scalar(mesh.handle, form, m.F64, pr.mat_kind, banded_input(pr.mat_a, off),
                         banded_input(pr.mat_b, off), banded_input(pr.u, off), lo, hi, val.view)
        torch.cuda.synchronize()
        assert val.intact()
        ue = pr.u[pr.dof_conn]                       # [E][nb] or [E][nb][D]
        ue = ue.reshape(pr.n_elems, pr.nb, -1).transpose(0, 2, 1).reshape(pr.n_elems, -1)
        ref = float(np.sum(oracle.problem_residual(pr)[lo:hi] * ue[lo:hi]))
        assert abs(val.view.item() - ref) <= 1e-11 * max(abs(ref), 1e-30)


@pytest.mark.parametrize("off", [GUARD - 1, GUARD])
@pytest.mark.parametrize("form,p", [(0, 1), (0, 2), (4, 2), (5, 2), (3, 4), (4, 1)])
def test_peer_window_guard_bands(form, p, off):
    """fe_eval_residual_peer: the two windows receive exactly their nodes' contributions at the
    requested node offsets of the destination buffers, nothing around them is written."""
    m = fe()
    pr = fi.make_problem(form, p, (4, 3, 5), 34000 + 7 * form + p)
    mesh = gpu_mesh(pr)
    D = pr.ncomp
    plane = pr.n_nodes // 7
    w0, w1 = (0, plane), (pr.n_nodes - plane - 3, pr.n_nodes)
    o0, o1 = 5, 11
    d0 = Banded((o0 + w0[1] - w0[0], D), off)
    d1 = Banded((o1 + w1[1] - w1[0], D), off)
    d0.view[o0:].zero_()
    d1.view[o1:].zero_()
    rg = Banded((pr.n_nodes, D), off)
    rg.view.zero_()
    m.fe_eval_residual_peer(mesh.handle, form, pr.mat_kind, banded_input(pr.mat_a, off),
                            banded_input(pr.mat_b, off), banded_input(pr.u, off), 0, pr.n_elems,
                            None, rg.view,
                            [(w0[0], w0[1], d0.view.data_ptr(), o0),
                             (w1[0], w1[1], d1.view.data_ptr(), o1)])
    torch.cuda.synchronize()
    assert rg.intact() and d0.intact() and d1.intact()
    assert d0.rows_untouched(0, o0) and d1.rows_untouched(0, o1)
    R = oracle.assemble(oracle.problem_residual(pr), pr.dof_conn, pr.n_nodes, D).reshape(-1, D)
    assert rel(rg.view.cpu().numpy(), R) <= TOL64
    assert rel(d0.view[o0:].cpu().numpy(), R[w0[0]:w0[1]]) <= TOL64
    assert rel(d1.view[o1:].cpu().numpy(), R[w1[0]:w1[1]]) <= TOL64

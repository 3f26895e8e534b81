"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Tolerances (BASELINE.json north_star): normwise relative
error <= 1e-12 in fp64 over the whole output array (stacked K in Frobenius
norm, residual vectors in 2-norm); <= 1e-5 for the fp32 residual path against
the fp64 oracle.  Atomic scatter order is the only allowed source of
difference.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import fe_inputs as fi
import oracle

pytestmark = pytest.mark.gpu

TOL64 = 1e-12
TOL32 = 1e-5


def fe():
    import paper_2107_04121_b200 as m
    return m


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300)


def rel_cell_max(a, b):
    """Diagnostic of SURVEY silent point 14: the largest per-cell relative error (each cell's
    K_e in Frobenius norm, or r_e in 2-norm, against the oracle's); a cell-local error that the
    normwise measure over all cells would dilute shows up here."""
    b = np.asarray(b, dtype=np.float64)
    b = b.reshape(b.shape[0], -1)
    a = np.asarray(a, dtype=np.float64).reshape(b.shape)
    nb = np.maximum(np.linalg.norm(b, axis=1), 1e-300)
    return float((np.linalg.norm(a - b, axis=1) / nb).max())


TOL64_CELL = 1e-11  # per cell: the same arithmetic, fewer terms in each norm


def gpu_mesh(prob):
    m = fe()
    return m.Mesh(torch.from_numpy(prob.coords), torch.from_numpy(prob.conn), prob.p, prob.q1d,
                  dof_conn=None if prob.p == 1 else torch.from_numpy(prob.dof_conn),
                  n_nodes=prob.n_nodes)


def dev(a, dtype=torch.float64):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)


# ragged element counts: several CTA batches plus a partial tail
SHAPES = [(5, 3, 4), (7, 2, 3)]
MATRIX_CASES = [(f, p) for f in (0, 1, 2, 3, 4, 5) for p in (1, 2)] + [(0, 3), (1, 3), (3, 3)] + \
               [(2, 3), (4, 3), (5, 3)]   # vector forms at p = 3: the dense DMMA kernel
RESIDUAL_CASES = [(f, p) for f in (0, 1, 2, 3, 4, 5) for p in (1, 2, 3)] + \
                 [(0, 4), (1, 4), (3, 4), (2, 4), (4, 4), (5, 4)]


@pytest.fixture(params=["default", "sf1", "dense"])
def matrix_impl(request, fe_opts):
    """default = sum-factorised kernels where built (warp-specialised pipeline for the scalar
    forms at p <= 2); sf1 = the single-stage sum-factorised kernel; dense = the DMMA kernels."""
    if request.param in ("dense", "sf1"):
        fe_opts(matrix_impl=request.param)
    else:
        fe_opts(matrix_impl="default")
    return request.param


@pytest.mark.parametrize("form,p", MATRIX_CASES)
@pytest.mark.parametrize("shape", SHAPES)
def test_matrix_parity(form, p, shape, matrix_impl):
    pr = fi.make_problem(form, p, shape, 1000 + 10 * form + p)
    Kref = oracle.problem_matrix(pr)
    mesh = gpu_mesh(pr)
    K = mesh.element_matrices(form, pr.mat_kind, dev(pr.mat_a), dev(pr.mat_b),
                              dev(pr.u) if form == fi.CONVECTIVE else None)
    torch.cuda.synchronize()
    assert rel(K.cpu().numpy(), Kref) <= TOL64
    assert rel_cell_max(K.cpu().numpy(), Kref) <= TOL64_CELL
    if form in (fi.DIFFUSION, fi.MASS, fi.MASS_DIFFUSION):
        Kn = K.cpu().numpy()
        assert np.abs(Kn - Kn.transpose(0, 2, 1)).max() <= 1e-14 * np.abs(Kn).max()


@pytest.mark.parametrize("kind", [fi.MAT_PER_ELEM, fi.MAT_PER_QP, fi.MAT_FULL_D])
def test_elasticity_material_kinds(kind):
    pr = fi.make_problem(fi.ELASTICITY, 2, (3, 3, 2), 77, mat_kind=kind)
    mesh = gpu_mesh(pr)
    K = mesh.element_matrices(fi.ELASTICITY, kind, dev(pr.mat_a), dev(pr.mat_b))
    assert rel(K.cpu().numpy(), oracle.problem_matrix(pr)) <= TOL64
    re_, rg = mesh.residual(fi.ELASTICITY, dev(pr.u), kind, dev(pr.mat_a), dev(pr.mat_b),
                            want_elem=True)
    assert rel(re_.cpu().numpy(), oracle.problem_residual(pr)) <= TOL64


@pytest.mark.parametrize("form,p", RESIDUAL_CASES)
@pytest.mark.parametrize("shape", SHAPES)
def test_residual_parity(form, p, shape):
    pr = fi.make_problem(form, p, shape, 2000 + 10 * form + p)
    r_ref = oracle.problem_residual(pr)
    R_ref = oracle.assemble(r_ref, pr.dof_conn, pr.n_nodes, pr.ncomp)
    mesh = gpu_mesh(pr)
    r_elem, r_glob = mesh.residual(form, dev(pr.u), pr.mat_kind, dev(pr.mat_a), dev(pr.mat_b),
                                   want_elem=True)
    torch.cuda.synchronize()
    assert rel(r_elem.cpu().numpy(), r_ref) <= TOL64
    assert rel_cell_max(r_elem.cpu().numpy(), r_ref) <= TOL64_CELL
    assert rel(r_glob.cpu().numpy().ravel(), R_ref) <= TOL64


@pytest.mark.parametrize("form,p", [(0, 1), (0, 2), (1, 2), (3, 2), (3, 4), (0, 4)])
def test_residual_fp32(form, p):
    pr = fi.make_problem(form, p, (5, 3, 4), 3000 + form)
    r_ref = oracle.problem_residual(pr)
    R_ref = oracle.assemble(r_ref, pr.dof_conn, pr.n_nodes, pr.ncomp)
    mesh = gpu_mesh(pr)
    r_elem, r_glob = mesh.residual(form, dev(pr.u, torch.float32), pr.mat_kind,
                                   dev(pr.mat_a, torch.float32), dev(pr.mat_b, torch.float32),
                                   want_elem=True)
    assert r_elem.dtype == torch.float32
    assert rel(r_elem.cpu().numpy(), r_ref) <= TOL32
    assert rel(r_glob.cpu().numpy().ravel(), R_ref) <= TOL32


@pytest.mark.parametrize("form,p", [(0, 2), (4, 2), (5, 2), (3, 4)])
def test_element_ranges(form, p):
    """elem_begin / elem_end split (boundary-first overlap) == one full call."""
    pr = fi.make_problem(form, p, (4, 3, 5), 4000 + form)
    mesh = gpu_mesh(pr)
    args = (pr.mat_kind, dev(pr.mat_a), dev(pr.mat_b))
    u = dev(pr.u)
    E = pr.n_elems
    cuts = [0, 7, 8, 31, E - 1, E]
    R = torch.zeros((pr.n_nodes, pr.ncomp), dtype=torch.float64, device="cuda")
    parts = []
    for a, b in zip(cuts[:-1], cuts[1:]):
        re_, _ = mesh.residual(form, u, *args, elem_begin=a, elem_end=b, r_global=R,
                               want_elem=True)
        parts.append(re_.cpu().numpy())
    r_ref = oracle.problem_residual(pr)
    assert rel(np.concatenate(parts), r_ref) <= TOL64
    R_ref = oracle.assemble(r_ref, pr.dof_conn, pr.n_nodes, pr.ncomp)
    assert rel(R.cpu().numpy().ravel(), R_ref) <= TOL64
    if p <= 2:
        Ks = [mesh.element_matrices(form, *args, state_u=u if form == 5 else None,
                                    elem_begin=a, elem_end=b).cpu().numpy()
              for a, b in zip(cuts[:-1], cuts[1:])]
        assert rel(np.concatenate(Ks), oracle.problem_matrix(pr)) <= TOL64
    # empty range is a no-op
    re_, _ = mesh.residual(form, u, *args, elem_begin=5, elem_end=5, r_global=R, want_elem=True)
    assert re_.shape[0] == 0


def test_assemble_vector():
    pr = fi.make_problem(fi.ELASTICITY, 2, (3, 4, 2), 55)
    r_ref = oracle.problem_residual(pr)
    mesh = gpu_mesh(pr)
    R = mesh.assemble(dev(r_ref), 3)
    R_ref = oracle.assemble(r_ref, pr.dof_conn, pr.n_nodes, 3)
    assert rel(R.cpu().numpy().ravel(), R_ref) <= TOL64
    r32 = mesh.assemble(dev(r_ref, torch.float32), 3)
    assert rel(r32.cpu().numpy().ravel(), R_ref) <= TOL32


@pytest.mark.parametrize("p", [1, 2, 4])
def test_geometry_materialized(p):
    pr = fi.make_problem(fi.DIFFUSION, p, (4, 3, 2), 66)
    detw_ref, jinv_ref = oracle.geometry(p + 1, pr.coords, pr.conn)
    mesh = gpu_mesh(pr)
    detw, jinv = mesh.geometry()
    assert rel(detw.cpu().numpy(), detw_ref) <= TOL64
    assert rel(jinv.cpu().numpy(), jinv_ref) <= TOL64
    assert abs(mesh.min_det_j - (detw_ref / oracle.tables(p, p + 1)[1]).min()) <= 1e-12


def test_degenerate_and_invalid():
    m = fe()
    pr = fi.make_problem(fi.DIFFUSION, 1, (3, 2, 1), 1)
    conn = pr.conn.copy()
    conn[4] = conn[4][[1, 0, 3, 2, 5, 4, 7, 6]]
    with pytest.raises(m.FEError) as ei:
        m.Mesh(pr.coords, conn, 1)
    assert ei.value.status == m.FE_ERR_DEGENERATE and ei.value.element == 4
    bad = pr.conn.copy()
    bad[2, 3] = pr.coords.shape[0]
    with pytest.raises(m.FEError) as ei:
        m.Mesh(pr.coords, bad, 1)
    assert ei.value.status == m.FE_ERR_INVALID_ARG
    with pytest.raises(m.FEError) as ei:
        m.Mesh(pr.coords, pr.conn, 5, dof_conn=pr.dof_conn, n_nodes=pr.n_nodes)
    assert ei.value.status == m.FE_ERR_UNSUPPORTED
    mesh = gpu_mesh(pr)
    with pytest.raises(m.FEError) as ei:
        mesh.residual(0, dev(pr.u), 0, dev(pr.mat_a), None, elem_begin=0, elem_end=pr.n_elems + 1)
    assert ei.value.status == m.FE_ERR_INVALID_ARG
    with pytest.raises(m.FEError) as ei:
        mesh.element_matrices(5, 0, None, None, None)   # convective without a state
    assert ei.value.status == m.FE_ERR_INVALID_ARG


def _sample_subproblem(pr, idx):
    return fi.Problem(pr.name, pr.form, pr.p, pr.q1d, pr.shape, pr.coords, pr.conn[idx],
                      pr.dof_conn[idx], pr.n_nodes, pr.mat_kind,
                      None if pr.mat_a is None else pr.mat_a[idx],
                      None if pr.mat_b is None else pr.mat_b[idx], pr.u)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_config_full_size(name):
    """BASELINE configs at full size in the bench launch configuration: matrices
    on a seeded sample of cells checked one by one against the oracle; the
    assembled residual checked in full (C1-C4) or on the slab of cells whose
    nodes are sampled (C5)."""
    pr = fi.make_config(name)
    mesh = gpu_mesh(pr)
    rng = np.random.default_rng(7)
    E = pr.n_elems
    idx = np.unique(np.concatenate([[0, E - 1], rng.choice(E, size=min(E, 48), replace=False)]))
    sub = _sample_subproblem(pr, idx)
    mat = (pr.mat_kind, dev(pr.mat_a), dev(pr.mat_b))
    u = dev(pr.u)
    if name != "C4":
        src = fi.corner_subproblem(pr, 64) if name == "C5" else pr
        mesh_m = gpu_mesh(src) if name == "C5" else mesh
        idx_m = idx[idx < src.n_elems]
        K = mesh_m.element_matrices(src.form, src.mat_kind, dev(src.mat_a), dev(src.mat_b),
                                    u if src.form == fi.CONVECTIVE else None)
        Kref = oracle.problem_matrix(_sample_subproblem(src, idx_m))
        Ks = K[torch.from_numpy(idx_m).cuda()].cpu().numpy()
        assert rel(Ks, Kref) <= TOL64
        assert rel_cell_max(Ks, Kref) <= TOL64_CELL
        del K
    r_elem, r_glob = mesh.residual(pr.form, u, *mat, want_elem=True)
    r_ref = oracle.problem_residual(sub)
    rs = r_elem[torch.from_numpy(idx).cuda()].cpu().numpy()
    assert rel(rs, r_ref) <= TOL64
    assert rel_cell_max(rs, r_ref) <= TOL64_CELL
    # the assembled global vector in full against the oracle's (C5: 2.1 M cells, 50.9 M
    # values; the OpenMP oracle does it in seconds)
    R_ref = oracle.problem_assembled_residual(pr)
    assert rel(r_glob.cpu().numpy().ravel(), R_ref) <= TOL64
    if name == "C4":
        r_elem32, r_glob32 = mesh.residual(pr.form, dev(pr.u, torch.float32), pr.mat_kind,
                                           dev(pr.mat_a, torch.float32),
                                           dev(pr.mat_b, torch.float32), want_elem=True)
        assert rel(r_glob32.cpu().numpy().ravel(), R_ref) <= TOL32


@pytest.mark.parametrize("form,p", [(0, 1), (0, 2), (1, 2), (2, 2), (3, 4), (4, 2), (5, 2), (5, 1)])
def test_eval_mode(form, p):
    """'eval' mode vs the oracle's plain quadrature sum of F(u, u)."""
    pr = fi.make_problem(form, p, (5, 3, 4), 5000 + form)
    ref = oracle.problem_eval_scalar(pr)
    mesh = gpu_mesh(pr)
    v = mesh.eval_scalar(form, dev(pr.u), pr.mat_kind, dev(pr.mat_a), dev(pr.mat_b))
    assert abs(v.item() - ref) <= TOL64 * abs(ref)
    if form in (0, 3):
        v32 = mesh.eval_scalar(form, dev(pr.u, torch.float32), pr.mat_kind,
                               dev(pr.mat_a, torch.float32), dev(pr.mat_b, torch.float32))
        assert abs(v32.item() - ref) <= TOL32 * abs(ref)


def _dense_global(pr, K):
    """Reference global matrix: plain scatter of element matrices (test infrastructure)."""
    D, nb = pr.ncomp, pr.nb
    n = pr.n_nodes * D
    A = np.zeros((n, n))
    dofs = (pr.dof_conn[:, None, :] * D + np.arange(D)[None, :, None]).reshape(pr.n_elems, D * nb)
    for e in range(pr.n_elems):
        A[np.ix_(dofs[e], dofs[e])] += K[e]
    return A


@pytest.mark.parametrize("form,p", [(0, 1), (0, 2), (3, 2), (4, 1), (4, 2), (5, 2)])
def test_csr_assembly(form, p):
    """N2: CSR pattern + assembly of the GPU element matrices == dense scatter of the
    oracle's element matrices (pattern = every node pair sharing a cell)."""
    import scipy.sparse as sp
    m = fe()
    pr = fi.make_problem(form, p, (3, 2, 3), 6000 + form)
    mesh = gpu_mesh(pr)
    K = mesh.element_matrices(form, pr.mat_kind, dev(pr.mat_a), dev(pr.mat_b),
                              dev(pr.u) if form == fi.CONVECTIVE else None)
    csr = m.CSR(mesh, pr.ncomp)
    vals = csr.assemble(K)
    rp, ci = csr.arrays()
    assert rp[0] == 0 and rp[-1] == csr.nnz and np.all(np.diff(rp) > 0)
    for r in range(csr.n_rows):  # sorted, unique columns per row
        c = ci[rp[r]:rp[r + 1]]
        assert np.all(np.diff(c) > 0)
    A = sp.csr_matrix((vals.cpu().numpy(), ci, rp), shape=(csr.n_rows, csr.n_rows)).toarray()
    Aref = _dense_global(pr, oracle.problem_matrix(pr))
    assert rel(A, Aref) <= TOL64
    # structural: the pattern is exactly the set of node pairs sharing a cell
    S = _dense_global(pr, np.ones_like(K.cpu().numpy())) != 0
    pattern = sp.csr_matrix((np.ones(csr.nnz), ci, rp), shape=A.shape).toarray() != 0
    assert np.array_equal(pattern, S)


def test_csr_full_size_c2():
    """C2 at full size: nnz of the Q2 lattice pattern and row sums of the assembled
    diffusion matrix (= 0 by partition of unity, P7)."""
    m = fe()
    pr = fi.make_config("C2")
    mesh = gpu_mesh(pr)
    K = mesh.element_matrices(fi.DIFFUSION, pr.mat_kind, dev(pr.mat_a))
    csr = m.CSR(mesh, 1)
    vals = csr.assemble(K)
    rp, ci = csr.arrays()
    # exact count: a node couples to the lattice nodes of all cells containing it
    M = 2 * 64 + 1
    idx = np.arange(M)
    span = np.where(idx % 2 == 0, np.minimum(idx + 2, M - 1) - np.maximum(idx - 2, 0) + 1, 3)
    assert csr.nnz == int(span.sum()) ** 3
    import scipy.sparse as sp
    A = sp.csr_matrix((vals.cpu().numpy(), ci, rp), shape=(csr.n_rows, csr.n_rows))
    rs = np.abs(A @ np.ones(csr.n_rows))
    assert rs.max() <= 1e-12 * np.abs(vals.cpu().numpy()).max()


@pytest.mark.parametrize("form,p,shape", [(0, 2, (6, 5, 4)), (3, 2, (5, 5, 3)), (1, 1, (9, 8, 7)),
                                          (4, 2, (4, 3, 5)), (5, 2, (4, 4, 3)), (0, 4, (4, 3, 3))])
@pytest.mark.parametrize("ctas", [1, 3])
def test_pipelined_many_batches_per_cta(form, p, shape, ctas, fe_opts):
    """FEB200_MAX_CTAS caps the persistent grids so that each CTA runs many batches: every
    ring slot and mbarrier phase of the warp-specialised kernels wraps several times (plus a
    ragged last batch); matrices and residuals still match the oracle in full."""
    fe_opts(max_ctas=ctas)
    pr = fi.make_problem(form, p, shape, 6000 + 10 * form + p)
    mesh = gpu_mesh(pr)
    mat = (pr.mat_kind, dev(pr.mat_a), dev(pr.mat_b))
    if p <= 2:
        K = mesh.element_matrices(form, *mat, dev(pr.u) if form == fi.CONVECTIVE else None)
        assert rel(K.cpu().numpy(), oracle.problem_matrix(pr)) <= TOL64
    r_elem, r_glob = mesh.residual(form, dev(pr.u), *mat, want_elem=True)
    r_ref = oracle.problem_residual(pr)
    assert rel(r_elem.cpu().numpy(), r_ref) <= TOL64
    R_ref = oracle.assemble(r_ref, pr.dof_conn, pr.n_nodes, pr.ncomp)
    assert rel(r_glob.cpu().numpy().ravel(), R_ref) <= TOL64


@pytest.mark.parametrize("form,p", [(0, 1), (0, 2), (3, 2), (4, 2)])
def test_csr_gather_deterministic(form, p, fe_opts):
    """FEB200_CSR_IMPL=gather: atomic-free row-owner assembly == the atomic one, and two runs
    are bitwise identical (fixed summation order)."""
    pr = fi.make_problem(form, p, (4, 3, 5), 8000 + form)
    mesh = gpu_mesh(pr)
    K = mesh.element_matrices(form, pr.mat_kind, dev(pr.mat_a), dev(pr.mat_b),
                              dev(pr.u) if form == fi.CONVECTIVE else None)
    csr = fe().CSR(mesh, pr.ncomp)
    ref = csr.assemble(K)
    fe_opts(csr_impl="gather")
    a = csr.assemble(K)
    b = csr.assemble(K)
    assert torch.equal(a, b)
    assert rel(a.cpu().numpy(), ref.cpu().numpy()) <= 1e-14
    # element ranges accumulate
    c = torch.zeros_like(a)
    csr.assemble(K[:7], elem_begin=0, elem_end=7, values=c)
    csr.assemble(K[7:], elem_begin=7, elem_end=pr.n_elems, values=c)
    assert rel(c.cpu().numpy(), ref.cpu().numpy()) <= 1e-14


@pytest.mark.parametrize("form,p", [(0, 1), (0, 2), (1, 2), (3, 2), (3, 1)])
@pytest.mark.parametrize("ctas", [0, 2])
def test_matrix_residual_fused(form, p, ctas, fe_opts):
    """fe_eval_matrix_residual: K as fe_eval_element_matrices and r_e = K_e u_e (Alg. 1 for a
    bilinear form, pin P8) with the fused scatter, against the oracle's direct residual."""
    if ctas:
        fe_opts(max_ctas=ctas)
    pr = fi.make_problem(form, p, (6, 4, 5), 9000 + 10 * form + p)
    mesh = gpu_mesh(pr)
    K, r_elem, r_glob = mesh.matrix_residual(form, dev(pr.u), pr.mat_kind, dev(pr.mat_a),
                                             dev(pr.mat_b), want_elem=True)
    assert rel(K.cpu().numpy(), oracle.problem_matrix(pr)) <= TOL64
    r_ref = oracle.problem_residual(pr)
    assert rel(r_elem.cpu().numpy(), r_ref) <= TOL64
    R_ref = oracle.assemble(r_ref, pr.dof_conn, pr.n_nodes, pr.ncomp)
    assert rel(r_glob.cpu().numpy().ravel(), R_ref) <= TOL64
    # element ranges (ragged) accumulate into one global vector
    R = torch.zeros_like(r_glob)
    for a, b in [(0, 9), (9, 10), (10, pr.n_elems)]:
        mesh.matrix_residual(form, dev(pr.u), pr.mat_kind, dev(pr.mat_a), dev(pr.mat_b),
                             elem_begin=a, elem_end=b, r_global=R)
    assert rel(R.cpu().numpy().ravel(), R_ref) <= TOL64


def test_matrix_residual_unsupported():
    m = fe()
    pr = fi.make_problem(fi.ELASTICITY, 2, (2, 2, 2), 1)
    mesh = gpu_mesh(pr)
    with pytest.raises(m.FEError) as ei:
        mesh.matrix_residual(fi.ELASTICITY, dev(pr.u), pr.mat_kind, dev(pr.mat_a), dev(pr.mat_b))
    assert ei.value.status == m.FE_ERR_UNSUPPORTED


@pytest.mark.parametrize("form,p", [(0, 1), (0, 2), (1, 2), (3, 2), (4, 2), (5, 2), (2, 2), (3, 4)])
def test_single_cell(form, p):
    """One cell: every persistent pipeline runs a single, ragged batch (TMA store fallback for
    the odd byte count) and the residual kernels a single partial group."""
    pr = fi.make_problem(form, p, (1, 1, 1), 11000 + 10 * form + p)
    mesh = gpu_mesh(pr)
    mat = (pr.mat_kind, dev(pr.mat_a), dev(pr.mat_b))
    if p <= 2:
        K = mesh.element_matrices(form, *mat, dev(pr.u) if form == fi.CONVECTIVE else None)
        assert rel(K.cpu().numpy(), oracle.problem_matrix(pr)) <= TOL64
    r_elem, r_glob = mesh.residual(form, dev(pr.u), *mat, want_elem=True)
    r_ref = oracle.problem_residual(pr)
    assert rel(r_elem.cpu().numpy(), r_ref) <= TOL64
    assert rel(r_glob.cpu().numpy().ravel(), oracle.assemble(r_ref, pr.dof_conn, pr.n_nodes, pr.ncomp)) <= TOL64


@pytest.mark.parametrize("form,p", [(0, 2), (3, 2), (4, 2), (5, 2)])
def test_unaligned_outputs(form, p):
    """K and r_elem written through views that start one cell in (8-byte, not 16-byte aligned
    for odd element counts): the bulk-store paths must fall back, results unchanged."""
    pr = fi.make_problem(form, p, (3, 3, 3), 12000 + form)
    mesh = gpu_mesh(pr)
    mat = (pr.mat_kind, dev(pr.mat_a), dev(pr.mat_b))
    nd = pr.ncomp * pr.nb
    big = torch.full((pr.n_elems + 1, nd, nd), float("nan"), dtype=torch.float64, device="cuda")
    Kv = big[1:]
    mesh.element_matrices(form, *mat, dev(pr.u) if form == fi.CONVECTIVE else None, out=Kv)
    assert rel(Kv.cpu().numpy(), oracle.problem_matrix(pr)) <= TOL64
    assert torch.isnan(big[0]).all()          # nothing written before the view
    rbig = torch.full((pr.n_elems * nd + 1,), float("nan"), dtype=torch.float64, device="cuda")
    rv = rbig[1:].view(pr.n_elems, nd)
    mesh.residual(form, dev(pr.u), *mat, r_elem=rv, want_elem=True)
    assert rel(rv.cpu().numpy(), oracle.problem_residual(pr)) <= TOL64


# ---- N3: the remaining Tab. 2 forms --------------------------------------------

@pytest.mark.parametrize("p", [1, 2, 3])
@pytest.mark.parametrize("shape", SHAPES)
def test_weighted_dot_matrix(p, shape):
    """'ij,i,j' matrix mode: 9 blocks of weight detw M_ab, M non-symmetric."""
    pr = fi.make_problem(fi.WEIGHTED_DOT, p, shape, 13000 + p)
    mesh = gpu_mesh(pr)
    K = mesh.element_matrices(fi.WEIGHTED_DOT, pr.mat_kind, dev(pr.mat_a))
    Kref = oracle.problem_matrix(pr)
    assert rel(K.cpu().numpy(), Kref) <= TOL64
    # K is not symmetric (M is not), but each (a, b) block is symmetric in (k, l)
    nb = pr.nb
    Kn = K.cpu().numpy().reshape(pr.n_elems, 3, nb, 3, nb)
    assert np.abs(Kn - Kn.transpose(0, 1, 4, 3, 2)).max() <= 1e-14 * np.abs(Kn).max()


@pytest.mark.parametrize("form", [fi.WEIGHTED_DOT, fi.DIVERGENCE])
@pytest.mark.parametrize("p", [1, 2, 3, 4])
@pytest.mark.parametrize("impl", ["default", "dense"])
def test_n3_residual(form, p, impl, fe_opts):
    """Residual mode of 'ij,i,j' (f0 = M u) and 'i.i' (r_k = int dphi_k/dx_a), sum-factorised
    and dense kernels, ragged cell counts."""
    if impl == "dense":
        fe_opts(residual_impl="dense")
    pr = fi.make_problem(form, p, (5, 3, 4) if p <= 2 else (3, 2, 3), 14000 + 10 * form + p)
    r_ref = oracle.problem_residual(pr)
    R_ref = oracle.assemble(r_ref, pr.dof_conn, pr.n_nodes, pr.ncomp)
    mesh = gpu_mesh(pr)
    r_elem, r_glob = mesh.residual(form, dev(pr.u), pr.mat_kind, dev(pr.mat_a), dev(pr.mat_b),
                                   want_elem=True)
    torch.cuda.synchronize()
    assert rel(r_elem.cpu().numpy(), r_ref) <= TOL64
    assert rel_cell_max(r_elem.cpu().numpy(), r_ref) <= TOL64_CELL
    assert rel(r_glob.cpu().numpy().ravel(), R_ref) <= TOL64


@pytest.mark.parametrize("form", [fi.WEIGHTED_DOT, fi.DIVERGENCE])
@pytest.mark.parametrize("p", [1, 2, 4])
def test_n3_eval(form, p):
    """'eval' mode: int u.M.u and int div u."""
    pr = fi.make_problem(form, p, (5, 3, 4), 15000 + 10 * form + p)
    ref = oracle.problem_eval_scalar(pr)
    mesh = gpu_mesh(pr)
    v = mesh.eval_scalar(form, dev(pr.u), pr.mat_kind, dev(pr.mat_a), dev(pr.mat_b))
    assert abs(v.item() - ref) <= TOL64 * max(abs(ref), 1.0)


def test_divergence_has_no_matrix_mode():
    m = fe()
    pr = fi.make_problem(fi.DIVERGENCE, 2, (2, 2, 2), 3)
    mesh = gpu_mesh(pr)
    with pytest.raises(m.FEError) as ei:
        mesh.element_matrices(fi.DIVERGENCE)
    assert ei.value.status == m.FE_ERR_UNSUPPORTED


@pytest.mark.parametrize("kind", [fi.MAT_PER_ELEM, fi.MAT_PER_QP, fi.MAT_FULL_D])
@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_stress(kind, p):
    """Cauchy stress 'IK,s(k:l)->K' at every qp, every material kind, plus an
    element sub-range and an empty one."""
    pr = fi.make_problem(fi.ELASTICITY, p, (4, 3, 2), 16000 + 10 * p + kind, mat_kind=kind)
    ref = oracle.problem_stress(pr)
    mesh = gpu_mesh(pr)
    mat = (kind, dev(pr.mat_a), dev(pr.mat_b))
    sig = mesh.stress(dev(pr.u), *mat)
    assert sig.shape == ref.shape
    assert rel(sig.cpu().numpy(), ref) <= TOL64
    sub = mesh.stress(dev(pr.u), *mat, elem_begin=5, elem_end=17)
    assert rel(sub.cpu().numpy(), ref[5:17]) <= TOL64
    empty = mesh.stress(dev(pr.u), *mat, elem_begin=3, elem_end=3)
    assert empty.shape[0] == 0
    # 'eval' mode of the Cauchy stress: the per-cell integral
    ref_i = oracle.eval_stress_integral(p, p + 1, pr.coords, pr.conn, pr.dof_conn, pr.u, kind,
                                        pr.mat_a, pr.mat_b)
    si = mesh.stress_integral(dev(pr.u), *mat)
    assert rel(si.cpu().numpy(), ref_i) <= TOL64
    si_sub = mesh.stress_integral(dev(pr.u), *mat, elem_begin=5, elem_end=17)
    assert rel(si_sub.cpu().numpy(), ref_i[5:17]) <= TOL64
    assert mesh.stress_integral(dev(pr.u), *mat, elem_begin=3, elem_end=3).shape[0] == 0


# ---- N3: Stokes coupling pair -------------------------------------------------

def _mixed(pv, pp, shape, seed):
    mp = fi.make_mixed_problem(pv, pp, shape, seed)
    mesh = gpu_mesh(mp.vel)
    pf = fe().PressureField(mesh, pp, torch.from_numpy(mp.p_dof_conn), n_nodes=mp.n_p_nodes)
    return mp, mesh, pf


@pytest.mark.parametrize("pv,pp", [(1, 1), (2, 1), (2, 2), (3, 2), (4, 3)])
def test_stokes_coupling(pv, pp):
    """Matrix, residual (element + fused scatter) and eval modes of the Stokes coupling and
    its transpose vs the oracle, ragged cell counts and a sub-range."""
    shape = (5, 3, 4) if pv <= 2 else (3, 2, 3)
    mp, mesh, pf = _mixed(pv, pp, shape, 17000 + 10 * pv + pp)
    v = mp.vel
    args = (pv, pp, pv + 1, v.coords, v.conn)
    for tr in (False, True):
        ref = oracle.coupling_matrix(*args, transposed=tr)
        assert rel(pf.coupling_matrices(transposed=tr).cpu().numpy(), ref) <= TOL64
        sub = pf.coupling_matrices(transposed=tr, elem_begin=3, elem_end=11)
        assert rel(sub.cpu().numpy(), ref[3:11]) <= TOL64
    u, p = dev(v.u), dev(mp.pres)
    # Stokes coupling residual: input p, velocity-shaped output
    rv_ref = oracle.coupling_residual(*args, v.dof_conn, mp.p_dof_conn, p=mp.pres)
    re_, rg = pf.coupling_residual(p, want_elem=True)
    assert rel(re_.cpu().numpy(), rv_ref) <= TOL64
    assert rel(rg.cpu().numpy().ravel(), oracle.assemble(rv_ref, v.dof_conn, v.n_nodes, 3)) <= TOL64
    # transposed: input u, pressure-shaped output
    rq_ref = oracle.coupling_residual(*args, v.dof_conn, mp.p_dof_conn, u=v.u, transposed=True)
    re_, rg = pf.coupling_residual(u, transposed=True, want_elem=True)
    assert rel(re_.cpu().numpy(), rq_ref) <= TOL64
    assert rel(rg.cpu().numpy(), oracle.assemble(rq_ref, mp.p_dof_conn, mp.n_p_nodes, 1)) <= TOL64
    ev_ref = oracle.coupling_eval(*args, v.dof_conn, mp.p_dof_conn, v.u, mp.pres)
    ev = pf.coupling_eval(u, p).item()
    assert abs(ev - ev_ref) <= TOL64 * max(abs(ev_ref), 1.0)


def test_stokes_coupling_errors():
    m = fe()
    mp, mesh, pf = _mixed(4, 1, (2, 2, 1), 5)          # (4, 1) pair not built
    with pytest.raises(m.FEError) as ei:
        pf.coupling_matrices()
    assert ei.value.status == m.FE_ERR_UNSUPPORTED
    with pytest.raises(m.FEError) as ei:                # pressure order above the mesh order
        m.PressureField(gpu_mesh(fi.make_problem(fi.DIVERGENCE, 1, (2, 2, 1), 1)), 2,
                        torch.from_numpy(mp.p_dof_conn))
    assert ei.value.status == m.FE_ERR_INVALID_ARG
    bad = torch.from_numpy(mp.p_dof_conn).clone()
    bad[1, 2] = mp.n_p_nodes + 5                        # out of range
    with pytest.raises(m.FEError) as ei:
        m.PressureField(mesh, 1, bad, n_nodes=mp.n_p_nodes)
    assert ei.value.status == m.FE_ERR_INVALID_ARG


# ---- N4: element-kind grouping ------------------------------------------------

def test_group_cells():
    m = fe()
    rng = np.random.default_rng(5)
    kind = rng.integers(0, 5, size=1001).astype(np.int32)
    perm, offs = m.fe_group_cells(torch.from_numpy(kind).cuda(), 5)
    ref = np.argsort(kind, kind="stable")
    assert np.array_equal(perm.cpu().numpy(), ref)
    assert offs == [0] + list(np.cumsum(np.bincount(kind, minlength=5)))
    with pytest.raises(m.FEError):
        m.fe_group_cells(torch.tensor([0, 7, 1], dtype=torch.int32).cuda(), 5)
    p0, o0 = m.fe_group_cells(torch.zeros(0, dtype=torch.int32).cuda(), 3)
    assert p0.numel() == 0 and o0 == [0, 0, 0, 0]


def test_mixed_order_mesh():
    """A p-mixed mesh (orders 1-3 per cell, each order's nodes on its own lattice): grouped
    evaluation == the oracle on each group's cells; the global residual == the sum of the
    groups' oracle scatters."""
    m = fe()
    shape = (4, 3, 3)
    base = fi.make_problem(fi.DIFFUSION, 1, shape, 19000)
    E = base.n_elems
    rng = np.random.default_rng(19001)
    orders = rng.integers(1, 4, size=E).astype(np.int32)
    lat = {p: fi.lattice_dof_conn(*shape, p) for p in (1, 2, 3)}
    off = {1: 0, 2: lat[1][1], 3: lat[1][1] + lat[2][1]}
    n_nodes = off[3] + lat[3][1]
    rows = [lat[p][0][e] + off[p] for e, p in enumerate(orders)]
    dof_ptr = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    dof_idx = np.concatenate(rows).astype(np.int32)
    kap_rows = [rng.uniform(1, 2, size=(p + 1) ** 3) for p in orders]
    kap = torch.from_numpy(np.concatenate(kap_rows)).cuda()
    u = rng.uniform(-1, 1, size=(n_nodes, 1))
    mm = m.MixedMesh(base.coords, base.conn, orders, dof_ptr, dof_idx, n_nodes)
    mats = mm.group_material(kap, row_ptr=torch.from_numpy(dof_ptr).cuda())
    Ks = mm.element_matrices(fi.DIFFUSION, fi.MAT_PER_QP, mats)
    R = mm.residual(fi.DIFFUSION, dev(u), fi.MAT_PER_QP, mats).cpu().numpy().ravel()
    R_ref = np.zeros(n_nodes)
    perm = mm.perm.cpu().numpy()
    assert np.array_equal(perm, np.argsort(orders, kind="stable"))
    for (p, b, e, _, _), K in zip(mm.groups, Ks):
        cells = perm[b:e]
        assert np.all(orders[cells] == p)
        dc = np.stack([rows[c] for c in cells]).astype(np.int32)
        ka = np.stack([kap_rows[c] for c in cells])
        Kref = oracle.eval_matrix(fi.DIFFUSION, p, p + 1, base.coords, base.conn[cells], dc, 0, ka)
        assert rel(K.cpu().numpy(), Kref) <= TOL64
        r = oracle.eval_residual(fi.DIFFUSION, p, p + 1, base.coords, base.conn[cells], dc, u, 0, ka)
        R_ref = oracle.assemble(r, dc, n_nodes, 1, R_ref)
    assert rel(R, R_ref) <= TOL64


@pytest.mark.parametrize("ctas", [1, 3])
def test_n3_n4_many_batches_per_cta(ctas, fe_opts):
    """Grid caps force many batches per CTA through the N3 / N4 kernels (weighted-dot matrix,
    FULL_D pipelined matrix and its D prefetch, divergence residual, stress, Stokes coupling)."""
    fe_opts(max_ctas=ctas)
    pr = fi.make_problem(fi.WEIGHTED_DOT, 2, (5, 4, 3), 18000)
    mesh = gpu_mesh(pr)
    K = mesh.element_matrices(fi.WEIGHTED_DOT, pr.mat_kind, dev(pr.mat_a))
    assert rel(K.cpu().numpy(), oracle.problem_matrix(pr)) <= TOL64
    pe = fi.make_problem(fi.ELASTICITY, 2, (5, 4, 3), 18001, mat_kind=fi.MAT_FULL_D)
    me = gpu_mesh(pe)
    K = me.element_matrices(fi.ELASTICITY, fi.MAT_FULL_D, dev(pe.mat_a))
    assert rel(K.cpu().numpy(), oracle.problem_matrix(pe)) <= TOL64
    re_, _ = me.residual(fi.ELASTICITY, dev(pe.u), fi.MAT_FULL_D, dev(pe.mat_a), want_elem=True)
    assert rel(re_.cpu().numpy(), oracle.problem_residual(pe)) <= TOL64
    sig = me.stress(dev(pe.u), fi.MAT_FULL_D, dev(pe.mat_a))
    assert rel(sig.cpu().numpy(), oracle.problem_stress(pe)) <= TOL64
    pd = fi.make_problem(fi.DIVERGENCE, 2, (5, 4, 3), 18002)
    md = gpu_mesh(pd)
    re_, _ = md.residual(fi.DIVERGENCE, dev(pd.u), want_elem=True)
    assert rel(re_.cpu().numpy(), oracle.problem_residual(pd)) <= TOL64
    mp, mesh2, pf = _mixed(2, 1, (5, 4, 3), 18003)
    v = mp.vel
    ref = oracle.coupling_matrix(2, 1, 3, v.coords, v.conn)
    assert rel(pf.coupling_matrices().cpu().numpy(), ref) <= TOL64


def test_full_d_config_sampled():
    """C3d (N4 bench workload: C3 with D[E][27][6][6]) at full size, in bench.py's launch
    configuration: sampled element matrices and residuals vs the oracle cell by cell."""
    import bench
    pr = bench.build_problem("C3d")
    mesh = gpu_mesh(pr)
    a = dev(pr.mat_a)
    K = mesh.element_matrices(fi.ELASTICITY, fi.MAT_FULL_D, a)
    re_, _ = mesh.residual(fi.ELASTICITY, dev(pr.u), fi.MAT_FULL_D, a, want_elem=True)
    idx = np.random.default_rng(7).choice(pr.n_elems, 24, replace=False)
    sub = _sample_subproblem(pr, idx)
    assert rel(K[torch.from_numpy(idx).cuda()].cpu().numpy(), oracle.problem_matrix(sub)) <= TOL64
    assert rel(re_[torch.from_numpy(idx).cuda()].cpu().numpy(), oracle.problem_residual(sub)) <= TOL64


@pytest.mark.parametrize("form,p,world", [(fi.DIFFUSION, 2, 2), (fi.DIFFUSION, 1, 4),
                                          (fi.ELASTICITY, 2, 2), (fi.MASS_DIFFUSION, 2, 4)])
def test_csr_row_ownership_ghost_layer(form, p, world):
    """Multi-GPU CSR with row ownership: each rank evaluates its z-slab plus the
    first cell layer of the rank above and assembles the CSR of that extended mesh; its owned
    block rows (global column ids) equal the single-GPU global matrix's rows exactly in pattern
    and to rounding in value, and the ranks' owned rows tile the global rows."""
    from paper_2107_04121_b200 import slabs
    m = fe()
    shape = (3, 2, 4)
    pr = fi.make_problem(form, p, shape, 22000 + 10 * form + p)
    D = pr.ncomp
    mat = lambda a, e0, e1: None if a is None else dev(a[e0:e1])
    mesh = gpu_mesh(pr)
    Kg = mesh.element_matrices(form, pr.mat_kind, dev(pr.mat_a), dev(pr.mat_b))
    cg = m.CSR(mesh, D)
    vg = cg.assemble(Kg).cpu().numpy()
    rpg, colg = cg.arrays()
    covered = 0
    for rank in range(world):
        gs = slabs.ghost_slab_of(shape, p, world, rank)
        lc, lconn, ldc = slabs.local_arrays(gs, pr.coords, pr.conn, pr.dof_conn)
        lm = m.Mesh(torch.from_numpy(lc), torch.from_numpy(lconn), p, dof_conn=torch.from_numpy(ldc),
                    n_nodes=gs.n_nodes)
        K = lm.element_matrices(form, pr.mat_kind, mat(pr.mat_a, gs.elem_begin, gs.elem_end),
                                mat(pr.mat_b, gs.elem_begin, gs.elem_end))
        c = m.CSR(lm, D)
        v = c.assemble(K).cpu().numpy()
        rp, col = c.arrays()
        g0, rpo, colo, vo = slabs.owned_block_rows(gs, rp, col, v, D)
        n = len(rpo) - 1
        a, b = rpg[g0], rpg[g0 + n]
        assert g0 == covered
        assert np.array_equal(rpo, rpg[g0:g0 + n + 1] - a)
        assert np.array_equal(colo, colg[a:b])
        assert rel(vo, vg[a:b]) <= TOL64
        covered += n
    assert covered == pr.n_nodes * D


@pytest.mark.parametrize("form", [fi.DIFFUSION, fi.MASS, fi.MASS_DIFFUSION])
def test_matrix_q4(form):
    """Matrix mode at p = 4 (single-stage SF kernel, one cell per CTA iteration, single K
    staging buffer of 125 KB), ragged cell count and a sub-range."""
    pr = fi.make_problem(form, 4, (3, 2, 2), 23000 + form)
    mesh = gpu_mesh(pr)
    mat = (pr.mat_kind, dev(pr.mat_a), dev(pr.mat_b))
    K = mesh.element_matrices(form, *mat)
    Kref = oracle.problem_matrix(pr)
    assert rel(K.cpu().numpy(), Kref) <= TOL64
    Ks = mesh.element_matrices(form, *mat, elem_begin=5, elem_end=12)
    assert rel(Ks.cpu().numpy(), Kref[5:12]) <= TOL64


@pytest.mark.parametrize("form,p", [(fi.MASS_DIFFUSION, 4), (fi.ELASTICITY, 2), (fi.DIFFUSION, 2),
                                    (fi.WEIGHTED_DOT, 2), (fi.MASS_DIFFUSION, 3)])
@pytest.mark.parametrize("ctas", [0, 2])
def test_residual_misaligned_inputs(form, p, ctas, fe_opts):
    """Material arrays passed as views that start 8 B past a 16-B boundary: the residual
    kernels' block fetches take the enclosing aligned range and read at the offset (and fall
    back to plain copies at the array end); results unchanged."""
    if ctas:
        fe_opts(max_ctas=ctas)
    pr = fi.make_problem(form, p, (5, 3, 3) if p <= 2 else (3, 2, 3), 24000 + 10 * form + p,
                         mat_kind=fi.MAT_PER_QP if form == fi.ELASTICITY else None)
    mesh = gpu_mesh(pr)

    def shifted(a):
        if a is None:
            return None
        flat = np.ascontiguousarray(a).ravel()
        big = torch.zeros(flat.size + 1, dtype=torch.float64, device="cuda")
        big[1:] = torch.from_numpy(flat).cuda()
        v = big[1:].view(a.shape)
        assert v.data_ptr() % 16 == 8
        return v

    r_elem, r_glob = mesh.residual(form, dev(pr.u), pr.mat_kind, shifted(pr.mat_a), shifted(pr.mat_b),
                                   want_elem=True)
    r_ref = oracle.problem_residual(pr)
    assert rel(r_elem.cpu().numpy(), r_ref) <= TOL64
    assert rel(r_glob.cpu().numpy().ravel(), oracle.assemble(r_ref, pr.dof_conn, pr.n_nodes, pr.ncomp)) <= TOL64


# ---- general D read as given (reading 23) -----------------------------------------

def _nonsym_D(pr, seed, scale=0.3):
    """The problem's SPD D plus a random skew part: a non-symmetric Voigt matrix per qp."""
    rng = np.random.default_rng(seed)
    S = rng.uniform(-1, 1, size=pr.mat_a.shape)
    return pr.mat_a + scale * (S - np.swapaxes(S, -1, -2))


@pytest.mark.parametrize("p", [1, 2])
@pytest.mark.parametrize("shape", SHAPES)
def test_full_d_nonsymmetric(p, shape, fe_opts):
    """A non-symmetric D[E][n_q][6][6] is read as given by matrix and residual mode at p = 1
    and 2 (at p = 2 the device-side symmetry check routes the matrix to the general 9-block
    kernel): K == oracle, K not symmetric, and K_e u_e == r_e (P8).  With many batches per
    CTA, and a symmetric-to-rounding D keeps the pipelined kernel's result within 1e-12."""
    pr = fi.make_problem(fi.ELASTICITY, p, shape, 17000 + p, mat_kind=fi.MAT_FULL_D)
    D = _nonsym_D(pr, 5 + p)
    pr_ns = fi.Problem(pr.name, pr.form, pr.p, pr.q1d, pr.shape, pr.coords, pr.conn, pr.dof_conn,
                       pr.n_nodes, pr.mat_kind, D, None, pr.u)
    Kref = oracle.problem_matrix(pr_ns)
    rref = oracle.problem_residual(pr_ns)
    assert rel(Kref, Kref.transpose(0, 2, 1)) > 1e-3
    mesh = gpu_mesh(pr)
    for ctas in (0, 2):
        fe_opts(max_ctas=ctas)
        K = mesh.element_matrices(fi.ELASTICITY, fi.MAT_FULL_D, dev(D), None).cpu().numpy()
        assert rel(K, Kref) <= TOL64
        re_, _ = mesh.residual(fi.ELASTICITY, dev(pr.u), fi.MAT_FULL_D, dev(D), None,
                               want_elem=True, want_global=False)
        re_ = re_.cpu().numpy()
        assert rel(re_, rref) <= TOL64
        ue = pr.u[pr.dof_conn].transpose(0, 2, 1).reshape(pr.n_elems, -1)
        assert rel(np.einsum("eij,ej->ei", K, ue), re_) <= 1e-12
    # one non-symmetric qp block among symmetric ones still routes the whole call
    D1 = pr.mat_a.copy()
    D1[-1, -1, 0, 5] += 0.5
    pr1 = fi.Problem(pr.name, pr.form, pr.p, pr.q1d, pr.shape, pr.coords, pr.conn, pr.dof_conn,
                     pr.n_nodes, pr.mat_kind, D1, None, pr.u)
    K1 = mesh.element_matrices(fi.ELASTICITY, fi.MAT_FULL_D, dev(D1), None).cpu().numpy()
    assert rel(K1, oracle.problem_matrix(pr1)) <= TOL64
    # a D whose transpose differs in the last bits only: the pipelined kernel (upper triangle)
    # stays within the parity tolerance
    Dr = pr.mat_a * (1 + 2.2e-16 * np.random.default_rng(3).integers(-2, 3, pr.mat_a.shape))
    prr = fi.Problem(pr.name, pr.form, pr.p, pr.q1d, pr.shape, pr.coords, pr.conn, pr.dof_conn,
                     pr.n_nodes, pr.mat_kind, Dr, None, pr.u)
    Kr = mesh.element_matrices(fi.ELASTICITY, fi.MAT_FULL_D, dev(Dr), None).cpu().numpy()
    assert rel(Kr, oracle.problem_matrix(prr)) <= TOL64


def test_concurrent_mesh_creation():
    """Two host threads create meshes of different orders at the same time (the per-order
    __constant__ tables are uploaded from per-call stack buffers) and evaluate them on their
    own streams; every result equals the oracle."""
    import threading
    probs = [fi.make_problem(fi.DIFFUSION, p, (4, 3, 3), 18000 + p) for p in (1, 2, 1, 2)]
    refs = [oracle.problem_matrix(pr) for pr in probs]
    errs, out = [], [None] * len(probs)

    def work(i):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for _ in range(5):
                    m = gpu_mesh(probs[i])
                    K = m.element_matrices(fi.DIFFUSION, 0, dev(probs[i].mat_a), None)
                    st.synchronize()
                    out[i] = K.cpu().numpy()
                    m.close()
        except Exception as ex:  # pragma: no cover - reported below
            errs.append(ex)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(len(probs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for K, Kr in zip(out, refs):
        assert rel(K, Kr) <= TOL64


def test_stream_ordered_destroy():
    """fe_destroy_mesh / fe_destroy_csr release on the caller's stream without a device
    synchronisation: work queued before on that stream still sees valid memory, and a
    mesh created right after works."""
    pr = fi.make_problem(fi.DIFFUSION, 2, (6, 5, 4), 18100)
    ref = oracle.problem_assembled_residual(pr)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3):
            m = gpu_mesh(pr)
            csr = fe().CSR(m, 1)
            _, rg = m.residual(fi.DIFFUSION, dev(pr.u), 0, dev(pr.mat_a), None)
            csr.close()
            m.close()          # queued behind the residual on st
            st.synchronize()
            assert rel(rg.cpu().numpy().ravel(), ref) <= TOL64


# ---- FE_F32 element matrices (scalar forms, p = 1, 2; reading 15) -------------------------

@pytest.mark.parametrize("form,p", [(fi.DIFFUSION, 1), (fi.DIFFUSION, 2), (fi.MASS, 2),
                                    (fi.MASS_DIFFUSION, 1), (fi.MASS_DIFFUSION, 2)])
@pytest.mark.parametrize("shape", SHAPES)
def test_matrix_fp32(form, p, shape, fe_opts):
    """fp32 coefficients -> fp32 K within 1e-5 of the fp64 oracle (also with many batches per
    CTA and an element sub-range); other forms / orders are FE_ERR_UNSUPPORTED."""
    pr = fi.make_problem(form, p, shape, 19000 + 10 * form + p)
    Kref = oracle.problem_matrix(pr)
    mesh = gpu_mesh(pr)
    for ctas in (0, 2):
        fe_opts(max_ctas=ctas)
        K = mesh.element_matrices(form, pr.mat_kind, dev(pr.mat_a, torch.float32),
                                  dev(pr.mat_b, torch.float32))
        assert K.dtype == torch.float32
        assert rel(K.cpu().numpy(), Kref) <= TOL32
    Ks = mesh.element_matrices(form, pr.mat_kind, dev(pr.mat_a, torch.float32),
                               dev(pr.mat_b, torch.float32), elem_begin=3, elem_end=pr.n_elems - 2)
    assert rel(Ks.cpu().numpy(), Kref[3:pr.n_elems - 2]) <= TOL32


def test_matrix_fp32_unsupported():
    m = fe()
    pr = fi.make_problem(fi.ELASTICITY, 2, (2, 2, 2), 19100)
    mesh = gpu_mesh(pr)
    with pytest.raises(m.FEError) as ei:
        mesh.element_matrices(fi.ELASTICITY, pr.mat_kind, dev(pr.mat_a, torch.float32),
                              dev(pr.mat_b, torch.float32))
    assert ei.value.status == m.FE_ERR_UNSUPPORTED

"""Maximum sizes: element-matrix outputs with more than 2^31 and 2^32 values.

The BASELINE configs stay below 2^31 values of K (C5t: 1.72e9), so a 32-bit flat index anywhere
in a matrix kernel's addressing would go unnoticed there.  Here K has 2.18e9 values (scalar Q2,
144^3 cells, 17 GB) and 4.47e9 values (elasticity Q2, 88^3 cells, 36 GB); the cells next to the
2^31- and 2^32-value boundaries, the first and last cells and a seeded sample are compared with
the oracle one by one, and a NaN-sentinel guard band behind K stays intact.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import fe_inputs as fi
import oracle
from test_gpu_parity import TOL64, TOL64_CELL, _sample_subproblem, dev, gpu_mesh, rel, rel_cell_max

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("form,n", [(fi.DIFFUSION, 144), (fi.ELASTICITY, 88)])
def test_matrix_beyond_32bit_indices(form, n):
    free, _ = torch.cuda.mem_get_info()
    pr = fi.make_problem(form, 2, (n, n, n), 51000 + form)
    E, nd = pr.n_elems, pr.ncomp * pr.nb
    vals = E * nd * nd
    assert vals > 2 ** 31
    if free < vals * 8 + (8 << 30):
        pytest.skip("not enough free device memory")
    mesh = gpu_mesh(pr)
    guard = 4096
    buf = torch.empty(vals + guard, dtype=torch.float64, device="cuda")
    buf[vals:] = float("nan")
    K = buf[:vals].view(E, nd, nd)
    mesh.element_matrices(form, pr.mat_kind, dev(pr.mat_a), dev(pr.mat_b), None, out=K)
    torch.cuda.synchronize()
    assert bool(torch.isnan(buf[vals:]).all())
    rng = np.random.default_rng(11)
    edges = [b // (nd * nd) + d for b in (2 ** 31, 2 ** 32) for d in (-1, 0, 1)]
    idx = np.unique(np.concatenate([[0, 1, E - 2, E - 1], [e for e in edges if 0 <= e < E],
                                    rng.choice(E, size=40, replace=False)]))
    Kref = oracle.problem_matrix(_sample_subproblem(pr, idx))
    Ks = K[torch.from_numpy(idx).cuda()].cpu().numpy()
    assert np.isfinite(Ks).all()
    assert rel(Ks, Kref) <= TOL64
    assert rel_cell_max(Ks, Kref) <= TOL64_CELL
    # every cell was written: a symmetric form's K_e has a positive diagonal
    diag = torch.diagonal(K, dim1=1, dim2=2)
    assert bool((diag > 0).all())
    del K, buf, diag
    torch.cuda.empty_cache()

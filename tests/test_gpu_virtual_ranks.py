"""Virtual ranks on one GPU: P z-slab meshes on the same
device exchange their interface planes by device copies (slabs.VirtualWorld) through the
multi-rank code path -- residual_overlapped's comm-stream exchange with the boundary-first
order (one host thread per rank), and the whole world's step captured into one CUDA graph
(slabs.virtual_world_step + StepGraph).  The gathered slabs must equal the oracle's
assembled global vector; the two copies of every shared plane must be bitwise equal.
No kernel waits on another rank's kernel: only stream / event order."""
from __future__ import annotations

import threading

import numpy as np
import pytest
import torch

import fe_inputs as fi
import oracle

pytestmark = pytest.mark.gpu
TOL64 = 1e-12

CASES = {"md_q4": (fi.MASS_DIFFUSION, 4, (3, 2, 8)), "diff_q2": (fi.DIFFUSION, 2, (4, 3, 8)),
         "elas_q2": (fi.ELASTICITY, 2, (3, 3, 4)), "conv_q2": (fi.CONVECTIVE, 2, (2, 3, 4))}


def _setup(case, P, seed=777, boundary_first=False):
    import paper_2107_04121_b200 as fe
    from paper_2107_04121_b200 import slabs
    form, p, shape = CASES[case]
    pr = fi.make_problem(form, p, shape, seed)
    ref = oracle.problem_assembled_residual(pr).reshape(pr.n_nodes, pr.ncomp)
    sls = [slabs.slab_of(shape, p, P, g) for g in range(P)]
    ranks = []
    for sl in sls:
        order = slabs.boundary_first_order(sl, shape) if boundary_first else None
        lc, lconn, ldc = slabs.local_arrays(sl, pr.coords, pr.conn, pr.dof_conn, order)
        e0, e1 = sl.elem_begin, sl.elem_end
        cells = np.arange(e0, e1) if order is None else e0 + order
        mesh = fe.Mesh(torch.from_numpy(lc), torch.from_numpy(lconn), p, p + 1,
                       dof_conn=torch.from_numpy(ldc), n_nodes=sl.n_nodes)
        cut = (lambda a: None if a is None else torch.from_numpy(
            np.ascontiguousarray(a[cells])).cuda())
        u = torch.from_numpy(np.ascontiguousarray(pr.u[sl.node_begin:sl.node_end])).cuda()
        r = torch.zeros((sl.n_nodes, pr.ncomp), dtype=torch.float64, device="cuda")
        ranks.append(dict(sl=sl, mesh=mesh, ma=cut(pr.mat_a), mb=cut(pr.mat_b), u=u, r=r,
                          main=torch.cuda.Stream(), comm=torch.cuda.Stream()))
    return fe, slabs, pr, ref, sls, ranks


def _evaluator(fe, pr, rk):
    def evaluate(a, b):
        fe.fe_eval_residual(rk["mesh"].handle, pr.form, fe.F64, pr.mat_kind, rk["ma"], rk["mb"],
                            rk["u"], a, b, None, rk["r"], torch.cuda.current_stream())
    return evaluate


def _check(pr, ref, ranks):
    torch.cuda.synchronize()
    scale = np.linalg.norm(ref)
    for g, rk in enumerate(ranks):
        sl, R = rk["sl"], rk["r"].cpu().numpy()
        assert np.linalg.norm(R - ref[sl.node_begin:sl.node_end]) <= TOL64 * scale, g
        if g + 1 < len(ranks):
            Rn = ranks[g + 1]["r"].cpu().numpy()
            assert np.array_equal(R[-sl.plane:], Rn[:sl.plane])  # both copies bitwise equal


@pytest.mark.parametrize("case,P,bf", [("md_q4", 2, False), ("md_q4", 4, False),
                                       ("md_q4", 8, False), ("diff_q2", 4, False),
                                       ("elas_q2", 2, False), ("conv_q2", 4, False),
                                       ("md_q4", 4, True), ("diff_q2", 2, True)])
def test_virtual_ranks_threaded(case, P, bf):
    """One host thread per virtual rank runs slabs.residual_overlapped (boundary layers,
    exchange on the comm stream, interior layers) with the device-copy exchange; two steps
    (re-zeroing and buffer reuse).  bf: cells in boundary_first_order (boundary layers in
    one launch)."""
    fe, slabs, pr, ref, sls, ranks = _setup(case, P, boundary_first=bf)
    world = slabs.VirtualWorld(sls, pr.ncomp, "cuda")
    errs = []

    def work(g):
        rk = rk_ = ranks[g]
        try:
            ev = torch.cuda.Event()
            with torch.cuda.stream(rk["main"]):
                for _ in range(2):
                    rk["r"].zero_()
                    slabs.residual_overlapped(_evaluator(fe, pr, rk_), rk["r"], rk["sl"],
                                              CASES[case][2], rk["comm"],
                                              exchange=world.exchange_for(g), events=ev,
                                              boundary_first=bf)
                    rk["main"].synchronize()
                    world.barrier.wait()  # nobody zeroes before everybody finished the step
        except Exception as ex:  # pragma: no cover - reported below
            errs.append(ex)
            world.barrier.abort()

    ts = [threading.Thread(target=work, args=(g,)) for g in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    _check(pr, ref, ranks)


@pytest.mark.parametrize("case,P", [("md_q4", 4), ("diff_q2", 2), ("elas_q2", 2)])
def test_virtual_ranks_graph(case, P):
    """The whole virtual world's step (every rank: zero, boundary, sends, interior, adds)
    captured into ONE CUDA graph and replayed three times."""
    fe, slabs, pr, ref, sls, ranks = _setup(case, P)
    world = slabs.VirtualWorld(sls, pr.ncomp, "cuda")
    evs = [_evaluator(fe, pr, rk) for rk in ranks]
    rs = [rk["r"] for rk in ranks]
    mains = [rk["main"] for rk in ranks]
    comms = [rk["comm"] for rk in ranks]
    bev = [torch.cuda.Event() for _ in ranks]

    def step():
        cur = torch.cuda.current_stream()
        for s in mains + comms:
            s.wait_stream(cur)
        slabs.virtual_world_step(sls, evs, rs, mains, comms, world, CASES[case][2], bev)
        for s in mains:
            cur.wait_stream(s)

    n0 = fe.fe_launch_count()
    g = slabs.StepGraph(step, torch.device("cuda"))
    n_capture = fe.fe_launch_count() - n0
    for r in rs:
        r.fill_(123.0)   # the replays must zero them
    for _ in range(3):
        g.replay()
    assert fe.fe_launch_count() - n0 == n_capture   # replays launch nothing from the host
    _check(pr, ref, ranks)

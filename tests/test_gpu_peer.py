"""Fused residual + interface exchange over peer memory (fe_eval_residual_peer).

Only one GPU is available here, so the two-rank test runs two processes on the SAME device:
each maps the other's IPC residual vector and the residual kernels add the interface planes
straight into it.  The ranks' kernels never wait on one another (host barriers order the
steps), so this exercises exactly the multi-GPU code path minus NVLink itself.
"""
import os
import socket

import numpy as np
import pytest
import torch

import fe_inputs as fi
import oracle

pytestmark = pytest.mark.gpu
TOL64 = 1e-12


def rel(a, b):
    return np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, form, p, shape, port, out_dir):
    import torch.distributed as dist
    import paper_2107_04121_b200 as fe
    from paper_2107_04121_b200 import slabs
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    pr = fi.make_problem(form, p, shape, 21000 + 10 * form + p)
    sl = slabs.slab_of(shape, p, world, rank)
    lc, lconn, ldc = slabs.local_arrays(sl, pr.coords, pr.conn, pr.dof_conn)
    mesh = fe.Mesh(torch.from_numpy(lc), torch.from_numpy(lconn), p, dof_conn=torch.from_numpy(ldc),
                   n_nodes=sl.n_nodes)
    e0, e1 = sl.elem_begin, sl.elem_end
    dv = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a[e0:e1])).cuda()
    u = torch.from_numpy(np.ascontiguousarray(pr.u[sl.node_begin:sl.node_end])).cuda()
    px = slabs.PeerExchange(sl, shape, p, pr.ncomp, "cuda:0")

    def barrier():
        torch.cuda.synchronize()
        dist.barrier()

    def evaluate(windows):
        fe.fe_eval_residual_peer(mesh.handle, form, pr.mat_kind, dv(pr.mat_a), dv(pr.mat_b), u, 0,
                                 sl.n_elems, None, px.r, windows)

    for _ in range(2):  # the second step checks that re-zeroing and the barriers order the ranks
        r = px.residual(evaluate, barrier)
    np.save(os.path.join(out_dir, f"r{rank}.npy"), r.cpu().numpy())
    barrier()
    px.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("form,p", [(fi.DIFFUSION, 2), (fi.ELASTICITY, 2), (fi.MASS_DIFFUSION, 4),
                                    (fi.DIFFUSION, 1), (fi.CONVECTIVE, 2)])
def test_peer_exchange_two_ranks(form, p, tmp_path):
    shape = (3, 4, 4)
    world = 2
    torch.multiprocessing.spawn(_worker, args=(world, form, p, shape, _free_port(), str(tmp_path)),
                                nprocs=world, join=True)
    pr = fi.make_problem(form, p, shape, 21000 + 10 * form + p)
    R = oracle.assemble(oracle.problem_residual(pr), pr.dof_conn, pr.n_nodes, pr.ncomp)
    R = R.reshape(pr.n_nodes, pr.ncomp)
    from paper_2107_04121_b200 import slabs
    for rank in range(world):
        sl = slabs.slab_of(shape, p, world, rank)
        r = np.load(os.path.join(tmp_path, f"r{rank}.npy"))
        # the rank's whole slice, both interface planes included, equals the global vector
        assert rel(r, R[sl.node_begin:sl.node_end]) <= TOL64


def test_peer_window_single_process():
    """Window into a plain local buffer: it receives exactly the window nodes' contributions
    (the same values the local vector gets), at the requested offset."""
    import paper_2107_04121_b200 as fe
    pr = fi.make_problem(fi.DIFFUSION, 2, (3, 3, 2), 21500)
    mesh = fe.Mesh(torch.from_numpy(pr.coords), torch.from_numpy(pr.conn), 2,
                   dof_conn=torch.from_numpy(pr.dof_conn), n_nodes=pr.n_nodes)
    u = torch.from_numpy(pr.u).cuda()
    a = torch.from_numpy(pr.mat_a).cuda()
    r = torch.zeros((pr.n_nodes, 1), dtype=torch.float64, device="cuda")
    side = torch.zeros((100 + 50, 1), dtype=torch.float64, device="cuda")
    fe.fe_eval_residual_peer(mesh.handle, fi.DIFFUSION, fi.MAT_PER_QP, a, None, u, 0, pr.n_elems,
                             None, r, [(10, 60, side.data_ptr(), 100)])
    torch.cuda.synchronize()
    assert rel(side[100:150].cpu().numpy(), r[10:60].cpu().numpy()) <= TOL64
    assert torch.count_nonzero(side[:100]) == 0
    R = oracle.assemble(oracle.problem_residual(pr), pr.dof_conn, pr.n_nodes, 1)
    assert rel(r.cpu().numpy().ravel(), R) <= TOL64
    m = fe
    with pytest.raises(m.FEError):
        fe.fe_eval_residual_peer(mesh.handle, fi.DIFFUSION, fi.MAT_PER_QP, a, None, u, 0,
                                 pr.n_elems, None, r, [(10, 5, side.data_ptr(), 0)])

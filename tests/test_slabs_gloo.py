"""Multi-rank z-slab path on CPU (gloo, world_size 2 and 4): partition bookkeeping and the
interface-plane summation of paper_2107_04121_b200.slabs.

The per-rank element residuals come from the oracle here (CPU test infrastructure stands in
for the kernel); what is tested is the product's plumbing: local renumbering, the contiguous
node slices and the NCCL/gloo exchange of the shared planes.  After the exchange every rank's
slice must equal the single-process assembled vector restricted to its node range.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import fe_inputs as fi
import oracle
from paper_2107_04121_b200 import slabs


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = {"diff_q2": (fi.DIFFUSION, 2, (3, 2, 4)), "elas_q2": (fi.ELASTICITY, 2, (2, 3, 4)),
         "conv_q1": (fi.CONVECTIVE, 1, (3, 3, 4)), "md_q4": (fi.MASS_DIFFUSION, 4, (2, 2, 4)),
         "diff_q2_deep": (fi.DIFFUSION, 2, (3, 2, 8))}


def _worker_overlap(rank, world, port, case, out):
    """Boundary layers, exchange, then interior (the order of residual_overlapped): the
    interior cells must not touch the interface planes, or the sums would be incomplete."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    form, p, shape = CASES[case]
    pr = fi.make_problem(form, p, shape, 4242)
    sl = slabs.slab_of(shape, p, world, rank)
    lc, lconn, ldc = slabs.local_arrays(sl, pr.coords, pr.conn, pr.dof_conn)
    e0, e1 = sl.elem_begin, sl.elem_end
    ma = None if pr.mat_a is None else pr.mat_a[e0:e1]
    mb = None if pr.mat_b is None else pr.mat_b[e0:e1]
    u_loc = pr.u[sl.node_begin:sl.node_end]
    R = torch.zeros((sl.n_nodes, pr.ncomp), dtype=torch.float64)

    def evaluate(a, b):
        r_el = oracle.eval_residual(form, p, p + 1, lc, lconn, ldc, u_loc, pr.mat_kind, ma, mb, a, b)
        Rn = oracle.assemble(r_el, ldc[a:b], sl.n_nodes, pr.ncomp)
        R.add_(torch.from_numpy(Rn.reshape(sl.n_nodes, pr.ncomp)))

    slabs.residual_overlapped(evaluate, R, sl, shape)
    out[rank] = (sl.node_begin, sl.node_end, R.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


def test_boundary_first_order_matches_global():
    world = 2
    form, p, shape = CASES["diff_q2_deep"]
    pr = fi.make_problem(form, p, shape, 4242)
    Rg = oracle.problem_assembled_residual(pr).reshape(pr.n_nodes, 1)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_overlap, args=(world, _free_port(), "diff_q2_deep", out), nprocs=world,
             join=True)
    for rank in range(world):
        a, b, R = out[rank]
        np.testing.assert_allclose(R, Rg[a:b], rtol=1e-13, atol=1e-15 * np.abs(Rg).max())


def _worker(rank, world, port, case, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    form, p, shape = CASES[case]
    pr = fi.make_problem(form, p, shape, 4242)
    sl = slabs.slab_of(shape, p, world, rank)
    lc, lconn, ldc = slabs.local_arrays(sl, pr.coords, pr.conn, pr.dof_conn)
    e0, e1 = sl.elem_begin, sl.elem_end
    ma = None if pr.mat_a is None else pr.mat_a[e0:e1]
    mb = None if pr.mat_b is None else pr.mat_b[e0:e1]
    u_loc = pr.u[sl.node_begin:sl.node_end]
    r_el = oracle.eval_residual(form, p, p + 1, lc, lconn, ldc, u_loc, pr.mat_kind, ma, mb)
    R = oracle.assemble(r_el, ldc, sl.n_nodes, pr.ncomp).reshape(sl.n_nodes, pr.ncomp)
    Rt = torch.from_numpy(R.copy())
    slabs.exchange_planes(Rt, sl)
    out[rank] = (sl.node_begin, sl.node_end, Rt.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case", ["conv_q1", "diff_q2", "elas_q2", "md_q4"])
def test_slab_exchange_matches_global(world, case):
    form, p, shape = CASES[case]
    pr = fi.make_problem(form, p, shape, 4242)
    Rg = oracle.problem_assembled_residual(pr).reshape(pr.n_nodes, pr.ncomp)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), case, out), nprocs=world, join=True)
    covered = np.zeros(pr.n_nodes, dtype=bool)
    for rank in range(world):
        a, b, R = out[rank]
        np.testing.assert_allclose(R, Rg[a:b], rtol=1e-13, atol=1e-15 * np.abs(Rg).max())
        covered[a:b] = True
    assert covered.all()
    # shared planes are bitwise equal on both neighbours
    for rank in range(world - 1):
        a0, b0, R0 = out[rank]
        a1, b1, R1 = out[rank + 1]
        assert b0 - a1 == slabs.slab_of(shape, p, world, rank).plane
        assert np.array_equal(R0[a1 - a0:], R1[: b0 - a1])


def test_slab_bookkeeping():
    shape, p = (4, 3, 8), 2
    pr = fi.make_problem(fi.DIFFUSION, p, shape, 1)
    for world in (1, 2, 4, 8):
        elems = []
        for r in range(world):
            sl = slabs.slab_of(shape, p, world, r)
            lc, lconn, ldc = slabs.local_arrays(sl, pr.coords, pr.conn, pr.dof_conn)
            np.testing.assert_array_equal(lc[lconn], pr.coords[pr.conn[sl.elem_begin:sl.elem_end]])
            np.testing.assert_array_equal(ldc + sl.node_begin, pr.dof_conn[sl.elem_begin:sl.elem_end])
            elems.append((sl.elem_begin, sl.elem_end))
        assert elems[0][0] == 0 and elems[-1][1] == pr.n_elems
        assert all(a[1] == b[0] for a, b in zip(elems[:-1], elems[1:]))
    with pytest.raises(ValueError):
        slabs.slab_of((4, 4, 6), 2, 4, 0)


@pytest.mark.parametrize("world,p", [(2, 2), (4, 1), (4, 3)])
def test_ghost_slabs_tile_rows(world, p):
    """Row ownership bookkeeping (N2 on several ranks): owned rows tile the global node rows,
    each extended slab holds its own cells plus exactly one layer above (not on the top rank),
    and every cell touching an owned row is inside the extended slab."""
    from paper_2107_04121_b200 import slabs
    shape = (3, 2, 8)
    pr = fi.make_problem(fi.DIFFUSION, p, shape, 5)
    nxy = shape[0] * shape[1]
    owner = np.full(pr.n_nodes, -1)
    for g in range(world):
        gs = slabs.ghost_slab_of(shape, p, world, g)
        sl = gs.slab
        assert gs.elem_begin == sl.elem_begin
        assert gs.elem_end == sl.elem_end + (nxy if g < world - 1 else 0)
        lo, hi = gs.node_begin + gs.row_begin, gs.node_begin + gs.row_end
        assert np.all(owner[lo:hi] == -1)
        owner[lo:hi] = g
        slabs.local_arrays(gs, pr.coords, pr.conn, pr.dof_conn)  # index ranges consistent
        touching = np.where(((pr.dof_conn >= lo) & (pr.dof_conn < hi)).any(axis=1))[0]
        assert touching.min() >= gs.elem_begin and touching.max() < gs.elem_end
    assert np.all(owner >= 0)


@pytest.mark.parametrize("world,p", [(2, 2), (4, 1), (3, 3)])
def test_peer_windows_map_shared_planes(world, p):
    """The peer windows map every shared interface node to the same GLOBAL node on the
    neighbour (index bookkeeping of the fused peer-memory exchange)."""
    from paper_2107_04121_b200 import slabs
    shape = (2, 3, 12)
    for g in range(world):
        sl = slabs.slab_of(shape, p, world, g)
        wins = slabs.peer_windows(sl, shape, p, "prev", "next")
        assert len(wins) == (g > 0) + (g < world - 1)
        for lo, hi, dst, off in wins:
            nb = slabs.slab_of(shape, p, world, g - 1 if dst == "prev" else g + 1)
            assert hi - lo == sl.plane
            for n in (lo, (lo + hi) // 2, hi - 1):
                assert sl.node_begin + n == nb.node_begin + (n - lo + off)


def test_boundary_first_order():
    """Boundary layers first: a permutation whose first 2L cells are the slab's first and last
    z-layers and whose rest is the interior in order (host bookkeeping, no exchange)."""
    shape, p = (3, 2, 8), 2
    for world in (1, 2, 4):
        for rank in range(world):
            sl = slabs.slab_of(shape, p, world, rank)
            o = slabs.boundary_first_order(sl, shape)
            assert sorted(o.tolist()) == list(range(sl.n_elems))
            L = shape[0] * shape[1]
            if world > 1 and sl.n_elems > 2 * L:
                ez = o // L
                nl = sl.n_elems // L
                assert set(ez[:2 * L].tolist()) == {0, nl - 1}
                assert (np.diff(o[2 * L:]) == 1).all()
    pr = fi.make_problem(fi.DIFFUSION, p, shape, 3)
    sl = slabs.slab_of(shape, p, 2, 1)
    o = slabs.boundary_first_order(sl, shape)
    lc, lconn, ldc = slabs.local_arrays(sl, pr.coords, pr.conn, pr.dof_conn, o)
    lc0, lconn0, ldc0 = slabs.local_arrays(sl, pr.coords, pr.conn, pr.dof_conn)
    assert (lconn == lconn0[o]).all() and (ldc == ldc0[o]).all()

"""Multi-GPU z-slab partition and interface-plane summation.

Elements of a structured nx*ny*nz grid (ez slowest) are split into contiguous
z-slabs, one per rank (BASELINE.json north_star: "Elements are partitioned as
contiguous slabs across the 8 GPUs ... Residual mode sums the shared
interface-plane DOFs with NCCL over NVLink").  Global node numbering is
z-slowest, so every rank's nodes are one contiguous slice of the global
vector, including both interface planes.  Matrix mode needs no
communication; residual mode adds, after the local scatter, the partial sums
of the two shared node planes with the neighbours (grouped NCCL send/recv of
contiguous slices; gloo on CPU tensors in the tests).  IEEE addition is
commutative, so both copies of a shared plane end up bitwise equal.

This module is plumbing only (index bookkeeping and torch.distributed calls);
all arithmetic of the method runs in libfeb200.so.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


@dataclass
class Slab:
    rank: int
    world: int
    elem_begin: int       # global element range [elem_begin, elem_end)
    elem_end: int
    vert_begin: int       # global vertex range [vert_begin, vert_end)
    vert_end: int
    node_begin: int       # global node range [node_begin, node_end)
    node_end: int
    plane: int            # nodes per interface plane

    @property
    def n_elems(self):
        return self.elem_end - self.elem_begin

    @property
    def n_nodes(self):
        return self.node_end - self.node_begin


def slab_of(shape, p: int, world: int, rank: int) -> Slab:
    nx, ny, nz = shape
    if nz % world != 0:
        raise ValueError(f"nz={nz} is not divisible by {world} ranks")
    z0, z1 = nz * rank // world, nz * (rank + 1) // world
    vplane = (nx + 1) * (ny + 1)
    plane = (p * nx + 1) * (p * ny + 1)
    return Slab(rank, world, z0 * nx * ny, z1 * nx * ny, z0 * vplane, (z1 + 1) * vplane,
                p * z0 * plane, (p * z1 + 1) * plane, plane)


def boundary_first_order(slab: Slab, shape) -> np.ndarray:
    """Local cell order with the slab's two boundary z-layers first (first layer, last
    layer, then the interior layers in order): the boundary cells are then ONE contiguous
    range [0, 2 L) and the step of residual_overlapped(boundary_first=True) needs two
    launches instead of three.  Returns the permutation of the slab's local cell ids."""
    L = layer_cells(shape, slab.world)
    n = slab.n_elems
    idx = np.arange(n)
    if slab.world == 1 or n <= 2 * L:
        return idx
    return np.concatenate([idx[:L], idx[n - L:], idx[L:n - L]])


def local_arrays(slab: Slab, coords, conn, dof_conn, order=None):
    """Rank-local mesh arrays: vertex/node ids renumbered into the slab's ranges; `order`
    (e.g. boundary_first_order) permutes the slab's cells (per-cell inputs such as the
    material must be permuted the same way)."""
    e0, e1 = slab.elem_begin, slab.elem_end
    lc = np.ascontiguousarray(coords[slab.vert_begin:slab.vert_end])
    cells = np.arange(e0, e1) if order is None else e0 + np.asarray(order)
    lconn = np.ascontiguousarray(conn[cells] - slab.vert_begin).astype(np.int32)
    ldc = np.ascontiguousarray(dof_conn[cells] - slab.node_begin).astype(np.int32)
    assert lconn.min() >= 0 and lconn.max() < slab.vert_end - slab.vert_begin
    assert ldc.min() >= 0 and ldc.max() < slab.n_nodes
    return lc, lconn, ldc


def exchange_planes(r: torch.Tensor, slab: Slab, group=None, bufs=None):
    """Sum the shared interface planes of the rank-local vector r [n_local][D] in place.

    Rank g sends its first plane to g-1 and its last plane to g+1 and adds what it
    receives.  Returns the list of receive buffers (reusable via `bufs`)."""
    if slab.world == 1:
        return bufs
    pl = slab.plane
    D = r.shape[1] if r.dim() > 1 else 1
    flat = r.view(-1)
    lo = flat[: pl * D]
    hi = flat[flat.numel() - pl * D:]
    if bufs is None:
        bufs = [torch.empty_like(lo), torch.empty_like(hi)]
    ops = []
    if slab.rank > 0:
        ops.append(dist.P2POp(dist.isend, lo.contiguous(), slab.rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, bufs[0], slab.rank - 1, group))
    if slab.rank < slab.world - 1:
        ops.append(dist.P2POp(dist.isend, hi.contiguous(), slab.rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, bufs[1], slab.rank + 1, group))
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    if slab.rank > 0:
        lo.add_(bufs[0])
    if slab.rank < slab.world - 1:
        hi.add_(bufs[1])
    return bufs


def layer_cells(shape, world: int) -> int:
    """Cells in one z-layer of a slab (nx * ny)."""
    return shape[0] * shape[1]


def residual_overlapped(evaluate, r: torch.Tensor, slab: Slab, shape, comm_stream=None, bufs=None,
                        exchange=None, events=None, boundary_first=False):
    """Boundary-first residual step with the interface exchange overlapped.

    evaluate(a, b) launches the fused residual kernel for local cells [a, b) on the current
    stream.  The two boundary z-layers are evaluated first; their node planes are then final,
    so the exchange of those planes (`exchange(r, slab, group, bufs)`, default the NCCL / gloo
    exchange_planes) runs on `comm_stream` while the interior layers are evaluated (the
    interior cells never touch the interface planes).  The current stream waits for the
    exchange before returning.  `events`: a preallocated torch.cuda.Event for the
    boundary -> exchange dependency (none is created per step when it is given).
    boundary_first: the local cells are in boundary_first_order (boundary cells = [0, 2L),
    one launch instead of two)."""
    exchange = exchange_planes if exchange is None else exchange
    n_local = slab.n_elems
    if slab.world == 1:
        evaluate(0, n_local)
        return bufs
    L = layer_cells(shape, slab.world)
    if comm_stream is None:  # CPU / gloo: same boundary-first order, no concurrency
        if n_local <= 2 * L:
            evaluate(0, n_local)
            return exchange(r, slab, None, bufs)
        evaluate(0, L)
        evaluate(n_local - L, n_local)
        bufs = exchange(r, slab, None, bufs)
        evaluate(L, n_local - L)
        return bufs
    main = torch.cuda.current_stream(r.device)
    if n_local <= 2 * L:
        evaluate(0, n_local)
        lo_hi_done = [(0, n_local)]
    elif boundary_first:
        evaluate(0, 2 * L)
        lo_hi_done = None
    else:
        evaluate(0, L)
        evaluate(n_local - L, n_local)
        lo_hi_done = None
    ev = torch.cuda.Event() if events is None else events
    ev.record(main)
    comm_stream.wait_event(ev)
    with torch.cuda.stream(comm_stream):
        bufs = exchange(r, slab, None, bufs)
    if lo_hi_done is None:
        if boundary_first:
            evaluate(2 * L, n_local)
        else:
            evaluate(L, n_local - L)
    main.wait_stream(comm_stream)
    return bufs


class VirtualWorld:
    """P z-slab "ranks" on ONE device in one process (one host thread per rank): the
    interface exchange of exchange_planes done by device copies instead of NCCL, so the
    multi-rank code path (residual_overlapped's comm-stream exchange, boundary-first order,
    plane adds, CUDA-graph capture) runs and is checked on a single GPU.

    exchange(r, slab, group, bufs) for rank g, on its comm stream: "send" = copy its first /
    last plane into the receive buffer that rank g-1 / g+1 owns, record an event; a host
    barrier (every rank has enqueued its sends and recorded its event); "receive" = wait for
    the neighbours' send events, add the buffers into its own planes -- the order of the NCCL
    send/recv + add.  No kernel waits on another rank's kernel (only stream-event order)."""

    def __init__(self, slabs_, ncomp, device, dtype=torch.float64):
        import threading
        self.slabs = slabs_
        P = len(slabs_)
        self.barrier = threading.Barrier(P, timeout=120)
        D = ncomp
        # recv[g] = [from g-1 (into my first plane), from g+1 (into my last plane)]
        self.recv = [[torch.empty(s.plane * D, dtype=dtype, device=device) for _ in range(2)]
                     for s in slabs_]
        self.sent = [torch.cuda.Event() for _ in range(P)]

    def exchange_for(self, rank):
        def exchange(r, slab, group, bufs):
            P = len(self.slabs)
            pl = slab.plane
            D = r.shape[1] if r.dim() > 1 else 1
            flat = r.view(-1)
            lo = flat[: pl * D]
            hi = flat[flat.numel() - pl * D:]
            if rank > 0:
                self.recv[rank - 1][1].copy_(lo)
            if rank < P - 1:
                self.recv[rank + 1][0].copy_(hi)
            self.sent[rank].record(torch.cuda.current_stream(r.device))
            self.barrier.wait()
            st = torch.cuda.current_stream(r.device)
            if rank > 0:
                st.wait_event(self.sent[rank - 1])
                lo.add_(self.recv[rank][0])
            if rank < P - 1:
                st.wait_event(self.sent[rank + 1])
                hi.add_(self.recv[rank][1])
            self.barrier.wait()  # no rank reuses a receive buffer of this step early
            return bufs
        return exchange


def virtual_world_step(slabs_, evaluators, rs, mains, comms, world: VirtualWorld, shape,
                       events=None):
    """One residual step of every virtual rank enqueued from ONE host thread, so that the
    whole world's step can be captured into a single CUDA graph: per rank, zero r and the
    boundary layers on its main stream; then the sends (device copies) on its comm stream;
    then the interior layers on the main stream while the comm stream adds the received
    planes; the main stream joins the comm stream.  The same order as residual_overlapped +
    exchange_planes, phase by phase over the ranks.  All streams must have been forked from
    the caller's current stream (mains[g] / comms[g] wait on it); the caller joins them."""
    P = len(slabs_)
    if events is None:
        events = [torch.cuda.Event() for _ in range(P)]
    L = layer_cells(shape, P)
    for g in range(P):
        with torch.cuda.stream(mains[g]):
            rs[g].zero_()
            n = slabs_[g].n_elems
            if n <= 2 * L:
                evaluators[g](0, n)
            else:
                evaluators[g](0, L)
                evaluators[g](n - L, n)
            events[g].record(mains[g])
    for g in range(P):
        comms[g].wait_event(events[g])
        with torch.cuda.stream(comms[g]):
            sl, r = slabs_[g], rs[g]
            D = r.shape[1] if r.dim() > 1 else 1
            flat = r.view(-1)
            if g > 0:
                world.recv[g - 1][1].copy_(flat[: sl.plane * D])
            if g < P - 1:
                world.recv[g + 1][0].copy_(flat[flat.numel() - sl.plane * D:])
            world.sent[g].record(comms[g])
    for g in range(P):
        n = slabs_[g].n_elems
        with torch.cuda.stream(mains[g]):
            if n > 2 * L:
                evaluators[g](L, n - L)
        with torch.cuda.stream(comms[g]):
            sl, r = slabs_[g], rs[g]
            D = r.shape[1] if r.dim() > 1 else 1
            flat = r.view(-1)
            if g > 0:
                comms[g].wait_event(world.sent[g - 1])
                flat[: sl.plane * D].add_(world.recv[g][0])
            if g < P - 1:
                comms[g].wait_event(world.sent[g + 1])
                flat[flat.numel() - sl.plane * D:].add_(world.recv[g][1])
        mains[g].wait_stream(comms[g])


class StepGraph:
    """A rank's whole step (e.g. zero r, boundary cells, exchange on the comm stream,
    interior cells, plane adds) captured once into a CUDA graph and replayed: one host call
    per step instead of ~10.  `step()` must issue its work on the current
    stream (torch.cuda.current_stream()), which is the capture stream while capturing; NCCL
    P2P inside the step is captured as well (NCCL >= 2.9.6).  warmup: eager runs on the
    capture stream before capturing (libraries / NCCL set up lazily)."""

    def __init__(self, step, device, warmup=2):
        self.device = device
        self.stream = torch.cuda.Stream(device)
        self.stream.wait_stream(torch.cuda.current_stream(device))
        with torch.cuda.stream(self.stream):
            for _ in range(warmup):
                step()
        torch.cuda.current_stream(device).wait_stream(self.stream)
        self.graph = torch.cuda.CUDAGraph()
        # thread_local: CUDA calls of other host threads (the NCCL watchdog) stay legal
        with torch.cuda.graph(self.graph, stream=self.stream, capture_error_mode="thread_local"):
            step()

    def replay(self):
        self.graph.replay()


def peer_windows(slab: Slab, shape, p: int, prev_ptr, next_ptr):
    """fe_eval_residual_peer windows of rank g: its first node plane is rank g-1's last plane
    (local offset n_prev - plane there), its last plane is rank g+1's first plane (offset 0)."""
    pl = slab.plane
    wins = []
    if slab.rank > 0:
        prev = slab_of(shape, p, slab.world, slab.rank - 1)
        wins.append((0, pl, prev_ptr, prev.n_nodes - pl))
    if slab.rank < slab.world - 1:
        wins.append((slab.n_nodes - pl, slab.n_nodes, next_ptr, 0))
    return wins


class PeerExchange:
    """Fused residual + interface exchange over peer memory.

    Every rank's residual vector lives in an IPC-shareable allocation (fe_ipc_alloc); each
    rank maps its neighbours' vectors (fe_ipc_open: NVLink peer memory on a multi-GPU node, or
    the same device) and passes two peer windows to fe_eval_residual_peer: its first node
    plane is also added into rank g-1's last plane, its last plane into rank g+1's first plane,
    by the residual kernel's own scatter (system-scope fp64 atomics).  No separate collective
    moves data; the step is ordered by two barriers (all vectors zeroed before any kernel;
    all kernels finished before any rank reads).  Plumbing only: the arithmetic is in the
    library's residual kernels."""

    def __init__(self, slab: Slab, shape, p: int, ncomp: int, device, group=None):
        import paper_2107_04121_b200 as fe
        self.fe, self.slab, self.group = fe, slab, group
        self.vec = fe.IpcVector((slab.n_nodes, ncomp), device)
        self.r = self.vec.tensor
        handles = [None] * slab.world
        dist.all_gather_object(handles, self.vec.handle, group=group)
        prev = fe.ipc_open(handles[slab.rank - 1]) if slab.rank > 0 else None
        nxt = fe.ipc_open(handles[slab.rank + 1]) if slab.rank < slab.world - 1 else None
        self.peers = [q for q in (prev, nxt) if q is not None]
        self.windows = peer_windows(slab, shape, p, prev, nxt)

    def residual(self, evaluate_peer, barrier):
        """One step: zero the own vector, barrier, fused residual + exchange over all local
        cells (evaluate_peer(windows) launches fe_eval_residual_peer), barrier."""
        self.r.zero_()
        barrier()
        evaluate_peer(self.windows)
        barrier()
        return self.r

    def close(self):
        for ptr in self.peers:
            self.fe.ipc_close(ptr)
        self.peers = []
        self.vec.close()


@dataclass
class GhostSlab:
    """A z-slab extended by the first cell layer of the rank above (matrix mode + CSR with row
    ownership): rank g owns the node rows of its planes p*z0+1 .. p*z1 (rank 0 also
    plane 0), so every owned row's cells are local or in the ghost layer, and the rank's block
    rows of the global CSR matrix are assembled without any communication; the ghost layer's
    element matrices are computed twice (by the owner of the cells and by the rank below)."""
    slab: Slab                # the rank's own cells
    elem_begin: int           # extended element range (own + ghost layer)
    elem_end: int
    vert_begin: int
    vert_end: int
    node_begin: int           # extended node range
    node_end: int
    row_begin: int            # owned rows, in the extended local numbering
    row_end: int

    @property
    def n_elems(self):
        return self.elem_end - self.elem_begin

    @property
    def n_nodes(self):
        return self.node_end - self.node_begin


def ghost_slab_of(shape, p: int, world: int, rank: int) -> GhostSlab:
    nx, ny, nz = shape
    sl = slab_of(shape, p, world, rank)
    z0, z1 = nz * rank // world, nz * (rank + 1) // world
    zg = z1 + 1 if rank < world - 1 else z1
    vplane = (nx + 1) * (ny + 1)
    pl = sl.plane
    row_begin = pl if rank > 0 else 0
    row_end = (p * (z1 - z0) + 1) * pl
    return GhostSlab(sl, z0 * nx * ny, zg * nx * ny, z0 * vplane, (zg + 1) * vplane,
                     p * z0 * pl, (p * zg + 1) * pl, row_begin, row_end)


def owned_block_rows(gs: GhostSlab, row_ptr, col, values, ncomp: int = 1):
    """The rank's block rows of the global CSR matrix from the CSR of its ghost-extended mesh:
    (global first row, row_ptr rebased to 0, GLOBAL column ids, values) of the owned rows.
    row_ptr / col / values: the local CSR (scalar rows when ncomp = 1; interleaved node-major
    rows node * ncomp + a otherwise, as fe_create_csr lays them out)."""
    r0, r1 = gs.row_begin * ncomp, gs.row_end * ncomp
    a, b = int(row_ptr[r0]), int(row_ptr[r1])
    rp = row_ptr[r0:r1 + 1] - a
    return gs.node_begin * ncomp + r0, rp, col[a:b] + gs.node_begin * ncomp, values[a:b]

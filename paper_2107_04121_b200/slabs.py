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


def local_arrays(slab: Slab, coords, conn, dof_conn):
    """Rank-local mesh arrays: vertex/node ids renumbered into the slab's ranges."""
    e0, e1 = slab.elem_begin, slab.elem_end
    lc = np.ascontiguousarray(coords[slab.vert_begin:slab.vert_end])
    lconn = np.ascontiguousarray(conn[e0:e1] - slab.vert_begin).astype(np.int32)
    ldc = np.ascontiguousarray(dof_conn[e0:e1] - slab.node_begin).astype(np.int32)
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


def residual_overlapped(evaluate, r: torch.Tensor, slab: Slab, shape, comm_stream=None, bufs=None):
    """Boundary-first residual step with the interface exchange overlapped.

    evaluate(a, b) launches the fused residual kernel for local cells [a, b) on the current
    stream.  The two boundary z-layers are evaluated first; their node planes are then final,
    so the NCCL exchange of those planes runs on `comm_stream` while the interior layers are
    evaluated (the interior cells never touch the interface planes).  The current stream
    waits for the exchange before returning."""
    n_local = slab.n_elems
    if slab.world == 1:
        evaluate(0, n_local)
        return bufs
    L = layer_cells(shape, slab.world)
    if comm_stream is None:  # CPU / gloo: same boundary-first order, no concurrency
        if n_local <= 2 * L:
            evaluate(0, n_local)
            return exchange_planes(r, slab, None, bufs)
        evaluate(0, L)
        evaluate(n_local - L, n_local)
        bufs = exchange_planes(r, slab, None, bufs)
        evaluate(L, n_local - L)
        return bufs
    main = torch.cuda.current_stream(r.device)
    if n_local <= 2 * L:
        evaluate(0, n_local)
        lo_hi_done = [(0, n_local)]
    else:
        evaluate(0, L)
        evaluate(n_local - L, n_local)
        lo_hi_done = None
    ev = torch.cuda.Event()
    ev.record(main)
    comm_stream.wait_event(ev)
    with torch.cuda.stream(comm_stream):
        bufs = exchange_planes(r, slab, None, bufs)
    if lo_hi_done is None:
        evaluate(L, n_local - L)
    main.wait_stream(comm_stream)
    return bufs


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

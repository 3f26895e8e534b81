"""Host cost of one rank's residual step, eager vs CUDA graph.

    python tools/host_overhead.py [--config C4] [--ranks 8] [--rank 3] [--steps 200]

One GPU.  The config's mesh is cut into P z-slabs (slabs.slab_of); rank g's slab (C4 at P = 8:
5 cell layers, 8000 cells) runs its step -- zero r, the two boundary layers, the interface
exchange on the comm stream (device copies: slabs.VirtualWorld's sends / adds for one rank),
the interior layers, the join -- (a) eagerly through slabs.residual_overlapped (~10 host calls
per step) and (b) captured once into a CUDA graph (slabs.StepGraph, one host call per step).
Reported: device time per step of each, host enqueue time per step of each, and the bare
kernel time of the rank's cells (one fe_eval_residual over all of them).  The whole P-rank
world's step captured into one graph (slabs.virtual_world_step) is timed too.  JSON on stdout.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import fe_inputs as fi  # noqa: E402
import paper_2107_04121_b200 as fe  # noqa: E402
from paper_2107_04121_b200 import slabs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--rank", type=int, default=3)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    args = ap.parse_args()
    P = args.ranks
    pr = fi.make_config(args.config)
    tdt = torch.float64 if args.dtype == "f64" else torch.float32
    dtc = fe.F64 if args.dtype == "f64" else fe.F32
    sls = [slabs.slab_of(pr.shape, pr.p, P, g) for g in range(P)]
    ranks = []
    for sl in sls:
        lc, lconn, ldc = slabs.local_arrays(sl, pr.coords, pr.conn, pr.dof_conn)
        e0, e1 = sl.elem_begin, sl.elem_end
        mesh = fe.Mesh(torch.from_numpy(lc), torch.from_numpy(lconn), pr.p, pr.q1d,
                       dof_conn=torch.from_numpy(ldc), n_nodes=sl.n_nodes)
        cut = (lambda a: None if a is None else torch.from_numpy(
            np.ascontiguousarray(a[e0:e1])).to("cuda", tdt))
        ranks.append(dict(sl=sl, mesh=mesh, ma=cut(pr.mat_a), mb=cut(pr.mat_b),
                          u=torch.from_numpy(np.ascontiguousarray(
                              pr.u[sl.node_begin:sl.node_end])).to("cuda", tdt),
                          r=torch.zeros((sl.n_nodes, pr.ncomp), dtype=tdt, device="cuda"),
                          main=torch.cuda.Stream(), comm=torch.cuda.Stream()))
    world = slabs.VirtualWorld(sls, pr.ncomp, "cuda", dtype=tdt)

    def evaluator(rk):
        def ev(a, b):
            fe.fe_eval_residual(rk["mesh"].handle, pr.form, dtc, pr.mat_kind, rk["ma"], rk["mb"],
                                rk["u"], a, b, None, rk["r"], torch.cuda.current_stream())
        return ev

    g = args.rank
    rk = ranks[g]
    sl = rk["sl"]
    D = pr.ncomp
    bufs_ev = torch.cuda.Event()

    def one_rank_exchange(r, slab, group, bufs):
        # the device work of one rank's exchange: sends into the neighbours' receive buffers,
        # adds of its own receive buffers (the neighbours' data is whatever they hold)
        flat = r.view(-1)
        lo, hi = flat[: slab.plane * D], flat[flat.numel() - slab.plane * D:]
        if slab.rank > 0:
            world.recv[slab.rank - 1][1].copy_(lo)
            lo.add_(world.recv[slab.rank][0])
        if slab.rank < slab.world - 1:
            world.recv[slab.rank + 1][0].copy_(hi)
            hi.add_(world.recv[slab.rank][1])
        return bufs

    evg = evaluator(rk)

    def step():
        rk["r"].zero_()
        slabs.residual_overlapped(evg, rk["r"], sl, pr.shape, rk["comm"], exchange=one_rank_exchange,
                                  events=bufs_ev)

    def timed(fn, n):
        st = torch.cuda.current_stream()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        a.record(st)
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        t1 = time.perf_counter()
        b.record(st)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n, (t1 - t0) / n * 1e6

    res = {"config": args.config, "ranks": P, "rank": g, "cells": sl.n_elems,
           "layers": sl.n_elems // (pr.shape[0] * pr.shape[1]), "dtype": args.dtype}
    # bare kernel: all the rank's cells in one call
    kern_ms, kern_host = timed(lambda: evg(0, sl.n_elems), args.steps)
    res["kernel_ms"] = kern_ms
    eager_ms, eager_host_us = timed(step, args.steps)
    res["eager"] = {"device_ms_per_step": eager_ms, "host_us_per_step": eager_host_us,
                    "launches_per_step": None}
    n0 = fe.fe_launch_count()
    step()
    torch.cuda.synchronize()
    res["eager"]["launches_per_step"] = fe.fe_launch_count() - n0
    gr = slabs.StepGraph(step, torch.device("cuda"))
    graph_ms, graph_host_us = timed(gr.replay, args.steps)
    res["graph"] = {"device_ms_per_step": graph_ms, "host_us_per_step": graph_host_us}
    res["graph_over_kernel"] = graph_ms / kern_ms
    res["eager_over_kernel"] = eager_ms / kern_ms
    # variants of the same step, graph-replayed: (b) the rank's cells in boundary-first order
    # (boundary layers one launch), (c) no overlap: all cells in one launch, then the exchange
    order = slabs.boundary_first_order(sl, pr.shape)
    lc, lconn, ldc = slabs.local_arrays(sl, pr.coords, pr.conn, pr.dof_conn, order)
    e0 = sl.elem_begin
    mesh_b = fe.Mesh(torch.from_numpy(lc), torch.from_numpy(lconn), pr.p, pr.q1d,
                     dof_conn=torch.from_numpy(ldc), n_nodes=sl.n_nodes)
    cutb = (lambda a: None if a is None else torch.from_numpy(
        np.ascontiguousarray(a[e0 + order])).to("cuda", tdt))
    rkb = dict(rk, mesh=mesh_b, ma=cutb(pr.mat_a), mb=cutb(pr.mat_b))
    evb = evaluator(rkb)

    def step_b():
        rk["r"].zero_()
        slabs.residual_overlapped(evb, rk["r"], sl, pr.shape, rk["comm"], exchange=one_rank_exchange,
                                  events=bufs_ev, boundary_first=True)

    def step_c():
        rk["r"].zero_()
        evg(0, sl.n_elems)
        one_rank_exchange(rk["r"], sl, None, None)

    # (d) the fused residual + exchange (fe_eval_residual_peer): the kernel's own scatter adds
    # the interface planes into the neighbours' vectors (here: the other virtual ranks' r on the
    # same GPU; NVLink peer memory across GPUs) -- one kernel per step plus the zeroing (the
    # two device barriers of the multi-GPU step, tiny NCCL all-reduces, are not in this number)
    prev_ptr = ranks[g - 1]["r"].data_ptr() if g > 0 else None
    next_ptr = ranks[g + 1]["r"].data_ptr() if g < P - 1 else None
    wins = slabs.peer_windows(sl, pr.shape, pr.p, prev_ptr, next_ptr)

    def step_d():
        rk["r"].zero_()
        fe.fe_eval_residual_peer(rk["mesh"].handle, pr.form, pr.mat_kind, rk["ma"], rk["mb"],
                                 rk["u"], 0, sl.n_elems, None, rk["r"], wins,
                                 torch.cuda.current_stream())

    variants = [("graph_boundary_first", step_b), ("graph_no_overlap", step_c)]
    if args.dtype == "f64":
        variants.append(("graph_peer_fused", step_d))
    for name, fn in variants:
        gx = slabs.StepGraph(fn, torch.device("cuda"))
        ms, hus = timed(gx.replay, args.steps)
        res[name] = {"device_ms_per_step": ms, "host_us_per_step": hus,
                     "over_kernel": ms / kern_ms}
    # the whole P-rank world in one graph (P slabs on one GPU: device time ~ P x one slab)
    evs = [evaluator(x) for x in ranks]
    rs = [x["r"] for x in ranks]
    mains = [x["main"] for x in ranks]
    comms = [x["comm"] for x in ranks]
    bev = [torch.cuda.Event() for _ in ranks]

    def world_step():
        cur = torch.cuda.current_stream()
        for s_ in mains + comms:
            s_.wait_stream(cur)
        slabs.virtual_world_step(sls, evs, rs, mains, comms, world, pr.shape, bev)
        for s_ in mains:
            cur.wait_stream(s_)

    wg = slabs.StepGraph(world_step, torch.device("cuda"))
    w_ms, w_host = timed(wg.replay, max(10, args.steps // 4))
    res["world_graph"] = {"device_ms_per_step": w_ms, "host_us_per_step": w_host,
                          "note": f"all {P} virtual ranks' steps (one GPU) in one graph"}
    print(json.dumps(res))


if __name__ == "__main__":
    main()

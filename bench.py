#!/usr/bin/env python
"""Benchmark of the hot path: batched FE weak-form evaluation on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One STEP = one pass of the whole hot path over the config's cells: geometry
(a1), physical gradients (b), element matrices (c1) and residual with gather
and fused scatter-add (c2, d) -- the modes the config names -- through the C
ABI of libfeb200.so, plus, for N > 1, the interface-plane summation (NCCL).
Default workload: BASELINE.json configs[1] = C2 (Q2 scalar diffusion, 64^3
perturbed cells, matrix + residual).  Metric: cells evaluated per second
(each cell gets its element matrix AND its residual every step).

Timing: W warm-up steps, then K steps bracketed by barrier + synchronize,
CUDA events on the launching stream (per-step and per-kernel events
preallocated), max over ranks.  Every step writes or reads more than the
126 MB L2 (C2: K = 1.53 GB), so no explicit flush.  Reported per step and
per kernel: mean, the paper's mean without the worst call T^ww,
median and minimum, plus the result throughput |K| or |r| / T^ww in MB/s
(P:1566-1572).  Clocks are sampled with nvidia-smi every 20 ms over a window
of >= 1.2 s that contains the timed region (untimed repeats of the same step
before and after it), so the record has samples even when K steps take a few
milliseconds.

The default line (--config C2) also carries `configs`: every other BASELINE
form and mode (C3 elasticity matrix + residual, C4 mass+Laplace residual in
fp64 and fp32, C5 convective residual, C5t convective tangent), each measured
the same way with its own kernel statistics, rooflines and clock record.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import fe_inputs as fi  # noqa: E402

# ----------------------------------------------------------------------------
# Algorithmic work per cell:
# flops of the lean dense-table formulation per qp (FMA = 2 flops) plus 120 per
# qp of geometry, bytes = minimal HBM traffic with perfect reuse.
GEOM = 120


def alg_flops(form: int, mode: str, nb: int, nq: int) -> float:
    if mode == "csr":
        return (fi.FORM_NCOMP[form] * nb) ** 2  # one add per element-matrix entry
    if mode == "matrix":
        per_qp = {fi.DIFFUSION: 6 * nb * nb + 21 * nb, fi.MASS: 2 * nb * nb + nb,
                  fi.MASS_DIFFUSION: 8 * nb * nb + 22 * nb,
                  fi.VECTOR_MASS: 2 * nb * nb + nb,
                  fi.ELASTICITY: 12 * nb * nb + 21 * nb,
                  fi.CONVECTIVE: 20 * nb * nb + 48 * nb}[form]
        per_el = {fi.ELASTICITY: 27 * nb * nb, fi.CONVECTIVE: 9 * nb * nb}.get(form, 0)
        return (per_qp + GEOM) * nq + per_el
    per_qp = {fi.DIFFUSION: 12 * nb + 40, fi.MASS: 4 * nb + 5, fi.MASS_DIFFUSION: 16 * nb + 45,
              fi.VECTOR_MASS: 12 * nb + 15, fi.ELASTICITY: 36 * nb + 137,
              fi.CONVECTIVE: 30 * nb + 75}[form]
    return (per_qp + GEOM) * nq


def sf_matrix_flops(form: int, p: int) -> float:
    """Flops per cell of the sum-factorised matrix kernel (k_matrix_sf.cu), FMA = 2."""
    n1 = q1 = p + 1
    nq = q1 ** 3
    nup = (6 if form != fi.MASS else 0) + (1 if form != fi.DIFFUSION else 0)
    nop = (9 if form != fi.MASS else 0) + (1 if form != fi.DIFFUSION else 0)
    tpe = n1 * n1 * (n1 * (n1 - 1) // 2) + n1 * (n1 * (n1 + 1) // 2)
    geo = (GEOM + 32) * nq
    z = nup * q1 * q1 * (q1 * n1 + 2 * n1 * n1 * q1)
    y = 2 * tpe * nop * q1 * q1
    x = tpe * q1 * 2 * (3 * n1 + 2 * n1 * n1)
    return geo + z + y + x


def sf_vector_matrix_flops(form: int, p: int) -> float:
    """Flops per cell of the pipelined vector SF matrix kernel (k_matrix_vp.cu), FMA = 2:
    phase 1 per qp (geometry + all pair weights W^{ab}_{mn}; convective: state interpolation),
    phase 2 stage z per pair, X stages y and x per (block, z pair, y pair) task."""
    n1 = q1 = p + 1
    nq = q1 ** 3
    sym_t = n1 * n1 * (n1 * (n1 - 1) // 2) + n1 * (n1 * (n1 + 1) // 2)
    full_t = n1 ** 4

    def x_task(nops):
        return 2 * nops * q1 * q1 + 4 * q1 + q1 * 2 * (3 * n1 + 2 * n1 * n1)
    if form == fi.ELASTICITY:
        per_qp, nwp = GEOM + 282, 45
        x = 3 * sym_t * x_task(9) + 3 * full_t * x_task(9)
    else:  # convective tangent: one item for the 3 diagonal blocks (shared advection + 3
        # reactions, stage x once for A and once per reaction), 6 off-diagonal reaction items
        per_qp, nwp = GEOM + 650, 12
        adv = 2 * 6 * q1 * q1 + 4 * q1 + q1 * 2 * (3 * n1 + 2 * n1 * n1) + 3 * q1 * 2 * (n1 + n1 * n1)
        x = full_t * adv + 6 * sym_t * x_task(1)
    z = nwp * q1 * q1 * (2 * n1 * n1 * q1)
    return per_qp * nq + z + x


def sf_residual_flops(form: int, p: int) -> float:
    """Flops per cell of the sum-factorised residual kernel (k_residual_sf.cu), FMA = 2:
    1D contractions 2 D (5 + V + 12 G) n^4 plus ~(100 + 40 D) per qp of geometry / flux; the
    convective backward pass tests against v only (no y^T / x^T gradient arrays: 5 fewer)."""
    n = p + 1
    D = fi.FORM_NCOMP[form]
    G = 0 if form in (fi.MASS, fi.VECTOR_MASS) else 1
    V = 1 if form in (fi.MASS, fi.VECTOR_MASS, fi.MASS_DIFFUSION, fi.CONVECTIVE) else 0
    back = -5 if form == fi.CONVECTIVE else 0
    return 2 * D * (5 + V + 12 * G + back) * n ** 4 + n ** 3 * (100 + 40 * D)


def uses_sf_residual(p: int) -> bool:
    return p <= 4 and os.environ.get("FEB200_RESIDUAL_IMPL", "") != "dense"


def uses_sf_matrix(form: int, p: int) -> bool:
    return (form in (fi.DIFFUSION, fi.MASS, fi.MASS_DIFFUSION) and p <= 3
            and os.environ.get("FEB200_MATRIX_IMPL", "") != "dense")


def alg_bytes(form: int, mode: str, p: int, nb: int, nq: int, D: int, mat_kind: int,
              esize: int = 8, csr_nnz_per_cell: float = 0.0) -> float:
    if mode == "csr":
        # essential traffic: read K_e once, read + write every global CSR value once (the
        # duplicate contributions of neighbouring cells merge in L2); the position map and the
        # row pointers are implementation overhead, not counted
        return (D * nb) ** 2 * 8 + 16 * csr_nnz_per_cell
    if form == fi.ELASTICITY:
        mat = (2 * esize if mat_kind == fi.MAT_PER_ELEM
               else 36 * nq * esize if mat_kind == fi.MAT_FULL_D else 2 * nq * esize)
    elif form == fi.MASS_DIFFUSION:
        mat = 2 * nq * esize
    elif form == fi.CONVECTIVE:
        mat = 0
    else:
        mat = nq * esize
    geo = 24 + 32                               # one vertex + 8 conn ids per cell
    if mode == "matrix":
        b = geo + mat + (D * nb) ** 2 * esize       # K in the call's type (fp32: FE_F32 path)
        if form == fi.CONVECTIVE:
            b += 4 * nb + D * p ** 3 * 8        # gather of the state
        return b
    return geo + mat + 4 * nb + D * p ** 3 * esize + 2 * D * p ** 3 * esize


# ----------------------------------------------------------------------------
FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "fp64_peak_r01.json")


def fp64_peak_tflops(key="dmma_m16n8k4_tflops_sustained"):
    """Measured FP64 peak (tools/fp64_peak.cu, profiles/fp64_peak_r01.json): DMMA for the
    tensor-core kernels, DFMA for the CUDA-core kernels.  MEASURED_PEAKS.json has no FP64 entry."""
    try:
        d = json.load(open(FP64_PEAK_FILE))
        return float(d[key]), f"measured: tools/fp64_peak {key} (4 s sustained, 1965 MHz)"
    except Exception:
        return 37.2, "derived: 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz"


def hbm_peak_gbs():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ----------------------------------------------------------------------------
WORKLOADS = {
    "C1": dict(modes=("matrix",)),
    "C2": dict(modes=("matrix", "residual")),
    "C3": dict(modes=("matrix", "residual")),
    "C4": dict(modes=("residual",)),
    "C5": dict(modes=("residual",)),
    "C5t": dict(modes=("matrix",)),
    "C2csr": dict(modes=("matrix", "csr")),   # N2: element matrices + global CSR assembly
    "C3csr": dict(modes=("matrix", "csr")),
    "C3d": dict(modes=("matrix", "residual")),  # N4: C3 with a general Voigt D[E][n_q][6][6]
}
# per-form sub-results carried by the default (C2) line: every BASELINE.json form and mode
SUB_CONFIGS = ("C3", "C4", "C4f32", "C5", "C5t")
L2_NOTE = ("no flush when a step moves more than 4 x the 126 MB L2 (C2: K = 1.53 GB); smaller "
           "steps (C4) flush L2 between timed steps: see l2_flush")


def split_cfg(name):
    """'C4f32' -> ('C4', 'f32'); 'C3' -> ('C3', None)."""
    return (name[:-3], "f32") if name.endswith("f32") else (name, None)


def build_problem(name):
    if name == "C5t":
        return fi.corner_subproblem(fi.make_config("C5"), 64)
    if name == "C3d":
        c = fi.CONFIGS["C3"]
        prob = fi.make_problem(c["form"], c["p"], (c["N"],) * 3, fi.SEED_BASE + c["index"],
                               mat_kind=fi.MAT_FULL_D, name="C3d")
        prob.meta["desc"] = c["desc"].replace("lambda,mu/elem U[0.5,2]", "D[E][27][6][6] SPD per qp")
        return prob
    if name.endswith("csr"):
        return fi.make_config(name[:-3])
    return fi.make_config(name)


def config_dict(cfg, prob, modes, world, exchange, dtype):
    """The `config` object of the JSON line -- identical in both arms (ours / reference)."""
    return {"workload": cfg, "desc": prob.meta.get("desc", ""), "cells": prob.n_elems,
            "order": prob.p, "q1d": prob.q1d, "form": fi.FORM_NAMES[prob.form],
            "modes": list(modes), "dtype": dtype, "parallelism": f"z-slabs x{world}",
            "exchange": exchange if world > 1 else None, "l2": L2_NOTE}


def step_stats(xs):
    """Timing statistics of repeated calls: mean, the paper's mean without the worst call
    T^ww, median and minimum."""
    xs = np.asarray(xs, dtype=np.float64)
    tww = float((xs.sum() - xs.max()) / (len(xs) - 1)) if len(xs) > 1 else float(xs[0])
    return {"mean": float(xs.mean()), "tww": tww, "median": float(np.median(xs)),
            "min": float(xs.min()), "n": int(len(xs))}


def result_bytes(prob, mode, esize):
    """Size of the resulting array the paper's throughput divides by T^ww:
    the element matrices (matrix mode) or the element residual vectors (residual mode)."""
    nd = prob.ncomp * prob.nb
    if mode == "residual":
        return prob.n_elems * nd * esize
    return prob.n_elems * nd * nd * 8


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.t0 = self.t1 = None

    def __enter__(self):
        self.t0 = time.perf_counter()
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.t1 = time.perf_counter()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        win = None if self.t1 is None else round(self.t1 - self.t0, 3)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "window_s": win}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "window_s": win,
                "note": "sampled every 20 ms over the timed region plus untimed repeats of the "
                        "same step before and after it (window >= 1.2 s)"}


# ----------------------------------------------------------------------------
def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_step(prob, n, modes):
    """One oracle pass over the first n cells of prob (matrix and/or residual)."""
    import oracle
    idx = slice(0, n)
    sub = fi.Problem(prob.name, prob.form, prob.p, prob.q1d, prob.shape, prob.coords,
                     prob.conn[idx], prob.dof_conn[idx], prob.n_nodes, prob.mat_kind,
                     None if prob.mat_a is None else prob.mat_a[idx],
                     None if prob.mat_b is None else prob.mat_b[idx], prob.u)
    t0 = time.perf_counter()
    if "matrix" in modes:
        oracle.problem_matrix(sub)
    if "residual" in modes:
        oracle.problem_assembled_residual(sub)
    return time.perf_counter() - t0


def oracle_sample_size(prob, modes, budget_s):
    n = min(64, prob.n_elems)
    t = oracle_step(prob, n, modes)
    while t < 0.2 and n < prob.n_elems:
        n = min(prob.n_elems, n * 4)
        t = oracle_step(prob, n, modes)
    per = t / n
    return int(max(1, min(prob.n_elems, budget_s / per))), per


def cpu_baseline(prob, modes, budget_s=12.0):
    """The oracle on the host cores: passes over (a prefix of) the workload until ~budget_s."""
    n, _ = oracle_sample_size(prob, modes, budget_s)
    passes, t = 0, 0.0
    while t < budget_s and passes < 50:
        t += oracle_step(prob, n, modes)
        passes += 1
    out = {"value": n * passes / t, "unit": "cells/s", "cores": cpu_cores(), "kind": "oracle",
           "sample": f"{passes} pass(es) over the first {n} of {prob.name}'s {prob.n_elems} cells, "
                     f"modes {'+'.join(modes)}, plain C oracle (-O2, OpenMP over cells), {t:.1f} s"}
    # the same oracle on one core, on a smaller prefix
    import oracle
    oracle.set_threads(1)
    try:
        n1 = max(1, n // max(1, cpu_cores()))
        t1 = oracle_step(prob, n1, modes)
        out["value_1core"] = n1 / t1
        out["sample_1core"] = f"first {n1} cells, 1 thread, {t1:.1f} s"
    finally:
        oracle.set_threads(cpu_cores())
    return out


def run_reference(args, cfg):
    """--impl reference: the oracle (this tier's reference arm) on the host cores, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    prob = build_problem(cfg)
    modes = WORKLOADS[cfg]["modes"]
    per_step_budget = max(0.5, min(6.0, 150.0 / max(1, args.steps + args.warmup)))
    n, _ = oracle_sample_size(prob, modes, per_step_budget)
    for _ in range(args.warmup):
        oracle_step(prob, n, modes)
    times = [oracle_step(prob, n, modes) for _ in range(args.steps)]
    T = float(np.sum(times))
    value = n * args.steps / T
    line = {
        "impl": "reference", "metric": f"{cfg} cells evaluated per second ({'+'.join(modes)})",
        "value": value, "unit": "cells/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": config_dict(cfg, prob, modes, world, args.exchange, args.dtype),
        "stats": {"step_ms_full_workload_equiv": step_stats(
            [1e3 * t * prob.n_elems / n for t in times])},
        "cpu_baseline": {"value": value, "unit": "cells/s", "cores": cpu_cores(), "kind": "oracle",
                         "sample": f"first {n} of {prob.n_elems} cells per step (plain C oracle, "
                                   f"-O2, OpenMP over cells)"},
        "e2e": {"value": value, "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
class Runner:
    """One config set up on this rank: mesh (z-slab for N > 1), inputs and outputs in HBM, and
    step() = one pass of the config's modes through the C ABI (plus, for N > 1, the interface
    exchange).  Kernel events are preallocated by the caller and passed in `rec`."""

    def __init__(self, cfg, dtype, world, rank, dev, exchange="nccl", fused=False):
        import torch

        import paper_2107_04121_b200 as fe
        from paper_2107_04121_b200 import slabs
        self.torch, self.fe, self.slabs = torch, fe, slabs
        self.cfg, self.world, self.rank, self.dev, self.dtype = cfg, world, rank, dev, dtype
        self.modes = WORKLOADS[cfg]["modes"]
        self.prob = prob = build_problem(cfg)
        self.fused = (fused and tuple(self.modes) == ("matrix", "residual") and dtype == "f64"
                      and prob.form in (fi.DIFFUSION, fi.MASS, fi.MASS_DIFFUSION) and prob.p <= 2)
        self.kmodes = ("matrix+residual",) if self.fused else tuple(self.modes)
        if cfg == "C5t" and world > 1:
            raise SystemExit("C5t (corner tangent) is single-GPU")
        if dtype == "f32" and "matrix" in self.modes and not (
                prob.form in (fi.DIFFUSION, fi.MASS, fi.MASS_DIFFUSION) and prob.p <= 2):
            raise SystemExit("fp32 matrices are built for the scalar forms at p <= 2")
        if dtype == "f32" and "csr" in self.modes:
            raise SystemExit("CSR assembly is built for fp64 element matrices")
        self.tdt = torch.float64 if dtype == "f64" else torch.float32
        self.dtc = fe.F64 if dtype == "f64" else fe.F32
        D, nb = prob.ncomp, prob.nb
        if cfg == "C5t":
            sl = slabs.Slab(0, 1, 0, prob.n_elems, 0, prob.coords.shape[0], 0, prob.n_nodes, 0)
            lc, lconn, ldc = prob.coords, prob.conn, prob.dof_conn
        elif "csr" in self.modes and world > 1:
            # N2 with row ownership: the slab plus the first cell layer above, so the rank's owned
            # block rows of the global CSR matrix are complete without communication
            sl = slabs.ghost_slab_of(prob.shape, prob.p, world, rank)
            lc, lconn, ldc = slabs.local_arrays(sl, prob.coords, prob.conn, prob.dof_conn)
        else:
            sl = slabs.slab_of(prob.shape, prob.p, world, rank)
            # N > 1: the slab's boundary layers first, so the boundary-first residual step
            # needs two launches instead of three (slabs.boundary_first_order)
            self.order = (slabs.boundary_first_order(sl, prob.shape)
                          if world > 1 and "residual" in self.modes else None)
            lc, lconn, ldc = slabs.local_arrays(sl, prob.coords, prob.conn, prob.dof_conn,
                                                self.order)
        self.sl = sl
        e0, e1 = sl.elem_begin, sl.elem_end
        self.El = El = e1 - e0
        order = getattr(self, "order", None)
        self.bfirst = order is not None
        cells = slice(e0, e1) if order is None else e0 + order
        self.mesh = fe.Mesh(torch.from_numpy(lc), torch.from_numpy(lconn), prob.p, prob.q1d,
                            dof_conn=torch.from_numpy(ldc), n_nodes=sl.n_nodes, device=dev)

        def dslice(a):
            return None if a is None else torch.from_numpy(np.ascontiguousarray(a[cells])).to(dev, self.tdt)

        self.mat_a, self.mat_b = dslice(prob.mat_a), dslice(prob.mat_b)
        self.u_loc = np.ascontiguousarray(prob.u[sl.node_begin:sl.node_end])
        self.u = torch.from_numpy(self.u_loc).to(dev, self.tdt)
        self.K = (torch.empty((El, D * nb, D * nb), dtype=self.tdt, device=dev)
                  if "matrix" in self.modes else None)
        self.peer = None
        if world > 1 and exchange == "peer" and "residual" in self.modes and not self.fused:
            if dtype != "f64":
                raise SystemExit("--exchange peer is built for fp64 residuals")
            self.peer = slabs.PeerExchange(sl, prob.shape, prob.p, D, dev)
            self.r = self.peer.r
            self.tiny = torch.zeros(1, dtype=torch.float32, device=dev)
        else:
            self.r = torch.zeros((sl.n_nodes, D), dtype=self.tdt, device=dev)
        self.csr = fe.CSR(self.mesh, D) if "csr" in self.modes else None
        self.csr_vals = (torch.zeros(self.csr.nnz, dtype=torch.float64, device=dev)
                         if self.csr is not None else None)
        self.stream = torch.cuda.current_stream(dev)
        self.comm_stream = torch.cuda.Stream(dev) if world > 1 else None
        self.bufs = [None]
        self.bev = torch.cuda.Event()   # boundary -> exchange dependency (preallocated)
        self.side = (torch.cuda.Stream(dev) if "matrix" in self.modes and "residual" in self.modes
                     and not self.fused and self.peer is None else None)
        # C2 step (B200, graph replay): forking the residual branch before the matrix kernel
        # 0.4876 -> 0.4804 ms (eager 0.5067 -> 0.4884); FEB200_BENCH_FORK=late forks after it
        self.fork_early = os.environ.get("FEB200_BENCH_FORK", "early") == "early"

    def events(self, n):
        """Preallocated kernel events: rec[i][mode] = (start, end) for step i."""
        E = self.torch.cuda.Event
        return [{m: (E(enable_timing=True), E(enable_timing=True)) for m in self.kmodes}
                for _ in range(n)]

    def step(self, rec=None):
        # every call goes to the CURRENT stream (the capture stream under --graph)
        fe, prob, mesh = self.fe, self.prob, self.mesh
        st = self.torch.cuda.current_stream(self.dev)
        mat = (prob.mat_kind, self.mat_a, self.mat_b)
        u, r, El, K = self.u, self.r, self.El, self.K
        comm = self.comm_stream if self.world > 1 else None
        if self.fused:
            r.zero_()
            if rec:
                rec["matrix+residual"][0].record(st)

            def evaluate_f(lo, hi):
                fe.fe_eval_matrix_residual(mesh.handle, prob.form, fe.F64, *mat, u, lo, hi,
                                           K[lo:hi], None, r, st)

            self.bufs[0] = self.slabs.residual_overlapped(evaluate_f, r, self.sl, prob.shape, comm,
                                                          self.bufs[0], events=self.bev,
                                                          boundary_first=self.bfirst)
            if rec:
                rec["matrix+residual"][1].record(st)
            return
        early = self.side is not None and self.fork_early
        if early:
            # the residual branch depends only on the step's inputs, not on K: fork it before
            # the matrix kernel, so that its zeroing runs beside the matrix kernel and its CTAs
            # take the SMs the matrix kernel's tail frees
            self.side.wait_stream(st)
        if "matrix" in self.modes:
            if rec:
                rec["matrix"][0].record(st)
            fe.fe_eval_element_matrices(mesh.handle, prob.form, self.dtc, *mat,
                                        u if prob.form == fi.CONVECTIVE else None, 0, El, K, st)
            if rec:
                rec["matrix"][1].record(st)
        if "csr" in self.modes:
            self.csr_vals.zero_()
            if rec:
                rec["csr"][0].record(st)
            self.csr.assemble(K, values=self.csr_vals, stream=st)
            if rec:
                rec["csr"][1].record(st)
        if "residual" in self.modes and self.peer is not None:
            if rec:
                rec["residual"][0].record(st)

            def evaluate_peer(windows):
                fe.fe_eval_residual_peer(mesh.handle, prob.form, *mat, u, 0, El, None, r, windows, st)

            # zero -> device barrier (tiny NCCL all-reduce) -> fused residual + exchange over
            # peer memory -> device barrier
            import torch.distributed as dist
            self.peer.residual(evaluate_peer, lambda: dist.all_reduce(self.tiny))
            if rec:
                rec["residual"][1].record(st)
        elif "residual" in self.modes:
            # matrix + residual steps: the residual runs on a side stream (forked before the
            # matrix kernel by default, see fork_early; else after it was queued); the current
            # stream joins it at the end of the step
            side = self.side
            if side is not None and not early:
                side.wait_stream(st)
            with self.torch.cuda.stream(side if side is not None else st):
                rst = self.torch.cuda.current_stream(self.dev)
                r.zero_()
                if rec:
                    rec["residual"][0].record(rst)

                def evaluate(lo, hi):
                    fe.fe_eval_residual(mesh.handle, prob.form, self.dtc, *mat, u, lo, hi, None, r,
                                        rst)

                # boundary-first residual; for N > 1 the interface exchange overlaps the interior
                self.bufs[0] = self.slabs.residual_overlapped(evaluate, r, self.sl, prob.shape, comm,
                                                              self.bufs[0], events=self.bev,
                                                              boundary_first=self.bfirst)
                if rec:
                    rec["residual"][1].record(rst)
            if side is not None:
                st.wait_stream(side)

    def close(self):
        if self.peer is not None:
            self.peer.close()
        if self.csr is not None:
            self.csr.close()
        self.mesh.close()


def _barrier(torch, dist, world, local_rank, dev):
    if world > 1:
        dist.barrier(device_ids=[local_rank])
    torch.cuda.synchronize(dev)


L2_BYTES = 126 * 2 ** 20


def step_bytes(run):
    """Algorithmic HBM bytes of one step of a Runner (all its modes): when they do not exceed a
    few L2 capacities, the timed loop flushes L2 between steps (timing rules)."""
    prob = run.prob
    esize = 8 if run.dtype == "f64" else 4
    tot = 0.0
    for m in run.modes:
        if m == "csr":
            continue
        tot += alg_bytes(prob.form, m, prob.p, prob.nb, prob.nq, prob.ncomp, prob.mat_kind,
                         esize) * run.El
    return tot


def timed_run(run, steps, warmup, world, local_rank, window_s=1.2, graph=False):
    """W warm-up steps; then, under the clock sampler, untimed repeats (>= 0.25 s), EXACTLY K
    timed steps bracketed by barrier + synchronize with CUDA events on the launching stream
    (per-step and per-kernel events preallocated), and untimed repeats until the sampler
    window is >= window_s.  Returns the max-over-ranks timings."""
    import torch
    import torch.distributed as dist
    dev, st = run.dev, run.stream
    for _ in range(warmup):
        run.step()
    _barrier(torch, dist, world, local_rank, dev)
    graph_error = None
    if graph:
        # the whole step captured once into a CUDA graph (slabs.StepGraph); the timed loop
        # replays it (per-kernel events are not recorded inside the graph: kernel times come
        # from an eager pass after the timed region).  A failed capture falls back to eager.
        try:
            gr = run.slabs.StepGraph(run.step, dev)
        except Exception as ex:  # noqa: BLE001 - reported in the JSON line
            graph, graph_error = False, f"{type(ex).__name__}: {ex}"[:300]
            print(f"bench: CUDA-graph capture failed, eager steps: {graph_error}", file=sys.stderr)
            torch.cuda.synchronize(dev)
        if world > 1:
            # every rank replays, or none does: the NCCL P2P calls of an eager step and the
            # captured ones of a replayed step must pair up across ranks
            ok = torch.tensor([1 if graph else 0], device=dev, dtype=torch.int32)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if graph and int(ok[0]) == 0:
                graph, graph_error = False, "capture failed on another rank: eager steps on all"
        _barrier(torch, dist, world, local_rank, dev)
    if graph:
        eager_step = run.step
        run.step = lambda rec=None: gr.replay()
    # step-time estimate (same on every rank: NCCL steps must match in count)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(2):
        run.step()
    b.record(st)
    _barrier(torch, dist, world, local_rank, dev)
    est = a.elapsed_time(b) / 2
    if world > 1:
        t = torch.tensor([est], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        est = float(t[0])
    est = max(est, 1e-3)
    n_pre = int(np.ceil(250.0 / est)) if window_s > 0 else 0
    n_post = max(0, int(np.ceil((window_s * 1e3 - 250.0 - steps * est) / est))) if window_s > 0 else 0
    ev_step = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    # L2 flush between timed steps when a step's working set is small (C4: ~260 MB f64, ~150 MB
    # f32): a write of 2 x L2 outside the per-step events; the step time is then the sum of the
    # per-step event times
    flush = step_bytes(run) < 4 * L2_BYTES
    fbuf = torch.empty(2 * L2_BYTES // 8, dtype=torch.float64, device=dev) if flush else None
    ev_beg = [torch.cuda.Event(enable_timing=True) for _ in range(steps)] if flush else None
    rec = run.events(steps)
    fe = run.fe
    with ClockSampler(local_rank) as clk:
        for _ in range(n_pre):
            run.step()
        _barrier(torch, dist, world, local_rank, dev)
        n_launch0 = fe.fe_launch_count()
        h0 = time.perf_counter()
        ev_step[0].record(st)
        for i in range(steps):
            if flush:
                fbuf.zero_()
                ev_beg[i].record(st)
            run.step(rec[i])
            ev_step[i + 1].record(st)
        h1 = time.perf_counter()
        _barrier(torch, dist, world, local_rank, dev)
        launches = fe.fe_launch_count() - n_launch0
        for _ in range(n_post):
            run.step()
        _barrier(torch, dist, world, local_rank, dev)
    host_us = (h1 - h0) / steps * 1e6
    if graph:
        run.step = eager_step
        # graph nodes: count the kernels of one eager step (the graph replays exactly these)
        n0 = fe.fe_launch_count()
        run.step()
        launches = (fe.fe_launch_count() - n0) * steps
        _barrier(torch, dist, world, local_rank, dev)
    early = getattr(run, "fork_early", False)
    if graph or early:
        # per-kernel times from an eager pass after the timed region, each kernel on its own:
        # with the early fork the residual's events would span the matrix kernel it waits
        # behind, so this pass runs the step with the two kernels serialised
        run.fork_early = False
        for i in range(steps):
            run.step(rec[i])
        _barrier(torch, dist, world, local_rank, dev)
        run.fork_early = early
    if flush:
        per_step = [ev_beg[i].elapsed_time(ev_step[i + 1]) for i in range(steps)]
        total = float(sum(per_step))
    else:
        total = ev_step[0].elapsed_time(ev_step[steps])
        per_step = [ev_step[i].elapsed_time(ev_step[i + 1]) for i in range(steps)]
    per_kern = {m: [rec[i][m][0].elapsed_time(rec[i][m][1]) for i in range(steps)]
                for m in run.kmodes}
    if world > 1:
        vec = [total] + per_step + [x for m in run.kmodes for x in per_kern[m]]
        t = torch.tensor(vec, device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t = t.tolist()
        total, per_step = t[0], t[1:1 + steps]
        off = 1 + steps
        for m in run.kmodes:
            per_kern[m], off = t[off:off + steps], off + steps
    return {"total_ms": total, "per_step": per_step, "per_kern": per_kern, "l2_flush": flush,
            "launches": launches, "clocks": clk.summary(), "host_us_per_step": host_us,
            "graph": graph, "graph_error": graph_error,
            "untimed_repeats": {"before": n_pre, "after": n_post}}


def roofline_for(prob, mode, kern_ms, El, dtype, csr_nnz=0.0, cfg=""):
    """Roofline of one kernel of the step: algorithmic bytes and flops per cell
    x cells per launch / the kernel's mean launch duration, against the measured HBM copy
    bandwidth or the measured FP64 (DFMA / DMMA) peak, whichever bounds it."""
    nb, nq, D = prob.nb, prob.nq, prob.ncomp
    esize = 8 if dtype == "f64" else 4
    pk_b, src_b = hbm_peak_gbs()
    t_s = kern_ms * 1e-3
    if mode == "matrix+residual":
        rf = roofline_for(prob, "matrix", kern_ms, El, dtype, csr_nnz, cfg)
        by = rf["alg_bytes_per_cell"] * El + (4 * nb + 3 * D * prob.p ** 3 * 8) * El
        fl = rf["alg_flops_per_cell"] * El + 2 * nb * nb * El      # r_e = K_e u_e
        fpk, fsrc = fp64_peak_tflops("dfma_tflops_sustained")
        if fl / (fpk * 1e12) >= by / (pk_b * 1e9):
            base = {"bound": "alu", "achieved": fl / t_s / 1e12, "peak": fpk, "unit": "TFLOP/s",
                    "frac": fl / t_s / 1e12 / fpk, "peak_source": fsrc}
        else:
            base = {"bound": "hbm", "achieved": by / t_s / 1e9, "peak": pk_b, "unit": "GB/s",
                    "frac": by / t_s / 1e9 / pk_b, "peak_source": src_b}
        rf.update(base)
        rf.update({"kernel": f"matrix+residual fused ({fi.FORM_NAMES[prob.form]}, Q{prob.p}, "
                             "sum-factorised, r_e = K_e u_e)",
                   "kernel_ms": kern_ms, "alg_flops_per_cell": fl / El,
                   "alg_bytes_per_cell": by / El, "achieved_gbs": by / t_s / 1e9,
                   "achieved_tflops": fl / t_s / 1e12, "traffic": None})
        return rf
    fl_lean = alg_flops(prob.form, mode, nb, nq) * El
    if mode == "matrix":
        sf = uses_sf_matrix(prob.form, prob.p) or (
            prob.form in (fi.ELASTICITY, fi.CONVECTIVE, fi.VECTOR_MASS) and prob.p <= 2
            and os.environ.get("FEB200_MATRIX_IMPL", "") != "dense")
    elif mode == "residual":
        sf = uses_sf_residual(prob.p)
    else:
        sf = False
    impl = "atomic-scatter" if mode == "csr" else ("sum-factorised" if sf else "dense-table")
    if not sf:
        fl = fl_lean
    elif mode == "matrix" and uses_sf_matrix(prob.form, prob.p):
        fl = sf_matrix_flops(prob.form, prob.p) * El
    elif mode == "matrix" and prob.form in (fi.ELASTICITY, fi.CONVECTIVE) and prob.p == 2:
        fl = sf_vector_matrix_flops(prob.form, prob.p) * El
        impl = "sum-factorised, pipelined"
    elif mode == "matrix":
        fl = fl_lean  # single-stage vector SF kernel: flop count not modelled, lean dense count
    else:
        fl = sf_residual_flops(prob.form, prob.p) * El
    by = alg_bytes(prob.form, mode, prob.p, nb, nq, D, prob.mat_kind, esize, csr_nnz) * El
    if dtype == "f32" and mode != "matrix":   # fp32 matrices contract in fp64
        # mixed precision: the 1D contractions run in fp32, the per-qp geometry and flux in fp64
        # (k_residual_sf keeps them fp64 for accuracy), so the ALU floor is the sum of the two
        # parts at their own peaks: fp32 74.4 TFLOP/s (derived) and the measured DFMA peak
        f64pk, _ = fp64_peak_tflops("dfma_tflops_sustained")
        n_ = prob.p + 1
        f_geo = n_ ** 3 * (100 + 40 * D)
        f_con = sf_residual_flops(prob.form, prob.p) - f_geo
        pk_f = (f_con + f_geo) / (f_con / 74.4 + f_geo / f64pk)
        src_f = (f"blended: contractions {f_con:.0f} flop/cell at the derived fp32 peak 74.4 TFLOP/s "
                 f"(148 SM x 128 lanes x 2 x 1.965 GHz) + geometry/flux {f_geo:.0f} flop/cell at the "
                 f"measured DFMA peak {f64pk:.2f} TFLOP/s")
        fbound = "alu"
    elif impl.startswith("sum-factorised") or mode == "csr":
        pk_f, src_f = fp64_peak_tflops("dfma_tflops_sustained")
        fbound = "alu"
    else:
        pk_f, src_f = fp64_peak_tflops("dmma_m16n8k4_tflops_sustained")
        fbound = "tensor"
    if fl / (pk_f * 1e12) >= by / (pk_b * 1e9):
        rf = {"bound": fbound, "achieved": fl / t_s / 1e12, "peak": pk_f, "unit": "TFLOP/s",
              "frac": (fl / t_s / 1e12) / pk_f, "peak_source": src_f}
    else:
        rf = {"bound": "hbm", "achieved": by / t_s / 1e9, "peak": pk_b, "unit": "GB/s",
              "frac": (by / t_s / 1e9) / pk_b, "peak_source": src_b}
    rf.update({"kernel": f"{mode} ({fi.FORM_NAMES[prob.form]}, Q{prob.p}, {impl})",
               "lean_dense_flops_per_cell": fl_lean / El,
               "effective_lean_tflops": fl_lean / t_s / 1e12,
               "kernel_ms": kern_ms, "alg_flops_per_cell": fl / El,
               "alg_bytes_per_cell": by / El, "cells_per_launch": El,
               "achieved_gbs": by / t_s / 1e9, "achieved_tflops": fl / t_s / 1e12,
               "traffic": None})
    prof_ = os.path.join(ROOT, "profiles", f"traffic_{cfg}_{mode}.json")
    if os.path.exists(prof_):
        try:
            rf["traffic"] = json.load(open(prof_)).get("dram_bytes_per_launch")
        except Exception:
            pass
    return rf


def summarize(run, res, dtype):
    """Per-mode kernel statistics, result throughput and rooflines of a run."""
    prob, El = run.prob, run.El
    esize = 8 if dtype == "f64" else 4
    csr_nnz = (run.csr.nnz / El) if run.csr is not None else 0.0
    modes = {}
    for m in run.kmodes:
        ks = step_stats(res["per_kern"][m])
        rf = roofline_for(prob, m, ks["mean"], El, dtype, csr_nnz, run.cfg)
        rb = sum(result_bytes(prob, mm, esize) for mm in m.split("+") if mm != "csr")
        modes[m] = {"kernel_ms": ks, "cells_per_s": El / (ks["mean"] * 1e-3),
                    "result_mb_per_s": (rb * El / prob.n_elems) / (ks["tww"] * 1e-3) / 1e6,
                    "roofline": rf}
    return modes


def measure_sub(cfg_name, args, world, rank, local_rank, dev):
    """A sub-result of the default line: one more BASELINE form / mode measured like the
    headline (warm-up, K timed steps, clocks over >= 1.2 s)."""
    import torch
    cfg, dt = split_cfg(cfg_name)
    dtype = dt or "f64"
    run = Runner(cfg, dtype, world, rank, dev, args.exchange)
    try:
        res = timed_run(run, args.steps, args.warmup, world, local_rank, args.clock_window,
                        graph=args.graph)
        modes = summarize(run, res, dtype)
        st = step_stats(res["per_step"])
        out = {"config": config_dict(cfg, run.prob, run.modes, world, args.exchange, dtype),
               "l2_flush": res["l2_flush"],
               "ms_per_step": res["total_ms"] / args.steps, "step_ms": st,
               "cells_per_s": run.prob.n_elems / (res["total_ms"] / args.steps * 1e-3),
               "modes": {m: {"kernel_ms": v["kernel_ms"], "cells_per_s": v["cells_per_s"],
                             "result_mb_per_s": v["result_mb_per_s"],
                             "roofline": {k: v["roofline"][k] for k in (
                                 "bound", "achieved", "peak", "unit", "frac", "kernel",
                                 "alg_bytes_per_cell", "alg_flops_per_cell", "traffic")}}
                         for m, v in modes.items()},
               "gpu_launches": int(res["launches"]), "clocks": res["clocks"],
               "host_us_per_step": res["host_us_per_step"], "graph": bool(res["graph"]),
               "graph_error": res["graph_error"]}
    finally:
        run.close()
        del run
        torch.cuda.synchronize(dev)
        torch.cuda.empty_cache()
    return out


# ----------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2", choices=sorted(WORKLOADS))
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--clock-window", type=float, default=1.2,
                    help="seconds of the clock-sampling window around the timed region (untimed "
                         "repeats before/after it); 0 = timed region only (profiler runs)")
    ap.add_argument("--sub-configs", default=None,
                    help="comma-separated per-form sub-results for the line (default with "
                         f"--config C2: {','.join(SUB_CONFIGS)}; 'none' to skip)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "peer"],
                    help="N > 1 residual: interface planes by NCCL send/recv overlapped with the "
                         "interior (default) or added by the residual kernel itself into the "
                         "neighbours' vectors over peer memory (fe_eval_residual_peer)")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="capture each rank's whole step (boundary cells, exchange on the comm "
                         "stream, interior cells, plane adds) into a CUDA graph and time its "
                         "replays (kernel times from an eager pass); auto = on (falls back to "
                         "eager steps if the capture fails; C2 N=1: 0.560 vs 0.574 ms)")
    ap.add_argument("--fused", action="store_true",
                    help="C2-type steps: fe_eval_matrix_residual (K_e and r_e = K_e u_e from one "
                         "pass) instead of the separate matrix and residual kernels")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args, args.config)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    dev = torch.device("cuda", local_rank)
    cfg = args.config
    args.graph = args.graph in ("on", "auto")
    run = Runner(cfg, args.dtype, world, rank, dev, args.exchange, args.fused)
    prob, modes, El = run.prob, run.modes, run.El
    fe = run.fe

    res = timed_run(run, args.steps, args.warmup, world, local_rank, args.clock_window,
                    graph=args.graph)
    ms_step = res["total_ms"] / args.steps
    value = prob.n_elems / (ms_step * 1e-3)
    mode_sum = summarize(run, res, args.dtype)

    # alternative path of the same step, timed outside the timed region for the record:
    # the fused kernel when the step ran unfused, the two kernels when it ran fused
    fusable = (tuple(modes) == ("matrix", "residual") and args.dtype == "f64" and world == 1
               and prob.form in (fi.DIFFUSION, fi.MASS, fi.MASS_DIFFUSION) and prob.p <= 2)
    mesh, st, u, r, K = run.mesh, run.stream, run.u, run.r, run.K
    mat = (prob.mat_kind, run.mat_a, run.mat_b)
    fused_alt = unfused = None
    if fusable and not run.fused:
        n_f = 20
        fa, fb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fe.fe_eval_matrix_residual(mesh.handle, prob.form, fe.F64, *mat, u, 0, El, K, None, r, st)
        torch.cuda.synchronize(dev)
        fa.record(st)
        for _ in range(n_f):
            r.zero_()
            fe.fe_eval_matrix_residual(mesh.handle, prob.form, fe.F64, *mat, u, 0, El, K, None, r, st)
        fb.record(st)
        torch.cuda.synchronize(dev)
        f_ms = fa.elapsed_time(fb) / n_f
        fused_alt = {"step_ms": f_ms, "cells_per_s": prob.n_elems / (f_ms * 1e-3),
                     "note": "fe_eval_matrix_residual: K_e and r_e = K_e u_e from one kernel pass "
                             "(linear form, pin P8), r zeroing included; not the timed step "
                             "(bench.py --fused times it)"}
    if run.fused and world == 1:
        n_u = 20
        ea = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        tm = tr = 0.0
        for _ in range(n_u):
            ea[0].record(st)
            fe.fe_eval_element_matrices(mesh.handle, prob.form, fe.F64, *mat, None, 0, El, K, st)
            ea[1].record(st)
            r.zero_()
            fe.fe_eval_residual(mesh.handle, prob.form, run.dtc, *mat, u, 0, El, None, r, st)
            ea[2].record(st)
            torch.cuda.synchronize(dev)
            tm += ea[0].elapsed_time(ea[1])
            tr += ea[1].elapsed_time(ea[2])
        unfused = {"matrix_ms": tm / n_u, "residual_ms": tr / n_u, "step_ms": (tm + tr) / n_u,
                   "note": "separate fe_eval_element_matrices + fe_eval_residual, not the timed step"}

    # ---- end-to-end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        h_u = torch.from_numpy(run.u_loc).to(run.tdt).pin_memory()
        h_a = None if run.mat_a is None else run.mat_a.cpu().pin_memory()
        h_b = None if run.mat_b is None else run.mat_b.cpu().pin_memory()
        h_r = torch.empty_like(r, device="cpu").pin_memory()
        h_K = torch.empty(K.shape, dtype=K.dtype).pin_memory() if K is not None else None
        n_e2e = max(3, min(args.steps, 10))
        # pipelined: the read-back of step i (r, then K, on a copy stream) overlaps the input
        # copies and the kernels of step i+1, which write the other of two device K buffers
        Kbuf = [K, torch.empty_like(K) if K is not None else None]
        cs = torch.cuda.Stream(dev)
        ev_r = [torch.cuda.Event() for _ in range(2)]
        ev_K = [torch.cuda.Event() for _ in range(2)]
        ev_c = torch.cuda.Event()
        nst = [0]

        def e2e_step():
            i = nst[0]
            j = i & 1
            if K is not None:
                run.K = Kbuf[j]
                if i >= 2:
                    st.wait_event(ev_K[j])          # step i-2's K read back from this buffer
            if i >= 1:
                st.wait_event(ev_r[(i - 1) & 1])    # step i-1's r read back before re-zeroing
            u.copy_(h_u, non_blocking=True)
            if h_a is not None:
                run.mat_a.copy_(h_a, non_blocking=True)
            if h_b is not None:
                run.mat_b.copy_(h_b, non_blocking=True)
            run.step()
            ev_c.record(st)
            cs.wait_event(ev_c)
            with torch.cuda.stream(cs):
                h_r.copy_(r, non_blocking=True)
                ev_r[j].record(cs)
                if h_K is not None:
                    h_K.copy_(run.K, non_blocking=True)
                    ev_K[j].record(cs)
            nst[0] += 1

        e2e_step()
        st.wait_stream(cs)
        _barrier(torch, dist, world, local_rank, dev)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(n_e2e):
            e2e_step()
        st.wait_stream(cs)
        b.record(st)
        _barrier(torch, dist, world, local_rank, dev)
        e_ms = a.elapsed_time(b)
        h2d = h_u.numel() * h_u.element_size() + sum(
            x.numel() * x.element_size() for x in (h_a, h_b) if x is not None)
        d2h = h_r.numel() * h_r.element_size() + (
            h_K.numel() * h_K.element_size() if h_K is not None else 0)
        if world > 1:
            tt = torch.tensor([e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_ms = float(tt[0])
            tt = torch.tensor([h2d, d2h], device=dev, dtype=torch.float64)
            dist.all_reduce(tt)
            h2d, d2h = int(tt[0]), int(tt[1])
        # the PCIe roofline of this leg: the same read-back as one plain D2H copy of this rank's
        # biggest result buffer (best of 3), timed after the e2e region
        link = None
        hb, db = (h_K, Kbuf[0]) if h_K is not None else (h_r, r)
        if hb.numel() * hb.element_size() >= (64 << 20):
            la, lb_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            best = float("inf")
            for _ in range(3):
                la.record(st)
                hb.copy_(db, non_blocking=True)
                lb_.record(st)
                torch.cuda.synchronize(dev)
                best = min(best, la.elapsed_time(lb_))
            peak = hb.numel() * hb.element_size() / (best * 1e-3) / 1e9
            ach = d2h / world / (e_ms / n_e2e * 1e-3) / 1e9
            link = {"bound": "pcie_d2h", "achieved_gbs": ach, "peak_gbs": peak, "frac": ach / peak,
                    "note": "achieved = D2H bytes per step per rank / e2e step time; peak = one "
                            "plain pinned D2H copy of the largest result buffer on this box"}
        e2e = {"value": prob.n_elems / (e_ms / n_e2e * 1e-3), "unit": "cells/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": e_ms / n_e2e, "steps": n_e2e, "link": link,
               "note": "every step: pinned host inputs (u, material) H2D, the step, D2H of r"
                       + (" and K" if K is not None else "") + "; the read-back of a step overlaps "
                       "the next step (copy stream, two device K buffers)"}
        run.K = K
        del h_K, Kbuf
    launches = int(res["launches"])
    fork_early, has_side = run.fork_early, run.side is not None
    run.close()
    del run, mesh, K, r, u
    torch.cuda.synchronize(dev)
    torch.cuda.empty_cache()

    # ---- the other BASELINE forms / modes, each measured like the headline
    subs_req = args.sub_configs if args.sub_configs is not None else (
        ",".join(SUB_CONFIGS) if cfg == "C2" and not args.fused else "none")
    subs = {}
    for name in [s for s in subs_req.split(",") if s and s != "none"]:
        if name == "C5t" and world > 1:
            continue
        subs[name] = measure_sub(name, args, world, rank, local_rank, dev)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    dom = max(mode_sum, key=lambda m: mode_sum[m]["kernel_ms"]["mean"])
    roof = mode_sum[dom]["roofline"]
    cb = None
    if not args.no_cpu_baseline and world == 1:
        cb = cpu_baseline(prob, modes)

    line = {
        "metric": f"{cfg} cells evaluated per second ({'+'.join(modes)})",
        "value": value, "unit": "cells/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": config_dict(cfg, prob, modes, world, args.exchange, args.dtype),
        "stats": {"step_ms": step_stats(res["per_step"]),
                  "note": "per-step CUDA-event times (max over ranks); tww = mean without the "
                          "worst call (P:1158-1163)"},
        "modes": {m: {"kernel_ms": v["kernel_ms"], "cells_per_s": v["cells_per_s"],
                      "result_mb_per_s": v["result_mb_per_s"],
                      "roofline": {k: v["roofline"][k] for k in ("bound", "achieved", "unit", "frac")}}
                  for m, v in mode_sum.items()},
        "roofline": roof,
        "unfused": unfused,
        "fused": fused_alt,
        "cpu_baseline": cb,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": res["clocks"],
        "untimed_repeats": res["untimed_repeats"],
        "graph": bool(res["graph"]),
        "graph_error": res["graph_error"],
        "residual_fork": ("early" if fork_early else "late") if has_side else None,
        "l2_flush": res["l2_flush"],
        "host_us_per_step": res["host_us_per_step"],
        "configs": subs,
        "options": fe.get_options(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Where the e2e step's time goes (C2, one GPU): the bench's pipelined e2e loop with parts
switched off.  python tools/e2e_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

dev = torch.device("cuda", 0)
run = bench.Runner("C2", "f64", 1, 0, dev, "nccl", False)
st = run.stream if hasattr(run, "stream") else torch.cuda.current_stream()
K, r, u = run.K, run.r, run.u
h_u = torch.from_numpy(run.u_loc).to(run.tdt).pin_memory()
h_a = run.mat_a.cpu().pin_memory()
h_r = torch.empty_like(r, device="cpu").pin_memory()
h_K = torch.empty(K.shape, dtype=K.dtype).pin_memory()
Kbuf = [K, torch.empty_like(K)]
cs = torch.cuda.Stream(dev)


def loop(n, do_step=True, do_h2d=True, alt=True, do_r=True):
    ev_r = [torch.cuda.Event() for _ in range(2)]
    ev_K = [torch.cuda.Event() for _ in range(2)]
    ev_c = torch.cuda.Event()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with torch.cuda.stream(st):
        a.record(st)
        for i in range(n):
            j = i & 1 if alt else 0
            run.K = Kbuf[j]
            if i >= 2:
                st.wait_event(ev_K[j])
            if i >= 1 and do_r:
                st.wait_event(ev_r[(i - 1) & 1])
            if do_h2d:
                u.copy_(h_u, non_blocking=True)
                run.mat_a.copy_(h_a, non_blocking=True)
            if do_step:
                run.step()
            ev_c.record(st)
            cs.wait_event(ev_c)
            with torch.cuda.stream(cs):
                if do_r:
                    h_r.copy_(r, non_blocking=True)
                    ev_r[j].record(cs)
                h_K.copy_(run.K, non_blocking=True)
                ev_K[j].record(cs)
        st.wait_stream(cs)
        b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


print("stream", st, "graph attr", getattr(run, "graph", None))
for kw in ({}, {"do_step": False}, {"do_h2d": False}, {"do_r": False}, {"alt": False},
           {"do_step": False, "do_h2d": False, "do_r": False}):
    loop(2, **kw)
    print(kw, f"{loop(10, **kw):.2f} ms/step")

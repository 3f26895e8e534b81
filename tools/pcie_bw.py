"""Host <-> device copy bandwidth for the e2e leg (pinned host memory, one GPU).

    python tools/pcie_bw.py"""
import torch

n = 1546 * 1024 * 1024 // 8  # ~ the C2 step's K read-back
d = torch.empty(n, dtype=torch.float64, device="cuda")
h = torch.empty(n, dtype=torch.float64).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def chunked(k, dst, src):
    def f():
        cur = torch.cuda.current_stream()
        ev = torch.cuda.Event()
        ev.record(cur)
        m = (n + k - 1) // k
        for i in range(k):
            s = (s1, s2)[i & 1]
            s.wait_event(ev)
            with torch.cuda.stream(s):
                dst[i * m:(i + 1) * m].copy_(src[i * m:(i + 1) * m], non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    return f


for name, f in (("D2H one copy", lambda: h.copy_(d, non_blocking=True)),
                ("H2D one copy", lambda: d.copy_(h, non_blocking=True)),
                ("D2H 2 streams x 8 chunks", chunked(16, h, d)),
                ("H2D 2 streams x 8 chunks", chunked(16, d, h))):
    ms = timeit(f)
    print(f"{name:28s} {8 * n / ms / 1e6:8.1f} GB/s ({ms:.2f} ms)")

# the e2e pattern: per step an H2D of the inputs on the compute stream and a D2H of K on a copy
# stream, pipelined (does the opposite-direction H2D slow the D2H?)
hin = torch.empty(74 * 1024 * 1024 // 8, dtype=torch.float64).pin_memory()
din = torch.empty_like(hin, device="cuda")
cs = torch.cuda.Stream()
for with_h2d in (False, True):
    def pattern():
        st = torch.cuda.current_stream()
        for _ in range(10):
            if with_h2d:
                din.copy_(hin, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(st)
            cs.wait_event(ev)
            with torch.cuda.stream(cs):
                h.copy_(d, non_blocking=True)
        st.wait_stream(cs)
    ms = timeit(pattern, reps=2) / 10
    print(f"e2e pattern, H2D {'on ' if with_h2d else 'off'}: {ms:.2f} ms per step ({8 * n / ms / 1e6:.1f} GB/s D2H)")

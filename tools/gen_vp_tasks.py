"""Generate csrc/vp_tasks.h: the X-thread -> (cell, z pair, y pair) task maps of the pipelined
vector matrix kernel (k_matrix_vp.cu, p = 2, E = 2 cells per batch, 192 X threads per group).

K_e is staged in shared memory in its global row-major layout (the TMA bulk store copies it
verbatim), so the bank of a thread's K store is fixed by its task; this script searches (seeded
simulated annealing over a half-warp bank model of the STS.64 stores) for a permutation of the
tasks over the 192 lanes that minimises store wavefronts.  Pure layout; no FE arithmetic.

    python tools/gen_vp_tasks.py [iterations]
"""
import collections
import math
import os
import random
import sys

E, LANES = 2, 192


def full_tasks():
    return [(el, zp // 3, zp % 3, yp // 3, yp % 3) for el in range(E) for zp in range(9) for yp in range(9)]


def sym_tasks():
    out = []
    for el in range(E):
        for r in range(45):
            if r < 27:
                c, yp = r // 9, r % 9
                iz, jz = [(0, 1), (0, 2), (1, 2)][c]
                iy, jy = yp // 3, yp % 3
            else:
                rr = r - 27
                iz = jz = rr // 6
                iy, jy = [(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)][rr % 6]
            out.append((el, iz, jz, iy, jy))
    return out


def addrs(t, a, bb):
    el, iz, jz, iy, jy = t
    ib, jb = 3 * (iy + 3 * iz), 3 * (jy + 3 * jz)
    return el * 6561 + (ib + a) * 81 + 27 + jb + bb, el * 6561 + (27 + jb + bb) * 81 + ib + a


def half_waves(lane_addr):
    tot = 0
    for h in (0, 1):
        cnt, seen = collections.Counter(), set()
        for lane, ad in lane_addr:
            if lane // 16 != h or ad in seen:
                continue
            seen.add(ad)
            cnt[ad % 16] += 1
        if cnt:
            tot += max(cnt.values())
    return tot


def quarter_waves(lane_addr):
    """LDS.128: a quarter warp (8 lanes) per wavefront, extra wavefronts for distinct
    16-B addresses that share a 4-bank group."""
    tot = 0
    for qq in range(4):
        cnt, seen = collections.Counter(), set()
        for lane, ad in lane_addr:
            if lane // 8 != qq or ad in seen:
                continue
            seen.add(ad)
            cnt[(ad // 2) % 8] += 1
        if cnt:
            tot += max(cnt.values())
    return tot


def pair_list(sym):
    """(m, n) ordered pairs read by a task and the T1 vector they use: (pidx, transposed)."""
    if sym:
        out = []
        for op in range(9):
            m, n = op // 3, op % 3
            mm, nn = min(m, n), max(m, n)
            out.append((nn if mm == 0 else (2 + nn if mm == 1 else 5), m > n))
        return out
    return [(op, False) for op in range(9)]


def warp_cost(ws, sym):
    c = 0
    # T1 vector loads: 4 x LDS.128 + 1 x LDS.64 per pair; T1 slot [el][9 pairs][9 zidx][10]
    for pidx, tr in pair_list(sym):
        for h in range(5):
            la = []
            for lane, t in enumerate(ws):
                if t is None:
                    continue
                el, iz, jz, iy, jy = t
                zidx = jz * 3 + iz if tr else iz * 3 + jz
                la.append((lane, (el * 9 + pidx) * 90 + zidx * 10 + 2 * h))
            c += quarter_waves(la) if h < 4 else half_waves(la)
    for a in range(3):
        for bb in range(3):
            d = [(lane, addrs(t, a, bb)[0]) for lane, t in enumerate(ws) if t is not None]
            m = [(lane, addrs(t, a, bb)[1]) for lane, t in enumerate(ws)
                 if t is not None and (not sym or t[1] < t[2] or t[3] < t[4])]
            c += half_waves(d) + half_waves(m)
    return c


def anneal(tasks, sym, iters, seed):
    rnd = random.Random(seed)
    slots = tasks + [None] * (LANES - len(tasks))
    wc = [warp_cost(slots[w:w + 32], sym) for w in range(0, LANES, 32)]
    start = cur = sum(wc)
    for k in range(iters):
        temp = 2.0 * (1 - k / iters) + 0.02
        a, b = rnd.randrange(LANES), rnd.randrange(LANES)
        wa, wb = a // 32, b // 32
        if a // 16 == b // 16:
            continue
        slots[a], slots[b] = slots[b], slots[a]
        na = warp_cost(slots[wa * 32:wa * 32 + 32], sym)
        nb = warp_cost(slots[wb * 32:wb * 32 + 32], sym) if wb != wa else na
        d = (na + nb - wc[wa] - wc[wb]) if wb != wa else (na - wc[wa])
        if d <= 0 or rnd.random() < math.exp(-d / temp):
            wc[wa] = na
            if wb != wa:
                wc[wb] = nb
            cur += d
        else:
            slots[a], slots[b] = slots[b], slots[a]
    return start, cur, slots


def pack(t):
    return -1 if t is None else t[0] | (t[1] << 4) | (t[2] << 8) | (t[3] << 12) | (t[4] << 16)


def main():
    """usage: gen_vp_tasks.py [ITERS] [--full ITERS:SEED] [--sym ITERS:SEED]
    (the committed header: --full 900000:21 --sym 400000:2107, about 1.5 h / 0.5 h of CPU)"""
    args = sys.argv[1:]
    iters = int(args.pop(0)) if args and not args[0].startswith("--") else 30000
    params = {"full": (iters, 2107), "sym": (iters, 2107)}
    while args:
        k, v = args.pop(0).lstrip("-"), args.pop(0)
        params[k] = tuple(int(x) for x in v.split(":"))
    lines = ["// Generated by tools/gen_vp_tasks.py -- X-thread task maps of k_matrix_vp.cu (p = 2, E = 2).",
             "// entry = el | iz << 4 | jz << 8 | iy << 12 | jy << 16, -1 = idle lane.", "#pragma once", ""]
    for name, tasks, sym in (("full", full_tasks(), False), ("sym", sym_tasks(), True)):
        it, seed = params[name]
        s, c, slots = anneal(tasks, sym, it, seed)
        print(f"{name}: shared wavefronts per item {s} -> {c}")
        vals = ", ".join(str(pack(t)) for t in slots)
        lines.append(f"// {name}: modelled shared wavefronts (T1 loads + K stores) per item {s} (natural order) -> {c}"
                     f" ({it} iterations, seed {seed})")
        lines.append(f"__device__ const int vp_tasks_{name}[{LANES}] = {{{vals}}};")
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "paper_2107_04121_b200", "csrc", "vp_tasks.h")
    open(out, "w").write("\n".join(lines) + "\n")
    print(out)


if __name__ == "__main__":
    main()

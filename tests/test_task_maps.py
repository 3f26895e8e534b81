"""CPU checks of the generated lane -> task maps of the pipelined matrix kernels (pure layout:
a map must assign every task of a batch to exactly one lane, or the kernel silently skips or
duplicates K blocks).  sfp_tasks.h: k_matrix_sfp's register-blocked X role (tools/gen_sfp_tasks.c);
vp_yb3_tasks.h: the YB3 X role of k_matrix_vp (tools/gen_vp_yb3_tasks.c)."""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2107_04121_b200", "csrc")


def _array(name, fname):
    src = open(os.path.join(CSRC, fname)).read()
    m = re.search(name + r"\[[^\]]*\](?:\[[^\]]*\])?\s*=\s*\{(.*?)\};", src, re.S)
    assert m, name
    return [int(v) for v in re.findall(r"-?\d+", m.group(1))]


def test_sfp_yb3_map_is_a_permutation_of_the_batch_tasks():
    # E = 8 cells x (9 off-diagonal (z pair, iy) tasks + 6 diagonal half tasks) = 120 tasks
    v = _array("sfp_tasks_yb3", "sfp_tasks.h")
    assert len(v) == 128
    tasks = [t for t in v if t >= 0]
    assert sorted(tasks) == list(range(120))
    assert v.count(-1) == 8


def _decode_sfp(t):
    """The decode of k_matrix_sf.cu (YB = 3): (cell, iz, jz, [(iy, jy)] x 3)."""
    if t < 72:
        el, r = divmod(t, 9)
        zp, iy = divmod(r, 3)
        iz, jz = zp >> 1, (1 if zp == 0 else 2)
        return el, iz, jz, [(iy, 0), (iy, 1), (iy, 2)]
    el, r = divmod(t - 72, 6)
    hf, iz = r & 1, r >> 1
    return el, iz, iz, [(hf, hf), (hf, hf + 1), (2 * hf, 2)]


def test_sfp_yb3_tasks_cover_the_symmetric_half_of_every_cell_once():
    """Each stored K block (z pair, y pair) of the upper triangle -- and through the mirror
    the whole 27 x 27 matrix -- is produced by exactly one (lane, k)."""
    seen = {}
    for t in range(120):
        el, iz, jz, yps = _decode_sfp(t)
        for iy, jy in yps:
            key = (el, iz, jz, iy, jy)
            assert key not in seen
            seen[key] = t
    for el in range(8):
        for iz in range(3):
            for jz in range(iz, 3):
                for iy in range(3):
                    for jy in range(3):
                        if iz == jz and jy < iy:
                            continue
                        assert (el, iz, jz, iy, jy) in seen


def test_vp_yb3_map_lanes_cover_both_item_kinds_once():
    v = _array("vp_yb3_tasks", "vp_yb3_tasks.h")
    assert len(v) == 3 * 64
    for g in range(3):
        full, sym = set(), set()
        for x in v[64 * g:64 * (g + 1)]:
            iy = x & 3
            if iy == 3:
                continue
            fel, fiz, fjz = (x >> 2) & 3, (x >> 4) & 3, (x >> 6) & 3
            sel, siz, sjz = (x >> 8) & 3, (x >> 10) & 3, (x >> 12) & 3
            if fel != 3:
                assert (fel, fiz, fjz, iy) not in full
                full.add((fel, fiz, fjz, iy))
            if sel != 3:
                assert siz <= sjz and (sel, siz, sjz, iy) not in sym
                sym.add((sel, siz, sjz, iy))
        # full items: every ordered z pair and iy of both cells; symmetric: z pairs iz <= jz
        assert full == {(e, a, b, y) for e in range(2) for a in range(3) for b in range(3) for y in range(3)}
        assert sym == {(e, a, b, y) for e in range(2) for a in range(3) for b in range(a, 3) for y in range(3)}

"""Per-role wait profile of the pipelined SF matrix kernel (build with -DFEB200_SFP_PROF).

    FEB200_LIB_PATH=.../lib_X.so python tools/sfp_prof.py [config]"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import fe_inputs as fi  # noqa: E402
import paper_2107_04121_b200 as fe  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
pr = fi.corner_subproblem(fi.make_config("C5"), 64) if cfg == "C5t" else fi.make_config(cfg)
VP = pr.form in (fi.ELASTICITY, fi.CONVECTIVE)
state = torch.from_numpy(pr.u).cuda() if pr.form == fi.CONVECTIVE else None
mesh = fe.Mesh(torch.from_numpy(pr.coords), torch.from_numpy(pr.conn), pr.p, pr.q1d,
               dof_conn=torch.from_numpy(pr.dof_conn), n_nodes=pr.n_nodes)
a = None if pr.mat_a is None else torch.from_numpy(pr.mat_a).cuda()
b = None if pr.mat_b is None else torch.from_numpy(pr.mat_b).cuda()
lib = fe.lib()
buf = (ctypes.c_ulonglong * 16)()
FUSED = os.environ.get("SFP_PROF_FUSED") == "1"
uu = torch.from_numpy(pr.u).cuda()


def run():
    if FUSED:
        mesh.matrix_residual(pr.form, uu, pr.mat_kind, a, b)
    else:
        mesh.element_matrices(pr.form, pr.mat_kind, a, b, state)


for _ in range(3):
    run()
(lib.fe_debug_vp_prof if VP else lib.fe_debug_sfp_prof)(buf, 1)
n = 20
for _ in range(n):
    run()
(lib.fe_debug_vp_prof if VP else lib.fe_debug_sfp_prof)(buf, 1)
v = np.array(list(buf), dtype=np.float64)
names = (["G bar", "L wait emptyL", "G wait fullL", "G wait emptyT", "X wait fullT", "X bar2", "X bar3"]
         if VP else ["L wait conn", "L wait emptyL", "G wait fullL", "G wait emptyT", "X wait fullT",
                     "X bar1", "X bar2", "X wait fullU"])
warps = {0: v[12], 1: v[13], 2: v[14]}
tot = {0: v[8], 1: v[9], 2: v[10]}
role = [1 if VP else 0, 0, 1, 1, 2, 2, 2, 2]
for k, nm in enumerate(names):
    r = role[k]
    print(f"{nm:16s} {v[k] / max(tot[r], 1):6.1%} of role time")
for r, nm in enumerate("LGX"):
    print(f"{nm}: warps {warps[r] / n:.0f}, mean cycles per warp per launch {tot[r] / max(warps[r], 1):.0f}")

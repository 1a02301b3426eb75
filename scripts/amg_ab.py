"""Time the config-3 block-AMG setup and hash its level operators (A/B of setup kernels via
environment switches, e.g. CF_SPGEMM_GROUPED=1).  usage: python scripts/amg_ab.py [cfg3|cfg2]"""
import hashlib
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1806_09924_b200 as cf

d, n0, r = {"cfg3": (3, 8, 4), "cfg2": (2, 8, 8)}[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
P = cf.Problem(d, 10.0, n0, r)
mat = cf.Material(eps_mode=1, eps_fixed=2 * P.h, kappa_factor=1e-12 / P.h)
reg = cf.resolve_regularization(P, mat, cf.slit_band_edge(P, mat))
st = cf.make_initial_state(P, mat).get()
x = torch.from_numpy(st["solution"]).cuda()
x[:P.n_u] = 1e-3 * torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, P.n_u)).cuda()
pt = torch.from_numpy(st["phi_old"]).cuda()
cs = cf.build_constraints(P)
J = cf.assemble_jacobian(P, cs, mat, reg, x, pt)
u = J.M_uu
A = cf.CsrMatrix(u.rows, u.cols, u.ptr, u.col, u.val)
B = cf.rigid_body_modes(P, cs)
node = np.repeat(np.arange(P.n_vertices, dtype=np.int32), d)
times = []
for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    h = cf.build_amg(A, node, B)
    torch.cuda.synchronize()
    times.append(1e3 * (time.perf_counter() - t))
hs = hashlib.sha256()
for lev in range(h.n_levels() - 1):
    for which in range(2):
        m = h.level_matrix(lev, which)
        for arr in (m.ptr, m.col, m.val):
            hs.update(np.ascontiguousarray(arr).tobytes())
print(f"build_amg(M_uu) ms: {' '.join(f'{t:.1f}' for t in times)}  levels {h.n_levels()}  hash {hs.hexdigest()[:16]}")
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    h = cf.build_amg(A, node, B)
    torch.cuda.synchronize()
rows = sorted(((getattr(e, "device_time_total", 0) or 0) / 1e3, e.count, e.key) for e in prof.key_averages())[::-1]
print(f"  kernel total {sum(r[0] for r in rows):.1f} ms")
for t, c, k in rows[:22]:
    print(f"  {t:8.2f} ms {c:5d} {k[:90]}")
for lev in range(h.n_levels() - 1):
    print("level", lev, h.level_info(lev))

"""Kernel breakdown of one config-3 u-V-cycle and one GMRES-iteration worth of operator applies,
with per-level sizes.  usage: python scripts/vcycle_profile.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import bench
import paper_1806_09924_b200 as cf

P, mat, reg = bench.sneddon_setup(cf, bench.CFG3)
st = cf.make_initial_state(P, mat)
cf.newton_active_set_step(st, mat, P, reg, cf.SolverOptions())
g = st.get()
x = torch.from_numpy(g["solution"]).cuda()
po = torch.from_numpy(g["phi_old"]).cuda()
s = torch.cuda.current_stream()
out = bench.vcycle_leg(cf, P, mat, reg, x, po, s)
print(out)
xs, pon = g["solution"], g["phi_old"]
act = np.nonzero(xs[P.n_u:] == pon)[0]
cs = cf.build_constraints(P, True, {int(P.n_u + v): float(pon[v]) for v in act})
J = cf.assemble_jacobian(P, cs, mat, reg, x, po)
node_u = np.repeat(np.arange(P.n_vertices, dtype=np.int32), P.dim)
hu = cf.build_amg(cf.CsrMatrix.from_block(J, 0), node_u, cf.rigid_body_modes(P, cs))
for lev in range(hu.n_levels() - 1):
    print("level", lev, hu.level_info(lev))
r = torch.randn(P.n_u, dtype=torch.float64, device="cuda")
for _ in range(3):
    hu.v_cycle(r)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(10):
        hu.v_cycle(r)
    torch.cuda.synchronize()
rows = sorted(((getattr(e, "device_time_total", 0) or 0) / 1e3 / 10, e.count // 10, e.key) for e in prof.key_averages())[::-1]
print(f"u V-cycle kernel total {sum(t[0] for t in rows):.3f} ms per application")
for t, c, k in rows[:25]:
    print(f"  {t:8.4f} ms {c:4d} {k[:100]}")

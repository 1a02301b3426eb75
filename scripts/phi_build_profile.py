"""Kernel breakdown (torch profiler) of one phi-hierarchy build at the converged config-3 state (the
shape of the builds in the late Newton iterations: most phi dofs active)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import bench
import paper_1806_09924_b200 as cf

s = torch.cuda.current_stream()
cf.set_stream(s)
P, mat, reg = bench.sneddon_setup(cf, bench.CFG3)
st = cf.make_initial_state(P, mat)
cf.newton_active_set_step(st, mat, P, reg, cf.SolverOptions())
g = st.get()
xs, po = g["solution"], g["phi_old"]
act = np.nonzero(xs[P.n_u:] == po)[0]
cs = cf.build_constraints(P, True, {int(P.n_u + v): float(po[v]) for v in act})
x = torch.from_numpy(xs).cuda()
pot = torch.from_numpy(po).cuda()
J = cf.assemble_jacobian(P, cs, mat, reg, x, pot)
free = 1.0 - np.isin(np.arange(P.n_vertices), act)
Ap = cf.CsrMatrix.from_block(J, 2)
idp = np.arange(P.n_vertices, dtype=np.int32)
B = free.reshape(-1, 1)
for _ in range(2):
    h = cf.build_amg(Ap, idp, B)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    h = cf.build_amg(Ap, idp, B)
    torch.cuda.synchronize()
rows = sorted(((getattr(e, "device_time_total", 0) or 0) / 1e3, e.count, e.key) for e in prof.key_averages())[::-1]
rows = [r for r in rows if r[0] > 0]
print(f"phi build at the converged state: {h.n_levels()} levels, kernel total {sum(r[0] for r in rows):.2f} ms, "
      f"launches {sum(r[1] for r in rows)}")
for lev in range(h.n_levels() - 1):
    print("level", lev, h.level_info(lev))
for t, c, k in rows[:30]:
    print(f"  {t:8.3f} ms {c:5d}  {k[:110]}")

"""Timing of the two config-3 hierarchy builds (run with CF_TIMING=1 for the per-phase split on
stderr): the u-hierarchy of the seeded state's M_uu and the phi-hierarchy at the converged state
(most phi dofs active).  Prints device ms per build (CUDA events, warm) and the top kernels."""
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
cases = {
    "phi": (cf.CsrMatrix.from_block(J, 2), np.arange(P.n_vertices, dtype=np.int32), free.reshape(-1, 1)),
    "u": (cf.CsrMatrix.from_block(J, 0), np.repeat(np.arange(P.n_vertices, dtype=np.int32), 3),
          cf.rigid_body_modes(P, cs)),
}
which = sys.argv[1:] or ["phi", "u"]
for name in which:
    A, nod, B = cases[name]
    nod_d = torch.from_numpy(nod).cuda()  # device arrays: the build times exclude staging copies
    B_d = torch.from_numpy(np.ascontiguousarray(B)).cuda()
    for _ in range(2):
        h = cf.build_amg(A, nod_d, B_d)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(3):
        h = cf.build_amg(A, nod_d, B_d)
    e1.record(s)
    torch.cuda.synchronize()
    print(f"{name}-build: {e0.elapsed_time(e1) / 3:.2f} ms per build (wall incl. host syncs), {h.n_levels()} levels")
    for lev in range(h.n_levels() - 1):
        print("  level", lev, h.level_info(lev))
    if os.environ.get("CF_TIMING"):
        continue
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        h = cf.build_amg(A, nod_d, B_d)
        torch.cuda.synchronize()
    rows = sorted(((getattr(e, "device_time_total", 0) or 0) / 1e3, e.count, e.key) for e in prof.key_averages())[::-1]
    rows = [r for r in rows if r[0] > 0]
    print(f"  kernel total {sum(r[0] for r in rows):.2f} ms, launches {sum(r[1] for r in rows)}")
    for t, c, k in rows[:25]:
        print(f"  {t:8.3f} ms {c:5d}  {k[:110]}")

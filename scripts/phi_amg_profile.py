"""Kernel profile of one phi-hierarchy build (M_phiphi at the converged config-3 state, active set =
the phi dofs sitting exactly at phi_old) and of the u / phi V-cycles."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import bench
import paper_1806_09924_b200 as cf

CFG = {"cfg3": bench.CFG3, "cfg2": dict(dim=2, half_width=10.0, n0=8, refinements=8)}[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
P, mat, reg = bench.sneddon_setup(cf, CFG)
st = cf.make_initial_state(P, mat)
s0 = st.get()
cf.newton_active_set_step(st, mat, P, reg, cf.SolverOptions())
s = st.get()
x, po = s["solution"], s0["phi_old"]
act = np.nonzero(x[P.n_u:] == po)[0]
print("active", act.size)
cs = cf.build_constraints(P, True, {int(P.n_u + v): float(po[v]) for v in act})
J = cf.assemble_jacobian(P, cs, mat, reg, x, po)
pp = J.M_phiphi
A = cf.CsrMatrix(pp.rows, pp.cols, pp.ptr, pp.col, pp.val)
B = (1.0 - np.isin(np.arange(P.n_vertices), act)).reshape(-1, 1)
node = np.arange(P.n_vertices, dtype=np.int32)
for rep in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    h = cf.build_amg(A, node, B)
    torch.cuda.synchronize()
    print(f"phi build {1e3 * (time.perf_counter() - t):.1f} ms, levels {h.n_levels()}")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    h = cf.build_amg(A, node, B)
    torch.cuda.synchronize()
rows = sorted(((getattr(e, "device_time_total", 0) or 0) / 1e3, e.count, e.key) for e in prof.key_averages())[::-1]
print(f"kernel total {sum(r[0] for r in rows):.1f} ms over {sum(r[1] for r in rows)} launches")
for t, c, k in rows[:25]:
    print(f"  {t:8.2f} ms {c:5d} {k[:90]}")
for lev in range(h.n_levels() - 1):
    print(lev, h.level_info(lev))

if os.environ.get("PHI_TRACE"):
    # chronological kernel list of one build (name, duration, gap before)
    evs = sorted((e for e in prof.events() if e.device_type.name == "CUDA"), key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    prev = t0
    with open(os.environ["PHI_TRACE"], "w") as f:
        for e in evs:
            f.write(f"{(e.time_range.start - t0) / 1e3:9.3f} ms  dur {e.time_range.elapsed_us():8.1f} us  gap {(e.time_range.start - prev):8.1f} us  {e.name[:80]}\n")
            prev = e.time_range.end

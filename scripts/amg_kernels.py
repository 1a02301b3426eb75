"""Per-kernel device time of one config-3 u-hierarchy build and one phi-hierarchy build (first
Jacobian of the step, torch profiler / CUPTI).  usage: python scripts/amg_kernels.py"""
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
st = cf.make_initial_state(P, mat).get()
x = torch.from_numpy(st["solution"]).cuda()
pt = torch.from_numpy(st["phi_old"]).cuda()
cs = cf.build_constraints(P)
J = cf.assemble_jacobian(P, cs, mat, reg, x, pt)
node_u = np.repeat(np.arange(P.n_vertices, dtype=np.int32), P.dim)
B = cf.rigid_body_modes(P, cs)
Au, Ap = cf.CsrMatrix.from_block(J, 0), cf.CsrMatrix.from_block(J, 2)
idp = np.arange(P.n_vertices, dtype=np.int32)
ones = np.ones((P.n_vertices, 1))
cf.build_amg(Au, node_u, B)  # warm-up (allocator, tables)
cf.build_amg(Ap, idp, ones)
torch.cuda.synchronize()
for name, fn in (("u", lambda: cf.build_amg(Au, node_u, B)), ("phi", lambda: cf.build_amg(Ap, idp, ones))):
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        h = fn()
        torch.cuda.synchronize()
    rows = sorted(((getattr(e, "device_time_total", 0) or 0) / 1e3, e.count, e.key) for e in prof.key_averages())[::-1]
    rows = [r for r in rows if r[0] > 0]
    print(f"== {name}-hierarchy build: {h.n_levels()} levels, kernel total {sum(r[0] for r in rows):.2f} ms")
    for t, c, k in rows[:30]:
        print(f"  {t:8.3f} ms {c:5d}  {k[:120]}")

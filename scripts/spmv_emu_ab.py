"""Focused timing of the emulated-lane stencil SpMV variants on config 1 (interleaved, many reps)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1806_09924_b200 as cf
from paper_1806_09924_b200._lib import check, load

s = torch.cuda.current_stream()
cf.set_stream(s)
P, cs, mat, reg, x, pt = bench.config1_inputs(cf)
J = cf.assemble_jacobian(P, cs, mat, reg, x, pt)
u = x[:P.n_u].contiguous()
y = torch.empty_like(u)
ref = J.spmv(0, u)
V = [(16, 141), (16, 142), (16, 143), (16, 144), (16, 181), (16, 182), (16, 183), (16, 184)]
res = {v: [] for v in V}
for rep in range(4):
    for tpr, un in V:
        f = lambda: check(load().cf_tune_spmv(J._h, 0, tpr, un, C.c_void_p(u.data_ptr()), C.c_void_p(y.data_ptr())))
        for _ in range(3):
            f()
        res[(tpr, un)].append(bench.time_events(f, 30, s))
        assert torch.equal(y, ref)
for v, t in res.items():
    print(v, " ".join(f"{a:.3f}" for a in t), f"min {min(t):.3f}")

"""Kernel times of the matrix-free M_uu apply on config 1."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import bench
import paper_1806_09924_b200 as cf

s = torch.cuda.current_stream()
cf.set_stream(s)
P, cs, mat, reg, x, pt = bench.config1_inputs(cf)
u = x[:P.n_u].contiguous()
y = torch.empty_like(u)
for _ in range(3):
    cf.mf_apply_uu(P, cs, mat, reg, pt, u, out=y)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        cf.mf_apply_uu(P, cs, mat, reg, pt, u, out=y)
    torch.cuda.synchronize()
for e in sorted(prof.key_averages(), key=lambda e: -(getattr(e, "device_time_total", 0) or 0))[:12]:
    print(f"{e.device_time_total / 1e3 / 5:8.3f} ms/apply  {e.count:4d}  {e.key[:80]}")

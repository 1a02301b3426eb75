"""Standalone M_uu apply of the config-3 Jacobian (seeded state): ms and GB/s in the stencil format."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1806_09924_b200 as cf

s = torch.cuda.current_stream()
cf.set_stream(s)
P, mat, reg = bench.sneddon_setup(cf, bench.CFG3)
st = cf.make_initial_state(P, mat).get()
x = torch.from_numpy(st["solution"]).cuda()
x[:P.n_u] = 1e-3 * torch.randn(P.n_u, dtype=torch.float64, device="cuda")
pt = torch.from_numpy(st["phi_old"]).cuda()
cs = cf.build_constraints(P)
J = cf.assemble_jacobian(P, cs, mat, reg, x, pt)
u = x[:P.n_u].contiguous()
y = torch.empty_like(u)
for _ in range(3):
    J.spmv(0, u, out=y)
ms = bench.time_events(lambda: J.spmv(0, u, out=y), 20, s)
nb = bench.stencil_bytes(P.n_u, P.n_u, J.nnz[0])
print(f"cfg3 M_uu ({J.format(0)}): {ms:.4f} ms, {nb / 1e9:.3f} GB -> {nb / ms / 1e6:.0f} GB/s; full apply:", flush=True)
z = torch.empty(P.n_total, dtype=torch.float64, device="cuda")
ms2 = bench.time_events(lambda: J.apply(x, out=z), 20, s)
print(f"  block apply {ms2:.4f} ms", flush=True)

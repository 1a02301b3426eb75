"""ncu target: one config-3 Jacobian + residual assembly (after a warm-up)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1806_09924_b200 as cf
P, mat, reg = bench.sneddon_setup(cf, bench.CFG3)
st = cf.make_initial_state(P, mat).get()
x = torch.from_numpy(st["solution"]).cuda()
x[:P.n_u] = 1e-3 * torch.randn(P.n_u, dtype=torch.float64, device="cuda")
pt = torch.from_numpy(st["phi_old"]).cuda()
cs = cf.build_constraints(P)
for _ in range(2):
    J = cf.assemble_jacobian(P, cs, mat, reg, x, pt)
    R = cf.assemble_residual(P, cs, mat, reg, x, pt)
    del J
torch.cuda.synchronize()
print("ok")

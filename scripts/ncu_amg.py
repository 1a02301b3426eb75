"""ncu target: one config-3 u-hierarchy build (M_uu of a perturbed seeded state) after a warm-up."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_1806_09924_b200 as cf
P, mat, reg = bench.sneddon_setup(cf, bench.CFG3)
st = cf.make_initial_state(P, mat).get()
x = torch.from_numpy(st["solution"]).cuda()
x[:P.n_u] = 1e-3 * torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, P.n_u)).cuda()
pt = torch.from_numpy(st["phi_old"]).cuda()
cs = cf.build_constraints(P)
J = cf.assemble_jacobian(P, cs, mat, reg, x, pt)
for _ in range(2):
    pre = cf.BlockPreconditioner.build(J, "amg", prob=P, constraints=cs)
    torch.cuda.synchronize()
print("ok")

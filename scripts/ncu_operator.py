"""Target for the ncu --set full capture of the CSR SpMV kernel on the config 1 operator."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1806_09924_b200 as cf
P, cs, mat, reg, x, pt = bench.config1_inputs(cf)
J = cf.assemble_jacobian(P, cs, mat, reg, x, pt)
u = x[:P.n_u].contiguous()
y = torch.empty_like(u)
for _ in range(3):
    J.spmv(0, u, out=y)
torch.cuda.synchronize()
print("ok", J.nnz[0])

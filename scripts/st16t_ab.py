"""Config-1 M_uu apply (3d stencil format) timed under the current environment; prints ms, GB/s of
the kernel's own format and the SHA-256 of y (the TMA-fed kernel must reproduce k_spmv_st16p bitwise).
usage: [CF_NO_ST16T=1 | CF_ST16T_STAGES=3|4|6] python scripts/st16t_ab.py"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1806_09924_b200 as cf

s = torch.cuda.current_stream()
cf.set_stream(s)
P, cs, mat, reg, x, pt = bench.config1_inputs(cf)
nu = P.n_u
u = x[:nu].contiguous()
J = cf.assemble_jacobian(P, cs, mat, reg, x, pt)
y = torch.empty(nu, dtype=torch.float64, device="cuda")
for _ in range(3):
    J.spmv(0, u, out=y)
ms = bench.time_events(lambda: J.spmv(0, u, out=y), 30, s)
nnz = J.nnz[0]
own = 8 * nnz + 8 * (nu + 1) + 16 * nu
tag = "st16p" if os.environ.get("CF_NO_ST16T") else "st16t S=" + os.environ.get("CF_ST16T_STAGES", "4")
print(f"{tag}: {ms:.3f} ms  {own / ms / 1e6:.0f} GB/s  sha {hashlib.sha256(y.cpu().numpy().tobytes()).hexdigest()[:16]}",
      flush=True)

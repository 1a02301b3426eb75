"""Config-1 matrix-free M_uu apply vs the assembled stencil SpMV (device ms, CUDA events) and their
agreement; CF_MF_TWO_PASS=1 selects the round-1 two-pass kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1806_09924_b200 as cf

s = torch.cuda.current_stream()
cf.set_stream(s)
P, cs, mat, reg, x, pt = bench.config1_inputs(cf)
u = x[:P.n_u].contiguous()
J = cf.assemble_jacobian(P, cs, mat, reg, x, pt)
y = torch.empty_like(u)
J.spmv(0, u, out=y)
ym = torch.empty_like(u)
cf.mf_apply_uu(P, cs, mat, reg, pt, u, out=ym)
rel = float(torch.linalg.norm(ym - y) / torch.linalg.norm(y))
ms_mf = bench.time_events(lambda: cf.mf_apply_uu(P, cs, mat, reg, pt, u, out=ym), 20, s)
ms_as = bench.time_events(lambda: J.spmv(0, u, out=y), 20, s)
fp64 = cf.fp64_peak_tflops()
fl = 2688.0 * P.n_cells
print(f"matrix-free {ms_mf:.3f} ms ({fl / ms_mf / 1e9:.1f} TF/s canonical = {fl / ms_mf / 1e9 / fp64:.3f} of "
      f"{fp64:.1f} TF/s FP64), assembled {ms_as:.3f} ms, rel diff {rel:.2e}")

"""Matrix-free M_uu apply: time per apply (CUDA events) on config 3 (128^3) and config 1 (192^3) and
the relative difference to the assembled apply (config 3).  Run under A/B builds (CF_LIB_PATH) or
with CF_MF_CELL=1 (the one-thread-per-cell kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1806_09924_b200 as cf

s = torch.cuda.current_stream()
cf.set_stream(s)
tag = os.environ.get("CF_LIB_PATH", "default") + (" CF_MF_CELL" if os.environ.get("CF_MF_CELL") else "")
for name, n0, r in (("cfg3", 8, 4), ("cfg1", 12, 4)):
    P = cf.Problem(3, 10.0, n0, r)
    g = torch.Generator(device="cuda").manual_seed(1)
    pt = torch.rand(P.n_vertices, dtype=torch.float64, device="cuda", generator=g)
    u = torch.randn(P.n_u, dtype=torch.float64, device="cuda", generator=g)
    cs = cf.build_constraints(P)
    mat, reg = cf.Material(), cf.Regularization(2 * P.h, 1e-12)
    y = torch.empty_like(u)
    cf.mf_apply_uu(P, cs, mat, reg, pt, u, out=y)
    ms = bench.time_events(lambda: cf.mf_apply_uu(P, cs, mat, reg, pt, u, out=y), 20, s)
    cells = (P.n_vertices ** (1 / 3) - 1) ** 3
    line = f"[{tag}] {name}: {ms:.3f} ms/apply, {2688 * cells / ms / 1e9:.2f} TFLOP/s canonical"
    if name == "cfg3":
        x = torch.zeros(P.n_total, dtype=torch.float64, device="cuda")
        x[P.n_u:] = pt
        J = cf.assemble_jacobian(P, cs, mat, reg, x, pt)
        ya = J.spmv(0, u)
        line += f", rel diff to assembled {float(torch.linalg.norm(y - ya) / torch.linalg.norm(ya)):.2e}"
        del J
    print(line, flush=True)

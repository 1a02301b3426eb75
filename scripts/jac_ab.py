"""A/B timing of the Jacobian fill variants on config 3 (CF_JAC_WARP=1 selects the slot-per-lane
kernel), with a bitwise comparison of the two results.  usage: python scripts/jac_ab.py [cfg3|cfg2]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1806_09924_b200 as cf

d, n0, r = {"cfg3": (3, 8, 4), "cfg2": (2, 8, 8), "cfg0": (2, 8, 5)}[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
P = cf.Problem(d, 10.0, n0, r)
mat = cf.Material(eps_mode=1, eps_fixed=2 * P.h, kappa_factor=1e-12 / P.h)
reg = cf.resolve_regularization(P, mat, cf.slit_band_edge(P, mat))
rng = np.random.default_rng(3)
x = np.zeros(P.n_total)
x[:P.n_u] = 1e-3 * rng.uniform(-1, 1, P.n_u)
x[P.n_u:] = rng.uniform(0, 1, P.n_vertices)
xd = torch.from_numpy(x).cuda()
pt = torch.from_numpy(rng.uniform(0, 1, P.n_vertices)).cuda()
cs = cf.build_constraints(P, True)
s = torch.cuda.current_stream()
cf.set_stream(s)
res = {}
for name in ("pair", "warp", "pair"):
    if name == "warp":
        os.environ["CF_JAC_WARP"] = "1"
    else:
        os.environ.pop("CF_JAC_WARP", None)
    J = cf.assemble_jacobian(P, cs, mat, reg, xd, pt)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(3):
        J = cf.assemble_jacobian(P, cs, mat, reg, xd, pt)
    e1.record(s)
    torch.cuda.synchronize()
    res[name] = [J.csr(w) for w in range(3)]
    print(f"{name}: assemble_jacobian {e0.elapsed_time(e1) / 3:.2f} ms", flush=True)
for w in range(3):
    a, b = res["pair"][w], res["warp"][w]
    same = np.array_equal(a.ptr, b.ptr) and np.array_equal(a.col, b.col) and np.array_equal(a.val, b.val)
    print(f"block {w}: identical={same}")

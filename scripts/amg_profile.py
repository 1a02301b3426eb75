"""AMG setup phase profile (CF_TIMING=1) on a config's first Jacobian, plus V-cycle and
block-apply timings.  usage: CF_TIMING=1 python scripts/amg_profile.py cfg3"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1806_09924_b200 as cf

CFG = {"cfg0": (2, 8, 5), "cfg2": (2, 8, 8), "cfg3": (3, 8, 4)}[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
d, n0, r = CFG
P = cf.Problem(d, 10.0, n0, r)
mat = cf.Material(eps_mode=1, eps_fixed=2 * P.h, kappa_factor=1e-12 / P.h)
reg = cf.resolve_regularization(P, mat, cf.slit_band_edge(P, mat))
st = cf.make_initial_state(P, mat)
s = st.get()
x = torch.from_numpy(s["solution"]).cuda()
pt = torch.from_numpy(s["phi_old"]).cuda()
cs = cf.build_constraints(P)
torch.cuda.synchronize()
t = time.perf_counter()
J = cf.assemble_jacobian(P, cs, mat, reg, x, pt)
torch.cuda.synchronize()
print(f"jacobian {1e3 * (time.perf_counter() - t):.2f} ms nnz {J.nnz}", flush=True)
t = time.perf_counter()
R = cf.assemble_residual(P, cs, mat, reg, x, pt)
torch.cuda.synchronize()
print(f"residual {1e3 * (time.perf_counter() - t):.2f} ms", flush=True)
for rep in range(2):
    t = time.perf_counter()
    pre = cf.BlockPreconditioner.build(J, "amg", prob=P, constraints=cs)
    torch.cuda.synchronize()
    print(f"prec build {1e3 * (time.perf_counter() - t):.2f} ms", flush=True)
os.environ.pop("CF_TIMING", None)
from torch.profiler import ProfilerActivity, profile
rhs = -R
for rep in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        res = cf.gmres(J, rhs, prec=pre)
        torch.cuda.synchronize()
    wall = 1e3 * (time.perf_counter() - t)
    ktot = sum((getattr(e, "device_time_total", 0) or 0) for e in prof.key_averages()) / 1e3
    print(f"gmres its {res['iterations']} wall {wall:.1f} ms kernels {ktot:.1f} ms", flush=True)
    if rep == 1:
        for e in sorted(prof.key_averages(), key=lambda e: -(getattr(e, "device_time_total", 0) or 0))[:12]:
            print(f"   {e.device_time_total / 1e3:8.2f} ms {e.count:6d} {e.key[:90]}")
r = torch.randn(P.n_total, dtype=torch.float64, device="cuda")
for name, f in (("block_apply", lambda: J.apply(r)), ("prec_apply", lambda: pre.apply(r))):
    f()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10):
        f()
    torch.cuda.synchronize()
    print(f"{name} {1e3 * (time.perf_counter() - t) / 10:.3f} ms", flush=True)

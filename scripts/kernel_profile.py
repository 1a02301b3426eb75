"""Per-kernel device-time breakdown of Newton iterations (CUPTI via torch.profiler).
usage: python scripts/kernel_profile.py cfg3 [newton_max_iter]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1806_09924_b200 as cf

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
its = int(sys.argv[2]) if len(sys.argv) > 2 else 3
d, n0, r = {"cfg0": (2, 8, 5), "cfg2": (2, 8, 8), "cfg3": (3, 8, 4)}[name]
P = cf.Problem(d, 10.0, n0, r)
mat = cf.Material(eps_mode=1, eps_fixed=2 * P.h, kappa_factor=1e-12 / P.h)
reg = cf.resolve_regularization(P, mat, cf.slit_band_edge(P, mat))
opts = cf.SolverOptions(newton_max_iter=its)
st = cf.make_initial_state(P, mat)
s = st.get()
cf.newton_active_set_step(cf.FractureState(P, s["solution"], s["phi_old"], s["phi_prev2"], 1), mat, P, reg, opts)
st = cf.FractureState(P, s["solution"], s["phi_old"], s["phi_prev2"], 1)  # measured: a warm second step
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    rep = cf.newton_active_set_step(st, mat, P, reg, opts)
    torch.cuda.synchronize()
rows = []
for e in prof.key_averages():
    t = getattr(e, "device_time_total", None) or getattr(e, "cuda_time_total", 0)
    if t > 0:
        rows.append((t / 1e3, e.count, e.key))
rows.sort(reverse=True)
tot = sum(r[0] for r in rows)
print(json.dumps(rep["times_ms"]))
print(f"total kernel time {tot:.1f} ms over {sum(r[1] for r in rows)} launches")
for t, c, k in rows[:int(os.environ.get("TOPN", "40"))]:
    print(f"{t:9.2f} ms {100 * t / tot:5.1f}% {c:7d}  {k[:110]}")
os.makedirs("gpurun_out", exist_ok=True)
with open(f"gpurun_out/kernels_{name}.json", "w") as f:
    json.dump(dict(config=name, newton_its=its, times=rep["times_ms"], kernels=[
        dict(ms=t, count=c, name=k) for t, c, k in rows]), f, indent=1)

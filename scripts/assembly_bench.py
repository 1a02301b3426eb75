"""Residual / Jacobian assembly timings (CUDA events) on config 3 and config 1."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1806_09924_b200 as cf
s = torch.cuda.current_stream()
cf.set_stream(s)
for name in sys.argv[1:] or ["cfg3", "cfg1"]:
    if name == "cfg1":
        P, cs, mat, reg, x, pt = bench.config1_inputs(cf)
    else:
        P, mat, reg = bench.sneddon_setup(cf, bench.CFG3)
        st = cf.make_initial_state(P, mat).get()
        x = torch.from_numpy(st["solution"]).cuda(); x[:P.n_u] = 1e-3 * torch.randn(P.n_u, dtype=torch.float64, device="cuda")
        pt = torch.from_numpy(st["phi_old"]).cuda()
        cs = cf.build_constraints(P)
    R = torch.empty(P.n_total, dtype=torch.float64, device="cuda")
    cf.assemble_residual(P, cs, mat, reg, x, pt, out=R)
    J = cf.assemble_jacobian(P, cs, mat, reg, x, pt); del J
    mr = bench.time_events(lambda: cf.assemble_residual(P, cs, mat, reg, x, pt, out=R), 5, s)
    mj = bench.time_events(lambda: cf.assemble_jacobian(P, cs, mat, reg, x, pt), 3, s)
    print(f"{name}: cells {P.n_cells} residual {mr:.2f} ms  jacobian {mj:.2f} ms", flush=True)
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    J = cf.assemble_jacobian(P, cs, mat, reg, x, pt)
    cf.assemble_residual(P, cs, mat, reg, x, pt, out=R)
    torch.cuda.synchronize()
for e in sorted(prof.key_averages(), key=lambda e: -(getattr(e, "device_time_total", 0) or 0))[:8]:
    print(f"   {e.device_time_total / 1e3:8.2f} ms {e.count:4d} {e.key[:90]}")

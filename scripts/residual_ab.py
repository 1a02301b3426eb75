"""Residual assembly time and output digest on config 3 at the initial state (u = 0) and at a
random displacement; run under two library builds (CF_LIB_PATH) and compare the digests."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1806_09924_b200 as cf

s = torch.cuda.current_stream()
cf.set_stream(s)
P, mat, reg = bench.sneddon_setup(cf, bench.CFG3)
st = cf.make_initial_state(P, mat).get()
pt = torch.from_numpy(st["phi_old"]).cuda()
cs = cf.build_constraints(P)
R = torch.empty(P.n_total, dtype=torch.float64, device="cuda")
gen = torch.Generator(device="cuda").manual_seed(3)
for name in ("u=0", "u random"):
    x = torch.from_numpy(st["solution"]).cuda()
    if name != "u=0":
        x[:P.n_u] = 1e-3 * torch.randn(P.n_u, dtype=torch.float64, device="cuda", generator=gen)
    cf.assemble_residual(P, cs, mat, reg, x, pt, out=R)
    ms = bench.time_events(lambda: cf.assemble_residual(P, cs, mat, reg, x, pt, out=R), 5, s)
    dig = hashlib.sha256(R.cpu().numpy().tobytes()).hexdigest()[:16]
    print(f"[{os.environ.get('CF_LIB_PATH', 'default')}] residual {name}: {ms:.3f} ms digest {dig}", flush=True)

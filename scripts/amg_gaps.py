"""GPU idle gaps inside one AMG build (torch.profiler CPU+CUDA trace): the largest gaps between
consecutive device activities and the CUDA runtime calls the host was in during them.
usage: python scripts/amg_gaps.py [u|phi]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import bench
import paper_1806_09924_b200 as cf

s = torch.cuda.current_stream()
cf.set_stream(s)
P, mat, reg = bench.sneddon_setup(cf, bench.CFG3)
st = cf.make_initial_state(P, mat)
cf.newton_active_set_step(st, mat, P, reg, cf.SolverOptions())
g = st.get()
xs, po = g["solution"], g["phi_old"]
act = np.nonzero(xs[P.n_u:] == po)[0]
cs = cf.build_constraints(P, True, {int(P.n_u + v): float(po[v]) for v in act})
x = torch.from_numpy(xs).cuda()
pot = torch.from_numpy(po).cuda()
J = cf.assemble_jacobian(P, cs, mat, reg, x, pot)
which = sys.argv[1] if len(sys.argv) > 1 else "u"
if which == "u":
    A = cf.CsrMatrix.from_block(J, 0)
    nod = torch.from_numpy(np.repeat(np.arange(P.n_vertices, dtype=np.int32), 3)).cuda()
    B = torch.from_numpy(np.ascontiguousarray(cf.rigid_body_modes(P, cs))).cuda()
else:
    A = cf.CsrMatrix.from_block(J, 2)
    nod = torch.from_numpy(np.arange(P.n_vertices, dtype=np.int32)).cuda()
    free = 1.0 - np.isin(np.arange(P.n_vertices), act)
    B = torch.from_numpy(free.reshape(-1, 1)).cuda()
for _ in range(2):
    h = cf.build_amg(A, nod, B)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    h = cf.build_amg(A, nod, B)
    torch.cuda.synchronize()
path = f"gpurun_out/amg_trace_{which}.json"
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
dev = sorted((e["ts"], e["ts"] + e.get("dur", 0), e["name"]) for e in ev
             if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset"))
host = [(e["ts"], e["ts"] + e.get("dur", 0), e["name"]) for e in ev
        if e.get("ph") == "X" and e.get("cat") == "cuda_runtime"]
t0, t1 = dev[0][0], dev[-1][1]
busy = sum(b - a for a, b, _ in dev)
gaps = []
for (a0, a1, n0), (b0, b1, n1) in zip(dev, dev[1:]):
    if b0 > a1:
        gaps.append((b0 - a1, a1, b0, n0[:50], n1[:50]))
gaps.sort(reverse=True)
print(f"{which}-build device span {(t1 - t0) / 1e3:.2f} ms, busy {busy / 1e3:.2f} ms, gaps {(t1 - t0 - busy) / 1e3:.2f} ms "
      f"in {len(gaps)} gaps")
calls = {}
for gdur, ga, gb, n0, n1 in gaps:
    for a, b, n in host:
        if b > ga and a < gb:
            ov = min(b, gb) - max(a, ga)
            calls[n] = calls.get(n, 0.0) + ov
for n, v in sorted(calls.items(), key=lambda kv: -kv[1])[:12]:
    print(f"  host in gaps: {v / 1e3:8.2f} ms  {n}")
for gdur, ga, gb, n0, n1 in gaps[:15]:
    print(f"  gap {gdur / 1e3:7.3f} ms after {n0} before {n1}")

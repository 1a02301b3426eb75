"""General-mesh path timing: a Sneddon mesh refined uniformly, then adaptively
around the slit (hanging nodes), one Newton step on the device vs the oracle (CPU, one thread), and a
device adaptive cycle.  usage: python scripts/mesh_bench.py [d] [r] [extra] [--oracle]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1806_09924_b200 as cf
import paper_1806_09924_b200.mesh as cm

d = int(sys.argv[1]) if len(sys.argv) > 1 else 2
r = int(sys.argv[2]) if len(sys.argv) > 2 else 5
extra = int(sys.argv[3]) if len(sys.argv) > 3 else 3
K, n0 = 10.0, 8
t0 = time.perf_counter()
M = cm.create_mesh(d, K, n0)
cm.uniform_refine(M, r)
marks = []
for _ in range(extra):
    xs = M.vertex_physical()
    cv = M.cell_vertices()
    ctr = xs[cv].mean(axis=1)
    near = (np.linalg.norm(ctr[:, :d - 1], axis=1) < 1.5) & (np.abs(ctr[:, d - 1]) < 0.6)
    ids = [int(c) for c in M.active_cells()[near]]
    marks.append(ids)
    cm.refine(M, ids)
t_mesh = time.perf_counter() - t0
mat = cf.Material()
reg = cm.resolve_regularization(M, mat, cm.slit_band_edge(M, mat))
st = cm.make_initial_state(M, mat)
torch.cuda.synchronize()
t0 = time.perf_counter()
rep = cm.newton_active_set_step(st, mat, M, reg, cf.SolverOptions())
torch.cuda.synchronize()
t_dev = time.perf_counter() - t0
st2 = cm.make_initial_state(M, mat)  # warm (plans and tables built)
torch.cuda.synchronize()
t0 = time.perf_counter()
rep2 = cm.newton_active_set_step(st2, mat, M, reg, cf.SolverOptions())
torch.cuda.synchronize()
t_dev2 = time.perf_counter() - t0
its = len(rep2["iterations"])
out = dict(dim=d, active_cells=M.n_active, dofs=M.n_total, max_level=M.max_level, mesh_s=t_mesh,
           newton_its=its, gmres=[q["gmres_iterations"] for q in rep2["iterations"]],
           device_step_s_cold=t_dev, device_step_s=t_dev2, device_dofs_per_s=M.n_total * its / t_dev2)
if "--oracle" in sys.argv:
    from oracle import orc
    O = orc.Mesh(d, K, n0)
    O.uniform_refine(r)
    for ids in marks:
        O.refine(ids)
    omat = orc.material()
    oreg = O.resolve_regularization(omat, O.slit_band_edge(omat))
    phi, _ = O.initial_crack(omat)
    sol = np.zeros(O.n_total)
    sol[O.n_u:] = phi
    t0 = time.perf_counter()
    orep = O.newton_step(omat, oreg, orc.solver_options(), sol, phi.copy(), phi.copy(), 0, shift=False)
    out["oracle_step_s"] = time.perf_counter() - t0
    out["oracle_dofs_per_s"] = O.n_total * len(orep["iterations"]) / out["oracle_step_s"]
    out["bitwise_vs_oracle"] = bool(np.array_equal(st2.get()["solution"], sol))
st3 = cm.make_initial_state(cm.create_mesh(d, K, n0), mat) if False else None
M2 = cm.create_mesh(d, K, n0)
cm.uniform_refine(M2, max(0, r - 2))
st3 = cm.make_initial_state(M2, mat)
torch.cuda.synchronize()
t0 = time.perf_counter()
recs = cm.adaptive_cycle(M2, st3, mat, cf._lib.AdaptiveOptions(cycles=2, n_steps=1))
torch.cuda.synchronize()
out["adaptive_cycle"] = dict(seconds=time.perf_counter() - t0, levels=[(q["dofs"], q["newton_iters"], round(q["tcv"], 8))
                                                                       for q in recs])
print(out, flush=True)

"""Run the Newton/active-set step on BASELINE configs 0, 2, 3 on the device and print per-phase
times, iteration counts and the Newton-step DoF/s (one JSON line per config)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1806_09924_b200 as cf

CFGS = {
    "cfg0": dict(d=2, n0=8, r=5, steps=1, gmres=dict(rtol=1e-8, restart=100)),
    "cfg2": dict(d=2, n0=8, r=8, steps=3, gmres=dict(rtol=1e-10, restart=50)),
    "cfg3": dict(d=3, n0=8, r=4, steps=1, gmres=dict(rtol=1e-8, restart=100)),
}

which = sys.argv[1:] or list(CFGS)
for name in which:
    c = CFGS[name]
    P = cf.Problem(c["d"], 10.0, c["n0"], c["r"])
    mat = cf.Material(eps_mode=1, eps_fixed=2 * P.h, kappa_factor=1e-12 / P.h)
    reg = cf.resolve_regularization(P, mat, cf.slit_band_edge(P, mat))
    opts = cf.SolverOptions(gmres=cf.GmresOptions(**c["gmres"]), log=1)
    st = cf.make_initial_state(P, mat)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    total_its, times, reps = 0, [], []
    for n in range(1, c["steps"] + 1):
        s = st.get()
        # shift history like solve_loading_sequence
        st2 = cf.FractureState(P, s["solution"], s["solution"][P.n_u:], s["phi_old"], n)
        st = st2
        rep = cf.newton_active_set_step(st, mat, P, reg, opts)
        reps.append(rep)
        total_its += len(rep["iterations"])
        times.append(rep["times_ms"])
    wall = time.perf_counter() - t0
    dev_ms = sum(t["total"] for t in times)
    out = dict(config=name, dofs=P.n_total, steps=c["steps"], newton_its=total_its,
               gmres=[[r["gmres_iterations"] for r in rep["iterations"]] for rep in reps],
               active=[rep["iterations"][-1]["active_size"] for rep in reps],
               converged=[rep["converged"] for rep in reps], wall_s=wall, device_ms=dev_ms,
               ms_per_newton_it=dev_ms / total_its, dofs_per_s=P.n_total * total_its / (dev_ms / 1e3),
               phases={k: sum(t[k] for t in times) for k in times[0]})
    print(json.dumps(out), flush=True)

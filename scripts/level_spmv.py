"""Per-operator SpMV bandwidth of the config-3 AMG hierarchies (u and phi) at the converged state:
every level's A, P and R = P^T through the production dispatch and through explicit variants
(k_spmv_b and the persistent pointer-prefetching k_spmv_pf), bitwise-checked against the
production result; then one V-cycle application per hierarchy with its algorithmic bytes.
usage: python scripts/level_spmv.py [--quick]   (CF_VCYCLE_UNFUSED=1 for the unfused V-cycle)"""
import ctypes as C
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_1806_09924_b200 as cf
from paper_1806_09924_b200._lib import check, load

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
node_u = np.repeat(np.arange(P.n_vertices, dtype=np.int32), P.dim)
hu = cf.build_amg(cf.CsrMatrix.from_block(J, 0), node_u, cf.rigid_body_modes(P, cs))
free = 1.0 - np.isin(np.arange(P.n_vertices), act)
hp = cf.build_amg(cf.CsrMatrix.from_block(J, 2), np.arange(P.n_vertices, dtype=np.int32), free.reshape(-1, 1))

VARIANTS = [(0, 0), (16, 4), (16, 204), (16, 206), (16, 202), (8, 4), (8, 204), (8, 206), (8, 202),
            (4, 5), (4, 205), (4, 203), (4, 208), (32, 204)]
if "--quick" in sys.argv:
    VARIANTS = [(0, 0)]
res = {"levels": {}}
vc_bytes = {}
for name, h in (("u", hu), ("phi", hp)):
    tot = 0
    for lev in range(h.n_levels() - 1):
        info = h.level_info(lev)
        n, nc = info["rows"], info["coarse"]
        tot += 56 * n  # pre-sweep 24n, residual reads b 8n, prolongation reads x 8n, post-sweep reads b, D^-1 16n
        for which, rows, cols, nnz in ((0, n, n, info["nnz_A"]), (1, n, nc, info["nnz_P"]), (2, nc, n, info["nnz_P"])):
            stencil = name == "u" and lev == 0 and which == 0
            nbytes = (bench.stencil_bytes if stencil else bench.csr_bytes)(rows, cols, nnz)
            # V-cycle traffic: 2 A applies (residual, fused sweep), R, P; vectors counted in the bytes
            tot += nbytes * (2 if which == 0 else 1)
            xin = torch.randn(cols, dtype=torch.float64, device="cuda")
            y = torch.empty(rows, dtype=torch.float64, device="cuda")
            ref = None
            row = {"rows": rows, "cols": cols, "nnz": nnz, "mean": nnz / max(rows, 1), "bytes": nbytes}
            for tpr, un in VARIANTS:
                if stencil and tpr != 0:
                    continue
                f = lambda: check(load().cf_tune_level_spmv(h._h, lev, which, tpr, un, C.c_void_p(xin.data_ptr()),
                                                            C.c_void_p(y.data_ptr())))
                for _ in range(3):
                    f()
                ms = bench.time_events(f, 20, s)
                if ref is None:
                    ref = y.clone()
                    eq = True
                else:
                    eq = bool(torch.equal(y, ref))
                row[f"{tpr}/{un}"] = {"ms": round(ms, 5), "gbs": round(nbytes / ms / 1e6, 1), "bitwise": eq}
            key = f"{name} L{lev} {'APR'[which]}"
            res["levels"][key] = row
            best = min((v for k, v in row.items() if isinstance(v, dict)), key=lambda v: v["ms"])
            print(f"{key:10s} rows {rows:9d} nnz {nnz:11d} mean {row['mean']:7.1f}  prod {row['0/0']['ms']:.4f} ms "
                  f"{row['0/0']['gbs']:7.1f} GB/s  best {best['ms']:.4f} ms {best['gbs']:7.1f} GB/s  "
                  + " ".join(f"{k}:{v['gbs']:.0f}{'' if v['bitwise'] else '!'}" for k, v in row.items()
                             if isinstance(v, dict) and k != '0/0'), flush=True)
    vc_bytes[name] = tot
for name, h, n in (("u", hu, P.n_u), ("phi", hp, P.n_phi)):
    gen = torch.Generator(device="cuda").manual_seed(5)
    r = torch.randn(n, dtype=torch.float64, device="cuda", generator=gen)
    out = h.v_cycle(r)
    ms = bench.time_events(lambda: h.v_cycle(r), 20, s)
    dig = hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()[:16]
    res[f"vcycle_{name}"] = {"ms": ms, "bytes": vc_bytes[name], "gbs": vc_bytes[name] / ms / 1e6, "sha": dig}
    print(f"V-cycle {name}: {ms:.4f} ms, {vc_bytes[name] / 1e9:.3f} GB algorithmic -> {vc_bytes[name] / ms / 1e6:.0f} GB/s, "
          f"output sha {dig}", flush=True)
os.makedirs("gpurun_out", exist_ok=True)
tag = "unfused" if os.environ.get("CF_VCYCLE_UNFUSED") else "fused"
with open(f"gpurun_out/level_spmv_{tag}.json", "w") as f:
    json.dump(res, f, indent=1)

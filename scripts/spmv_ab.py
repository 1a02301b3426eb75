"""A/B of the stencil-implicit-column SpMV against the CSR SpMV (CF_NO_STENCIL_COLS=1) on the
config-1 operator and the config-3 block apply; results must be bitwise equal."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1806_09924_b200 as cf

s = torch.cuda.current_stream()
cf.set_stream(s)
P, cs, mat, reg, x, pt = bench.config1_inputs(cf)
nu = P.n_u
u = x[:nu].contiguous()
out = {}
for mode in ("stencil", "csr"):
    if mode == "csr":
        os.environ["CF_NO_STENCIL_COLS"] = "1"
    else:
        os.environ.pop("CF_NO_STENCIL_COLS", None)
    J = cf.assemble_jacobian(P, cs, mat, reg, x, pt)
    y = torch.empty(nu, dtype=torch.float64, device="cuda")
    for _ in range(3):
        J.spmv(0, u, out=y)
    ms = bench.time_events(lambda: J.spmv(0, u, out=y), 20, s)
    out[mode] = y.clone()
    nnz = J.nnz[0]
    own = 8 * nnz + 8 * (nu + 1) + 16 * nu if mode == "stencil" else bench.csr_bytes(nu, nu, nnz)
    print(f"cfg1 M_uu {mode}: {ms:.3f} ms  own-format {own / ms / 1e6:.0f} GB/s  "
          f"CSR-equivalent {bench.csr_bytes(nu, nu, nnz) / ms / 1e6:.0f} GB/s", flush=True)
    del J
    torch.cuda.empty_cache()
print("cfg1 bitwise equal:", bool(torch.equal(out["stencil"], out["csr"])))
del x, pt, u
torch.cuda.empty_cache()
P, mat, reg = bench.sneddon_setup(cf, bench.CFG3)
st = cf.make_initial_state(P, mat).get()
x = torch.from_numpy(st["solution"]).cuda()
x[:P.n_u] = 1e-3 * torch.randn(P.n_u, dtype=torch.float64, device="cuda")
pt = torch.from_numpy(st["phi_old"]).cuda()
cs = cf.build_constraints(P)
z = torch.randn(P.n_total, dtype=torch.float64, device="cuda")
for mode in ("stencil", "csr"):
    if mode == "csr":
        os.environ["CF_NO_STENCIL_COLS"] = "1"
    else:
        os.environ.pop("CF_NO_STENCIL_COLS", None)
    J = cf.assemble_jacobian(P, cs, mat, reg, x, pt)
    y = torch.empty(P.n_total, dtype=torch.float64, device="cuda")
    J.apply(z, out=y)
    ms = bench.time_events(lambda: J.apply(z, out=y), 20, s)
    out[mode] = y.clone()
    print(f"cfg3 block apply {mode}: {ms:.3f} ms", flush=True)
print("cfg3 bitwise equal:", bool(torch.equal(out["stencil"], out["csr"])))

"""SpMV kernel-variant sweep on the config 1 M_uu (and a 2d config-2-size M_uu)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C

import torch

import bench
import paper_1806_09924_b200 as cf
from paper_1806_09924_b200._lib import check, load

s = torch.cuda.current_stream()
cf.set_stream(s)
res = {}
CASES = (("cfg1_3d192", {}), ("2d2048", dict(dim=2, half_width=10.0, n0=8, refinements=8)))
if len(sys.argv) > 1:
    CASES = CASES[:int(sys.argv[1])]
for name, over in CASES:
    P, cs, mat, reg, x, pt = bench.config1_inputs(cf, **over)
    J = cf.assemble_jacobian(P, cs, mat, reg, x, pt)
    u = x[:P.n_u].contiguous()
    y = torch.empty_like(u)
    ref = J.spmv(0, u)
    nb = bench.csr_bytes(P.n_u, P.n_u, J.nnz[0])
    for tpr, un in ((32, 0), (16, 0), (8, 0), (32, 1), (32, 2), (32, 3), (32, 4), (16, 2), (16, 4), (16, 6),
                    (8, 4), (8, 6), (8, 11), (4, 4), (4, 5), (16, 141), (16, 142), (16, 181), (16, 182),
                    (16, 121), (16, 111)):
        f = lambda: check(load().cf_tune_spmv(J._h, 0, tpr, un, C.c_void_p(u.data_ptr()), C.c_void_p(y.data_ptr())))
        for _ in range(3):
            f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(10):
            f()
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        err = ((y - ref).abs().max() / ref.abs().max()).item()
        res[f"{name} tpr{tpr} u{un}"] = (round(ms, 3), round(nb / ms / 1e6, 1), err)
        print(name, tpr, un, f"{ms:.3f} ms  {nb / ms / 1e6:.1f} GB/s  err {err:.2e}", flush=True)
    del J, x, pt, u, y, ref
    torch.cuda.empty_cache()
tag = "_csr" if os.environ.get("CF_NO_STENCIL_COLS") else ""
json.dump(res, open(f"gpurun_out/spmv_sweep{tag}.json", "w"), indent=1)

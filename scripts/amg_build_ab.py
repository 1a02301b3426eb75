"""Timing and a digest of every level operator of the config-3 u- and phi-hierarchy builds (first
Jacobian of the step): run under two kernel settings (environment switches) and compare the
digests for bitwise equality.  usage: python scripts/amg_build_ab.py"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import ctypes as C

import bench
import paper_1806_09924_b200 as cf
from paper_1806_09924_b200._lib import check, load


def build(A, nod, Bcm, m):
    """cf_amg_build with device node ids and a device column-major nullspace (no host copies)."""
    h = cf.AmgHierarchy.__new__(cf.AmgHierarchy)
    h.A, h.opts, h._h = A, cf.AmgOptions(), C.c_void_p()
    check(load().cf_amg_build(A._h, C.c_void_p(nod.data_ptr()), C.c_void_p(Bcm.data_ptr()), m, C.byref(h.opts),
                              C.byref(h._h)))
    nl, cd = C.c_int(), C.c_int64()
    check(load().cf_amg_info(h._h, C.byref(nl), C.byref(cd)))
    h._n_levels, h._coarse = nl.value, cd.value
    return h

s = torch.cuda.current_stream()
cf.set_stream(s)
P, mat, reg = bench.sneddon_setup(cf, bench.CFG3)
st = cf.make_initial_state(P, mat).get()
x = torch.from_numpy(st["solution"]).cuda()
pt = torch.from_numpy(st["phi_old"]).cuda()
cs = cf.build_constraints(P)
J = cf.assemble_jacobian(P, cs, mat, reg, x, pt)
node_u = torch.from_numpy(np.repeat(np.arange(P.n_vertices, dtype=np.int32), P.dim)).cuda()
B = torch.from_numpy(np.ascontiguousarray(cf.rigid_body_modes(P, cs).T)).cuda()  # column-major n_u x 6
Au, Ap = cf.CsrMatrix.from_block(J, 0), cf.CsrMatrix.from_block(J, 2)
idp = torch.arange(P.n_vertices, dtype=torch.int32, device="cuda")
ones = torch.ones(P.n_vertices, dtype=torch.float64, device="cuda")
tag = " ".join(k for k in os.environ if k.startswith("CF_")) or "default"
for name, fn in (("u", lambda: build(Au, node_u, B, 6)), ("phi", lambda: build(Ap, idp, ones, 1))):
    fn()
    ms = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        h = fn()
        e1.record(s)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    dig = hashlib.sha256()
    for lev in range(h.n_levels() - 1):
        for which in (0, 1):
            M = h.level_matrix(lev, which)
            for a in (M.ptr, M.col, M.val):
                dig.update(np.ascontiguousarray(a).tobytes())
    print(f"[{tag}] {name}-hierarchy build {min(ms):.1f} ms (of {[round(m, 1) for m in ms]}), levels {h.n_levels()}, "
          f"digest {dig.hexdigest()[:16]}", flush=True)

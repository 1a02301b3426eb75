"""Row-pattern groups of the config-3 u-hierarchy SpGEMM operands: how many consecutive rows share
their column pattern with the previous row (A_l, P_l and R_l = P_l^T).  usage: python scripts/group_stats.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1806_09924_b200 as cf

P = cf.Problem(3, 10.0, 8, 4)
mat = cf.Material(eps_mode=1, eps_fixed=2 * P.h, kappa_factor=1e-12 / P.h)
reg = cf.resolve_regularization(P, mat, cf.slit_band_edge(P, mat))
st = cf.make_initial_state(P, mat).get()
x = torch.from_numpy(st["solution"]).cuda()
x[:P.n_u] = 1e-3 * torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, P.n_u)).cuda()
pt = torch.from_numpy(st["phi_old"]).cuda()
cs = cf.build_constraints(P)
J = cf.assemble_jacobian(P, cs, mat, reg, x, pt)
u = J.M_uu
A = cf.CsrMatrix(u.rows, u.cols, u.ptr, u.col, u.val)
h = cf.build_amg(A, np.repeat(np.arange(P.n_vertices, dtype=np.int32), 3), cf.rigid_body_modes(P, cs))


def stats(name, rows, ptr, col):
    ptr = torch.as_tensor(ptr).cuda()
    col = torch.as_tensor(col).cuda().long()
    ln = ptr[1:] - ptr[:-1]
    rid = torch.repeat_interleave(torch.arange(rows, device="cuda"), ln)
    same_len = torch.zeros(rows, dtype=torch.bool, device="cuda")
    same_len[1:] = ln[1:] == ln[:-1]
    e = torch.arange(col.numel(), device="cuda")
    prev = e - ln[rid]
    ok = same_len[rid] & (prev >= 0)
    mism = torch.zeros(rows, dtype=torch.int64, device="cuda")
    bad = ok & (col[prev.clamp(min=0)] != col)
    mism.index_add_(0, rid, bad.long())
    same = same_len & (mism == 0)
    same[ln == 0] = False
    heads = int(rows - same.sum())
    print(f"{name:8s} rows {rows:9d} nnz {col.numel():11d} heads {heads:9d} mean group {rows / max(heads, 1):.2f}")


for lev in range(h.n_levels() - 1):
    for which, nm in ((0, "A"), (1, "P")):
        m = h.level_matrix(lev, which)
        stats(f"{nm}{lev}", m.rows, m.ptr, m.col)
        if which == 1:
            ptr = torch.as_tensor(m.ptr).cuda()
            rid = torch.repeat_interleave(torch.arange(m.rows, device="cuda"), ptr[1:] - ptr[:-1])
            c = torch.as_tensor(m.col).cuda().long()
            key = c * m.rows + rid
            key, _ = torch.sort(key)
            rc = key // m.rows
            rr = (key % m.rows).int()
            cnt = torch.bincount(rc, minlength=m.cols)
            rptr = torch.zeros(m.cols + 1, dtype=torch.int64, device="cuda")
            rptr[1:] = torch.cumsum(cnt, 0)
            stats(f"R{lev}", m.cols, rptr, rr)

"""world_size-2 gloo test (CPU) of the slab decomposition's host protocol.

The multi-GPU step (paper_1806_09924_b200/csrc/newton.cu: rank_slab, halo_global, to_ext,
Comm::sum_ordered; block-Jacobi preconditioner over the slabs) cannot run here, so this test runs
the same protocol on CPU with the oracle's Jacobian as data and torch.distributed/gloo as the
transport:
  * the plane split and ghost ranges (rank_slab / make_slab);
  * every owned row's columns lie in the owned + one-ghost-plane range, so the ext layout
    [u_ext | phi_ext] is complete, and the halo exchange fills exactly those planes;
  * a slab's rows times the ext vector are bitwise the rows of the undivided product;
  * rank-ordered sums are bitwise identical on every rank;
  * GMRES with rank-ordered dots and the preconditioners of the product — restricted additive
    Schwarz with one overlap plane (default) and block-Jacobi (CF_BLOCK_JACOBI=1) — converges to
    the undivided solution.
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rank_slab(d, nn, rank, size):  # newton.cu rank_slab + assembly.cu make_slab
    pl = nn ** (d - 1)
    p_lo, p_hi = nn * rank // size, nn * (rank + 1) // size
    return dict(v_lo=p_lo * pl, v_hi=p_hi * pl, ve_lo=max(p_lo - 1, 0) * pl, ve_hi=min(p_hi + 1, nn) * pl, plane=pl)


def to_ext(z, s, d, rank, size):  # newton.cu to_ext
    import torch
    import torch.distributed as dist
    nv, ne, pl = s["v_hi"] - s["v_lo"], s["ve_hi"] - s["ve_lo"], s["plane"]
    lo, nul, nue = s["v_lo"] - s["ve_lo"], d * nv, d * ne
    e = torch.zeros((d + 1) * ne, dtype=torch.float64)
    zt = torch.from_numpy(np.ascontiguousarray(z))
    e[d * lo:d * lo + nul] = zt[:nul]
    e[nue + lo:nue + lo + nv] = zt[nul:]
    recv, ops = [], []
    if rank > 0:
        for snd, (a, b) in ((zt[:d * pl], (0, d * pl)), (zt[nul:nul + pl], (nue, nue + pl))):
            buf = torch.empty(b - a, dtype=torch.float64)
            ops += [dist.P2POp(dist.isend, snd.clone(), rank - 1), dist.P2POp(dist.irecv, buf, rank - 1)]
            recv.append((buf, a, b))
    if rank + 1 < size:
        for snd, (a, b) in ((zt[nul - d * pl:nul], (d * (ne - pl), nue)), (zt[nul + nv - pl:], (nue + ne - pl, nue + ne))):
            buf = torch.empty(b - a, dtype=torch.float64)
            ops += [dist.P2POp(dist.isend, snd.clone(), rank + 1), dist.P2POp(dist.irecv, buf, rank + 1)]
            recv.append((buf, a, b))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    for buf, a, b in recv:
        e[a:b] = buf
    return e.numpy()


def sum_ordered(vals, size):  # comm.cu Comm::sum_ordered: all-gather, then left-to-right in rank order
    import torch
    import torch.distributed as dist
    t = torch.tensor(np.atleast_1d(vals), dtype=torch.float64)
    parts = [torch.empty_like(t) for _ in range(size)]
    dist.all_gather(parts, t)
    s = parts[0].clone()
    for p in parts[1:]:
        s = s + p
    return s.numpy()


def _worker(rank, size, port, out_dir, ras):
    sys.path.insert(0, ROOT)
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    import torch.distributed as dist
    from oracle import orc
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    d, n0, r = 2, 4, 2
    O = orc.Problem(d, 1.0, n0, r)
    nn, V = (n0 << r) + 1, O.V
    nu, nt = d * V, (d + 1) * V
    rng = np.random.default_rng(11)  # identical global data on every rank
    x = np.zeros(nt)
    x[:nu] = 1e-2 * rng.uniform(-1, 1, nu)
    x[nu:] = rng.uniform(0, 1, V)
    pt = rng.uniform(0, 1, V)
    act = rng.choice(V, V // 8, replace=False)
    cs = O.constraints(True, [int(nu + v) for v in act], list(rng.uniform(0, 1, act.size)))
    mat, reg = orc.material(pressure=2e-3), orc.Regularization(0.3, 1e-6)
    Jo = O.jacobian(cs, mat, reg, x, pt)
    Muu, Mpu, Mpp = (Jo.csr(w).to_scipy().tocsr() for w in range(3))
    s = rank_slab(d, nn, rank, size)
    lo, hi, elo, ehi = s["v_lo"], s["v_hi"], s["ve_lo"], s["ve_hi"]
    nv, ne = hi - lo, ehi - elo

    # slab rows, columns shifted to the ext layout; nothing may fall outside the ghost planes
    def slab_block(M, rlo, rhi, clo, chi):
        B = M[rlo:rhi].tocoo()
        assert B.col.min(initial=clo) >= clo and B.col.max(initial=clo) < chi, "column outside owned + ghost planes"
        return sp.csr_matrix((B.data, (B.row, B.col - clo)), shape=(rhi - rlo, chi - clo))
    Suu = slab_block(Muu, d * lo, d * hi, d * elo, d * ehi)
    Spu = slab_block(Mpu, lo, hi, d * elo, d * ehi)
    Spp = slab_block(Mpp, lo, hi, elo, ehi)

    def own(v):
        return np.concatenate([v[d * lo:d * hi], v[nu + lo:nu + hi]])

    def apply(zl):
        e = to_ext(zl, s, d, rank, size)
        return np.concatenate([Suu @ e[:d * ne], Spu @ e[:d * ne] + Spp @ e[d * ne:]])

    z = rng.standard_normal(nt)
    e = to_ext(own(z), s, d, rank, size)
    assert np.array_equal(e, np.concatenate([z[d * elo:d * ehi], z[nu + elo:nu + ehi]])), "halo planes"
    yg = np.concatenate([Muu @ z[:nu], Mpu @ z[:nu] + Mpp @ z[nu:]])
    assert np.array_equal(apply(own(z)), own(yg)), "slab rows differ from the undivided product"

    # rank-ordered sum (compared across ranks by the parent)
    tot = sum_ordered([own(z) @ own(z)], size)

    # preconditioner (exact local solves in place of the per-slab AMG) + MGS GMRES, rank-ordered dots
    if ras:  # restricted additive Schwarz: the block of the planes plus one overlap plane each side
        Xuu = sp.csc_matrix(Muu[d * elo:d * ehi, d * elo:d * ehi])
        Xpp = sp.csc_matrix(Mpp[elo:ehi, elo:ehi])
        Luu, Lpp = spla.splu(Xuu), spla.splu(Xpp)

        def prec(rl):
            e = to_ext(rl, s, d, rank, size)
            zu, zp = Luu.solve(e[:d * ne]), Lpp.solve(e[d * ne:])
            return np.concatenate([zu[d * (lo - elo):d * (hi - elo)], zp[lo - elo:hi - elo]])
    else:  # block-Jacobi: the diagonal block of the slab
        Luu = spla.splu(sp.csc_matrix(Suu[:, d * (lo - elo):d * (hi - elo)]))
        Lpp = spla.splu(sp.csc_matrix(Spp[:, lo - elo:hi - elo]))

        def prec(rl):
            return np.concatenate([Luu.solve(rl[:d * nv]), Lpp.solve(rl[d * nv:])])

    def gdot(a, b):
        return float(sum_ordered([a @ b], size)[0])

    b = own(rng.standard_normal(nt))
    xl, m, rtol = np.zeros_like(b), 40, 1e-11
    bn = np.sqrt(gdot(b, b))
    its = 0
    for _cycle in range(20):
        rr = b - apply(prec(xl)) if its else b.copy()
        beta = np.sqrt(gdot(rr, rr))
        if beta <= rtol * bn:
            break
        Vb, H = [rr / beta], np.zeros((m + 1, m))
        for j in range(m):
            w = apply(prec(Vb[j]))
            for i in range(j + 1):
                H[i, j] = gdot(w, Vb[i])
                w = w - H[i, j] * Vb[i]
            H[j + 1, j] = np.sqrt(gdot(w, w))
            its += 1
            Vb.append(w / H[j + 1, j])
            g = np.zeros(j + 2)
            g[0] = beta
            y = np.linalg.lstsq(H[:j + 2, :j + 1], g, rcond=None)[0]
            if np.linalg.norm(H[:j + 2, :j + 1] @ y - g) <= rtol * bn:
                break
        xl = xl + sum(yi * vi for yi, vi in zip(y, Vb))
    sol = prec(xl)
    res = b - apply(sol)
    rel = np.sqrt(gdot(res, res)) / bn
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), np.concatenate([[rel, its, tot[0]], sol]))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


@pytest.mark.parametrize("size,ras", [(2, True), (2, False)])
def test_slab_protocol_gloo(orc, tmp_path, size, ras):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(size, _free_port(), str(tmp_path), ras), nprocs=size, join=True)
    outs = [np.load(tmp_path / f"rank{r}.npy") for r in range(size)]
    assert all(o[0] <= 1e-9 for o in outs), [o[0] for o in outs]
    assert len({o[1] for o in outs}) == 1, "ranks disagree on the iteration count"
    assert len({o[2] for o in outs}) == 1, "rank-ordered sums differ between ranks"
    # the distributed solution solves the undivided system
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    d, n0, r = 2, 4, 2
    O = orc.Problem(d, 1.0, n0, r)
    V = O.V
    nu, nt = d * V, (d + 1) * V
    rng = np.random.default_rng(11)
    x = np.zeros(nt)
    x[:nu] = 1e-2 * rng.uniform(-1, 1, nu)
    x[nu:] = rng.uniform(0, 1, V)
    pt = rng.uniform(0, 1, V)
    act = rng.choice(V, V // 8, replace=False)
    cs = O.constraints(True, [int(nu + v) for v in act], list(rng.uniform(0, 1, act.size)))
    Jo = O.jacobian(cs, orc.material(pressure=2e-3), orc.Regularization(0.3, 1e-6), x, pt)
    Muu, Mpu, Mpp = (Jo.csr(w).to_scipy().tocsr() for w in range(3))
    J = sp.bmat([[Muu, None], [Mpu, Mpp]]).tocsc()
    rng.standard_normal(nt)  # z of the workers
    b = rng.standard_normal(nt)
    ref = spla.spsolve(J, b)
    nn = (n0 << r) + 1
    sol_u, sol_p = np.zeros(nu), np.zeros(V)
    for rank, o in enumerate(outs):
        s = rank_slab(d, nn, rank, size)
        nv = s["v_hi"] - s["v_lo"]
        sol_u[d * s["v_lo"]:d * s["v_hi"]] = o[3:3 + d * nv]
        sol_p[s["v_lo"]:s["v_hi"]] = o[3 + d * nv:]
    got = np.concatenate([sol_u, sol_p])
    assert np.linalg.norm(got - ref) <= 1e-6 * np.linalg.norm(ref)

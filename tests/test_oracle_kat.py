"""Pin the CPU oracle against the reference's own known-answer tests.

Each test names the reference test it ports (file:line).  These run on CPU only
(`-m "not gpu"`); the GPU parity tests then compare the CUDA path against this oracle.
"""
import math

import numpy as np
import pytest


def _setup(orc, d, n0, K=1.0, clamp=True):
    P = orc.Problem(d, K, n0, 0)
    cs = P.constraints(clamp=clamp)
    reg = orc.Regularization(0.25, 1e-10)
    return P, cs, reg


def _interp(P, f):
    """fem.cpp:269-279 interpolate: f(x, comp), comp == d selects phi."""
    xyz = P.coords()
    sol = np.zeros(P.n_total)
    for c in range(P.d):
        sol[c:P.n_u:P.d] = [f(x, c) for x in xyz]
    sol[P.n_u:] = [f(x, P.d) for x in xyz]
    return sol


def test_lame_and_sigma(orc):  # model_test.cpp:39-84
    m = orc.material()
    mu, lam = orc.lame(m)
    assert mu == pytest.approx(5.0 / 12.0, rel=1e-15)
    assert lam == pytest.approx(5.0 / 18.0, rel=1e-15)
    assert np.linalg.norm(orc.sigma(np.zeros((3, 3)), m, 2)) == 0.0
    I2 = np.diag([1.0, 1.0, 0.0])
    s = orc.sigma(I2, m, 2)
    assert s[0, 0] == pytest.approx(1.38888888888888884, rel=1e-14)
    assert s[1, 1] == pytest.approx(2 * mu + 2 * lam, rel=1e-14)
    rot = np.zeros((3, 3))
    rot[0, 1], rot[1, 0] = 1.0, -1.0
    assert np.linalg.norm(orc.sigma(rot, m, 2)) <= 1e-15
    rng = np.random.default_rng(3)
    for d in (2, 3):
        for _ in range(20):
            g = np.zeros((3, 3))
            g[:d, :d] = rng.uniform(-1, 1, (d, d))
            t = orc.sigma(g, m, d)
            assert np.linalg.norm(t - t.T) <= 1e-14


def test_dof_counts(orc):  # fem_test.cpp:82-101
    assert orc.Problem(2, 1.0, 1, 0).n_total == 12
    P = orc.Problem(2, 20.0, 8, 5)
    assert P.V == 257 * 257 and P.n_total == 198147
    assert orc.Problem(2, 20.0, 8, 6).n_total == 789507


def test_quadrature_and_shape(orc):  # fem_test.cpp:40-80 (rule sums, Kronecker property)
    for d in (2, 3):
        pts, w, s, g = orc.qp_tables(d)
        assert w.sum() == pytest.approx(1.0, abs=1e-15)
        assert np.allclose(s.sum(axis=1), 1.0, atol=1e-15)
        assert np.allclose(g[:, :, :d].sum(axis=1), 0.0, atol=1e-15)
        a = 1.0 / math.sqrt(3.0)
        assert pts[0, 0] == 0.5 * (-a + 1.0) and pts[1, 0] == 0.5 * (a + 1.0)  # x fastest


def test_dirichlet_constraints(orc):  # fem_test.cpp:123-142
    P = orc.Problem(2, 1.0, 4, 0)
    f, g = P.constraints().flags()
    xyz = P.coords()
    bnd = (np.abs(np.abs(xyz[:, 0]) - 1) < 1e-12) | (np.abs(np.abs(xyz[:, 1]) - 1) < 1e-12)
    assert bnd.sum() == 16 and f.sum() == 32
    assert np.array_equal(f[0:P.n_u:2].astype(bool), bnd) and np.array_equal(f[1:P.n_u:2].astype(bool), bnd)
    assert not f[P.n_u:].any() and np.all(g == 0.0)


def test_active_set_pinning(orc):  # fem_test.cpp:213-225
    P = orc.Problem(2, 1.0, 2, 0)
    cs = P.constraints(True, [P.n_u + 0, P.n_u + 3], [0.25, 1.0])
    v = cs.distribute(np.zeros(P.n_total))
    assert v[P.n_u + 0] == 0.25 and v[P.n_u + 3] == 1.0
    inc = cs.distribute(np.ones(P.n_total), homogeneous=True)
    assert inc[P.n_u + 0] == 0.0


def test_residual_intact_and_mass_rows(orc):  # model_test.cpp:118-144
    P, cs, reg = _setup(orc, 2, 4)
    m = orc.material(pressure=0.0)
    sol = np.zeros(P.n_total)
    sol[P.n_u:] = 1.0
    r = P.residual(cs, m, reg, sol, np.ones(P.V))
    assert np.abs(r).max() <= 1e-14
    r0 = P.residual(cs, m, reg, np.zeros(P.n_total), np.zeros(P.V))
    h = P.h
    xyz = P.coords()
    nb = (np.abs(np.abs(xyz[:, 0]) - 1) < 1e-12).astype(int) + (np.abs(np.abs(xyz[:, 1]) - 1) < 1e-12).astype(int)
    expect = -m.G_c / reg.eps * h * h / (2.0 ** nb)
    assert np.allclose(r0[P.n_u:], expect, rtol=1e-12, atol=0)


def test_residual_single_cell_hand_integral(orc):  # model_test.cpp:146-188
    P = orc.Problem(2, 0.5, 1, 0)
    cs = P.constraints(clamp=False)
    m = orc.material(pressure=2.5e-3)
    reg = orc.Regularization(0.5, 1e-3)
    a, b, c = 0.3, -0.2, 0.6
    sol = _interp(P, lambda x, k: a * x[0] if k == 0 else (b * x[1] if k == 1 else c))
    r = P.residual(cs, m, reg, sol, c * np.ones(P.V))
    g = np.zeros((3, 3))
    g[0, 0], g[1, 1] = a, b
    sig = orc.sigma(g, m, 2)
    deg = (1.0 - reg.kappa) * c * c + reg.kappa
    for k in range(4):  # corner k == vertex k on the single cell
        sx = 0.5 if k & 1 else -0.5
        sy = 0.5 if k & 2 else -0.5
        ex = deg * (sig[0, 0] * sx + sig[0, 1] * sy) + c * c * m.pressure * sx
        ey = deg * (sig[1, 0] * sx + sig[1, 1] * sy) + c * c * m.pressure * sy
        assert r[2 * k] == pytest.approx(ex, rel=1e-12)
        assert r[2 * k + 1] == pytest.approx(ey, rel=1e-12)


def test_rigid_translation_zero_residual(orc):  # model_test.cpp:190-209
    P = orc.Problem(2, 1.0, 3, 0)
    cs = P.constraints(clamp=False)
    m = orc.material(pressure=0.0)
    reg = orc.Regularization(0.25, 1e-10)
    rng = np.random.default_rng(9)
    phi = rng.uniform(0, 1, P.V)
    sol = np.zeros(P.n_total)
    sol[0:P.n_u:2], sol[1:P.n_u:2] = 1.7, -0.4
    sol[P.n_u:] = phi
    r = P.residual(cs, m, reg, sol, phi)
    assert np.abs(r[:P.n_u]).max() <= 1e-13


def _random_state(P, cs, rng):
    sol = np.zeros(P.n_total)
    sol[:P.n_u] = 1e-2 * rng.uniform(-1, 1, P.n_u)
    sol[P.n_u:] = rng.uniform(0, 1, P.V)
    pt = rng.uniform(0, 1, P.V)
    return cs.distribute(sol, homogeneous=True), pt


@pytest.mark.parametrize("d", [2, 3])
def test_jacobian_vs_finite_differences(orc, d):  # model_test.cpp:211-240
    rng = np.random.default_rng(13)
    P, cs, reg = _setup(orc, d, 4 if d == 2 else 2)
    m = orc.material(pressure=1e-3)
    sol, pt = _random_state(P, cs, rng)
    J = P.jacobian(cs, m, reg, sol, pt)
    for _ in range(3):
        delta = cs.distribute(rng.uniform(-1, 1, P.n_total), homogeneous=True)
        t = 1e-6 * max(1.0, np.abs(sol).max())
        fd = (P.residual(cs, m, reg, sol + t * delta, pt) - P.residual(cs, m, reg, sol - t * delta, pt)) / (2 * t)
        jd = J.apply(delta)
        assert np.linalg.norm(fd - jd) / np.linalg.norm(jd) <= 1e-5


def test_jacobian_block_structure(orc):  # model_test.cpp:242-269
    rng = np.random.default_rng(21)
    P, cs, reg = _setup(orc, 2, 4)
    m = orc.material()
    sol, pt = _random_state(P, cs, rng)
    J = P.jacobian(cs, m, reg, sol, pt)
    uu = J.csr(0).to_scipy().toarray()
    pp = J.csr(2).to_scipy().toarray()
    assert np.linalg.norm(uu - uu.T) <= 1e-12 * np.linalg.norm(uu)
    assert np.linalg.norm(pp - pp.T) <= 1e-12 * np.linalg.norm(pp)
    np.linalg.cholesky(uu)  # SPD
    sol2 = sol.copy()
    sol2[P.n_u:] += 0.1 * rng.uniform(0, 1, P.V)
    r1 = P.residual(cs, m, reg, sol, pt)
    r2 = P.residual(cs, m, reg, sol2, pt)
    assert np.abs(r1[:P.n_u] - r2[:P.n_u]).max() <= 1e-15


def test_muu_plain_elasticity(orc):  # model_test.cpp:271-322
    P = orc.Problem(2, 1.0, 3, 0)
    cs = P.constraints()
    m = orc.material()
    mu, lam = orc.lame(m)
    J = P.jacobian(cs, m, orc.Regularization(0.25, 0.0), np.zeros(P.n_total), np.ones(P.V))
    uu = J.csr(0).to_scipy().toarray()
    pts, w, s, g = orc.qp_tables(2)
    h = P.h
    nn = 4
    K = np.zeros((P.n_u, P.n_u))
    for cy in range(3):
        for cx in range(3):
            verts = [cx + (k & 1) + nn * (cy + (k >> 1 & 1)) for k in range(4)]
            for q in range(4):
                for a in range(4):
                    for ca in range(2):
                        ga = np.zeros((3, 3))
                        ga[ca, :2] = g[q, a, :2] / h
                        ea = 0.5 * (ga + ga.T)
                        for b in range(4):
                            for cb in range(2):
                                gb = np.zeros((3, 3))
                                gb[cb, :2] = g[q, b, :2] / h
                                eb = 0.5 * (gb + gb.T)
                                sb = 2 * mu * eb + lam * np.trace(eb) * np.diag([1.0, 1.0, 0.0])
                                K[2 * verts[a] + ca, 2 * verts[b] + cb] += w[q] * h * h * (sb * ea).sum()
    f, _ = cs.flags()
    con = f[:P.n_u].astype(bool)
    free = ~con
    assert np.allclose(uu[np.ix_(free, free)], K[np.ix_(free, free)], rtol=1e-10, atol=1e-10)
    off = uu.copy()
    np.fill_diagonal(off, 0.0)
    assert np.abs(off[con, :]).max() <= 1e-14 and np.abs(off[:, con]).max() <= 1e-14


@pytest.mark.parametrize("d", [2, 3])
def test_initial_crack_slab(orc, d):  # model_test.cpp:324-362
    P = orc.Problem(d, 2.0, 4, 2 if d == 2 else 1)
    m = orc.material()
    phi, be = P.initial_crack(m)
    assert be == pytest.approx(P.h)
    xyz = P.coords()
    if d == 2:
        inslab = (np.abs(xyz[:, 0]) <= m.l0 + 1e-12) & (np.abs(xyz[:, 1]) <= be + 1e-12)
    else:
        inslab = (np.hypot(xyz[:, 0], xyz[:, 1]) <= m.l0 + 1e-12) & (np.abs(xyz[:, 2]) <= be + 1e-12)
    assert np.array_equal(phi == 0.0, inslab) and np.all((phi == 0) | (phi == 1)) and inslab.sum() > 0
    origin = np.argmin(np.linalg.norm(xyz, axis=1))
    assert phi[origin] == 0.0


def test_regularization(orc):  # model_test.cpp:364-391 (uniform part)
    P = orc.Problem(2, 2.0, 4, 0)
    m = orc.material()
    assert P.slit_band_edge(m) == pytest.approx(1.0)
    r = P.resolve_regularization(m, 0.5)
    assert r.eps == pytest.approx(2.0 * 0.5 * math.sqrt(2.0))
    assert r.kappa == pytest.approx(1e-12 * P.h)
    mf = orc.material(eps_mode=1, eps_fixed=0.1234)
    assert P.resolve_regularization(mf, 0.5).eps == pytest.approx(0.1234)


def _small_jacobian(orc, rng, n0=3):  # linsolve_test.cpp:46-67
    P = orc.Problem(2, 1.0, n0, 0)
    cs = P.constraints()
    m = orc.material()
    reg = orc.Regularization(0.25, 1e-10)
    sol, pt = _random_state(P, cs, rng)
    J = P.jacobian(cs, m, reg, sol, pt)
    rhs = cs.distribute(rng.uniform(-1, 1, P.n_total), homogeneous=True)
    return P, cs, J, rhs


def _dense(J, nu, np_):
    D = np.zeros((nu + np_, nu + np_))
    D[:nu, :nu] = J.csr(0).to_scipy().toarray()
    D[nu:, :nu] = J.csr(1).to_scipy().toarray()
    D[nu:, nu:] = J.csr(2).to_scipy().toarray()
    return D


def test_block_apply(orc):  # linsolve_test.cpp:133-145
    rng = np.random.default_rng(1)
    P, cs, J, _ = _small_jacobian(orc, rng)
    x = rng.uniform(-1, 1, P.n_total)
    assert np.abs(J.apply(x) - _dense(J, P.n_u, P.V) @ x).max() <= 1e-14


def test_gmres_identity_and_spd(orc):  # linsolve_test.cpp:194-217
    I = orc.Csr.from_scipy(__import__("scipy.sparse", fromlist=["x"]).identity(20, format="csr"))
    b = np.linspace(1.0, 20.0, 20)
    res = orc.gmres(b, csr=orc.CsrHandle(I))
    assert res["converged"] and res["iterations"] == 1 and np.abs(res["x"] - b).max() <= 1e-12
    rng = np.random.default_rng(4)
    import scipy.sparse as sp
    for _ in range(5):
        B = rng.uniform(-1, 1, (50, 50))
        A = B @ B.T + 50 * np.eye(50)
        b = rng.uniform(-1, 1, 50)
        res = orc.gmres(b, csr=orc.CsrHandle(orc.Csr.from_scipy(sp.csr_matrix(A))))
        assert res["converged"]
        ex = np.linalg.solve(A, b)
        assert np.linalg.norm(res["x"] - ex) / np.linalg.norm(ex) <= 1e-7
        h = res["history"]
        assert np.all(h[1:] <= h[:-1] * (1 + 1e-12))


def test_gmres_exact_block_prec(orc):  # linsolve_test.cpp:219-237
    rng = np.random.default_rng(8)
    for _ in range(20):
        P, cs, J, rhs = _small_jacobian(orc, rng)
        pre = orc.Prec(J, 0)
        res = orc.gmres(rhs, block=J, prec=pre)
        assert res["converged"]
        ex = np.linalg.solve(_dense(J, P.n_u, P.V), rhs)
        assert np.linalg.norm(res["x"] - ex) / np.linalg.norm(ex) <= 1e-8
        assert res["iterations"] <= 5


def test_block_prec_diagonal_structure(orc):  # linsolve_test.cpp:239-263
    rng = np.random.default_rng(12)
    P, cs, J, _ = _small_jacobian(orc, rng)
    pre = orc.Prec(J, 0)
    r = np.zeros(P.n_total)
    r[:P.n_u] = rng.uniform(-1, 1, P.n_u)
    z = pre.apply(r)
    assert np.abs(z[P.n_u:]).max() == 0.0
    uu = J.csr(0).to_scipy()
    assert np.abs(uu @ z[:P.n_u] - r[:P.n_u]).max() <= 1e-10
    za = orc.Prec(J, 1).apply(r)
    assert np.linalg.norm(za - z) / np.linalg.norm(z) < 1.0
    assert np.abs(za[P.n_u:]).max() == 0.0


def _chain(n):
    import scipy.sparse as sp
    return orc_csr_from(sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1], format="csr"))


def orc_csr_from(M):
    from oracle import orc
    return orc.Csr.from_scipy(M)


def test_amg_diagonal_one_level(orc):  # linsolve_test.cpp:265-276
    import scipy.sparse as sp
    rng = np.random.default_rng(6)
    dg = rng.uniform(1, 5, 30)
    amg = orc.Amg(orc.Csr.from_scipy(sp.diags(dg, format="csr")))
    assert amg.n_levels == 1
    b = rng.uniform(1, 5, 30)
    assert np.allclose(amg.vcycle(b), b / dg, rtol=1e-12)


def test_amg_linear_and_chain(orc):  # linsolve_test.cpp:278-300
    rng = np.random.default_rng(14)
    A = _chain(200)
    amg = orc.Amg(A)
    assert amg.n_levels >= 2
    r, s = rng.uniform(-1, 1, 200), rng.uniform(-1, 1, 200)
    lhs = amg.vcycle(1.7 * r - 0.3 * s)
    rhs = 1.7 * amg.vcycle(r) - 0.3 * amg.vcycle(s)
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * max(1.0, np.linalg.norm(rhs))
    A64 = _chain(64)
    res = orc.gmres(rng.uniform(-1, 1, 64), csr=orc.CsrHandle(A64), amg=orc.Amg(A64))
    assert res["converged"] and res["iterations"] <= 25


def _q1_laplacian(orc, nv):  # linsolve_test.cpp:82-118
    import scipy.sparse as sp
    P = orc.Problem(2, 1.0, 2, int(round(math.log2((nv - 1) / 2))))
    pts, w, s, g = orc.qp_tables(2)
    local = sum(w[q] * g[q, :, :2] @ g[q, :, :2].T for q in range(4))
    n = P.nn if hasattr(P, "nn") else nv
    rows, cols, vals = [], [], []
    bnd = np.zeros(nv * nv, bool)
    for v in range(nv * nv):
        x, y = v % nv, v // nv
        bnd[v] = x in (0, nv - 1) or y in (0, nv - 1)
    for cy in range(nv - 1):
        for cx in range(nv - 1):
            verts = [cx + (k & 1) + nv * (cy + (k >> 1 & 1)) for k in range(4)]
            for a in range(4):
                for b in range(4):
                    if bnd[verts[a]] or bnd[verts[b]]:
                        continue
                    rows.append(verts[a]); cols.append(verts[b]); vals.append(local[a, b])
    for v in np.nonzero(bnd)[0]:
        rows.append(v); cols.append(v); vals.append(1.0)
    M = sp.csr_matrix((vals, (rows, cols)), shape=(nv * nv, nv * nv))
    return orc.Csr.from_scipy(M)


def test_amg_mesh_independence(orc):  # linsolve_test.cpp:302-308
    rng = np.random.default_rng(16)
    its = []
    for nv in (65, 129):
        A = _q1_laplacian(orc, nv)
        res = orc.gmres(rng.uniform(-1, 1, A.rows), csr=orc.CsrHandle(A), amg=orc.Amg(A))
        assert res["converged"]
        its.append(res["iterations"])
    assert its[1] <= 1.5 * its[0] and its[0] <= 1.5 * its[1]


def test_rigid_body_modes(orc):  # linsolve_test.cpp:310-334
    P = orc.Problem(2, 1.0, 3, 0)
    cs = P.constraints()
    B = P.rigid_body_modes(cs)
    assert B.shape == (P.n_u, 3)
    xyz = P.coords()
    f, _ = cs.flags()
    for v in range(P.V):
        if f[2 * v]:
            assert np.all(B[2 * v:2 * v + 2] == 0.0)
        else:
            assert B[2 * v, 0] == 1.0 and B[2 * v + 1, 0] == 0.0 and B[2 * v + 1, 1] == 1.0
            assert abs(B[2 * v, 2] * xyz[v, 0] + B[2 * v + 1, 2] * xyz[v, 1]) <= 1e-12


def test_colpiv_qr_reconstructs(orc):  # ColPivHouseholderQR contract used at linsolve.cpp:217-222
    rng = np.random.default_rng(5)
    for rows, cols in ((18, 3), (81, 6), (4, 6), (27, 6)):
        A = rng.standard_normal((rows, cols))
        A[rows // 2:, 0] = 0.0
        rk, Q, R, perm = orc.colpiv_qr(A)
        assert rk == min(rows, cols)
        assert np.allclose(Q.T @ Q, np.eye(rk), atol=1e-13)
        assert np.allclose(Q @ R, A, atol=1e-12)
    A = np.zeros((6, 3))
    A[:, 0] = 1.0
    A[:, 1] = 2.0  # rank 1
    rk, Q, R, _ = orc.colpiv_qr(A)
    assert rk == 1 and np.allclose(Q @ R, A)
    assert orc.colpiv_qr(np.zeros((5, 3)))[0] == 0


def test_detect_cycles(orc):  # solver_test.cpp:58-88
    out = orc.detect_cycles([[1, 1, 1, 1], [1, 0, 1, 0], [0, 0, 1, 1]], 8, 3)
    assert list(out) == [0, 1, 0]
    rng = np.random.default_rng(42)
    for _ in range(50):
        hs = [list(rng.integers(0, 2, rng.integers(1, 13))) for _ in range(30)]
        exp = []
        for b in hs:
            st = max(0, len(b) - 8)
            exp.append(int(sum(b[k] != b[k - 1] for k in range(st + 1, len(b))) >= 3))
        assert list(orc.detect_cycles(hs, 8, 3)) == exp


def test_newton_intact_converges_immediately(orc):  # solver_test.cpp:90-110
    P = orc.Problem(2, 1.0, 4, 0)
    m = orc.material(pressure=0.0)
    reg = orc.Regularization(0.25, 1e-10)
    sol = np.zeros(P.n_total)
    sol[P.n_u:] = 1.0
    po, pp = np.ones(P.V), np.ones(P.V)
    rep = P.newton_step(m, reg, orc.solver_options(prec_kind=0), sol, po, pp, 1, shift=False)
    assert rep["converged"] and len(rep["iterations"]) == 1
    assert np.abs(sol[:P.n_u]).max() <= 1e-12 and np.abs(sol[P.n_u:] - 1).max() <= 1e-12
    assert rep["feasibility"] <= 1e-10


def _sneddon(orc, d=2, K=5.0, n0=10, r=2, fixed=False):
    P = orc.Problem(d, K, n0, r)
    m = orc.material(eps_mode=1, eps_fixed=2 * P.h, kappa_factor=1e-12 / P.h) if fixed else orc.material()
    reg = P.resolve_regularization(m, P.slit_band_edge(m))
    phi, _ = P.initial_crack(m)
    sol = np.zeros(P.n_total)
    sol[P.n_u:] = phi
    return P, m, reg, sol, phi.copy(), phi.copy()


def test_sneddon_feasibility_and_opening(orc):  # solver_test.cpp:112-150 (uniform mesh)
    P, m, reg, sol, po, pp = _sneddon(orc, r=1)
    rep = P.newton_step(m, reg, orc.solver_options(prec_kind=0), sol, po, pp, 1)
    assert rep["converged"] and rep["feasibility"] <= 1e-10
    assert rep["iterations"][-1, 2] == 0
    assert np.all(np.isfinite(rep["iterations"][:, 0]))
    phi = sol[P.n_u:]
    assert (phi - po).max() <= 1e-10
    xyz = P.coords()
    col = np.abs(xyz[:, 0]) < 1e-12
    above = col & (xyz[:, 1] > 1.4 * reg.eps) & (xyz[:, 1] < 2.0 * reg.eps + P.h)
    below = col & (xyz[:, 1] < -1.4 * reg.eps) & (xyz[:, 1] > -2.0 * reg.eps - P.h)
    assert sol[2 * np.nonzero(above)[0] + 1].min() > 0 and sol[2 * np.nonzero(below)[0] + 1].max() < 0


def test_newton_determinism_and_amg_vs_exact(orc):  # solver_test.cpp:178-210
    runs = []
    for kind in (1, 1, 0):
        P, m, reg, sol, po, pp = _sneddon(orc, r=1)
        rep = P.newton_step(m, reg, orc.solver_options(prec_kind=kind), sol, po, pp, 1)
        assert rep["converged"]
        runs.append((rep, sol))
    (ra, xa), (rb, xb), (re, xe) = runs
    assert np.array_equal(ra["iterations"], rb["iterations"]) and np.array_equal(xa, xb)
    assert np.abs(xa - xe).max() <= 1e-6 * np.abs(xe).max()
    assert ra["iterations"][:, 3].sum() >= 1


def test_gmres_trend_criterion6(orc):  # acceptance_test.cpp:164-187 (r = 1..3 here)
    first = []
    for r in (1, 2, 3):
        P, m, reg, sol, po, pp = _sneddon(orc, r=r)
        rep = P.newton_step(m, reg, orc.solver_options(), sol, po, pp, 1)
        assert rep["converged"]
        first.append(rep["iterations"][0, 3])
    for a, b in zip(first, first[1:]):
        assert b <= 1.3 * a
    assert first[-1] <= 2.5 * first[0]


def test_tcv_manufactured(orc):  # postproc_test.cpp:35-55
    P = orc.Problem(2, 0.5, 1, 2)
    flat = _interp(P, lambda x, c: 0.7 if c == 2 else x[0] + x[1])
    assert abs(P.tcv(flat)) <= 1e-14
    f = _interp(P, lambda x, c: x[0] + 0.5 if c == 0 else (0.0 if c == 1 else x[0]))
    assert P.tcv(f) == pytest.approx(0.5, rel=1e-13)


def test_cod_constant_phi_and_validation(orc):  # postproc_test.cpp:92-105
    P = orc.Problem(2, 2.0, 4, 0)
    f = _interp(P, lambda x, c: 1.0 if c == 2 else x[0] * x[1])
    assert np.abs(P.cod(f, [-1.0, 0.0, 1.0])).max() <= 1e-14
    with pytest.raises(RuntimeError):
        P.cod(f, [0.0, 0.0])
    with pytest.raises(RuntimeError):
        P.cod(f, [-3.0, 0.0])


def test_tcv_closed_form_convergence(orc):  # reference_test.cpp:21-40, PAPER.md:321 (TCV_2d = 6.0319e-3)
    exact = 2 * math.pi * 1e-3 * (1 - 0.2 ** 2) * 1.0
    assert exact == pytest.approx(6.0319e-3, rel=1e-4)
    P, m, reg, sol, po, pp = _sneddon(orc, K=10.0, n0=8, r=3, fixed=True)
    rep = P.newton_step(m, reg, orc.solver_options(), sol, po, pp, 1)
    assert rep["converged"]
    tcv = abs(P.tcv(sol))
    assert 0.5 * exact < tcv < 1.5 * exact


def test_oracle_threads_bitwise(orc):
    """The row-parallel SpMV of the oracle (orc_set_threads) leaves every Newton result bitwise
    unchanged: a 2d Sneddon step (80x80, SpMVs above the pool's 4096-row threshold) with 1 and
    with 4 host threads."""
    O = orc.Problem(2, 5.0, 10, 3)
    m = orc.material()
    reg = O.resolve_regularization(m, O.slit_band_edge(m))
    phi, _ = O.initial_crack(m)
    out = []
    for t in (1, 4):
        orc.set_threads(t)
        sol = np.zeros(O.n_total)
        sol[O.n_u:] = phi
        rep = O.newton_step(m, reg, orc.solver_options(), sol, phi.copy(), phi.copy(), 0, shift=False)
        out.append((rep["iterations"], sol))
    orc.set_threads(1)
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])

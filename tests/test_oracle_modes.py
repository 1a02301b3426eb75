"""The oracle's two execution knobs (CPU only, `-m "not gpu"`):

* thread count — the multi-threaded forms (vertex-owned assembly rows, row-chunked SpGEMM,
  parallel aggregate QR, ...) must reproduce the single-threaded restatement of the reference
  bit for bit, so a config-3-sized check can run on all host cores;
* reduction order — ORDER_REFERENCE must be the reference's arithmetic as written: a CSR row
  is one left-to-right sum (Eigen RowMajor sparse x dense, linsolve.cpp:16-17), a dot one
  sequential sum (linsolve.cpp:30,38,57,60).  scipy's CSR mat-vec and numpy's cumsum are
  exactly those sequential sums, so they pin the mode bitwise.
"""
import numpy as np
import pytest


def _state(orc, d, n0, r, seed, frac_active=5):
    P = orc.Problem(d, 10.0, n0, r)
    m = orc.material(eps_mode=1, eps_fixed=2 * P.h, kappa_factor=1e-12 / P.h)
    reg = P.resolve_regularization(m, P.slit_band_edge(m))
    rng = np.random.default_rng(seed)
    x = np.zeros(P.n_total)
    x[:P.n_u] = 1e-3 * rng.uniform(-1, 1, P.n_u)
    x[P.n_u:] = rng.uniform(0, 1, P.V)
    pt = rng.uniform(0, 1, P.V)
    act = np.arange(0, P.V, frac_active)
    cs = P.constraints(True, P.n_u + act, x[P.n_u + act])
    return P, m, reg, x, pt, cs


@pytest.mark.parametrize("d,n0,r", [(2, 8, 2), (3, 4, 1), (3, 3, 2)])
def test_assembly_thread_invariant(orc, d, n0, r):
    P, m, reg, x, pt, cs = _state(orc, d, n0, r, 11 + d)
    with orc.threads(1):
        R1 = P.residual(cs, m, reg, x, pt)
        J1 = P.jacobian(cs, m, reg, x, pt)
    with orc.threads(5):
        R5 = P.residual(cs, m, reg, x, pt)
        J5 = P.jacobian(cs, m, reg, x, pt)
    assert np.array_equal(R1, R5)
    for w in range(3):
        a, b = J1.csr(w), J5.csr(w)
        assert np.array_equal(a.ptr, b.ptr) and np.array_equal(a.col, b.col)
        assert np.array_equal(a.val, b.val), (w, np.abs(a.val - b.val).max())


def test_amg_and_newton_thread_invariant(orc):
    P, m, reg, x, pt, cs = _state(orc, 3, 4, 1, 5)
    J = P.jacobian(cs, m, reg, x, pt)
    u = J.csr(0)
    node = np.repeat(np.arange(P.V, dtype=np.int32), 3)
    B = P.rigid_body_modes(cs)
    rhs = np.random.default_rng(4).uniform(-1, 1, P.n_u)
    out = []
    for th in (1, 6):
        with orc.threads(th):
            h = orc.Amg(u, node, B)
            levels = [(h.level(l), h.aggregates(l), h.level_matrix(l, 0).val, h.level_matrix(l, 1).val)
                      for l in range(h.n_levels - 1)]
            out.append((levels, h.vcycle(rhs)))
    (l1, v1), (l6, v6) = out
    assert len(l1) == len(l6) and np.array_equal(v1, v6)
    for a, b in zip(l1, l6):
        assert a[0] == b[0] and np.array_equal(a[1], b[1])
        assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3])
    # a whole Newton step on the 3d penny (rebuilds both hierarchies every iteration)
    Q = orc.Problem(3, 10.0, 8, 1)
    mq = orc.material(eps_mode=1, eps_fixed=2 * Q.h, kappa_factor=1e-12 / Q.h)
    rq = Q.resolve_regularization(mq, Q.slit_band_edge(mq))
    phi, _ = Q.initial_crack(mq)
    res = []
    for th in (1, 6):
        with orc.threads(th):
            sol = np.zeros(Q.n_total)
            sol[Q.n_u:] = phi
            rep = Q.newton_step(mq, rq, orc.solver_options(), sol, phi.copy(), phi.copy(), 1)
            res.append((rep["iterations"], sol))
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])


def test_reference_order_is_sequential(orc):
    P, m, reg, x, pt, cs = _state(orc, 3, 4, 1, 9)
    J = P.jacobian(cs, m, reg, x, pt)
    blocks = [J.csr(w).to_scipy() for w in range(3)]
    nu = P.n_u
    with orc.reference_order():
        assert orc.get_order() == orc.ORDER_REFERENCE
        y = J.apply(x)
    assert orc.get_order() == orc.ORDER_PRODUCT
    yu = blocks[0] @ x[:nu]
    yp = blocks[1] @ x[:nu] + blocks[2] @ x[nu:]
    assert np.array_equal(y[:nu], yu) and np.array_equal(y[nu:], yp)
    yprod = J.apply(x)  # the device's lane-split order: equal to rounding, not bitwise
    assert np.linalg.norm(yprod - y) <= 1e-14 * np.linalg.norm(y)
    # GMRES on a CSR operator without preconditioner: iterate 1 is r/||r||, ||r|| a sequential sum
    A = blocks[2].tocsr()
    rhs = np.random.default_rng(3).uniform(-1, 1, A.shape[0])
    with orc.reference_order():
        g = orc.gmres(rhs, csr=orc.CsrHandle(orc.Csr.from_scipy(A)), opts=orc.gmres_options(max_iter=1, restart=1))
    bnorm = np.sqrt(np.cumsum(rhs * rhs)[-1])
    assert g["iterations"] == 1
    v0 = rhs / bnorm
    w = A @ v0
    h00 = np.cumsum(w * v0)[-1]
    w = w - h00 * v0
    h10 = np.sqrt(np.cumsum(w * w)[-1])
    rel = abs(-(h10 / np.hypot(h00, h10)) * bnorm) / bnorm
    assert g["history"][0] == rel


def test_reference_order_newton_close_to_product_order(orc):
    """The two orders run the same algorithm; on a small penny they agree to far below the
    north-star tolerances (this is the oracle-side half of the GPU reference-order tests)."""
    Q = orc.Problem(3, 10.0, 8, 1)
    mq = orc.material(eps_mode=1, eps_fixed=2 * Q.h, kappa_factor=1e-12 / Q.h)
    rq = Q.resolve_regularization(mq, Q.slit_band_edge(mq))
    phi, _ = Q.initial_crack(mq)
    out = []
    for order in (orc.ORDER_PRODUCT, orc.ORDER_REFERENCE):
        orc.set_order(order)
        try:
            sol = np.zeros(Q.n_total)
            sol[Q.n_u:] = phi
            rep = Q.newton_step(mq, rq, orc.solver_options(), sol, phi.copy(), phi.copy(), 1)
        finally:
            orc.set_order(orc.ORDER_PRODUCT)
        out.append((rep["iterations"], sol))
    (i0, s0), (i1, s1) = out
    assert i0.shape == i1.shape and np.array_equal(i0[:, 1:3], i1[:, 1:3])
    assert np.linalg.norm(s0 - s1) <= 1e-10 * np.linalg.norm(s0)

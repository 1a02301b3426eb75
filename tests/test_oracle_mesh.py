"""The general-mesh oracle (oracle/oracle_mesh.inc) pinned by ports of the
reference's own known-answer tests: mesh_test.cpp (forest, closure, faces, point location),
fem_test.cpp:144-359 (hanging constraints, transfer), adapt_test.cpp (estimator, marking,
adaptive cycle), and by bitwise agreement with the uniform-grid oracle on uniformly refined
meshes (the general path reduces to it there)."""
import math

import numpy as np
import pytest

KUNIT = 1 << 16


def hanging_mesh(orc, d):  # adapt_test.cpp:20-24 / fem_test.cpp: K = 1, 2^d cells, cell 0 refined
    m = orc.Mesh(d, 1.0, 2)
    m.refine([0])
    return m


def balance_ok(m):  # mesh_test.cpp:27-34
    cells = m.cells()
    for cell, axis, side, nb, rel in m.faces():
        if nb < 0:
            continue
        dl = cells["level"][cell] - cells["level"][nb]
        if abs(dl) > 1 or rel != -dl:
            return False
    return True


def brute_pairs(m):  # mesh_test.cpp:38-66
    cells = m.cells()
    act = m.active()
    d = m.d
    out = set()
    for i, a in enumerate(act):
        for b in act[i + 1:]:
            touch, ok = -1, True
            for ax in range(d):
                alo = cells["anchor"][a][ax]
                ahi = alo + (KUNIT >> cells["level"][a])
                blo = cells["anchor"][b][ax]
                bhi = blo + (KUNIT >> cells["level"][b])
                if ahi < blo or bhi < alo:
                    ok = False
                    break
                if ahi == blo or bhi == alo:
                    if touch >= 0:
                        ok = False
                        break
                    touch = ax
            if ok and touch >= 0:
                out.add((min(a, b), max(a, b)))
    return out


def test_mesh_create_refine_closure(orc):  # mesh_test.cpp:78-151
    m = orc.Mesh(2, 1.0, 1)
    m.refine([])
    assert m.n_active == 1
    m.refine([m.active()[0]])
    assert m.n_active == 4
    with pytest.raises(RuntimeError):
        m.refine([9999])
    m = orc.Mesh(2, 1.0, 2)
    ll = m.find_cell([-0.5, -0.5])
    m.refine([ll])
    m.refine([m.find_cell([-0.75, -0.75])])
    assert balance_ok(m)
    assert m.max_level == 2
    assert 1 in set(m.cells()["level"][m.active()])
    m = orc.Mesh(2, 20.0, 8)
    m.uniform_refine(5)
    assert m.n_active == 65536 and m.h_min == pytest.approx(40.0 / 256.0)
    m = orc.Mesh(3, 5.0, 2)
    m.uniform_refine(1)
    assert m.n_active == 64
    with pytest.raises(RuntimeError):
        orc.Mesh(4, 1.0, 2)


@pytest.mark.parametrize("d", [2, 3])
def test_active_faces_match_brute_force(orc, d):  # mesh_test.cpp:173-201
    rng = np.random.default_rng(2024 + d)
    m = orc.Mesh(d, 1.0, 2)
    for _ in range(3 if d == 2 else 2):
        act = m.active()
        marked = [c for c in act if rng.integers(3) == 0] or [act[0]]
        m.refine(marked)
        assert balance_ok(m)
        rep = {}
        cells = m.cells()
        for cell, axis, side, nb, rel in m.faces():
            if nb < 0:
                continue
            key = (min(cell, nb), max(cell, nb))
            rep[key] = rep.get(key, 0) + 1
            if rel == -1:
                assert cells["level"][cell] == cells["level"][nb] + 1
        assert all(v == 1 for v in rep.values())
        assert set(rep) == brute_pairs(m)


@pytest.mark.parametrize("d", [2, 3])
def test_tiling_and_determinism(orc, d):  # mesh_test.cpp:203-230
    rng = np.random.default_rng(99)
    m = orc.Mesh(d, 7.5 if d == 2 else 2.5, 3 if d == 2 else 2)
    for _ in range(4 if d == 2 else 2):
        act = m.active()
        m.refine([c for c in act if rng.integers(4) == 0])
        cells = m.cells()
        lev = cells["level"][m.active()]
        meas = np.sum((2.0 * m.K / (m.n0 * 2.0 ** lev)) ** d)
        assert meas == pytest.approx((2.0 * m.K) ** d, rel=1e-12)
        assert balance_ok(m)

    def run():
        mm = orc.Mesh(2, 1.0, 2)
        a = mm.active()
        mm.refine([a[0], a[3]])
        mm.refine([mm.active()[2]])
        return mm.active()

    assert np.array_equal(run(), run())


def test_point_location(orc):  # mesh_test.cpp:245-266
    m = orc.Mesh(2, 1.0, 2)
    m.refine([m.find_cell([-0.5, -0.5])])
    cid = m.find_cell([0.6, 0.6])
    assert cid >= 0 and m.cells()["active"][cid]
    # the level-0/level-1 corner at the origin: the smallest containing id
    act = m.active()
    cells = m.cells()
    at = [c for c in act if all(cells["anchor"][c][a] <= KUNIT <= cells["anchor"][c][a] + (KUNIT >> cells["level"][c])
                                for a in range(2))]
    assert len(at) >= 3 and m.find_cell([0.0, 0.0]) == min(at)
    assert m.find_cell([-1.5, 0.0]) == -1


@pytest.mark.parametrize("d", [2, 3])
def test_hanging_constraints_conform(orc, d):  # fem_test.cpp:144-211
    m = hanging_mesh(orc, d)
    cs = m.constraints(clamp=False)
    dofs, ptr, masters, w, inh = cs.lines()
    keys = m.vertex_keys()
    xyz = np.stack([keys & ((1 << 21) - 1), (keys >> 21) & ((1 << 21) - 1), (keys >> 42) & ((1 << 21) - 1)], 1)
    phys = -1.0 + xyz * (2.0 / (2 * KUNIT))
    if d == 2:
        phys[:, 2] = 0.0

    def lin(x, c):
        return (c + 1.0) * x[:, 0] + 2.0 * x[:, 1] - 0.75 * x[:, 2] + 0.25 * c

    f = np.zeros(m.n_total)
    for c in range(d):
        f[c:m.n_u:d] = lin(phys, c)
    f[m.n_u:] = lin(phys, d)
    g = cs.distribute(f)
    assert len(dofs) > 0
    for i, dof in enumerate(dofs):
        ww = w[ptr[i]:ptr[i + 1]]
        assert np.all((ww == 0.5) | (ww == 0.25))
        assert abs(ww.sum() - 1.0) <= 1e-14
        assert not np.isin(masters[ptr[i]:ptr[i + 1]], dofs).any()  # closed form
        assert g[dof] == pytest.approx(f[dof], rel=1e-13, abs=1e-13)
    assert np.array_equal(cs.distribute(g), g)  # idempotent


@pytest.mark.parametrize("d", [2, 3])
def test_transfer_exact_on_nested_spaces(orc, d):  # fem_test.cpp:302-359
    old = hanging_mesh(orc, d)
    rng = np.random.default_rng(31)
    v = old.constraints(clamp=False).distribute(rng.uniform(-1, 1, old.n_total))
    new = old.copy()
    new.refine(old.active()[::2])
    moved = old.transfer_to(v, new)
    one_new = old.transfer_to(np.ones(old.n_total), new)
    assert np.abs(one_new - 1.0).max() <= 1e-14
    # old vertices keep their values exactly (they are vertices of the refinement too)
    ko, kn = old.vertex_keys(), new.vertex_keys()
    idx = np.searchsorted(kn, ko)
    assert np.array_equal(kn[idx], ko)
    assert np.abs(moved[new.n_u + idx] - v[old.n_u + np.arange(old.V)]).max() <= 1e-15


@pytest.mark.parametrize("d", [2, 3])
def test_estimator_kats(orc, d):  # adapt_test.cpp:100-128
    m = hanging_mesh(orc, d)
    keys = m.vertex_keys()
    xyz = np.stack([keys & ((1 << 21) - 1), (keys >> 21) & ((1 << 21) - 1), (keys >> 42) & ((1 << 21) - 1)], 1)
    x = -1.0 + xyz * (2.0 / (2 * KUNIT))
    if d == 2:
        x[:, 2] = 0.0
    lin = np.zeros(m.n_total)
    for c in range(d):
        lin[c:m.n_u:d] = 0.7 + 1.3 * x[:, 0] - 0.4 * x[:, 1] + (0.9 * x[:, 2] if d == 3 else 0.0) + 0.1 * c
    lin[m.n_u:] = 0.3 * x[:, 0]
    assert np.all(m.estimator(lin) <= 1e-12)
    m = orc.Mesh(d, 1.0, 2)
    kk = m.vertex_keys()
    xx = -1.0 + (kk & ((1 << 21) - 1)) * (2.0 / (2 * KUNIT))
    kink = np.zeros(m.n_total)
    kink[0:m.n_u:d] = np.abs(xx)
    eta = m.estimator(kink)
    assert len(eta) == 1 << d and np.allclose(eta, 1.0, rtol=1e-12)


def test_mark_cells_kats(orc):  # adapt_test.cpp:171-259
    m = hanging_mesh(orc, 2)
    keys = m.vertex_keys()
    x0 = -1.0 + (keys & ((1 << 21) - 1)) * (2.0 / (2 * KUNIT))
    x1 = -1.0 + ((keys >> 21) & ((1 << 21) - 1)) * (2.0 / (2 * KUNIT))
    sol = np.zeros(m.n_total)
    sol[m.n_u:] = np.where((x0 < -0.4) & (x1 < -0.4), 0.1, 1.0)
    marked = m.mark(sol, estimator=False)
    cv = m.cell_vertices()
    expect = sorted(int(c) for c, vs in zip(m.active(), cv) if sol[m.n_u + vs].min() < 0.8)
    assert list(marked) == expect and len(marked) > 0
    assert len(m.mark(sol, estimator=False, h_target=2.0)) == 0
    m = orc.Mesh(2, 1.0, 4)
    intact = np.zeros(m.n_total)
    intact[m.n_u:] = 1.0
    act = m.active()
    eta = np.zeros(len(act))
    assert len(m.mark(intact, eta)) == 0
    eta[5] = 2.0
    assert list(m.mark(intact, eta)) == [act[5]]
    assert list(m.mark(intact, np.ones(len(act)), theta=1.0)) == sorted(act)
    eta = np.zeros(len(act))
    eta[:3] = [3.0, 2.0, 1.0]
    assert list(m.mark(intact, eta, theta=0.5)) == [act[0]]
    assert list(m.mark(intact, eta, theta=0.75)) == sorted([act[0], act[1]])


def test_adaptive_cycle_kats(orc):  # adapt_test.cpp:293-349
    mat = orc.material()
    so = orc.solver_options(prec_kind=0)
    m = orc.Mesh(2, 5.0, 10)
    with pytest.raises(RuntimeError):
        m.adaptive_cycle(mat, so, cycles=-1)
    rec, _ = m.adaptive_cycle(mat, so, cycles=0)
    assert len(rec) == 1 and rec[0][7] == 1.0 and rec[0][0] == 0 and rec[0][1] == m.n_total and rec[0][4] > 0
    m = orc.Mesh(2, 5.0, 10)
    rec, sol = m.adaptive_cycle(mat, so, cycles=2, n_steps=2, theta=0.3)
    assert len(rec) == 3
    exact = 2.0 * math.pi * 1e-3 * (1 - 0.04) / 1.0
    for i in range(3):
        assert rec[i][7] == 1.0 and rec[i][0] == i and rec[i][4] > 0
        if i:
            assert rec[i][2] == pytest.approx(0.5 * rec[i - 1][2], rel=1e-12)
            assert rec[i][3] <= rec[i - 1][3]
            assert rec[i - 1][1] < rec[i][1] < 4 * rec[i - 1][1]
    assert abs(rec[-1][4] - exact) < abs(rec[0][4] - exact)


@pytest.mark.parametrize("d,n0,r", [(2, 4, 2), (3, 2, 1)])
def test_uniform_mesh_equals_grid_oracle(orc, d, n0, r):
    """On a uniformly refined mesh the general path (triplets + setFromTriplets, constraint lines)
    is bitwise the uniform-grid oracle (residual, Jacobian); a whole Newton step agrees to rounding."""
    m = orc.Mesh(d, 1.0, n0)
    m.uniform_refine(r)
    P = orc.Problem(d, 1.0, n0, r)
    assert m.V == P.V
    rng = np.random.default_rng(5 + d)
    x = np.zeros(P.n_total)
    x[:P.n_u] = 1e-2 * rng.uniform(-1, 1, P.n_u)
    x[P.n_u:] = rng.uniform(0, 1, P.V)
    pt = rng.uniform(0, 1, P.V)
    act = list(range(P.n_u, P.n_total, 5))
    vals = [float(x[i]) for i in act]
    mat, reg = orc.material(pressure=1e-3), orc.Regularization(0.25, 1e-10)
    a, b = m.constraints(True, act, vals), P.constraints(True, act, vals)
    assert np.array_equal(m.residual(a, mat, reg, x, pt), P.residual(b, mat, reg, x, pt))
    Ja, Jb = m.jacobian(a, mat, reg, x, pt), P.jacobian(b, mat, reg, x, pt)
    for w in range(3):
        A, B = Ja.csr(w), Jb.csr(w)
        assert np.array_equal(A.ptr, B.ptr) and np.array_equal(A.col, B.col) and np.array_equal(A.val, B.val)
    # Newton step on a Sneddon slit
    m2 = orc.Mesh(2, 5.0, 10)
    m2.uniform_refine(1)
    P2 = orc.Problem(2, 5.0, 10, 1)
    mat = orc.material()
    reg2 = m2.resolve_regularization(mat, m2.slit_band_edge(mat))
    phi, _ = m2.initial_crack(mat)
    phi_p, _ = P2.initial_crack(mat)
    assert np.array_equal(phi, phi_p)
    s1 = np.zeros(m2.n_total)
    s1[m2.n_u:] = phi
    s2 = s1.copy()
    r1 = m2.newton_step(mat, reg2, orc.solver_options(), s1, phi.copy(), phi.copy(), 0, shift=False)
    r2 = P2.newton_step(mat, reg2, orc.solver_options(), s2, phi.copy(), phi.copy(), 0, shift=False)
    # the Newton dots of a general mesh reduce each block in flat 8192-chunks (one "plane"), the
    # grid's per vertex plane: the same sums in another order, so the step agrees to rounding
    i1, i2 = r1["iterations"], r2["iterations"]
    assert np.array_equal(i1[:, 1:], i2[:, 1:])
    assert np.allclose(i1[:-1, 0], i2[:-1, 0], rtol=1e-9, atol=0)
    assert np.abs(s1 - s2).max() <= 1e-12 * np.abs(s2).max()
    assert m2.tcv(s1) == pytest.approx(P2.tcv(s2), rel=1e-10)

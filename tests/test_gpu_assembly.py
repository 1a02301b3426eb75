"""GPU parity of K1/K2/K4 (residual, Jacobian, block apply) against the CPU oracle.

Assembly is bit-exact: same pattern (int64 row pointers, int32 columns) and the same IEEE
doubles, because the kernels reproduce the reference's expression order and cell order
(model.cpp:127-322).  SpMV/apply is compared within 1e-13 relative (different summation order).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cf():
    import paper_1806_09924_b200 as cf
    return cf


def _pair(cf, orc, d, K, n0, r):
    return cf.Problem(d, K, n0, r), orc.Problem(d, K, n0, r)


def _state(P, rng, uscale=1e-2):
    x = np.zeros(P.n_total)
    x[:P.n_u] = uscale * rng.uniform(-1, 1, P.n_u)
    x[P.n_u:] = rng.uniform(0, 1, P.n_vertices)
    return x, rng.uniform(0, 1, P.n_vertices)


def _assert_blocks_equal(J, Jo):
    for w in range(3):
        a, b = J.csr(w), Jo.csr(w)
        assert np.array_equal(a.ptr, b.ptr), f"row pointers differ in block {w}"
        assert np.array_equal(a.col, b.col), f"columns differ in block {w}"
        bad = np.nonzero(a.val != b.val)[0]
        assert bad.size == 0, f"block {w}: {bad.size} values differ, max {np.abs(a.val - b.val).max()}"


CASES = [
    (2, 1.0, 4, 2, True, 0.0, 0),   # 16x16, clamp
    (2, 1.0, 3, 1, False, 0.0, 0),  # unconstrained
    (2, 1.0, 4, 2, True, 0.2, 1),   # with an active set, current pressure coupling
    (3, 1.0, 2, 1, True, 0.0, 0),   # 4^3
    (3, 1.0, 3, 1, True, 0.15, 0),  # 6^3 + active set
    (3, 2.0, 2, 2, False, 0.1, 1),  # 8^3 unconstrained + active
]


@pytest.mark.parametrize("d,K,n0,r,clamp,frac_active,coupling", CASES)
def test_assembly_bit_exact(cf, orc, d, K, n0, r, clamp, frac_active, coupling):
    P, O = _pair(cf, orc, d, K, n0, r)
    rng = np.random.default_rng(100 + d * 10 + n0 + r)
    x, pt = _state(P, rng)
    nact = int(frac_active * P.n_vertices)
    verts = rng.choice(P.n_vertices, nact, replace=False) if nact else np.zeros(0, dtype=np.int64)
    act = {int(P.n_u + v): float(rng.uniform(0, 1)) for v in verts}
    cs = cf.build_constraints(P, clamp, act)
    ocs = O.constraints(clamp, list(act.keys()), list(act.values()))
    mat = cf.Material(pressure=2e-3, pressure_coupling=coupling)
    omat = orc.material(pressure=2e-3, pressure_coupling=coupling)
    reg, oreg = cf.Regularization(0.3, 1e-6), orc.Regularization(0.3, 1e-6)
    R = cf.assemble_residual(P, cs, mat, reg, x, pt)
    Ro = O.residual(ocs, omat, oreg, x, pt)
    assert np.array_equal(R, Ro), np.abs(R - Ro).max()
    J = cf.assemble_jacobian(P, cs, mat, reg, x, pt)
    Jo = O.jacobian(ocs, omat, oreg, x, pt)
    _assert_blocks_equal(J, Jo)
    z = rng.standard_normal(P.n_total)
    y, yo = J.apply(z), Jo.apply(z)
    assert np.linalg.norm(y - yo) <= 1e-13 * np.linalg.norm(yo)
    for w, (rows, cols) in enumerate(((P.n_u, P.n_u), (P.n_phi, P.n_u), (P.n_phi, P.n_phi))):
        xin = rng.standard_normal(cols)
        ref = Jo.csr(w).to_scipy() @ xin
        got = J.spmv(w, xin)
        assert np.linalg.norm(got - ref) <= 1e-13 * max(np.linalg.norm(ref), 1e-300)


def _sneddon(cf, orc, d, n0, r, K=10.0):
    P, O = _pair(cf, orc, d, K, n0, r)
    h = P.h
    kw = dict(eps_mode=1, eps_fixed=2 * h, kappa_factor=1e-12 / h)
    omat = orc.material(**kw)
    phi, _ = O.initial_crack(omat)
    oreg = O.resolve_regularization(omat, O.slit_band_edge(omat))
    return P, O, cf.Material(**kw), omat, cf.Regularization(oreg.eps, oreg.kappa), oreg, phi


def test_config0_sneddon_bit_exact(cf, orc):
    """BASELINE config 0 (2d 256^2, eps=2h, kappa=1e-12): initial and perturbed states."""
    P, O, mat, omat, reg, oreg, phi = _sneddon(cf, orc, 2, 8, 5)
    assert P.n_total == 198147
    rng = np.random.default_rng(0)
    x = np.zeros(P.n_total)
    x[P.n_u:] = phi
    for trial in range(2):
        cs, ocs = cf.build_constraints(P), O.constraints()
        R, Ro = cf.assemble_residual(P, cs, mat, reg, x, phi), O.residual(ocs, omat, oreg, x, phi)
        assert np.array_equal(R, Ro)
        J, Jo = cf.assemble_jacobian(P, cs, mat, reg, x, phi), O.jacobian(ocs, omat, oreg, x, phi)
        _assert_blocks_equal(J, Jo)
        x[:P.n_u] += 1e-3 * rng.standard_normal(P.n_u)
        ocs.distribute(x, homogeneous=True)
        x = ocs.distribute(x, homogeneous=True)


def test_3d_penny_bit_exact(cf, orc):
    """3d penny crack on 32^3 (config 3 family)."""
    P, O, mat, omat, reg, oreg, phi = _sneddon(cf, orc, 3, 8, 2)
    rng = np.random.default_rng(1)
    x = np.zeros(P.n_total)
    x[:P.n_u] = 1e-3 * rng.standard_normal(P.n_u)
    x[P.n_u:] = phi
    act = {int(P.n_u + v): 0.0 for v in np.nonzero(phi == 0)[0]}
    cs, ocs = cf.build_constraints(P, True, act), O.constraints(True, list(act.keys()), list(act.values()))
    x = ocs.distribute(x)
    R, Ro = cf.assemble_residual(P, cs, mat, reg, x, phi), O.residual(ocs, omat, oreg, x, phi)
    assert np.array_equal(R, Ro)
    _assert_blocks_equal(cf.assemble_jacobian(P, cs, mat, reg, x, phi), O.jacobian(ocs, omat, oreg, x, phi))


def test_jacobian_fd_on_device(cf):
    """model_test.cpp:211-240 on the device path: J delta vs central differences <= 1e-5."""
    rng = np.random.default_rng(13)
    for d, n0 in ((2, 4), (3, 2)):
        P = cf.Problem(d, 1.0, n0, 1)
        cs = cf.build_constraints(P)
        mat, reg = cf.Material(pressure=1e-3), cf.Regularization(0.25, 1e-10)
        x, pt = _state(P, rng)
        cs.distribute_homogeneous(x)
        J = cf.assemble_jacobian(P, cs, mat, reg, x, pt)
        for _ in range(3):
            dl = rng.uniform(-1, 1, P.n_total)
            cs.distribute_homogeneous(dl)
            t = 1e-6 * max(1.0, np.abs(x).max())
            fd = (cf.assemble_residual(P, cs, mat, reg, x + t * dl, pt)
                  - cf.assemble_residual(P, cs, mat, reg, x - t * dl, pt)) / (2 * t)
            jd = J.apply(dl)
            assert np.linalg.norm(fd - jd) / np.linalg.norm(jd) <= 1e-5


def test_device_pointer_path_matches_host(cf):
    import torch
    P = cf.Problem(3, 1.0, 2, 2)
    rng = np.random.default_rng(3)
    x, pt = _state(P, rng)
    cs = cf.build_constraints(P)
    mat, reg = cf.Material(), cf.Regularization(0.25, 1e-10)
    Rh = cf.assemble_residual(P, cs, mat, reg, x, pt)
    xd, ptd = torch.from_numpy(x).cuda(), torch.from_numpy(pt).cuda()
    Rd = cf.assemble_residual(P, cs, mat, reg, xd, ptd)
    torch.cuda.synchronize()
    assert np.array_equal(Rd.cpu().numpy(), Rh)
    J = cf.assemble_jacobian(P, cs, mat, reg, xd, ptd)
    yd = J.apply(xd)
    torch.cuda.synchronize()
    assert np.array_equal(yd.cpu().numpy(), J.apply(x))


def test_constraints_distribute(cf, orc):  # fem_test.cpp:213-225
    P = cf.Problem(2, 1.0, 2, 0)
    cs = cf.build_constraints(P, True, {P.phi_dof(0): 0.25, P.phi_dof(3): 1.0})
    v = np.zeros(P.n_total)
    cs.distribute(v)
    assert v[P.phi_dof(0)] == 0.25 and v[P.phi_dof(3)] == 1.0
    inc = np.ones(P.n_total)
    cs.distribute_homogeneous(inc)
    assert inc[P.phi_dof(0)] == 0.0
    O = orc.Problem(2, 1.0, 2, 0)
    ocs = O.constraints(True, [P.phi_dof(0), P.phi_dof(3)], [0.25, 1.0])
    w = np.ones(P.n_total)
    assert np.array_equal(cs.distribute(w.copy()), ocs.distribute(w))
    with pytest.raises(ValueError):
        cf.build_constraints(P, True, {10 ** 9: 0.0})


@pytest.mark.slow
def test_config1_operator_properties(cf):
    """Config 1 at full size (3d 192^3, 21.5M u dofs): the exact nnz of SURVEY §8(a) and
    size-independent properties of y = M_uu u (symmetry, rigid-translation kernel)."""
    import torch
    from bench import config1_inputs
    P, cs, mat, reg, x, pt = config1_inputs(cf, device="cuda")
    J = cf.assemble_jacobian(P, cs, mat, reg, x, pt)
    assert J.nnz[0] == 1_676_188_257
    u = x[:P.n_u].contiguous()
    g = torch.Generator(device="cuda").manual_seed(5)
    w = torch.randn(P.n_u, dtype=torch.float64, device="cuda", generator=g)
    Mu, Mw = J.spmv(0, u), J.spmv(0, w)
    a, b = torch.dot(w, Mu).item(), torch.dot(u, Mw).item()
    assert abs(a - b) <= 1e-10 * (abs(a) + abs(b))
    t = torch.zeros(P.n_u, dtype=torch.float64, device="cuda")
    t[0::3] = 1.0
    Mt = J.spmv(0, t)
    n = P.nodes_per_side
    idx = torch.arange(P.n_vertices, device="cuda")
    xi, yi, zi = idx % n, (idx // n) % n, idx // (n * n)
    interior = (xi > 1) & (xi < n - 2) & (yi > 1) & (yi < n - 2) & (zi > 1) & (zi < n - 2)
    rows = Mt.view(-1, 3)[interior]
    assert rows.abs().max().item() <= 1e-12 * Mu.abs().max().item() + 1e-14


@pytest.mark.parametrize("d,n0,r,frac", [(2, 2, 1, 0.0), (2, 3, 1, 0.2), (3, 2, 1, 0.15)])
def test_assemble_pattern_covers_support_overlaps(cf, d, n0, r, frac):
    """linsolve_test.cpp:147-190: dofs couple when their vertices share a cell, routed through the
    constraint masters (Dirichlet / active lines have none); constrained dofs keep their diagonal."""
    P = cf.Problem(d, 1.0, n0, r)
    rng = np.random.default_rng(5 + d)
    nact = int(frac * P.n_vertices)
    act = {int(P.n_u + v): 0.5 for v in rng.choice(P.n_vertices, nact, replace=False)}
    cs = cf.build_constraints(P, True, act)
    pat = cf.assemble_pattern(P, cs)
    nn = P.nodes_per_side
    nc = nn - 1
    xyz = lambda v: (v % nn, (v // nn) % nn, v // (nn * nn) if d == 3 else 0)
    bnd = lambda v: any(c in (0, nc) for c in xyz(v)[:d])
    cons = set(act)
    for v in range(P.n_vertices):
        if bnd(v):
            cons.update(v * d + a for a in range(d))
    uu, pu, pp = set(), set(), set()
    for cz in range(nc if d == 3 else 1):
        for cy in range(nc):
            for cx in range(nc):
                verts = [(cx + (k & 1)) + nn * ((cy + ((k >> 1) & 1)) + nn * (cz + ((k >> 2) & 1)))
                         for k in range(1 << d)]
                for a in verts:
                    for b in verts:
                        for ca in range(d):
                            for cb in range(d):
                                i, j = a * d + ca, b * d + cb
                                if i not in cons and j not in cons:
                                    uu.add((i, j))
                        for cb in range(d):
                            i, j = P.n_u + a, b * d + cb
                            if i not in cons and j not in cons:
                                pu.add((a, j))
                        if P.n_u + a not in cons and P.n_u + b not in cons:
                            pp.add((a, b))
    for dof in cons:
        if dof < P.n_u:
            uu.add((dof, dof))
        else:
            pp.add((dof - P.n_u, dof - P.n_u))
    for w, ref in enumerate((uu, pu, pp)):
        A = pat.csr(w)
        got = {(i, int(A.col[k])) for i in range(A.rows) for k in range(A.ptr[i], A.ptr[i + 1])}
        assert got == ref, f"block {w}"
        for i in range(A.rows):  # ascending columns
            assert np.all(np.diff(A.col[A.ptr[i]:A.ptr[i + 1]]) > 0)
        assert not A.val.any()
    # the Jacobian's pattern is the same except constrained diagonals that sum to exactly zero
    x = np.zeros(P.n_total)
    x[P.n_u:] = rng.uniform(0, 1, P.n_vertices)
    J = cf.assemble_jacobian(P, cs, cf.Material(), cf.Regularization(0.3, 1e-6), x, rng.uniform(0, 1, P.n_vertices))
    for w in range(3):
        A, B = J.csr(w), pat.csr(w)
        ja = {(i, int(A.col[k])) for i in range(A.rows) for k in range(A.ptr[i], A.ptr[i + 1])}
        jb = {(i, int(B.col[k])) for i in range(B.rows) for k in range(B.ptr[i], B.ptr[i + 1])}
        assert ja <= jb and all(i == j for i, j in jb - ja)


def test_extrapolate_phi(cf):
    """model.cpp:60-64: phi_old for step <= 2, else clip(2 phi_old - phi_prev2, [0, 1])."""
    P = cf.Problem(2, 1.0, 4, 1)
    rng = np.random.default_rng(8)
    po, pp = rng.uniform(-0.2, 1.2, P.n_vertices), rng.uniform(-0.2, 1.2, P.n_vertices)
    for step in (0, 2, 3, 7):
        st = cf.FractureState(P, np.zeros(P.n_total), po, pp, step)
        got = cf.extrapolate_phi(st)
        ref = po if step <= 2 else np.minimum(np.maximum(2.0 * po - pp, 0.0), 1.0)
        assert np.array_equal(got, ref)


@pytest.mark.parametrize("d,n0,r,clamp", [(2, 4, 2, True), (2, 3, 2, False), (3, 3, 1, True), (3, 2, 2, True),
                                          (3, 5, 2, True), (3, 3, 2, False), (3, 9, 1, True)])
def test_matrix_free_apply_equals_assembled(cf, d, n0, r, clamp):
    """BASELINE config 1's matrix-free operator: y = M_uu x from phi_tilde cell by cell, equal to the
    assembled block's apply (Dirichlet condensation included) to 1e-12 relative."""
    P = cf.Problem(d, 1.0, n0, r)
    rng = np.random.default_rng(21 + d + n0)
    cs = cf.build_constraints(P, clamp)
    pt = rng.uniform(0, 1, P.n_vertices)
    x = np.zeros(P.n_total)
    x[P.n_u:] = pt
    mat, reg = cf.Material(pressure=1e-3), cf.Regularization(0.3, 1e-12)
    J = cf.assemble_jacobian(P, cs, mat, reg, x, pt)
    u = rng.standard_normal(P.n_u)
    ref = J.spmv(0, u)
    got = cf.mf_apply_uu(P, cs, mat, reg, pt, u)
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)


@pytest.mark.parametrize("h", [20.0 / 256, 20.0 / 128, 20.0 / 2048, 20.0 / 192, 2.0 / 16, 10.0 / 40, 0.3, 1.0 / 3.0])
def test_div_by_h_is_ieee_division(cf, h):
    """The residual kernel divides every gradient product by the cell size h through a reciprocal
    and two Markstein corrections (assembly.cu DivBy); it must be the IEEE quotient a / h bit for bit:
    4M random dividends over 2^-70..2^70 of both signs, mantissas uniform, plus zeros, subnormals,
    extreme exponents, infinities and NaN."""
    import ctypes as C
    from paper_1806_09924_b200._lib import check, load
    rng = np.random.default_rng(int(h * 1e6))
    n = 1 << 22
    a = rng.uniform(1.0, 2.0, n) * np.exp2(rng.integers(-70, 71, n)) * rng.choice([-1.0, 1.0], n)
    # products of shape-gradient-like factors, as in the kernel
    a[: n // 4] = rng.normal(size=n // 4) * rng.uniform(-0.8, 0.8, n // 4)
    special = np.array([0.0, -0.0, 5e-324, -5e-324, 2.2250738585072014e-308, 1e-300, 1e300, 1.7976931348623157e308,
                        np.inf, -np.inf, np.nan, 2.0 ** -900, 2.0 ** 900, h, -h, 2 * h, h / 3])
    a[: special.size] = special
    q = np.empty_like(a)
    check(load().cf_test_div_by(C.c_double(h), a.ctypes.data_as(C.c_void_p), C.c_int64(n), q.ctypes.data_as(C.c_void_p)))
    ref = a / h
    same = (q.view(np.uint64) == ref.view(np.uint64)) | (np.isnan(q) & np.isnan(ref))
    assert same.all(), f"{(~same).sum()} quotients differ, e.g. a={a[~same][:3]} q={q[~same][:3]} ref={ref[~same][:3]}"

"""GPU parity of the solver stack: AMG setup (K7) and V-cycle (K8), GMRES (K6), the block
preconditioner and the Newton / active-set step (K9, K10) against the CPU oracle.

The device path and the oracle share one documented reduction order, so the
comparisons are bit-for-bit: aggregates, every level operator, lambda_max, V-cycle outputs,
GMRES iterates, Newton transcripts and solutions.
"""
import math

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cf():
    import paper_1806_09924_b200 as cf
    return cf


def _chain(n):
    return sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1], format="csr")


def _assert_amg_equal(h, ho, exact=True):
    assert h.n_levels() == ho.n_levels and h.coarse_dim() == ho.coarse_dim
    for lev in range(ho.n_levels - 1):
        a, b = h.level_info(lev), ho.level(lev)
        for k in ("rows", "nnz_A", "nnz_P", "coarse", "n_nodes", "n_aggregates"):
            assert a[k] == b[k], (lev, k, a[k], b[k])
        assert np.array_equal(h.aggregates(lev), ho.aggregates(lev)), f"aggregates differ on level {lev}"
        if exact:
            assert a["lam"] == b["lam"], (lev, a["lam"], b["lam"])
            for w in (0, 1):
                m1, m2 = h.level_matrix(lev, w), ho.level_matrix(lev, w)
                assert np.array_equal(m1.ptr, m2.ptr) and np.array_equal(m1.col, m2.col)
                assert np.array_equal(m1.val, m2.val), (lev, w, np.abs(m1.val - m2.val).max())


def test_amg_scalar_chain_and_diag(cf, orc):  # linsolve_test.cpp:265-300
    rng = np.random.default_rng(6)
    dg = rng.uniform(1, 5, 30)
    h = cf.build_amg(cf.CsrMatrix.from_scipy(sp.diags(dg, format="csr")))
    assert h.n_levels() == 1
    b = rng.uniform(1, 5, 30)
    assert np.allclose(h.v_cycle(b), b / dg, rtol=1e-12)
    A = _chain(200)
    h = cf.build_amg(cf.CsrMatrix.from_scipy(A))
    ho = orc.Amg(orc.Csr.from_scipy(A))
    _assert_amg_equal(h, ho)
    r = rng.uniform(-1, 1, 200)
    assert np.array_equal(h.v_cycle(r), ho.vcycle(r))
    s = rng.uniform(-1, 1, 200)
    lhs, rhs = h.v_cycle(1.7 * r - 0.3 * s), 1.7 * h.v_cycle(r) - 0.3 * h.v_cycle(s)
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * max(1.0, np.linalg.norm(rhs))
    A64 = cf.CsrMatrix.from_scipy(_chain(64))
    res = cf.gmres(A64, rng.uniform(-1, 1, 64), prec=cf.build_amg(A64))
    assert res["converged"] and res["iterations"] <= 25


def _random_graph_spd(n, deg, seed):
    rng = np.random.default_rng(seed)
    rows = np.repeat(np.arange(n), deg)
    cols = rng.integers(0, n, n * deg)
    vals = -rng.uniform(0.5, 1.0, n * deg)
    S = sp.csr_matrix((vals, (rows, cols)), shape=(n, n))
    S = S + S.T
    S.setdiag(0.0)
    S.eliminate_zeros()
    d = np.asarray(abs(S).sum(axis=1)).ravel() + 1.0
    return (S + sp.diags(d)).tocsr()


def test_amg_high_degree_tiers_bit_exact(cf, orc):
    """Random graph (~80 neighbours per row, a fully dense 2752^2 coarse level): strength/N2 overflow
    tiers and SpGEMM rows beyond the 384- and 1024-column tiers must still reproduce the oracle's
    hierarchy bit for bit."""
    A = _random_graph_spd(4000, 40, 5)
    h = cf.build_amg(cf.CsrMatrix.from_scipy(A))
    ho = orc.Amg(orc.Csr.from_scipy(A))
    _assert_amg_equal(h, ho)
    r = np.random.default_rng(2).uniform(-1, 1, A.shape[0])
    assert np.array_equal(h.v_cycle(r), ho.vcycle(r))


def _q1_laplacian(nv):
    pts = [0.5 * (-1 / math.sqrt(3) + 1), 0.5 * (1 / math.sqrt(3) + 1)]
    local = np.zeros((4, 4))
    for qy in pts:
        for qx in pts:
            g = np.array([[-(1 - qy), -(1 - qx)], [(1 - qy), -qx], [-qy, (1 - qx)], [qy, qx]])
            local += 0.25 * g @ g.T
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
                    if not (bnd[verts[a]] or bnd[verts[b]]):
                        rows.append(verts[a]); cols.append(verts[b]); vals.append(local[a, b])
    for v in np.nonzero(bnd)[0]:
        rows.append(v); cols.append(v); vals.append(1.0)
    return sp.csr_matrix((vals, (rows, cols)), shape=(nv * nv, nv * nv))


def test_amg_laplacian_parity_and_mesh_independence(cf, orc):  # linsolve_test.cpp:302-308
    rng = np.random.default_rng(16)
    its = []
    for nv in (65, 129):
        A = _q1_laplacian(nv)
        h = cf.build_amg(cf.CsrMatrix.from_scipy(A))
        ho = orc.Amg(orc.Csr.from_scipy(A))
        _assert_amg_equal(h, ho)
        b = rng.uniform(-1, 1, A.shape[0])
        res = cf.gmres(cf.CsrMatrix.from_scipy(A), b, prec=h)
        reso = orc.gmres(b, csr=orc.CsrHandle(orc.Csr.from_scipy(A)), amg=ho)
        assert res["converged"] and res["iterations"] == reso["iterations"]
        assert np.array_equal(res["x"], reso["x"])
        its.append(res["iterations"])
    assert its[1] <= 1.5 * its[0] and its[0] <= 1.5 * its[1]


def test_amg_empty_coarse_nodes_reference_numbering(cf, orc):
    """A phi-like block: most rows constrained (identity rows with a zero near-nullspace entry), so
    most level-0 aggregates carry no coarse dof and are empty nodes of every coarser level.  The
    device build leaves them out (amg.cu, "empty coarse nodes") and must still report the
    reference's node counts, aggregate counts and aggregate ids (linsolve.cpp:146-154: an empty
    node seeds its own aggregate in pass 1), and produce the same operators and V-cycle."""
    rng = np.random.default_rng(23)
    for nv, keep in ((97, 0.25), (129, 0.6)):
        A = _q1_laplacian(nv).tolil()
        n = nv * nv
        con = rng.uniform(0, 1, n) > keep
        # constrained rows and columns become identity (Scatter condensation of a Dirichlet value)
        A = A.tocsr()
        D = sp.diags((~con).astype(float))
        A = (D @ A @ D + sp.diags(con.astype(float))).tocsr()
        A.eliminate_zeros()
        A.sort_indices()
        B = (~con).astype(float).reshape(n, 1)
        nod = np.arange(n, dtype=np.int32)
        opts = cf.AmgOptions(coarse_size=16)
        h = cf.build_amg(cf.CsrMatrix.from_scipy(A), nod, B, opts)
        ho = orc.Amg(orc.Csr.from_scipy(A), nod, B, orc.amg_options(coarse_size=16))
        assert ho.n_levels >= 3
        # the case must contain empty nodes below the last non-empty one on a coarse level
        assert any(ho.level(l)["n_aggregates"] > ho.level(l)["coarse"] for l in range(1, ho.n_levels - 1))
        _assert_amg_equal(h, ho)
        r = rng.uniform(-1, 1, n)
        assert np.array_equal(h.v_cycle(r), ho.vcycle(r))


def test_gmres_identity_spd_and_validation(cf, orc):  # linsolve_test.cpp:194-217
    I = cf.CsrMatrix.from_scipy(sp.identity(20, format="csr"))
    b = np.linspace(1.0, 20.0, 20)
    res = cf.gmres(I, b)
    assert res["converged"] and res["iterations"] == 1 and np.abs(res["x"] - b).max() <= 1e-12
    rng = np.random.default_rng(4)
    for _ in range(5):
        B = rng.uniform(-1, 1, (50, 50))
        A = B @ B.T + 50 * np.eye(50)
        b = rng.uniform(-1, 1, 50)
        res = cf.gmres(cf.CsrMatrix.from_scipy(sp.csr_matrix(A)), b)
        reso = orc.gmres(b, csr=orc.CsrHandle(orc.Csr.from_scipy(sp.csr_matrix(A))))
        assert res["converged"] and np.array_equal(res["x"], reso["x"])
        assert np.array_equal(res["residual_history"], reso["history"])
        ex = np.linalg.solve(A, b)
        assert np.linalg.norm(res["x"] - ex) / np.linalg.norm(ex) <= 1e-7
    with pytest.raises(ValueError, match="rtol"):
        cf.gmres(I, b, opts=cf.GmresOptions(rtol=0.0))


def _small_jacobian(cf, orc, rng, n0=3, r=0, d=2):
    P, O = cf.Problem(d, 1.0, n0, r), orc.Problem(d, 1.0, n0, r)
    x = np.zeros(P.n_total)
    x[:P.n_u] = 1e-2 * rng.uniform(-1, 1, P.n_u)
    x[P.n_u:] = rng.uniform(0, 1, P.n_vertices)
    pt = rng.uniform(0, 1, P.n_vertices)
    cs, ocs = cf.build_constraints(P), O.constraints()
    cs.distribute_homogeneous(x)
    J = cf.assemble_jacobian(P, cs, cf.Material(), cf.Regularization(0.25, 1e-10), x, pt)
    Jo = O.jacobian(ocs, orc.material(), orc.Regularization(0.25, 1e-10), x, pt)
    rhs = rng.uniform(-1, 1, P.n_total)
    cs.distribute_homogeneous(rhs)
    return P, O, cs, ocs, J, Jo, rhs


def test_exact_block_prec_gmres(cf, orc):  # linsolve_test.cpp:219-237
    rng = np.random.default_rng(8)
    for _ in range(10):
        P, O, cs, ocs, J, Jo, rhs = _small_jacobian(cf, orc, rng)
        pre = cf.BlockPreconditioner.build(J, "exact")
        res = cf.gmres(J, rhs, prec=pre)
        reso = orc.gmres(rhs, block=Jo, prec=orc.Prec(Jo, 0))
        assert res["converged"] and res["iterations"] <= 5
        assert res["iterations"] == reso["iterations"]
        assert np.linalg.norm(res["x"] - reso["x"]) <= 1e-12 * np.linalg.norm(reso["x"])


@pytest.mark.parametrize("d,n0,r", [(2, 4, 2), (3, 2, 1)])
def test_block_prec_amg_with_nullspace_bit_exact(cf, orc, d, n0, r):
    rng = np.random.default_rng(12 + d)
    P, O, cs, ocs, J, Jo, rhs = _small_jacobian(cf, orc, rng, n0=n0, r=r, d=d)
    for kind in (1, 2):
        pre = cf.BlockPreconditioner.build(J, kind, prob=P, constraints=cs)
        preo = orc.Prec(Jo, kind, prob=O, cs=ocs)
        assert np.array_equal(pre.apply(rhs), preo.apply(rhs)), kind
    res = cf.gmres(J, rhs, prec=cf.BlockPreconditioner.build(J, 1, prob=P, constraints=cs))
    reso = orc.gmres(rhs, block=Jo, prec=orc.Prec(Jo, 1, prob=O, cs=ocs))
    assert res["iterations"] == reso["iterations"] and np.array_equal(res["x"], reso["x"])


def test_rigid_body_modes(cf, orc):  # linsolve_test.cpp:310-334
    for d in (2, 3):
        P, O = cf.Problem(d, 1.0, 3, 0), orc.Problem(d, 1.0, 3, 0)
        act = {P.n_u + 1: 0.5}
        B = cf.rigid_body_modes(P, cf.build_constraints(P, True, act))
        Bo = O.rigid_body_modes(O.constraints(True, list(act), list(act.values())))
        assert np.array_equal(B, Bo)


def _sneddon_pair(cf, orc, d=2, K=5.0, n0=10, r=1, fixed=False):
    P, O = cf.Problem(d, K, n0, r), orc.Problem(d, K, n0, r)
    kw = dict(eps_mode=1, eps_fixed=2 * P.h, kappa_factor=1e-12 / P.h) if fixed else {}
    mat, omat = cf.Material(**kw), orc.material(**kw)
    reg = cf.resolve_regularization(P, mat, cf.slit_band_edge(P, mat))
    oreg = O.resolve_regularization(omat, O.slit_band_edge(omat))
    assert (reg.eps, reg.kappa) == (oreg.eps, oreg.kappa)
    phi, _ = cf.initial_crack(P, mat)
    ophi, _ = O.initial_crack(omat)
    assert np.array_equal(phi, ophi)
    return P, O, mat, omat, reg, oreg, phi


def _run_pair(cf, orc, P, O, mat, omat, reg, oreg, phi, steps=1, **optkw):
    st = cf.make_initial_state(P, mat)
    reps = cf.solve_loading_sequence(st, mat, P, reg, cf.SolverOptions(**dict(dict(operator_kind=0), **optkw)), steps)
    sol = np.zeros(O.n_total)
    sol[O.n_u:] = phi
    po, pp = phi.copy(), phi.copy()
    oreps = []
    okw = dict(optkw)
    if "gmres" in okw:
        g = okw["gmres"]
        okw["gmres"] = orc.gmres_options(rtol=g.rtol, max_iter=g.max_iter, restart=g.restart)
    for n in range(1, steps + 1):
        oreps.append(O.newton_step(omat, oreg, orc.solver_options(**okw), sol, po, pp, n))
    return reps, st.get()["solution"], oreps, sol


def _same_transcript(rep, orep):
    its = np.array([[r["residual_norm"], r["active_size"], r["set_changes"], r["gmres_iterations"]]
                    for r in rep["iterations"]])
    assert its.shape == orep["iterations"].shape, (its, orep["iterations"])
    assert np.array_equal(its, orep["iterations"]), (its, orep["iterations"])
    assert rep["converged"] == orep["converged"]
    assert rep["feasibility_violation"] == orep["feasibility"]


@pytest.mark.parametrize("r", [1, 2])
def test_newton_step_bit_exact_small(cf, orc, r):  # solver_test.cpp:112-150, 178-195
    P, O, mat, omat, reg, oreg, phi = _sneddon_pair(cf, orc, r=r)
    reps, x, oreps, xo = _run_pair(cf, orc, P, O, mat, omat, reg, oreg, phi)
    _same_transcript(reps[0], oreps[0])
    assert np.array_equal(x, xo)
    assert reps[0]["converged"] and reps[0]["feasibility_violation"] <= 1e-10
    assert reps[0]["iterations"][-1]["set_changes"] == 0


def test_newton_determinism_and_exact_prec(cf, orc):  # solver_test.cpp:178-210
    P, O, mat, omat, reg, oreg, phi = _sneddon_pair(cf, orc, r=1)
    runs = [_run_pair(cf, orc, P, O, mat, omat, reg, oreg, phi)[:2] for _ in range(2)]
    assert np.array_equal(runs[0][1], runs[1][1])
    xe = _run_pair(cf, orc, P, O, mat, omat, reg, oreg, phi, prec_kind=0)[1]
    assert np.abs(runs[0][1] - xe).max() <= 1e-6 * np.abs(xe).max()


def test_loading_sequence_three_steps(cf, orc):  # solver.cpp:190-204, config 2 semantics (step 3 extrapolates)
    P, O, mat, omat, reg, oreg, phi = _sneddon_pair(cf, orc, r=1, fixed=True)
    reps, x, oreps, xo = _run_pair(cf, orc, P, O, mat, omat, reg, oreg, phi, steps=3,
                                   gmres=cf.GmresOptions(rtol=1e-10, restart=50))
    assert len(reps) == 3
    for a, b in zip(reps, oreps):
        _same_transcript(a, b)
    assert np.array_equal(x, xo)
    with pytest.raises(ValueError, match="n_steps"):
        cf.solve_loading_sequence(cf.make_initial_state(P, mat), mat, P, reg, cf.SolverOptions(), 0)


def test_config0_newton_parity(cf, orc):
    """BASELINE config 0 (2d 256^2, eps = 2h, kappa = 1e-12): full Newton step vs the oracle,
    then TCV and COD on the 64 stations x = -1.575 + 0.05 i computed on the device."""
    P, O, mat, omat, reg, oreg, phi = _sneddon_pair(cf, orc, d=2, K=10.0, n0=8, r=5, fixed=True)
    assert P.n_total == 198147
    reps, x, oreps, xo = _run_pair(cf, orc, P, O, mat, omat, reg, oreg, phi)
    _same_transcript(reps[0], oreps[0])
    assert np.array_equal(x, xo)
    st = -1.575 + 0.05 * np.arange(64)
    cod, codo = cf.compute_cod(P, x, st), O.cod(xo, st)
    assert np.allclose(cod, codo, rtol=1e-12, atol=1e-18)
    tcv, tcvo = cf.compute_tcv(P, x), O.tcv(xo)
    assert abs(tcv - tcvo) <= 1e-12 * abs(tcvo)
    exact = 2 * math.pi * 1e-3 * (1 - 0.2 ** 2)  # PAPER.md:321, 6.0319e-3
    assert 0.8 * exact < abs(tcv) < 1.2 * exact
    assert 1.6e-3 < cod[np.argmin(np.abs(st))] < 2.1e-3  # COD(0) ~ 1.92e-3


@pytest.mark.parametrize("d", [2, 3])
def test_functionals_random_fields(cf, orc, d):  # postproc_test.cpp:35-105
    rng = np.random.default_rng(31 + d)
    P, O = cf.Problem(d, 2.0, 4, 1), orc.Problem(d, 2.0, 4, 1)
    x = rng.uniform(-1, 1, P.n_total)
    assert abs(cf.compute_tcv(P, x) - O.tcv(x)) <= 1e-12 * max(1.0, abs(O.tcv(x)))
    st = np.array([-2.0, -1.3, -0.25, 0.0, 0.6, 1.9, 2.0])
    assert np.allclose(cf.compute_cod(P, x, st), O.cod(x, st), rtol=1e-12, atol=1e-14)
    flat = x.copy()
    flat[P.n_u:] = 0.7  # constant phi: zero TCV and zero profile
    assert abs(cf.compute_tcv(P, flat)) <= 1e-13 and np.abs(cf.compute_cod(P, flat, st)).max() <= 1e-13
    with pytest.raises(ValueError, match="strictly increasing"):
        cf.compute_cod(P, x, [0.0, 0.0])
    with pytest.raises(ValueError, match="outside"):
        cf.compute_cod(P, x, [-3.0, 0.0])


def test_3d_penny_newton_bit_exact(cf, orc):
    """3d penny crack (config 3 physics) on 16^3: full Newton step vs the oracle."""
    P, O, mat, omat, reg, oreg, phi = _sneddon_pair(cf, orc, d=3, K=10.0, n0=8, r=1, fixed=True)
    reps, x, oreps, xo = _run_pair(cf, orc, P, O, mat, omat, reg, oreg, phi)
    _same_transcript(reps[0], oreps[0])
    assert np.array_equal(x, xo)
    assert reps[0]["converged"] and reps[0]["feasibility_violation"] <= 1e-10


def test_amg_large_diagonal_coarsest(cf):
    """A diagonal matrix beyond the dense-LU size (the all-active phi block of a slab far from the
    crack): aggregation stops at once and the coarsest 'LU' is the diagonal itself."""
    import scipy.sparse as sp
    n = 20000
    d = np.random.default_rng(2).uniform(1.0, 3.0, n)
    h = cf.build_amg(cf.CsrMatrix.from_scipy(sp.diags(d).tocsr()))
    assert h.n_levels() == 1
    r = np.random.default_rng(3).standard_normal(n)
    assert np.array_equal(h.v_cycle(r), r / d)


def test_u_amg_3d_bit_exact(cf, orc):
    """u-block hierarchy of a 3d Jacobian (16^3 mesh, rigid-body near-nullspace): the products run
    through the row-group SpGEMM (rows of one node / one aggregate share their pattern) and must
    reproduce the oracle's level operators bit for bit."""
    P, O = cf.Problem(3, 10.0, 8, 1), orc.Problem(3, 10.0, 8, 1)
    rng = np.random.default_rng(21)
    x = np.zeros(P.n_total)
    x[:P.n_u] = 1e-3 * rng.uniform(-1, 1, P.n_u)
    x[P.n_u:] = rng.uniform(0.2, 1.0, P.n_phi)
    pt = rng.uniform(0.2, 1.0, P.n_phi)
    mat = cf.Material()
    reg = cf.resolve_regularization(P, mat, cf.slit_band_edge(P, mat))
    cs = cf.build_constraints(P)
    J = cf.assemble_jacobian(P, cs, mat, reg, x, pt)
    u = J.M_uu
    node = np.repeat(np.arange(P.n_vertices, dtype=np.int32), 3)
    B = cf.rigid_body_modes(P, cs)
    h = cf.build_amg(cf.CsrMatrix(u.rows, u.cols, u.ptr, u.col, u.val), node, B)
    ho = orc.Amg(orc.Csr(u.rows, u.cols, u.ptr, u.col, u.val), node, B)
    _assert_amg_equal(h, ho)
    r = rng.uniform(-1, 1, P.n_u)
    assert np.array_equal(h.v_cycle(r), ho.vcycle(r))


def test_amg_grouped_spgemm_everywhere(cf):
    """CF_SPGEMM_GROUP_ALL=1 sends every product the row-group kernel can take through it (tiny
    matrices, single-row groups, runs chunked at 6 rows); the AMG parity tests must still pass."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CF_SPGEMM_GROUP_ALL="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", os.path.join(root, "tests", "test_gpu_solver.py"),
                        "-k", "amg and not everywhere or block_prec or penny"], env=env, capture_output=True, text=True,
                       timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("env", [
    {"CF_SPGEMM_FORCE_PATHS": "1"},
    {"CF_SPGEMM_NO_FLAGS": "1", "CF_SPGEMM_NO_CTA_PF": "1", "CF_SPGEMM_NO_SHORT_GROUP": "1",
     "CF_VCYCLE_UNFUSED": "1"},
], ids=["forced-coarse-paths", "legacy-paths"])
def test_amg_paths_forced_and_disabled(cf, env):
    """The structure-aware SpGEMM paths (byte-flag symbolic, CTA-per-row prefetching numeric) forced
    onto every product they can take, and, separately, every fast path switched off (generic hash
    SpGEMM, unfused V-cycle): the oracle AMG / preconditioner / Newton parity tests must pass
    bit for bit either way."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", os.path.join(root, "tests", "test_gpu_solver.py"),
                        "-k", "amg and not everywhere and not forced or block_prec or penny"],
                       env=dict(os.environ, **env), capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def _np_vcycle_cheb(levels, Ac, b, deg, sweeps=1):
    """numpy restatement of the opt-in Chebyshev V-cycle (amg.cu vcycle_range, smoother 1): on each
    level `sweeps` Chebyshev passes of degree `deg` on D^-1 A over [hi / 10, hi], hi the Gershgorin
    bound max_i |d_i| sum_j |a_ij|, restrict the residual, dense solve on the coarsest level,
    prolongate and post-smooth."""
    def cheb(A, dinv, bl, x, zero):
        hi = (abs(A) @ np.ones(A.shape[1]) * abs(dinv)).max()
        lo = hi / 10.0
        theta, delta = 0.5 * (hi + lo), 0.5 * (hi - lo)
        sigma = theta / delta
        for s in range(sweeps):
            r = bl if (zero and s == 0) else bl - A @ x
            d = dinv * r / theta
            x = d.copy() if (zero and s == 0) else x + d
            rho = 1.0 / sigma
            for _ in range(1, deg):
                rho_new = 1.0 / (2.0 * sigma - rho)
                d = rho_new * rho * d + 2.0 * rho_new / delta * (dinv * (bl - A @ x))
                x = x + d
                rho = rho_new
        return x

    def rec(l, bl):
        if l == len(levels):
            return np.linalg.solve(Ac, bl)
        A, P = levels[l]
        dinv = 1.0 / A.diagonal()
        x = cheb(A, dinv, bl, None, True)
        xc = rec(l + 1, P.T @ (bl - A @ x))
        return cheb(A, dinv, bl, x + P @ xc, False)
    return rec(0, b)


@pytest.mark.parametrize("deg,sweeps", [(1, 1), (2, 1), (3, 2)])
def test_amg_chebyshev_smoother_matches_numpy(cf, deg, sweeps):
    """The opt-in Chebyshev smoother (AmgOptions.smoother = 1; the reference smooths with damped
    Jacobi only, so this is outside the bitwise contract) against its numpy restatement on the
    16^3 u-block hierarchy, to 1e-10 relative."""
    P = cf.Problem(3, 10.0, 8, 1)
    rng = np.random.default_rng(31)
    x = np.zeros(P.n_total)
    x[:P.n_u] = 1e-3 * rng.uniform(-1, 1, P.n_u)
    x[P.n_u:] = rng.uniform(0.2, 1.0, P.n_phi)
    mat = cf.Material()
    reg = cf.resolve_regularization(P, mat, cf.slit_band_edge(P, mat))
    cs = cf.build_constraints(P)
    u = cf.assemble_jacobian(P, cs, mat, reg, x, x[P.n_u:].copy()).M_uu
    node = np.repeat(np.arange(P.n_vertices, dtype=np.int32), 3)
    opts = cf.AmgOptions(smoother=1, chebyshev_degree=deg, smoothing_sweeps=sweeps)
    h = cf.build_amg(cf.CsrMatrix(u.rows, u.cols, u.ptr, u.col, u.val), node, cf.rigid_body_modes(P, cs), opts)
    levels = []
    for lev in range(h.n_levels() - 1):
        A, Pm = h.level_matrix(lev, 0), h.level_matrix(lev, 1)
        levels.append((sp.csr_matrix((A.val, A.col, A.ptr), shape=(A.rows, A.cols)),
                       sp.csr_matrix((Pm.val, Pm.col, Pm.ptr), shape=(Pm.rows, Pm.cols))))
    assert len(levels) >= 2
    Ac = levels[-1][0]
    Pl = levels[-1][1]
    Ac = (Pl.T @ Ac @ Pl).toarray()
    r = rng.uniform(-1, 1, P.n_u)
    got = h.v_cycle(r)
    ref = _np_vcycle_cheb(levels, Ac, r, deg, sweeps)
    assert np.linalg.norm(got - ref) <= 1e-10 * np.linalg.norm(ref)
    # a linear operator (fixed polynomial), and a better smoother than none at all
    s = rng.uniform(-1, 1, P.n_u)
    lhs, rhs = h.v_cycle(0.6 * r + 1.3 * s), 0.6 * got + 1.3 * h.v_cycle(s)
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(rhs)
    A0 = levels[0][0]
    assert np.linalg.norm(r - A0 @ got) < np.linalg.norm(r)


@pytest.mark.parametrize("opkind", [0, 1])
def test_newton_step_chebyshev_smoother(cf, orc, opkind):
    """The whole 3d penny Newton step with Chebyshev-smoothed AMG (assembled and matrix-free finest
    level) converges to the same solution as the reference's Jacobi-smoothed run, to the Newton
    tolerance, with the same final active set."""
    P, O, mat, omat, reg, oreg, phi = _sneddon_pair(cf, orc, d=3, K=10.0, n0=8, r=1, fixed=True)
    out = {}
    for sm in (0, 1):
        st = cf.make_initial_state(P, mat)
        o = cf.SolverOptions(operator_kind=opkind, amg=cf.AmgOptions(smoother=sm, chebyshev_degree=2))
        rep = cf.newton_active_set_step(st, mat, P, reg, o)
        assert rep["converged"] and rep["feasibility_violation"] <= 1e-10
        out[sm] = (rep, st.get()["solution"])
    (rj, xj), (rc, xc) = out[0], out[1]
    assert np.abs(xc - xj).max() <= 1e-6 * np.abs(xj).max()
    assert rc["iterations"][-1]["active_size"] == rj["iterations"][-1]["active_size"]
    assert max(q["gmres_iterations"] for q in rc["iterations"]) <= 4 * max(q["gmres_iterations"]
                                                                        for q in rj["iterations"])

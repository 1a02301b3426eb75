"""General (adaptive) meshes on the B200 against the CPU oracle
(oracle/oracle_mesh.inc): DofMap, faces, hanging-node constraint lines, distribute, residual and
Jacobian (condensation through masters + setFromTriplets sums), rigid modes, a whole Newton step,
TCV/COD, the jump estimator, marking, transfer and the adaptive cycle — bitwise wherever the
reference's arithmetic is reproduced operation by operation (everything but the TCV/COD sums,
which are tree reductions on the device and are checked to 1e-12)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cm():
    import paper_1806_09924_b200 as cf
    import paper_1806_09924_b200.mesh as m
    cf._lib.load()
    return m


def twin(orc, cm, d, K, n0, rounds, seed, frac):
    """The same refinement sequence on the device mesh and on the oracle mesh."""
    M = cm.create_mesh(d, K, n0)
    O = orc.Mesh(d, K, n0)
    rng = np.random.default_rng(seed)
    for _ in range(rounds):
        act = M.active_cells()
        assert np.array_equal(act, O.active())
        marked = [int(c) for c in act if rng.integers(frac) == 0] or [int(act[0])]
        cm.refine(M, marked)
        O.refine(marked)
    return M, O


def rand_state(M, rng, phi_lo=0.0):
    x = np.zeros(M.n_total)
    x[:M.n_u] = 1e-2 * rng.uniform(-1, 1, M.n_u)
    x[M.n_u:] = rng.uniform(phi_lo, 1, M.n_vertices)
    return x


# (d, K, n0, rounds, seed, frac): random refinement sequences (each active cell marked with
# probability 1/frac per round); the 3d seed-0 case has chained hanging lines (a vertex hanging on a
# hanging vertex across a 2-level edge jump: closed weights 1/8, 3/8, 3/4, five masters)
CASES = [(2, 1.0, 2, 3, 11, 3), (2, 5.0, 4, 4, 12, 3), (3, 1.0, 2, 2, 13, 3), (3, 1.0, 2, 3, 0, 4)]


@pytest.mark.parametrize("d,K,n0,rounds,seed,frac", CASES)
def test_mesh_topology(orc, cm, d, K, n0, rounds, seed, frac):
    M, O = twin(orc, cm, d, K, n0, rounds, seed, frac)
    assert (M.n_cells, M.n_active, M.max_level, M.n_vertices) == (O.n_cells, O.n_active, O.max_level, O.V)
    c1, c2 = M.cells(), O.cells()
    for k in ("level", "parent", "active", "anchor"):
        assert np.array_equal(c1[k], c2[k]), k
    assert np.array_equal(M.vertex_keys(), O.vertex_keys())
    assert np.array_equal(M.cell_vertices(), O.cell_vertices())
    assert np.array_equal(M.faces(), O.faces())
    rng = np.random.default_rng(seed)
    for _ in range(20):
        x = rng.uniform(-K, K, 3)
        assert M.find_active_cell(x[:d]) == O.find_cell(x[:d])


@pytest.mark.parametrize("d,K,n0,rounds,seed,frac", CASES)
@pytest.mark.parametrize("clamp", [True, False])
def test_constraint_lines_and_distribute(orc, cm, d, K, n0, rounds, seed, frac, clamp):
    M, O = twin(orc, cm, d, K, n0, rounds, seed, frac)
    rng = np.random.default_rng(seed + 1)
    act = sorted(set(int(v) for v in rng.integers(0, M.n_vertices, M.n_vertices // 6)))
    adofs = [M.n_u + v for v in act]
    avals = [float(rng.uniform()) for _ in act]
    dc = cm.build_constraints(M, clamp, dict(zip(adofs, avals)))
    oc = O.constraints(clamp, adofs, avals)
    # the device exports the lines with entries; the oracle's include the entry-free ones
    dd, dp, dm, dw, di = dc.lines()
    od, op, om, ow, oi = oc.lines()
    keep = op[1:] > op[:-1]
    keep |= np.isin(od, dd)  # lines that lost every master to the active set stay lines on the device
    sel = np.nonzero(keep)[0]
    assert np.array_equal(dd, od[sel])
    assert np.array_equal(di, oi[sel])
    for i, j in enumerate(sel):
        assert np.array_equal(dm[dp[i]:dp[i + 1]], om[op[j]:op[j + 1]])
        assert np.array_equal(dw[dp[i]:dp[i + 1]], ow[op[j]:op[j + 1]])
    v = rng.uniform(-1, 1, M.n_total)
    assert np.array_equal(dc.distribute(v.copy()), oc.distribute(v))
    assert np.array_equal(dc.distribute_homogeneous(v.copy()), oc.distribute(v, homogeneous=True))


@pytest.mark.parametrize("d,K,n0,rounds,seed,frac", CASES)
def test_assembly_bitwise(orc, cm, d, K, n0, rounds, seed, frac):
    import paper_1806_09924_b200 as cf
    M, O = twin(orc, cm, d, K, n0, rounds, seed, frac)
    rng = np.random.default_rng(seed + 2)
    x = rand_state(M, rng)
    pt = rng.uniform(0, 1, M.n_vertices)
    act = sorted(set(int(v) for v in rng.integers(0, M.n_vertices, M.n_vertices // 5)))
    adofs = [M.n_u + v for v in act]
    avals = [float(x[a]) for a in adofs]
    for clamp, (ad, av) in ((True, ([], [])), (True, (adofs, avals)), (False, (adofs, avals))):
        dc = cm.build_constraints(M, clamp, dict(zip(ad, av)))
        oc = O.constraints(clamp, ad, av)
        mat, reg = cf.Material(pressure=1e-3), cf.Regularization(0.25, 1e-10)
        omat, oreg = orc.material(pressure=1e-3), orc.Regularization(0.25, 1e-10)
        R = cm.assemble_residual(M, dc, mat, reg, x, pt)
        Ro = O.residual(oc, omat, oreg, x, pt)
        assert np.array_equal(R, Ro), np.abs(R - Ro).max()
        J = cm.assemble_jacobian(M, dc, mat, reg, x, pt)
        Jo = O.jacobian(oc, omat, oreg, x, pt)
        for w in range(3):
            a, b = J.csr(w), Jo.csr(w)
            assert np.array_equal(a.ptr, b.ptr) and np.array_equal(a.col, b.col), f"pattern {w}"
            assert np.array_equal(a.val, b.val), f"values {w}: {np.abs(a.val - b.val).max()}"
        y, yo = J.apply(x), Jo.apply(x)
        assert np.array_equal(y, yo)
        assert np.array_equal(cm.rigid_body_modes(M, dc), O.rigid_body_modes(oc))


def sneddon_twin(orc, cm, d, K, n0, r, extra):
    """A Sneddon mesh refined uniformly r times, then `extra` rounds of refinement around the slit."""
    M = cm.create_mesh(d, K, n0)
    O = orc.Mesh(d, K, n0)
    cm.uniform_refine(M, r)
    O.uniform_refine(r)
    for _ in range(extra):
        xs = M.vertex_physical()
        cv = M.cell_vertices()
        act = M.active_cells()
        near = np.linalg.norm(xs[cv].mean(axis=1)[:, :d - 1], axis=1) < 1.6
        flat = np.abs(xs[cv].mean(axis=1)[:, d - 1]) < 1.0
        marked = [int(c) for c in act[near & flat]]
        cm.refine(M, marked)
        O.refine(marked)
    return M, O


@pytest.mark.parametrize("d,K,n0,r,extra", [(2, 5.0, 10, 0, 2), (3, 4.0, 4, 1, 1), (2, 10.0, 8, 3, 3)])
def test_newton_step_bitwise(orc, cm, d, K, n0, r, extra):
    import paper_1806_09924_b200 as cf
    M, O = sneddon_twin(orc, cm, d, K, n0, r, extra)
    mat, omat = cf.Material(), orc.material()
    be = cm.slit_band_edge(M, mat)
    assert be == O.slit_band_edge(omat)
    reg = cm.resolve_regularization(M, mat, be)
    oreg = O.resolve_regularization(omat, be)
    assert (reg.eps, reg.kappa) == (oreg.eps, oreg.kappa)
    phi, _ = cm.initial_crack(M, mat)
    ophi, _ = O.initial_crack(omat)
    assert np.array_equal(phi, ophi)
    st = cm.make_initial_state(M, mat)
    rep = cm.newton_active_set_step(st, mat, M, reg, cf.SolverOptions())
    sol = np.zeros(O.n_total)
    sol[O.n_u:] = ophi
    orep = O.newton_step(omat, oreg, orc.solver_options(), sol, ophi.copy(), ophi.copy(), 0, shift=False)
    its = np.array([[q["residual_norm"], q["active_size"], q["set_changes"], q["gmres_iterations"]]
                    for q in rep["iterations"]])
    assert rep["converged"] and orep["converged"]
    assert np.array_equal(its, orep["iterations"]), (its, orep["iterations"])
    got = st.get()["solution"]
    assert np.array_equal(got, sol)
    assert cm.compute_tcv(M, got) == pytest.approx(O.tcv(sol), rel=1e-12, abs=1e-300)
    stations = np.linspace(-0.9, 0.9, 7)
    assert np.allclose(cm.compute_cod(M, got, stations), O.cod(sol, stations), rtol=1e-12, atol=1e-18)


@pytest.mark.parametrize("d,K,n0,rounds,seed,frac", CASES)
def test_estimator_marking_transfer_bitwise(orc, cm, d, K, n0, rounds, seed, frac):
    M, O = twin(orc, cm, d, K, n0, rounds, seed, frac)
    rng = np.random.default_rng(seed + 3)
    x = rand_state(M, rng)
    x = O.constraints(True).distribute(x)
    eta = cm.jump_estimator(M, x)
    assert np.array_equal(eta, O.estimator(x))
    for theta in (0.3, 0.7):
        for est in (True, False):
            kw = dict(phi_threshold=0.5, h_target=0.0, theta=theta, max_level=M.max_level + 1, estimator=est)
            import paper_1806_09924_b200 as cf
            pol = cf._lib.RefinementPolicy(phi_threshold=0.5, h_target=0.0, theta=theta, max_level=M.max_level + 1,
                                           estimator=1 if est else 0)
            assert np.array_equal(cm.mark_cells(M, x, eta, pol), O.mark(x, eta, **kw))
    marked = O.mark(x, eta, theta=0.4)
    M2, O2 = M.copy(), O.copy()
    cm.refine(M2, marked)
    O2.refine(marked)
    assert np.array_equal(cm.transfer(M, x, M2), O.transfer_to(x, O2))


def test_adaptive_cycle_matches_oracle(orc, cm):
    import paper_1806_09924_b200 as cf
    M = cm.create_mesh(2, 5.0, 10)
    O = orc.Mesh(2, 5.0, 10)
    mat = cf.Material()
    st = cm.make_initial_state(M, mat)
    opts = cf._lib.AdaptiveOptions(cycles=2, n_steps=2)
    recs = cm.adaptive_cycle(M, st, mat, opts)
    orec, osol = O.adaptive_cycle(orc.material(), orc.solver_options(), cycles=2, n_steps=2)
    assert len(recs) == len(orec) == 3
    for r, o in zip(recs, orec):
        assert (r["level"], r["dofs"], r["eps"], r["h_min"], r["newton_iters"], r["converged"]) == \
            (o[0], o[1], o[2], o[3], o[5], bool(o[7]))
        assert r["gmres_mean"] == o[6]
        assert r["tcv"] == pytest.approx(o[4], rel=1e-12)
    assert M.n_total == O.n_total
    assert np.array_equal(st.get()["solution"], osol)


def test_chained_lines_present(orc):
    """The seed-0 3d case really has chained hanging lines (so the closure is exercised)."""
    O = orc.Mesh(3, 1.0, 2)
    rng = np.random.default_rng(0)
    for _ in range(3):
        act = O.active()
        O.refine([int(c) for c in act if rng.integers(4) == 0] or [int(act[0])])
    dd, p, m, w, inh = O.constraints(False).lines()
    assert {0.125, 0.375}.issubset(set(w.tolist())) and max(p[1:] - p[:-1]) > 4

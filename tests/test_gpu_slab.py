"""Slab decomposition on one GPU: every rank's rows, assembled from its planes plus one
ghost plane, must be bitwise the rows of the undivided system; the block apply of a slab reads
the ext layout [u_ext | phi_ext]; a size-1 communicator is the single-GPU step exactly.

The multi-rank NCCL transport needs one GPU per rank; the decomposition it moves data for is
checked here rank by rank (the host-side protocol of the halo exchange and rank-ordered sums is
checked over gloo in tests/test_slab_protocol.py)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cf():
    import paper_1806_09924_b200 as cf
    return cf


def _rows(A, lo, hi):
    p = A.ptr[lo:hi + 1]
    return p - p[0], A.col[p[0]:p[-1]], A.val[p[0]:p[-1]]


def _setup(cf, d, n0, r, frac_active, seed):
    P = cf.Problem(d, 1.0, n0, r)
    rng = np.random.default_rng(seed)
    x = np.zeros(P.n_total)
    x[:P.n_u] = 1e-2 * rng.uniform(-1, 1, P.n_u)
    x[P.n_u:] = rng.uniform(0, 1, P.n_vertices)
    pt = rng.uniform(0, 1, P.n_vertices)
    nact = int(frac_active * P.n_vertices)
    verts = rng.choice(P.n_vertices, nact, replace=False)
    cs = cf.build_constraints(P, True, {int(P.n_u + v): float(rng.uniform(0, 1)) for v in verts})
    mat = cf.Material(pressure=2e-3)
    reg = cf.Regularization(0.3, 1e-6)
    return P, x, pt, cs, mat, reg, rng


@pytest.mark.parametrize("d,n0,r,size", [(2, 4, 2, 2), (2, 4, 2, 5), (3, 3, 1, 2), (3, 3, 1, 3), (3, 2, 2, 4)])
def test_slab_rows_bit_exact(cf, d, n0, r, size):
    P, x, pt, cs, mat, reg, rng = _setup(cf, d, n0, r, 0.15, 7 * d + size)
    R = cf.assemble_residual(P, cs, mat, reg, x, pt)
    J = cf.assemble_jacobian(P, cs, mat, reg, x, pt)
    G = [J.csr(w) for w in range(3)]
    y_glob = J.apply(z := rng.standard_normal(P.n_total))
    covered = 0
    for rank in range(size):
        s = cf.slab_info(P, rank, size)
        planes = (s["v_lo"] // s["plane"], s["v_hi"] // s["plane"])
        nv, lo, hi, elo, ehi = s["v_hi"] - s["v_lo"], s["v_lo"], s["v_hi"], s["ve_lo"], s["ve_hi"]
        covered += nv
        Rs = cf.assemble_residual(P, cs, mat, reg, x, pt, planes=planes)
        assert np.array_equal(Rs, np.concatenate([R[d * lo:d * hi], R[P.n_u + lo:P.n_u + hi]]))
        Js = cf.assemble_jacobian(P, cs, mat, reg, x, pt, planes=planes)
        assert Js.n_u() == d * nv and Js.n_phi() == nv and Js.n_in() == (d + 1) * (ehi - elo)
        for w, (rlo, rhi, shift) in enumerate(((d * lo, d * hi, d * elo), (lo, hi, d * elo), (lo, hi, elo))):
            A = Js.csr(w)
            gp, gc, gv = _rows(G[w], rlo, rhi)
            assert np.array_equal(A.ptr, gp), f"rank {rank} block {w}: row pointers differ"
            assert np.array_equal(A.col + shift, gc), f"rank {rank} block {w}: columns differ"
            assert np.array_equal(A.val, gv), f"rank {rank} block {w}: values differ"
        xe = np.concatenate([z[d * elo:d * ehi], z[P.n_u + elo:P.n_u + ehi]])
        ys = Js.apply(xe)
        ref = np.concatenate([y_glob[d * lo:d * hi], y_glob[P.n_u + lo:P.n_u + hi]])
        assert np.linalg.norm(ys - ref) <= 1e-13 * np.linalg.norm(ref)
    assert covered == P.n_vertices


def test_slab_info_partition(cf):
    P = cf.Problem(3, 1.0, 2, 2)  # 9 planes
    for size in (1, 2, 4, 9):
        prev_hi = 0
        for rank in range(size):
            s = cf.slab_info(P, rank, size)
            assert s["v_lo"] == prev_hi and s["v_hi"] > s["v_lo"]
            assert s["ve_lo"] == max(s["v_lo"] - s["plane"], 0)
            assert s["ve_hi"] == min(s["v_hi"] + s["plane"], P.n_vertices)
            prev_hi = s["v_hi"]
        assert prev_hi == P.n_vertices
    with pytest.raises(NotImplementedError):
        cf.slab_info(P, 0, 10)  # fewer planes than ranks


def test_single_rank_communicator_is_the_single_gpu_step(cf):
    P = cf.Problem(2, 10.0, 8, 2)
    mat = cf.Material(eps_mode=1, eps_fixed=2 * P.h, kappa_factor=1e-12 / P.h)
    reg = cf.resolve_regularization(P, mat, cf.slit_band_edge(P, mat))
    opts = cf.SolverOptions(operator_kind=0)
    a, b = cf.make_initial_state(P, mat), cf.make_initial_state(P, mat)
    comm = cf.Communicator(0, 1)
    ra = cf.newton_active_set_step(a, mat, P, reg, opts)
    rb = cf.newton_active_set_step(b, mat, P, reg, opts, comm=comm)
    assert ra["iterations"] == rb["iterations"] and ra["converged"] and rb["converged"]
    sa, sb = a.get(), b.get()
    assert np.array_equal(sa["solution"], sb["solution"])

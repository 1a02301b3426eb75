"""Sizes and options where the reference has no limit (round-1 hard limits removed), each
compared bit for bit with the oracle:

* GMRES restart beyond 255 (the basis combination stages its coefficients 256 at a time);
* cycle-detection windows beyond 64 entries (multi-word toggle history per dof);
* coarsest dense LU beyond one CTA (the multi-CTA factorisation; forced onto a 2000-row system
  with CF_LU_MULTICTA_MIN so the oracle's unblocked LU finishes in seconds);
* SpGEMM output rows beyond the 16384-slot hash tier (the sort-based long-row tier).
"""
import os
import subprocess
import sys

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cf():
    import paper_1806_09924_b200 as cf
    return cf


def test_gmres_restart_beyond_255(cf, orc):
    n = 400
    A = sp.diags([-np.ones(n - 1), 2.0 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1], format="csr")
    b = np.random.default_rng(1).uniform(-1, 1, n)
    opts = cf.GmresOptions(rtol=1e-10, restart=300, max_iter=1000)
    res = cf.gmres(cf.CsrMatrix.from_scipy(A), b, opts=opts)
    reso = orc.gmres(b, csr=orc.CsrHandle(orc.Csr.from_scipy(A)),
                     opts=orc.gmres_options(rtol=1e-10, restart=300, max_iter=1000))
    assert res["iterations"] > 255 and res["iterations"] == reso["iterations"]
    assert np.array_equal(res["x"], reso["x"])
    assert np.array_equal(res["residual_history"], reso["history"])
    with pytest.raises(ValueError, match="restart"):
        cf.gmres(cf.CsrMatrix.from_scipy(A), b, opts=cf.GmresOptions(restart=0))


@pytest.mark.parametrize("window,toggles", [(100, 1), (130, 2)])
def test_cycle_window_beyond_64(cf, orc, window, toggles):
    P, O = cf.Problem(2, 5.0, 10, 1), orc.Problem(2, 5.0, 10, 1)
    mat, omat = cf.Material(), orc.material()
    reg = cf.resolve_regularization(P, mat, cf.slit_band_edge(P, mat))
    oreg = O.resolve_regularization(omat, O.slit_band_edge(omat))
    phi, _ = cf.initial_crack(P, mat)
    st = cf.make_initial_state(P, mat)
    rep = cf.newton_active_set_step(st, mat, P, reg, cf.SolverOptions(cycle_window=window, cycle_toggles=toggles, operator_kind=0))
    sol = np.zeros(O.n_total)
    sol[O.n_u:] = phi
    orep = O.newton_step(omat, oreg, orc.solver_options(cycle_window=window, cycle_toggles=toggles), sol,
                         phi.copy(), phi.copy(), 0, shift=False)
    its = np.array([[r["residual_norm"], r["active_size"], r["set_changes"], r["gmres_iterations"]]
                    for r in rep["iterations"]])
    assert np.array_equal(its, orep["iterations"])
    assert np.array_equal(st.get()["solution"], sol)


def test_dense_lu_multi_cta(orc):
    r = subprocess.run([sys.executable, "-c", _LU_SCRIPT], env=dict(os.environ, CF_LU_MULTICTA_MIN="512"),
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


_LU_SCRIPT = r'''
import sys; sys.path.insert(0, ".")
import numpy as np, scipy.sparse as sp
import paper_1806_09924_b200 as cf
from oracle import orc
rng = np.random.default_rng(3)
n = 2000
rows = np.repeat(np.arange(n), 6); cols = rng.integers(0, n, 6 * n)
S = sp.csr_matrix((-rng.uniform(0.5, 1.0, 6 * n), (rows, cols)), shape=(n, n)); S = S + S.T; S.setdiag(0.0)
S.eliminate_zeros(); A = (S + sp.diags(np.asarray(abs(S).sum(axis=1)).ravel() + 1.0)).tocsr()
# a non-symmetric perturbation so that pivoting swaps rows
A = (A + sp.diags(rng.uniform(-0.5, 0.5, n - 1), 1)).tocsr(); A.sort_indices()
opts = cf.AmgOptions(max_levels=0)
h = cf.build_amg(cf.CsrMatrix.from_scipy(A), opts=opts)
ho = orc.Amg(orc.Csr.from_scipy(A), opts=orc.amg_options(max_levels=0))
assert h.n_levels() == 1 and h.coarse_dim() == n == ho.coarse_dim
b = rng.uniform(-1, 1, n)
x, xo = h.v_cycle(b), ho.vcycle(b)
assert np.array_equal(x, xo), np.abs(x - xo).max()
assert np.linalg.norm(A @ x - b) <= 1e-10 * np.linalg.norm(b)
print("OK")
'''


def _rand_csr(rows, cols, per_row, seed):
    rng = np.random.default_rng(seed)
    r = np.repeat(np.arange(rows), per_row)
    c = rng.integers(0, cols, rows * per_row)
    M = sp.csr_matrix((rng.uniform(-1, 1, rows * per_row), (r, c)), shape=(rows, cols))
    M.sum_duplicates()
    M.sort_indices()
    return M


@pytest.mark.parametrize("case", ["giant", "mixed", "giant_hash"])
def test_spgemm_any_row_length(cf, orc, case):
    """Output rows beyond 12288 columns (the sort tier) and, mixed in, rows of every other tier;
    with and without a row scale: pattern and values bitwise the oracle's Gustavson product."""
    if case == "giant":
        A = _rand_csr(40, 30000, 300, 1)     # ~ 300 x 100 products over 60000 columns per row
        B = _rand_csr(30000, 60000, 100, 2)
    elif case == "mixed":
        A = sp.vstack([_rand_csr(3000, 30000, 8, 3), _rand_csr(20, 30000, 250, 4)]).tocsr()
        B = _rand_csr(30000, 60000, 90, 5)
    else:  # beyond the byte-flag column space and with many rows: the hash tiers, then the sort tier
        A = sp.vstack([_rand_csr(40000, 30000, 4, 7), _rand_csr(30, 30000, 300, 8)]).tocsr()
        B = _rand_csr(30000, 200000, 100, 9)
    rs = np.random.default_rng(6).uniform(0.5, 2.0, A.shape[0])
    for scale in (None, rs):
        Cd = cf.CsrMatrix.from_scipy(A).matmul(cf.CsrMatrix.from_scipy(B), scale).export()
        Co = orc.spgemm(orc.Csr.from_scipy(A), orc.Csr.from_scipy(B), scale)
        assert np.array_equal(Cd.ptr, Co.ptr) and np.array_equal(Cd.col, Co.col)
        assert np.array_equal(Cd.val, Co.val), np.abs(Cd.val - Co.val).max()
    assert np.diff(Co.ptr).max() > 12288

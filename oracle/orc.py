"""ctypes bindings of the CPU oracle (liborc.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs, as the checker and the CPU baseline.  The
product package (paper_1806_09924_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liborc.so")


def build(force: bool = False) -> str:
    srcs = [os.path.join(HERE, f) for f in ("crackfield_oracle.cpp", "oracle_mesh.inc")]
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(map(os.path.getmtime, srcs)):
        subprocess.check_call(["make", "-s", "-C", HERE, "liborc.so"])
    return LIB_PATH


class Material(C.Structure):
    _fields_ = [("E", C.c_double), ("nu", C.c_double), ("G_c", C.c_double), ("pressure", C.c_double),
                ("l0", C.c_double), ("kappa_factor", C.c_double), ("eps_mode", C.c_int),
                ("c_eps", C.c_double), ("eps_fixed", C.c_double), ("pressure_coupling", C.c_int)]


def material(**kw) -> Material:
    """Material defaults of model.hpp:14-30 (eps_mode 0 = tied, 1 = fixed)."""
    m = Material(E=1.0, nu=0.2, G_c=1.0, pressure=1e-3, l0=1.0, kappa_factor=1e-12, eps_mode=0,
                 c_eps=2.0, eps_fixed=0.0625, pressure_coupling=0)
    for k, v in kw.items():
        setattr(m, k, v)
    return m


class Regularization(C.Structure):
    _fields_ = [("eps", C.c_double), ("kappa", C.c_double)]


class AmgOptions(C.Structure):
    _fields_ = [("strength_threshold", C.c_double), ("prolongation_omega", C.c_double),
                ("jacobi_omega", C.c_double), ("smoothing_sweeps", C.c_int), ("coarse_size", C.c_int),
                ("max_levels", C.c_int)]


def amg_options(**kw) -> AmgOptions:
    o = AmgOptions(0.02, 2.0 / 3.0, 2.0 / 3.0, 1, 64, 25)
    for k, v in kw.items():
        setattr(o, k, v)
    return o


class GmresOptions(C.Structure):
    _fields_ = [("rtol", C.c_double), ("max_iter", C.c_int), ("restart", C.c_int)]


def gmres_options(**kw) -> GmresOptions:
    o = GmresOptions(1e-8, 1000, 100)
    for k, v in kw.items():
        setattr(o, k, v)
    return o


class SolverOptions(C.Structure):
    _fields_ = [("newton_tol", C.c_double), ("newton_abs_floor", C.c_double), ("newton_max_iter", C.c_int),
                ("active_set_c_scale", C.c_double), ("cycle_window", C.c_int), ("cycle_toggles", C.c_int),
                ("damping", C.c_int), ("prec_kind", C.c_int), ("freeze_preconditioner", C.c_int),
                ("log", C.c_int), ("gmres", GmresOptions), ("amg", AmgOptions)]


def solver_options(**kw) -> SolverOptions:
    o = SolverOptions(1e-8, 1e-11, 50, 100.0, 8, 3, 0, 1, 0, 0, gmres_options(), amg_options())
    for k, v in kw.items():
        setattr(o, k, v)
    return o


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        L.orc_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    """Host threads of the oracle's row-parallel SpMV (1 = the single-threaded reference; results
    are bitwise independent of the count)."""
    lib().orc_set_threads(int(n))


def get_threads() -> int:
    return int(lib().orc_get_threads())


ORDER_PRODUCT, ORDER_REFERENCE = 0, 1


def set_order(order: int) -> None:
    """Reduction order: ORDER_PRODUCT (the device's documented order; bitwise checks) or
    ORDER_REFERENCE (the reference's sequential CSR row sums and dots; tolerance checks)."""
    _chk(lib().orc_set_order(int(order)))


def get_order() -> int:
    return int(lib().orc_get_order())


class reference_order:
    """with orc.reference_order(): ... runs the oracle in the reference's arithmetic order."""

    def __enter__(self):
        self.prev = get_order()
        set_order(ORDER_REFERENCE)
        return self

    def __exit__(self, *exc):
        set_order(self.prev)


class threads:
    """with orc.threads(n): ... runs the oracle on n host threads (results are unchanged)."""

    def __init__(self, n: int):
        self.n = int(n)

    def __enter__(self):
        self.prev = get_threads()
        set_threads(self.n)
        return self

    def __exit__(self, *exc):
        set_threads(self.prev)


def _p(a, ct=C.c_double):
    return a.ctypes.data_as(C.POINTER(ct)) if a is not None else None


def _chk(rc):
    if rc != 0:
        raise RuntimeError(lib().orc_last_error().decode())


class Problem:
    """Uniform grid: create_mesh(d, K, n0) + uniform_refine(r) + build_dof_map."""

    def __init__(self, d: int, K: float, n0: int, r: int):
        self.h_ = C.c_void_p()
        _chk(lib().orc_problem_create(d, C.c_double(K), n0, r, C.byref(self.h_)))
        V, nc, h, dj = C.c_int64(), C.c_int64(), C.c_double(), C.c_double()
        lib().orc_problem_info(self.h_, C.byref(V), C.byref(nc), C.byref(h), C.byref(dj))
        self.d, self.K, self.n0, self.r = d, K, n0, r
        self.V, self.ncells, self.h, self.detJ = V.value, nc.value, h.value, dj.value
        self.n_u, self.n_phi = d * self.V, self.V
        self.n_total = (d + 1) * self.V

    def __del__(self):
        try:
            lib().orc_problem_destroy(self.h_)
        except Exception:
            pass

    def coords(self):
        xyz = np.zeros((self.V, 3))
        lib().orc_vertex_coords(self.h_, _p(xyz))
        return xyz

    def cell_order(self):
        out = np.zeros(self.ncells, dtype=np.int64)
        lib().orc_cell_order(self.h_, _p(out, C.c_int64))
        return out

    def initial_crack(self, mat, band_half=0.0):
        phi = np.zeros(self.V)
        be = C.c_double()
        _chk(lib().orc_initial_crack(self.h_, C.byref(mat), C.c_double(band_half), _p(phi), C.byref(be)))
        return phi, be.value

    def slit_band_edge(self, mat):
        out = C.c_double()
        _chk(lib().orc_slit_band_edge(self.h_, C.byref(mat), C.byref(out)))
        return out.value

    def resolve_regularization(self, mat, band_edge):
        reg = Regularization()
        _chk(lib().orc_resolve_regularization(self.h_, C.byref(mat), C.c_double(band_edge), C.byref(reg)))
        return reg

    def constraints(self, clamp=True, active_dofs=(), active_vals=()):
        return Constraints(self, clamp, active_dofs, active_vals)

    def residual(self, cs, mat, reg, x, pt):
        R = np.zeros(self.n_total)
        _chk(lib().orc_assemble_residual(self.h_, cs.h_, C.byref(mat), C.byref(reg),
                                         _p(np.ascontiguousarray(x, dtype=np.float64)),
                                         _p(np.ascontiguousarray(pt, dtype=np.float64)), _p(R)))
        return R

    def jacobian(self, cs, mat, reg, x, pt):
        h = C.c_void_p()
        _chk(lib().orc_assemble_jacobian(self.h_, cs.h_, C.byref(mat), C.byref(reg),
                                         _p(np.ascontiguousarray(x, dtype=np.float64)),
                                         _p(np.ascontiguousarray(pt, dtype=np.float64)), C.byref(h)))
        return Block(h)

    def rigid_body_modes(self, cs):
        m = 3 if self.d == 2 else 6
        B = np.zeros((m, self.n_u))  # column-major n_u x m == row-major m x n_u
        lib().orc_rigid_body_modes(self.h_, cs.h_, _p(B))
        return B.T.copy()

    def tcv(self, sol):
        out = C.c_double()
        _chk(lib().orc_tcv(self.h_, _p(np.ascontiguousarray(sol, dtype=np.float64)), C.byref(out)))
        return out.value

    def cod(self, sol, stations):
        st = np.ascontiguousarray(stations, dtype=np.float64)
        out = np.zeros(len(st))
        _chk(lib().orc_cod(self.h_, _p(np.ascontiguousarray(sol, dtype=np.float64)), _p(st), len(st), _p(out)))
        return out

    def newton_step(self, mat, reg, opts, solution, phi_old, phi_prev2, step, shift=True, max_its=64):
        its = np.zeros((max_its, 4))
        n_its, conv, feas = C.c_int(), C.c_int(), C.c_double()
        _chk(lib().orc_newton_step(self.h_, C.byref(mat), C.byref(reg), C.byref(opts), _p(solution), _p(phi_old),
                                   _p(phi_prev2), step, int(shift), max_its, _p(its), C.byref(n_its),
                                   C.byref(conv), C.byref(feas)))
        return dict(iterations=its[:n_its.value].copy(), converged=bool(conv.value), feasibility=feas.value)


class Constraints:
    def __init__(self, prob: Problem, clamp, dofs, vals):
        self.prob = prob
        dofs = np.ascontiguousarray(dofs, dtype=np.int64)
        vals = np.ascontiguousarray(vals, dtype=np.float64)
        self.h_ = C.c_void_p()
        _chk(lib().orc_constraints_build(prob.h_, int(clamp), len(dofs), _p(dofs, C.c_int64), _p(vals),
                                         C.byref(self.h_)))

    def __del__(self):
        try:
            lib().orc_constraints_destroy(self.h_)
        except Exception:
            pass

    def flags(self):
        f = np.zeros(self.prob.n_total, dtype=np.uint8)
        g = np.zeros(self.prob.n_total)
        lib().orc_constraints_flags(self.h_, _p(f, C.c_uint8), _p(g))
        return f, g

    def distribute(self, v, homogeneous=False):
        v = np.array(v, dtype=np.float64)
        lib().orc_distribute(self.h_, _p(v), int(homogeneous))
        return v


class Csr:
    """Plain CSR triple (int64 row pointer, int32 columns, float64 values)."""

    def __init__(self, rows, cols, ptr, col, val):
        self.rows, self.cols = int(rows), int(cols)
        self.ptr = np.ascontiguousarray(ptr, dtype=np.int64)
        self.col = np.ascontiguousarray(col, dtype=np.int32)
        self.val = np.ascontiguousarray(val, dtype=np.float64)

    @property
    def nnz(self):
        return int(self.ptr[-1])

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.val, self.col, self.ptr), shape=(self.rows, self.cols))

    @staticmethod
    def from_scipy(M):
        M = M.tocsr()
        M.sort_indices()
        return Csr(M.shape[0], M.shape[1], M.indptr, M.indices, M.data)


class Block:
    def __init__(self, h):
        self.h_ = h

    def __del__(self):
        try:
            lib().orc_block_destroy(self.h_)
        except Exception:
            pass

    def nnz(self, which: int):
        """(rows, cols, nnz) of block `which` (0 M_uu, 1 M_phiu, 2 M_phiphi)."""
        r, c, n = C.c_int64(), C.c_int64(), C.c_int64()
        lib().orc_block_nnz(self.h_, which, C.byref(r), C.byref(c), C.byref(n))
        return r.value, c.value, n.value

    def csr(self, which: int) -> Csr:
        r, c, n = C.c_int64(), C.c_int64(), C.c_int64()
        lib().orc_block_nnz(self.h_, which, C.byref(r), C.byref(c), C.byref(n))
        ptr = np.zeros(r.value + 1, dtype=np.int64)
        col = np.zeros(n.value, dtype=np.int32)
        val = np.zeros(n.value)
        lib().orc_block_export(self.h_, which, _p(ptr, C.c_int64), _p(col, C.c_int32), _p(val))
        return Csr(r.value, c.value, ptr, col, val)

    def apply(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros_like(x)
        lib().orc_block_apply(self.h_, _p(x), _p(y))
        return y

    def spmv(self, which, x, y):
        lib().orc_block_spmv(self.h_, which, _p(x), _p(y))


class CsrHandle:
    def __init__(self, A: Csr):
        self.A = A
        self.h_ = C.c_void_p()
        _chk(lib().orc_csr_create(A.rows, A.cols, _p(A.ptr, C.c_int64), _p(A.col, C.c_int32), _p(A.val),
                                  C.byref(self.h_)))

    def __del__(self):
        try:
            lib().orc_csr_destroy(self.h_)
        except Exception:
            pass


def spgemm(A: Csr, B: Csr, row_scale=None) -> Csr:
    """C = diag(row_scale) A B (the oracle's Gustavson product, linsolve.cpp:248-263)."""
    ha, hb = CsrHandle(A), CsrHandle(B)
    h = C.c_void_p()
    rs = np.ascontiguousarray(row_scale, dtype=np.float64) if row_scale is not None else None
    _chk(lib().orc_csr_spgemm(ha.h_, hb.h_, _p(rs), C.byref(h)))
    r, c, n = C.c_int64(), C.c_int64(), C.c_int64()
    lib().orc_csr_info(h, C.byref(r), C.byref(c), C.byref(n))
    ptr = np.zeros(r.value + 1, dtype=np.int64)
    col = np.zeros(n.value, dtype=np.int32)
    val = np.zeros(n.value)
    lib().orc_csr_export(h, _p(ptr, C.c_int64), _p(col, C.c_int32), _p(val))
    lib().orc_csr_destroy(h)
    return Csr(r.value, c.value, ptr, col, val)


class Amg:
    def __init__(self, A: Csr, node_of_dof=None, B=None, opts=None):
        self.csr = CsrHandle(A)
        opts = opts or amg_options()
        self.h_ = C.c_void_p()
        if node_of_dof is not None:
            nod = np.ascontiguousarray(node_of_dof, dtype=np.int32)
            Bc = np.asfortranarray(B, dtype=np.float64)
            m = Bc.shape[1]
            _chk(lib().orc_amg_build(self.csr.h_, _p(nod, C.c_int32), Bc.ctypes.data_as(C.POINTER(C.c_double)), m,
                                     C.byref(opts), C.byref(self.h_)))
        else:
            _chk(lib().orc_amg_build(self.csr.h_, None, None, 1, C.byref(opts), C.byref(self.h_)))
        nl, cd = C.c_int(), C.c_int64()
        lib().orc_amg_info(self.h_, C.byref(nl), C.byref(cd))
        self.n_levels, self.coarse_dim = nl.value, cd.value
        self.n = A.rows

    def __del__(self):
        try:
            lib().orc_amg_destroy(self.h_)
        except Exception:
            pass

    def level(self, lev):
        info = np.zeros(6, dtype=np.int64)
        lam, jw = C.c_double(), C.c_double()
        lib().orc_amg_level(self.h_, lev, _p(info, C.c_int64), C.byref(lam), C.byref(jw))
        return dict(rows=int(info[0]), nnz_A=int(info[1]), nnz_P=int(info[2]), coarse=int(info[3]),
                    n_nodes=int(info[4]), n_aggregates=int(info[5]), lam=lam.value, jacobi_weight=jw.value)

    def aggregates(self, lev):
        n = self.level(lev)["n_nodes"]
        out = np.zeros(n, dtype=np.int32)
        lib().orc_amg_level_aggregates(self.h_, lev, _p(out, C.c_int32))
        return out

    def level_matrix(self, lev, which):
        info = self.level(lev)
        rows = info["rows"]
        nnz = info["nnz_A"] if which == 0 else info["nnz_P"]
        cols = rows if which == 0 else info["coarse"]
        ptr = np.zeros(rows + 1, dtype=np.int64)
        col = np.zeros(nnz, dtype=np.int32)
        val = np.zeros(nnz)
        lib().orc_amg_level_export(self.h_, lev, which, _p(ptr, C.c_int64), _p(col, C.c_int32), _p(val))
        return Csr(rows, cols, ptr, col, val)

    def vcycle(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        x = np.zeros(self.n)
        _chk(lib().orc_amg_vcycle(self.h_, _p(r), _p(x)))
        return x


class Prec:
    def __init__(self, block: Block, kind: int, opts=None, prob: Problem | None = None, cs: Constraints | None = None):
        opts = opts or amg_options()
        self.block = block
        self.h_ = C.c_void_p()
        _chk(lib().orc_prec_build(block.h_, kind, C.byref(opts), int(prob is not None),
                                  prob.h_ if prob else None, cs.h_ if cs else None, C.byref(self.h_)))

    def __del__(self):
        try:
            lib().orc_prec_destroy(self.h_)
        except Exception:
            pass

    def apply(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.zeros_like(r)
        _chk(lib().orc_prec_apply(self.h_, _p(r), _p(z)))
        return z


def gmres(rhs, block: Block | None = None, csr: CsrHandle | None = None, prec: Prec | None = None,
          amg: Amg | None = None, opts=None):
    opts = opts or gmres_options()
    rhs = np.ascontiguousarray(rhs, dtype=np.float64)
    x = np.zeros_like(rhs)
    it, conv, brk, res = C.c_int(), C.c_int(), C.c_int(), C.c_double()
    hist = np.zeros(max(opts.max_iter, 1))
    _chk(lib().orc_gmres(block.h_ if block else None, csr.h_ if csr else None, prec.h_ if prec else None,
                         amg.h_ if amg else None, _p(rhs), C.byref(opts), _p(x), C.byref(it), C.byref(conv),
                         C.byref(brk), C.byref(res), _p(hist)))
    return dict(x=x, iterations=it.value, converged=bool(conv.value), breakdown=bool(brk.value),
                residual=res.value, history=hist[:it.value].copy())


def detect_cycles(histories, window=8, toggles=3):
    lens = np.array([len(h) for h in histories], dtype=np.int32)
    bits = np.concatenate([np.asarray(h, dtype=np.int8) for h in histories]) if len(histories) else np.zeros(0, np.int8)
    out = np.zeros(len(histories), dtype=np.int32)
    lib().orc_detect_cycles(len(histories), _p(lens, C.c_int32), _p(bits, C.c_int8), window, toggles,
                            _p(out, C.c_int32))
    return out


def qp_tables(d):
    nq = 1 << d
    pts = np.zeros((nq, 3))
    wts = np.zeros(nq)
    shape = np.zeros((nq, nq))
    grads = np.zeros((nq, nq, 3))
    lib().orc_qp_tables(d, _p(pts), _p(wts), _p(shape), _p(grads))
    return pts, wts, shape, grads


def colpiv_qr(A, threshold=1e-10):
    A = np.asfortranarray(A, dtype=np.float64)
    rows, cols = A.shape
    rank = C.c_int()
    Q = np.zeros((cols, rows))  # column-major rows x cols storage, generous
    R = np.zeros(cols * cols)
    perm = np.zeros(cols, dtype=np.int32)
    lib().orc_colpiv_qr(rows, cols, A.ctypes.data_as(C.POINTER(C.c_double)), C.c_double(threshold), C.byref(rank),
                        _p(Q), _p(R), _p(perm, C.c_int32))
    rk = rank.value
    Qm = Q.reshape(-1)[: rows * rk].reshape(rk, rows).T.copy()
    Rm = R[: rk * cols].reshape(cols, rk).T.copy()
    return rk, Qm, Rm, perm


def lame(mat):
    mu, lam = C.c_double(), C.c_double()
    lib().orc_lame(C.byref(mat), C.byref(mu), C.byref(lam))
    return mu.value, lam.value


def sigma(grad, mat, d):
    g = np.ascontiguousarray(np.asarray(grad, dtype=np.float64).reshape(3, 3))
    out = np.zeros((3, 3))
    lib().orc_sigma(_p(g), C.byref(mat), d, _p(out))
    return out


# ------------------------------------------------------------------ general (adaptive) meshes
class Mesh:
    """Adaptive forest mesh + its DofMap (mesh.cpp, fem.cpp:98-146): create_mesh(d, K, n0),
    refine / uniform_refine; cell ids in creation order, vertices = sorted packed keys."""

    def __init__(self, d: int, K: float, n0: int, _h=None):
        self.h_ = C.c_void_p()
        if _h is None:
            _chk(lib().orc_mesh_create(d, C.c_double(K), n0, C.byref(self.h_)))
        else:
            self.h_ = _h
        self.d, self.K, self.n0 = d, K, n0
        self._info()

    def _info(self):
        info = np.zeros(4, dtype=np.int64)
        hmin = C.c_double()
        lib().orc_mesh_info(self.h_, _p(info, C.c_int64), C.byref(hmin))
        self.n_cells, self.n_active, self.max_level, self.V = (int(v) for v in info)
        self.h_min = hmin.value
        self.n_u, self.n_phi, self.n_total = self.d * self.V, self.V, (self.d + 1) * self.V

    def __del__(self):
        try:
            lib().orc_mesh_destroy(self.h_)
        except Exception:
            pass

    def copy(self):
        h = C.c_void_p()
        _chk(lib().orc_mesh_copy(self.h_, C.byref(h)))
        return Mesh(self.d, self.K, self.n0, _h=h)

    def refine(self, ids):
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        _chk(lib().orc_mesh_refine(self.h_, _p(ids, C.c_int32), C.c_int64(len(ids))))
        self._info()

    def uniform_refine(self, times):
        _chk(lib().orc_mesh_uniform_refine(self.h_, int(times)))
        self._info()

    def cells(self):
        n = self.n_cells
        lev = np.zeros(n, dtype=np.int32)
        par = np.zeros(n, dtype=np.int32)
        act = np.zeros(n, dtype=np.int8)
        anc = np.zeros((n, 3), dtype=np.int64)
        lib().orc_mesh_cells(self.h_, _p(lev, C.c_int32), _p(par, C.c_int32), _p(act, C.c_int8), _p(anc, C.c_int64))
        return dict(level=lev, parent=par, active=act.astype(bool), anchor=anc)

    def active(self):
        out = np.zeros(self.n_active, dtype=np.int32)
        lib().orc_mesh_active(self.h_, _p(out, C.c_int32))
        return out

    def vertex_keys(self):
        out = np.zeros(self.V, dtype=np.int64)
        lib().orc_mesh_vertex_keys(self.h_, _p(out, C.c_int64))
        return out

    def cell_vertices(self):
        out = np.zeros((self.n_active, 1 << self.d), dtype=np.int64)
        _chk(lib().orc_mesh_cell_vertices(self.h_, _p(out, C.c_int64)))
        return out

    def faces(self):
        n = C.c_int64()
        lib().orc_mesh_faces(self.h_, C.byref(n), None)
        out = np.zeros((n.value, 5), dtype=np.int32)
        lib().orc_mesh_faces(self.h_, C.byref(n), _p(out, C.c_int32))
        return out

    def find_cell(self, x):
        x = np.ascontiguousarray(list(x) + [0.0] * (3 - len(x)), dtype=np.float64)
        out = C.c_int32()
        lib().orc_mesh_find_cell(self.h_, _p(x), C.byref(out))
        return out.value

    def constraints(self, clamp=True, active_dofs=(), active_vals=()):
        return MeshConstraints(self, clamp, active_dofs, active_vals)

    def residual(self, cs, mat, reg, x, pt):
        R = np.zeros(self.n_total)
        _chk(lib().orc_mesh_residual(self.h_, cs.h_, C.byref(mat), C.byref(reg),
                                     _p(np.ascontiguousarray(x, dtype=np.float64)),
                                     _p(np.ascontiguousarray(pt, dtype=np.float64)), _p(R)))
        return R

    def jacobian(self, cs, mat, reg, x, pt):
        h = C.c_void_p()
        _chk(lib().orc_mesh_jacobian(self.h_, cs.h_, C.byref(mat), C.byref(reg),
                                     _p(np.ascontiguousarray(x, dtype=np.float64)),
                                     _p(np.ascontiguousarray(pt, dtype=np.float64)), C.byref(h)))
        return Block(h)

    def rigid_body_modes(self, cs):
        m = 3 if self.d == 2 else 6
        B = np.zeros((m, self.n_u))
        lib().orc_mesh_rigid_body_modes(self.h_, cs.h_, _p(B))
        return B.T.copy()

    def slit_band_edge(self, mat):
        out = C.c_double()
        _chk(lib().orc_mesh_slit_band_edge(self.h_, C.byref(mat), C.byref(out)))
        return out.value

    def resolve_regularization(self, mat, band_edge):
        reg = Regularization()
        _chk(lib().orc_mesh_resolve_regularization(self.h_, C.byref(mat), C.c_double(band_edge), C.byref(reg)))
        return reg

    def initial_crack(self, mat, band_half=0.0):
        phi = np.zeros(self.V)
        be = C.c_double()
        _chk(lib().orc_mesh_initial_crack(self.h_, C.byref(mat), C.c_double(band_half), _p(phi), C.byref(be)))
        return phi, be.value

    def newton_step(self, mat, reg, opts, solution, phi_old, phi_prev2, step, shift=True, max_its=64):
        its = np.zeros((max_its, 4))
        n_its, conv, feas = C.c_int(), C.c_int(), C.c_double()
        _chk(lib().orc_mesh_newton_step(self.h_, C.byref(mat), C.byref(reg), C.byref(opts), _p(solution),
                                        _p(phi_old), _p(phi_prev2), step, int(shift), max_its, _p(its),
                                        C.byref(n_its), C.byref(conv), C.byref(feas)))
        return dict(iterations=its[:n_its.value].copy(), converged=bool(conv.value), feasibility=feas.value)

    def tcv(self, sol):
        out = C.c_double()
        _chk(lib().orc_mesh_tcv(self.h_, _p(np.ascontiguousarray(sol, dtype=np.float64)), C.byref(out)))
        return out.value

    def cod(self, sol, stations):
        st = np.ascontiguousarray(stations, dtype=np.float64)
        out = np.zeros(len(st))
        _chk(lib().orc_mesh_cod(self.h_, _p(np.ascontiguousarray(sol, dtype=np.float64)), _p(st), len(st),
                                _p(out)))
        return out

    def estimator(self, sol):
        eta = np.zeros(self.n_active)
        _chk(lib().orc_mesh_estimator(self.h_, _p(np.ascontiguousarray(sol, dtype=np.float64)), _p(eta)))
        return eta

    def mark(self, sol, eta=None, phi_threshold=0.8, h_target=0.0, theta=0.3, max_level=16, estimator=True):
        pol = np.array([phi_threshold, h_target, theta, max_level, 1.0 if estimator else 0.0])
        out = np.zeros(self.n_active, dtype=np.int32)
        n = C.c_int64()
        e = None if eta is None else np.ascontiguousarray(eta, dtype=np.float64)
        _chk(lib().orc_mesh_mark(self.h_, _p(np.ascontiguousarray(sol, dtype=np.float64)), _p(e), _p(pol),
                                 _p(out, C.c_int32), C.byref(n)))
        return out[:n.value].copy()

    def transfer_to(self, vec, new_mesh):
        out = np.zeros(new_mesh.n_total)
        _chk(lib().orc_mesh_transfer(self.h_, _p(np.ascontiguousarray(vec, dtype=np.float64)), new_mesh.h_,
                                     _p(out)))
        return out

    def adaptive_cycle(self, mat, opts, cycles=1, n_steps=1, estimator_rounds=1, halve_band_target=True,
                       seed_band=0.0, phi_threshold=0.8, h_target=0.0, theta=0.3, max_level=16, estimator=True,
                       sol_cap=1 << 24):
        pol = np.array([phi_threshold, h_target, theta, max_level, 1.0 if estimator else 0.0])
        rec = np.zeros((cycles + 1, 8))
        n = C.c_int()
        sol = np.zeros(sol_cap)
        _chk(lib().orc_mesh_adaptive_cycle(self.h_, C.byref(mat), C.byref(opts), _p(pol), cycles, n_steps,
                                           estimator_rounds, int(halve_band_target), C.c_double(seed_band),
                                           cycles + 1, _p(rec), C.byref(n), _p(sol), C.c_int64(sol_cap)))
        self._info()
        return rec[:n.value].copy(), sol[:self.n_total].copy()


class MeshConstraints:
    """ConstraintSet of a general mesh (fem.cpp:189-267): closed lines in ascending dof order."""

    def __init__(self, mesh: Mesh, clamp, dofs, vals):
        self.mesh = mesh
        dofs = np.ascontiguousarray(dofs, dtype=np.int64)
        vals = np.ascontiguousarray(vals, dtype=np.float64)
        self.h_ = C.c_void_p()
        _chk(lib().orc_mesh_constraints(mesh.h_, int(clamp), C.c_int64(len(dofs)), _p(dofs, C.c_int64), _p(vals),
                                        C.byref(self.h_)))

    def __del__(self):
        try:
            lib().orc_mcs_destroy(self.h_)
        except Exception:
            pass

    def lines(self):
        """dofs, ptr, masters, weights, inhomogeneities (CSR of the closed lines)."""
        nl, ne = C.c_int64(), C.c_int64()
        lib().orc_mcs_info(self.h_, C.byref(nl), C.byref(ne))
        dofs = np.zeros(nl.value, dtype=np.int64)
        ptr = np.zeros(nl.value + 1, dtype=np.int64)
        m = np.zeros(ne.value, dtype=np.int64)
        w = np.zeros(ne.value)
        inh = np.zeros(nl.value)
        lib().orc_mcs_export(self.h_, _p(dofs, C.c_int64), _p(ptr, C.c_int64), _p(m, C.c_int64), _p(w), _p(inh))
        return dofs, ptr, m, w, inh

    def distribute(self, v, homogeneous=False):
        v = np.array(v, dtype=np.float64)
        lib().orc_mcs_distribute(self.h_, _p(v), C.c_int64(len(v)), int(homogeneous))
        return v

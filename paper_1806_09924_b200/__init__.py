"""crackfield_b200: B200-native Newton/active-set hot path of the pressurized phase-field fracture
solver of arXiv 1806.09924, behind the reference's own operator interface.

Host-side mirror of the reference C++ API on the hot path, over the C ABI of
include/crackfield_b200.h.  Names, argument meaning and error behaviour follow
/root/reference/proj/include/crackfield/{model,linsolve,solver,fem}.hpp:

    prob = Problem(dim=2, half_width=10.0, n0=8, refinements=5)   # create_mesh + uniform_refine + DofMap
    cs   = build_constraints(prob, active_set={dof: value})       # fem.cpp:205-267
    R    = assemble_residual(prob, cs, mat, reg, x, phi_tilde)    # model.cpp:127-202
    J    = assemble_jacobian(prob, cs, mat, reg, x, phi_tilde)    # model.cpp:204-322
    y    = J.apply(x)                                             # linsolve.cpp:13-19

Arrays may be numpy (host; copied in/out per call, synchronous) or torch CUDA tensors (device
resident; stream-ordered on the library stream, see set_stream).  Outputs follow the kind of
the first array argument.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import (AmgOptions, CfError, GmresOptions, Material, Regularization, SolverOptions, check, load)

__all__ = ["Material", "Regularization", "AmgOptions", "GmresOptions", "SolverOptions", "Problem",
           "ConstraintSet", "BlockSystem", "build_constraints", "assemble_residual", "assemble_jacobian",
           "set_stream", "synchronize", "kernel_launches", "device_info", "CfError"]


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


def _ptr(a):
    """Raw pointer of a numpy array or torch tensor (must be contiguous float64/int64)."""
    if a is None:
        return None
    if _is_torch(a):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return C.c_void_p(a.data_ptr())
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("array must be C-contiguous")
    return C.c_void_p(a.ctypes.data)


def _as_f64(a):
    if _is_torch(a):
        import torch
        return a.to(torch.float64).contiguous()
    return np.ascontiguousarray(a, dtype=np.float64)


def _empty_like_kind(ref, n):
    if _is_torch(ref):
        import torch
        return torch.empty(n, dtype=torch.float64, device=ref.device)
    return np.empty(n, dtype=np.float64)


def set_stream(stream) -> None:
    """Order all library work on `stream` (a torch.cuda.Stream, a raw handle, or None)."""
    h = getattr(stream, "cuda_stream", stream)
    check(load().cf_set_stream(C.c_void_p(h) if h else None))


def synchronize() -> None:
    check(load().cf_synchronize())


def kernel_launches() -> int:
    return int(load().cf_kernel_launches())


def device_info():
    dev, sms, mem = C.c_int(), C.c_int(), C.c_int64()
    check(load().cf_device_info(C.byref(dev), C.byref(sms), C.byref(mem)))
    return dict(device=dev.value, sm_count=sms.value, total_mem=mem.value)


class Problem:
    """Uniform mesh + DofMap: create_mesh(DomainSpec{dim, half_width, n0}) + uniform_refine(refinements)
    + build_dof_map (mesh.cpp:18-34, 209-215; fem.cpp:98-116).  Vertices are lexicographic (x fastest);
    u dofs v*d+c, phi dofs n_u+v (fem.hpp:35-43)."""

    def __init__(self, dim: int = 2, half_width: float = 20.0, n0: int = 8, refinements: int = 0):
        self._h = C.c_void_p()
        check(load().cf_problem_create_uniform(dim, float(half_width), n0, refinements, C.byref(self._h)))
        V, nc, h = C.c_int64(), C.c_int64(), C.c_double()
        check(load().cf_problem_info(self._h, C.byref(V), C.byref(nc), C.byref(h)))
        self.dim, self.half_width, self.n0, self.refinements = dim, float(half_width), n0, refinements
        self.n_vertices, self.n_cells, self.h = V.value, nc.value, h.value
        self.n_u, self.n_phi = dim * self.n_vertices, self.n_vertices
        self.n_total = self.n_u + self.n_phi
        self.nodes_per_side = (n0 << refinements) + 1

    def __del__(self):
        try:
            load().cf_problem_destroy(self._h)
        except Exception:
            pass

    # DofMap accessors (fem.hpp:39-43)
    def u_dof(self, vertex: int, component: int) -> int:
        return vertex * self.dim + component

    def phi_dof(self, vertex: int) -> int:
        return self.n_u + vertex

    def vertex_physical(self):
        """Physical vertex coordinates (V x 3), mesh.hpp:73-75 arithmetic."""
        n = self.nodes_per_side
        unit = 2.0 * self.half_width / (self.n0 * float(1 << 16))
        c = -self.half_width + (np.arange(n, dtype=np.int64) * (1 << (16 - self.refinements))).astype(np.float64) * unit
        idx = np.arange(self.n_vertices)
        xyz = np.zeros((self.n_vertices, 3))
        xyz[:, 0] = c[idx % n]
        xyz[:, 1] = c[(idx // n) % n]
        if self.dim == 3:
            xyz[:, 2] = c[idx // (n * n)]
        return xyz


class ConstraintSet:
    """ConstraintSet built by build_constraints (fem.cpp:205-267); device resident."""

    def __init__(self, prob: Problem, clamp: bool = True, active_set: dict | None = None):
        self.prob = prob
        active_set = active_set or {}
        dofs = np.fromiter(active_set.keys(), dtype=np.int64, count=len(active_set))
        vals = np.fromiter(active_set.values(), dtype=np.float64, count=len(active_set))
        self._h = C.c_void_p()
        check(load().cf_constraints_build(prob._h, int(clamp), len(dofs), _ptr(dofs), _ptr(vals), C.byref(self._h)))
        self.n_active = len(dofs)

    def __del__(self):
        try:
            load().cf_constraints_destroy(self._h)
        except Exception:
            pass

    def distribute(self, v):
        """In place (fem.cpp:189-195)."""
        check(load().cf_constraints_distribute(self._h, _ptr(v), 0))
        return v

    def distribute_homogeneous(self, v):
        """In place (fem.cpp:197-203)."""
        check(load().cf_constraints_distribute(self._h, _ptr(v), 1))
        return v


def build_constraints(prob: Problem, clamp_displacement_on_boundary: bool = True, active_set: dict | None = None):
    return ConstraintSet(prob, clamp_displacement_on_boundary, active_set)


class Csr:
    def __init__(self, rows, cols, ptr, col, val):
        self.rows, self.cols, self.ptr, self.col, self.val = rows, cols, ptr, col, val

    @property
    def nnz(self):
        return int(self.ptr[-1])

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.val, self.col, self.ptr), shape=(self.rows, self.cols))


class BlockSystem:
    """Device-resident BlockSystem (linsolve.hpp:17-28): [M_uu 0; M_phiu M_phiphi]."""

    def __init__(self, handle):
        self._h = handle
        nu, np_, nnz = C.c_int64(), C.c_int64(), (C.c_int64 * 3)()
        check(load().cf_block_info(self._h, C.byref(nu), C.byref(np_), nnz))
        self._n_u, self._n_phi = nu.value, np_.value
        self.nnz = tuple(int(v) for v in nnz)

    def __del__(self):
        try:
            load().cf_block_destroy(self._h)
        except Exception:
            pass

    def n_u(self):
        return self._n_u

    def n_phi(self):
        return self._n_phi

    def n_total(self):
        return self._n_u + self._n_phi

    def apply(self, x, out=None):
        """BlockSystem::apply (linsolve.cpp:13-19)."""
        x = _as_f64(x)
        y = out if out is not None else _empty_like_kind(x, self.n_total())
        check(load().cf_block_apply(self._h, _ptr(x), _ptr(y)))
        return y

    def spmv(self, which: int, x, out=None):
        """One block times a vector (which: 0 M_uu, 1 M_phiu, 2 M_phiphi)."""
        rows = self._n_u if which == 0 else self._n_phi
        y = out if out is not None else _empty_like_kind(x, rows)
        check(load().cf_block_spmv(self._h, which, _ptr(x), _ptr(y)))
        return y

    def csr(self, which: int) -> Csr:
        rows = self._n_u if which == 0 else self._n_phi
        cols = self._n_phi if which == 2 else self._n_u
        nnz = self.nnz[which]
        ptr = np.empty(rows + 1, dtype=np.int64)
        col = np.empty(nnz, dtype=np.int32)
        val = np.empty(nnz, dtype=np.float64)
        check(load().cf_block_export(self._h, which, _ptr(ptr), _ptr(col), _ptr(val)))
        return Csr(rows, cols, ptr, col, val)

    @property
    def M_uu(self):
        return self.csr(0)

    @property
    def M_phiu(self):
        return self.csr(1)

    @property
    def M_phiphi(self):
        return self.csr(2)


def assemble_residual(prob: Problem, constraints: ConstraintSet, mat: Material, reg: Regularization, solution,
                      phi_tilde, out=None):
    """model.hpp:62-64: residual (F_u, F_phi), condensed (constrained entries 0)."""
    x, pt = _as_f64(solution), _as_f64(phi_tilde)
    R = out if out is not None else _empty_like_kind(x, prob.n_total)
    check(load().cf_assemble_residual(prob._h, constraints._h, C.byref(mat), C.byref(reg), _ptr(x), _ptr(pt),
                                      _ptr(R)))
    return R


def assemble_jacobian(prob: Problem, constraints: ConstraintSet, mat: Material, reg: Regularization, solution,
                      phi_tilde) -> BlockSystem:
    """model.hpp:68-70: exact Gateaux derivative with phi_tilde frozen (M_uphi = 0)."""
    x, pt = _as_f64(solution), _as_f64(phi_tilde)
    h = C.c_void_p()
    check(load().cf_assemble_jacobian(prob._h, constraints._h, C.byref(mat), C.byref(reg), _ptr(x), _ptr(pt),
                                      C.byref(h)))
    return BlockSystem(h)

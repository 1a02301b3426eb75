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
        # vertex planes along the slowest axis (z in 3d, y in 2d): the slab decomposition unit
        self.n_planes = self.nodes_per_side
        self.plane = self.nodes_per_side ** (dim - 1)

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
        shape = (C.c_int64 * 4)()
        check(load().cf_block_shape(self._h, shape))
        self._in_u, self._in_phi = int(shape[2]), int(shape[3])  # > rows for a slab (ghost planes)

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

    def n_in(self):
        """Input length of apply: n_total, or the ext layout [u_ext | phi_ext] of a slab."""
        return self._in_u + self._in_phi

    def apply(self, x, out=None):
        """BlockSystem::apply (linsolve.cpp:13-19)."""
        x = _as_f64(x)
        y = out if out is not None else _empty_like_kind(x, self.n_total())
        check(load().cf_block_apply(self._h, _ptr(x), _ptr(y)))
        return y

    def format(self, which: int) -> str:
        """Storage the SpMV of a block streams: "csr" or "stencil" (values only, implicit columns)."""
        f = C.c_int()
        check(load().cf_block_format(self._h, which, C.byref(f)))
        return "stencil" if f.value == 1 else "csr"

    def spmv(self, which: int, x, out=None):
        """One block times a vector (which: 0 M_uu, 1 M_phiu, 2 M_phiphi)."""
        rows = self._n_u if which == 0 else self._n_phi
        y = out if out is not None else _empty_like_kind(x, rows)
        check(load().cf_block_spmv(self._h, which, _ptr(x), _ptr(y)))
        return y

    def csr(self, which: int) -> Csr:
        rows = self._n_u if which == 0 else self._n_phi
        cols = self._in_phi if which == 2 else self._in_u
        nnz = self.nnz[which]
        ptr = np.empty(rows + 1, dtype=np.int64)
        col = np.empty(nnz, dtype=np.int32)
        val = np.empty(nnz, dtype=np.float64)
        check(load().cf_block_export(self._h, which, _ptr(ptr), _ptr(col), _ptr(val)))
        return Csr(rows, cols, ptr, col, val)

    def write_matrix_market(self, which: int, path: str) -> None:
        """write_matrix_market (linsolve.cpp:478-490) of one block, byte-identical text."""
        check(load().cf_block_write_matrix_market(self._h, int(which), str(path).encode()))

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
                      phi_tilde, out=None, planes=None):
    """model.hpp:62-64: residual (F_u, F_phi), condensed (constrained entries 0).

    planes=(p_lo, p_hi): only the rows of the vertex planes [p_lo, p_hi) along the slowest axis
    (a slab), in the local layout [u_own | phi_own]."""
    x, pt = _as_f64(solution), _as_f64(phi_tilde)
    if planes is None:
        R = out if out is not None else _empty_like_kind(x, prob.n_total)
        check(load().cf_assemble_residual(prob._h, constraints._h, C.byref(mat), C.byref(reg), _ptr(x), _ptr(pt),
                                          _ptr(R)))
        return R
    nv = (planes[1] - planes[0]) * prob.plane
    R = out if out is not None else _empty_like_kind(x, (prob.dim + 1) * nv)
    check(load().cf_assemble_residual_planes(prob._h, constraints._h, C.byref(mat), C.byref(reg), _ptr(x),
                                             _ptr(pt), int(planes[0]), int(planes[1]), _ptr(R)))
    return R


def assemble_jacobian(prob: Problem, constraints: ConstraintSet, mat: Material, reg: Regularization, solution,
                      phi_tilde, planes=None) -> BlockSystem:
    """model.hpp:68-70: exact Gateaux derivative with phi_tilde frozen (M_uphi = 0).

    planes=(p_lo, p_hi): the slab's rows, columns over its planes plus one ghost plane each side."""
    x, pt = _as_f64(solution), _as_f64(phi_tilde)
    h = C.c_void_p()
    if planes is None:
        check(load().cf_assemble_jacobian(prob._h, constraints._h, C.byref(mat), C.byref(reg), _ptr(x), _ptr(pt),
                                          C.byref(h)))
    else:
        check(load().cf_assemble_jacobian_planes(prob._h, constraints._h, C.byref(mat), C.byref(reg), _ptr(x),
                                                 _ptr(pt), int(planes[0]), int(planes[1]), C.byref(h)))
    return BlockSystem(h)


def mf_apply_uu(prob: Problem, constraints: ConstraintSet, mat: Material, reg: Regularization, phi_tilde, x,
                out=None):
    """Matrix-free y_u = M_uu x_u (BASELINE config 1's matrix-free operator; equal to the assembled
    apply to rounding)."""
    xx, pt = _as_f64(x), _as_f64(phi_tilde)
    y = out if out is not None else _empty_like_kind(xx, prob.n_u)
    check(load().cf_mf_apply_uu(prob._h, constraints._h, C.byref(mat), C.byref(reg), _ptr(pt), _ptr(xx), _ptr(y)))
    return y


def fp64_peak_tflops() -> float:
    """FP64 FMA throughput of the device (DFMA loop), TFLOP/s."""
    v = C.c_double()
    check(load().cf_fp64_peak(C.byref(v)))
    return v.value


def sigma(grad_u, mat: Material, d: int) -> np.ndarray:
    """model.cpp:19-26: sigma = 2 mu e + lambda tr(e) I, e = sym(grad u) (3x3, first d x d used)."""
    g = np.ascontiguousarray(np.asarray(grad_u, dtype=np.float64).reshape(3, 3))
    out = np.zeros((3, 3))
    check(load().cf_sigma(_ptr(g), C.byref(mat), int(d), _ptr(out)))
    return out


def q1_shape(d: int, xi):
    """fem.cpp:76-96: Q1 values (2^d) and gradients (2^d x d) at reference point xi."""
    x = np.zeros(3)
    x[:len(xi)] = xi
    vals, grads = np.zeros(1 << d), np.zeros((1 << d, d))
    check(load().cf_q1_shape(int(d), _ptr(x), _ptr(vals), _ptr(grads)))
    return vals, grads


def detect_cycles(history: dict, window: int = 8, toggles: int = 3) -> set:
    """solver.cpp:10-22: dofs whose membership history toggles >= `toggles` times within the last
    `window` entries."""
    dofs = np.fromiter(history.keys(), dtype=np.int32, count=len(history))
    lens = np.array([len(history[int(k)]) for k in dofs], dtype=np.int64)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    bits = np.concatenate([np.asarray(history[int(k)], dtype=np.uint8) for k in dofs]) if len(dofs) else \
        np.zeros(1, dtype=np.uint8)
    out = np.zeros(max(1, len(dofs)), dtype=np.int32)
    n = C.c_int()
    check(load().cf_detect_cycles(len(dofs), _ptr(dofs), _ptr(offs), _ptr(bits), int(window), int(toggles),
                                  _ptr(out), C.byref(n)))
    return set(int(v) for v in out[:n.value])


def extrapolate_phi(state) -> np.ndarray:
    """model.cpp:60-64: phi_tilde of a FractureState (host copy)."""
    out = np.zeros(state.prob.n_phi)
    check(load().cf_extrapolate_phi(state._h, _ptr(out)))
    return out


def assemble_pattern(prob: Problem, constraints: ConstraintSet) -> BlockSystem:
    """linsolve.hpp:138 / linsolve.cpp:417-476: the block sparsity after condensation (values 0)."""
    h = C.c_void_p()
    check(load().cf_assemble_pattern(prob._h, constraints._h, C.byref(h)))
    return BlockSystem(h)


def slab_info(prob: Problem, rank: int, size: int) -> dict:
    """The slab of rank `rank` of `size` (cf_slab_info): owned / ext vertex ranges, cell range."""
    info = (C.c_int64 * 7)()
    check(load().cf_slab_info(prob._h, int(rank), int(size), info))
    keys = ("v_lo", "v_hi", "ve_lo", "ve_hi", "c_lo", "c_hi", "plane")
    return {k: int(v) for k, v in zip(keys, info)}


class Communicator:
    """NCCL communicator of the slab-decomposed Newton step (one process per GPU).

    from_torch_distributed(): rank 0 makes the NCCL id, torch.distributed broadcasts it, every
    rank creates its communicator on its current CUDA device (set it first)."""

    def __init__(self, rank: int, size: int, uid: bytes | None = None):
        self._h = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(uid) if uid is not None else None
        check(load().cf_comm_create(buf, int(rank), int(size), C.byref(self._h)))
        self.rank, self.size = int(rank), int(size)

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(load().cf_comm_unique_id(buf))
        return bytes(buf)

    @staticmethod
    def nccl_selftest() -> int:
        """Every NCCL entry point of the decomposed step on a one-rank communicator on the current
        device (cf_comm_selftest); returns the number of failed checks (0 = all hold)."""
        bad = C.c_int(-1)
        check(load().cf_comm_selftest(C.byref(bad)))
        return bad.value

    @classmethod
    def from_torch_distributed(cls, group=None) -> "Communicator":
        import torch.distributed as dist
        rank, size = dist.get_rank(group), dist.get_world_size(group)
        if size == 1:
            return cls(0, 1)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(rank, size, obj[0])

    @classmethod
    def from_gloo(cls, group=None) -> "Communicator":
        """TEST ONLY: a communicator whose transport is torch.distributed on host memory (e.g. gloo),
        so several ranks can share one GPU to exercise the decomposed step's control flow.  Device
        data is staged through the host; never used for a measurement."""
        import torch
        import torch.distributed as dist
        from ._lib import AllgatherF64, AllreduceI64, Bcast, HostTransport, SendRecv
        rank, size = dist.get_rank(group), dist.get_world_size(group)

        def buf(ptr, n, ctype):
            return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), shape=(n,)) if n else np.zeros(0)

        def allgather(_ctx, send, recv, k):
            try:
                t = torch.from_numpy(buf(send, k, C.c_double).copy())
                parts = [torch.empty_like(t) for _ in range(size)]
                dist.all_gather(parts, t, group=group)
                buf(recv, size * k, C.c_double)[:] = torch.cat(parts).numpy()
                return 0
            except Exception:
                return 1

        def allreduce(_ctx, vals, k, op):
            try:
                a = buf(vals, k, C.c_longlong)
                t = torch.from_numpy(a.astype(np.int64))
                dist.all_reduce(t, op=dist.ReduceOp.SUM if op == 0 else dist.ReduceOp.MAX, group=group)
                a[:] = t.numpy()
                return 0
            except Exception:
                return 1

        def sendrecv(_ctx, n, send, recv, nbytes, peer):
            try:
                ops, outs = [], []
                for j in range(n):
                    b = int(nbytes[j])
                    if send[j]:
                        t = torch.from_numpy(buf(send[j], b, C.c_uint8).copy())
                        ops.append(dist.P2POp(dist.isend, t, int(peer[j]), group=group))
                    if recv[j]:
                        t = torch.empty(b, dtype=torch.uint8)
                        ops.append(dist.P2POp(dist.irecv, t, int(peer[j]), group=group))
                        outs.append((recv[j], b, t))
                if ops:
                    for w in dist.batch_isend_irecv(ops):
                        w.wait()
                for p, b, t in outs:
                    buf(p, b, C.c_uint8)[:] = t.numpy()
                return 0
            except Exception:
                return 1

        def bcast(_ctx, p, nbytes, root):
            try:
                a = buf(p, int(nbytes), C.c_uint8)
                t = torch.from_numpy(a.copy())
                dist.broadcast(t, src=root, group=group)
                a[:] = t.numpy()
                return 0
            except Exception:
                return 1

        obj = cls.__new__(cls)
        obj._callbacks = (AllgatherF64(allgather), AllreduceI64(allreduce), SendRecv(sendrecv), Bcast(bcast))
        obj._transport = HostTransport(None, *obj._callbacks)
        obj._h = C.c_void_p()
        check(load().cf_comm_create_host(rank, size, C.byref(obj._transport), C.byref(obj._h)))
        obj.rank, obj.size = rank, size
        return obj

    def __del__(self):
        try:
            load().cf_comm_destroy(self._h)
        except Exception:
            pass


# ---------------------------------------------------------------------------- linear algebra
class CsrMatrix:
    """Device CSR matrix (types.hpp:12); from host (rows, cols, rowptr, col, val) or a block."""

    def __init__(self, rows=None, cols=None, rowptr=None, col=None, val=None, _handle=None):
        if _handle is not None:
            self._h = _handle
        else:
            rp = np.ascontiguousarray(rowptr, dtype=np.int64)
            ci = np.ascontiguousarray(col, dtype=np.int32)
            vv = np.ascontiguousarray(val, dtype=np.float64)
            self._h = C.c_void_p()
            check(load().cf_csr_create(int(rows), int(cols), _ptr(rp), _ptr(ci), _ptr(vv), C.byref(self._h)))
        r, c, n = C.c_int64(), C.c_int64(), C.c_int64()
        check(load().cf_csr_info(self._h, C.byref(r), C.byref(c), C.byref(n)))
        self.rows, self.cols, self.nnz = r.value, c.value, n.value

    @staticmethod
    def from_scipy(M):
        M = M.tocsr()
        M.sort_indices()
        return CsrMatrix(M.shape[0], M.shape[1], M.indptr, M.indices, M.data)

    @staticmethod
    def from_block(J: BlockSystem, which: int):
        h = C.c_void_p()
        check(load().cf_block_csr(J._h, which, C.byref(h)))
        return CsrMatrix(_handle=h)

    def __del__(self):
        try:
            load().cf_csr_destroy(self._h)
        except Exception:
            pass

    def __matmul__(self, x):
        x = _as_f64(x)
        y = _empty_like_kind(x, self.rows)
        check(load().cf_csr_spmv(self._h, _ptr(x), _ptr(y)))
        return y

    def export(self) -> Csr:
        """Host copy (rowptr, col, val) of the device matrix."""
        rp = np.zeros(self.rows + 1, dtype=np.int64)
        ci = np.zeros(self.nnz, dtype=np.int32)
        vv = np.zeros(self.nnz)
        check(load().cf_csr_export(self._h, _ptr(rp), _ptr(ci), _ptr(vv)))
        return Csr(self.rows, self.cols, rp, ci, vv)

    def matmul(self, B: "CsrMatrix", row_scale=None) -> "CsrMatrix":
        """C = diag(row_scale) self B (linsolve.cpp:248-263, the AMG setup's sparse products)."""
        h = C.c_void_p()
        rs = _as_f64(row_scale) if row_scale is not None else None
        check(load().cf_csr_spgemm(self._h, B._h, _ptr(rs) if rs is not None else None, C.byref(h)))
        return CsrMatrix(_handle=h)


class AmgHierarchy:
    """AmgHierarchy (linsolve.hpp:64-85) built by build_amg on the device."""

    def __init__(self, A: CsrMatrix, node_of_dof=None, near_nullspace=None, opts: AmgOptions | None = None):
        self.A = A
        self.opts = opts or AmgOptions()
        self._h = C.c_void_p()
        if node_of_dof is not None and _is_torch(node_of_dof):  # device arrays: no staging copies
            import torch
            nod = node_of_dof.to(torch.int32).contiguous()
            B = near_nullspace.to(torch.float64)
            m = 1 if B.dim() == 1 else B.shape[1]
            Bf = B.t().contiguous().reshape(-1) if B.dim() == 2 else B.contiguous()
            check(load().cf_amg_build(A._h, _ptr(nod), _ptr(Bf), m, C.byref(self.opts), C.byref(self._h)))
        elif node_of_dof is not None:
            nod = np.ascontiguousarray(node_of_dof, dtype=np.int32)
            B = np.asfortranarray(near_nullspace, dtype=np.float64)
            m = 1 if B.ndim == 1 else B.shape[1]
            Bf = np.ascontiguousarray(B.T).reshape(-1) if B.ndim == 2 else B
            check(load().cf_amg_build(A._h, _ptr(nod), _ptr(np.ascontiguousarray(Bf)), m, C.byref(self.opts),
                                      C.byref(self._h)))
        else:
            check(load().cf_amg_build(A._h, None, None, 1, C.byref(self.opts), C.byref(self._h)))
        nl, cd = C.c_int(), C.c_int64()
        check(load().cf_amg_info(self._h, C.byref(nl), C.byref(cd)))
        self._n_levels, self._coarse = nl.value, cd.value

    def __del__(self):
        try:
            load().cf_amg_destroy(self._h)
        except Exception:
            pass

    def n_levels(self):
        return self._n_levels

    def coarse_dim(self):
        return self._coarse

    def set_matrix_free(self, prob, constraints, mat, reg, phi_tilde):
        """Apply the finest level (a 3d u-block) matrix-free in the V-cycles (operator_kind 1)."""
        pt = _as_f64(phi_tilde)
        check(load().cf_amg_set_matrix_free(self._h, prob._h, constraints._h, C.byref(mat), C.byref(reg), _ptr(pt)))

    def v_cycle(self, r):
        r = _as_f64(r)
        x = _empty_like_kind(r, self.A.rows)
        check(load().cf_amg_vcycle(self._h, _ptr(r), _ptr(x)))
        return x

    def level_info(self, lev: int) -> dict:
        info = np.zeros(8, dtype=np.int64)
        lam, jw = C.c_double(), C.c_double()
        check(load().cf_amg_level_info(self._h, lev, _ptr(info), C.byref(lam), C.byref(jw)))
        keys = ("rows", "nnz_A", "nnz_P", "coarse", "n_nodes", "n_aggregates", "strong_edges", "lfmis_rounds")
        d = {k: int(v) for k, v in zip(keys, info)}
        d.update(lam=lam.value, jacobi_weight=jw.value)
        return d

    def aggregates(self, lev: int):
        n = self.level_info(lev)["n_nodes"]
        out = np.zeros(n, dtype=np.int32)
        check(load().cf_amg_level_aggregates(self._h, lev, _ptr(out)))
        return out

    def level_matrix(self, lev: int, which: int) -> Csr:
        info = self.level_info(lev)
        rows = info["rows"]
        nnz = info["nnz_A"] if which == 0 else info["nnz_P"]
        ptr = np.zeros(rows + 1, dtype=np.int64)
        col = np.zeros(nnz, dtype=np.int32)
        val = np.zeros(nnz)
        check(load().cf_amg_level_export(self._h, lev, which, _ptr(ptr), _ptr(col), _ptr(val)))
        return Csr(rows, rows if which == 0 else info["coarse"], ptr, col, val)


def build_amg(A: CsrMatrix, node_of_dof=None, near_nullspace=None, opts: AmgOptions | None = None) -> AmgHierarchy:
    """linsolve.hpp:90-94 (node_of_dof + near-nullspace) or the scalar overload (both None)."""
    return AmgHierarchy(A, node_of_dof, near_nullspace, opts)


PREC_KINDS = {"exact": 0, "amg": 1, "diagonal": 2}


def preconditioner_kind_from_string(s: str) -> int:
    """linsolve.cpp:345-350."""
    if s not in PREC_KINDS:
        raise ValueError(f"unknown preconditioner kind: {s}")
    return PREC_KINDS[s]


class BlockPreconditioner:
    """linsolve.hpp:106-128: diag(M_uu^-1, M_phiphi^-1) approximations, frozen at build."""

    def __init__(self, handle, n):
        self._h, self.n = handle, n

    @staticmethod
    def build(J: BlockSystem, kind=1, amg_opts: AmgOptions | None = None, prob: Problem | None = None,
              constraints: ConstraintSet | None = None):
        kind = preconditioner_kind_from_string(kind) if isinstance(kind, str) else int(kind)
        h = C.c_void_p()
        o = amg_opts or AmgOptions()
        check(load().cf_prec_build(J._h, kind, C.byref(o), prob._h if prob else None,
                                   constraints._h if constraints else None, C.byref(h)))
        return BlockPreconditioner(h, J.n_total())

    def __del__(self):
        try:
            load().cf_prec_destroy(self._h)
        except Exception:
            pass

    def apply(self, r):
        r = _as_f64(r)
        z = _empty_like_kind(r, self.n)
        check(load().cf_prec_apply(self._h, _ptr(r), _ptr(z)))
        return z


def rigid_body_modes(prob: Problem, constraints: ConstraintSet):
    """linsolve.cpp:320-343: n_u x m (m = 3 in 2d, 6 in 3d)."""
    m = 3 if prob.dim == 2 else 6
    B = np.zeros(m * prob.n_u)
    check(load().cf_rigid_body_modes(prob._h, constraints._h, _ptr(B)))
    return B.reshape(m, prob.n_u).T.copy()


def gmres(op, rhs, prec=None, opts: GmresOptions | None = None):
    """linsolve.hpp:48-49.  op: BlockSystem or CsrMatrix; prec: BlockPreconditioner, AmgHierarchy
    or None.  Returns dict(x, iterations, converged, breakdown, residual, residual_history)."""
    from ._lib import GmresResultC
    o = opts or GmresOptions()
    b = _as_f64(rhs)
    x = _empty_like_kind(b, len(b))
    res = GmresResultC()
    hist = np.zeros(max(1, o.max_iter))
    J = op._h if isinstance(op, BlockSystem) else None
    A = op._h if isinstance(op, CsrMatrix) else None
    P = prec._h if isinstance(prec, BlockPreconditioner) else None
    M = prec._h if isinstance(prec, AmgHierarchy) else None
    check(load().cf_gmres(J, A, P, M, _ptr(b), C.byref(o), _ptr(x), C.byref(res), _ptr(hist), len(hist)))
    return dict(x=x, iterations=res.iterations, converged=bool(res.converged), breakdown=bool(res.breakdown),
                residual=res.residual, residual_history=hist[:res.iterations].copy())


# ---------------------------------------------------------------------------- functionals
def compute_tcv(prob: Problem, solution) -> float:
    """postproc.cpp:12-28: signed total crack volume."""
    x = _as_f64(solution)
    out = C.c_double()
    check(load().cf_compute_tcv(prob._h, _ptr(x), C.byref(out)))
    return out.value


def default_cod_stations():
    """postproc.cpp:30-34: -1.5 .. 1.5 step 0.05 (61 stations)."""
    return [0.05 * i for i in range(-30, 31)]


def compute_cod(prob: Problem, solution, stations) -> np.ndarray:
    """postproc.cpp:70-99 (line-integral method): crack opening at each station."""
    x = _as_f64(solution)
    st = np.ascontiguousarray(stations, dtype=np.float64)
    out = np.zeros(len(st))
    check(load().cf_compute_cod(prob._h, _ptr(x), _ptr(st), len(st), _ptr(out)))
    return out


# ---------------------------------------------------------------------------- Newton / active set
def write_matrix_market(path: str, A) -> None:
    """linsolve.cpp:478-490 for a CsrMatrix (use BlockSystem.write_matrix_market for a block)."""
    check(load().cf_csr_write_matrix_market(A._h, str(path).encode()))


def write_vtk(path: str, prob: Problem, solution, phi_old=None, binary: bool = False) -> None:
    """postproc.cpp:111-167: legacy VTK of the solution (ASCII = the reference's text; binary = the
    same dataset in big-endian BINARY encoding)."""
    x = _as_f64(solution)
    po = _as_f64(phi_old) if phi_old is not None else None
    check(load().cf_write_vtk(prob._h, _ptr(x), _ptr(po), str(path).encode(), int(bool(binary))))


def slit_band_edge(prob: Problem, mat: Material) -> float:
    out = C.c_double()
    check(load().cf_slit_band_edge(prob._h, C.byref(mat), C.byref(out)))
    return out.value


def resolve_regularization(prob: Problem, mat: Material, band_edge: float) -> Regularization:
    reg = Regularization()
    check(load().cf_resolve_regularization(prob._h, C.byref(mat), float(band_edge), C.byref(reg)))
    return reg


def initial_crack(prob: Problem, mat: Material, band_half: float = 0.0):
    """model.cpp:324-349: (phi seed, band edge)."""
    phi = np.zeros(prob.n_vertices)
    be = C.c_double()
    check(load().cf_initial_crack(prob._h, C.byref(mat), float(band_half), _ptr(phi), C.byref(be)))
    return phi, be.value


class FractureState:
    """model.hpp:50-55 on the device: solution (u, phi), phi_old, phi_prev2, step."""

    def __init__(self, prob: Problem, solution=None, phi_old=None, phi_prev2=None, step=0, _handle=None):
        self.prob = prob
        if _handle is not None:
            self._h = _handle
        else:
            arrs = [None if a is None else _as_f64(a) for a in (solution, phi_old, phi_prev2)]
            self._h = C.c_void_p()
            check(load().cf_state_create(prob._h, *[_ptr(a) for a in arrs], int(step), C.byref(self._h)))

    def __del__(self):
        try:
            load().cf_state_destroy(self._h)
        except Exception:
            pass

    def get(self):
        p = self.prob
        sol, po, pp = np.zeros(p.n_total), np.zeros(p.n_vertices), np.zeros(p.n_vertices)
        step = C.c_int()
        check(load().cf_state_get(self._h, _ptr(sol), _ptr(po), _ptr(pp), C.byref(step)))
        return dict(solution=sol, phi_old=po, phi_prev2=pp, step=step.value)

    @property
    def solution(self):
        return self.get()["solution"]


def make_initial_state(prob: Problem, mat: Material, seed_band: float = 0.0) -> FractureState:
    """solver.cpp:24-35: u = 0, phi = phi_old = phi_prev2 = initial crack, step 0."""
    h = C.c_void_p()
    check(load().cf_make_initial_state(prob._h, C.byref(mat), float(seed_band), C.byref(h)))
    return FractureState(prob, _handle=h)


def _report(its, n, conv, feas, times=None):
    rows = [dict(residual_norm=its[i].residual_norm, active_size=its[i].active_size,
                 set_changes=its[i].set_changes, gmres_iterations=its[i].gmres_iterations) for i in range(n)]
    out = dict(iterations=rows, converged=bool(conv), feasibility_violation=float(feas))
    if times is not None:
        out["times_ms"] = dict(residual=times.residual_ms, active_set=times.active_set_ms,
                               jacobian=times.jacobian_ms, amg_setup=times.amg_setup_ms, gmres=times.gmres_ms,
                               total=times.total_ms)
    return out


def newton_active_set_step(state: FractureState, mat: Material, prob: Problem, reg: Regularization,
                           opts: SolverOptions | None = None, max_its: int = 256,
                           comm: Communicator | None = None) -> dict:
    """solver.cpp:49-188 (the state is updated in place on the device).

    comm: run this rank's slab of the decomposed step (every rank calls it with the same state)."""
    from ._lib import NewtonIterationC, PhaseTimesC
    o = opts or SolverOptions()
    its = (NewtonIterationC * max_its)()
    n, conv, feas, times = C.c_int(), C.c_int(), C.c_double(), PhaseTimesC()
    if comm is None:
        check(load().cf_newton_active_set_step(prob._h, state._h, C.byref(mat), C.byref(reg), C.byref(o), its,
                                               max_its, C.byref(n), C.byref(conv), C.byref(feas), C.byref(times)))
    else:
        check(load().cf_newton_active_set_step_comm(prob._h, state._h, C.byref(mat), C.byref(reg), C.byref(o),
                                                    comm._h, its, max_its, C.byref(n), C.byref(conv), C.byref(feas),
                                                    C.byref(times)))
    return _report(its, n.value, conv.value, feas.value, times)


def solve_loading_sequence(state: FractureState, mat: Material, prob: Problem, reg: Regularization,
                           opts: SolverOptions | None, n_steps: int, max_its: int = 1024,
                           comm: Communicator | None = None) -> list:
    """solver.cpp:190-204: list of per-step reports; stops after a non-converged step."""
    from ._lib import NewtonIterationC
    o = opts or SolverOptions()
    its = (NewtonIterationC * max_its)()
    n_its = (C.c_int * max(1, n_steps))()
    conv = (C.c_int * max(1, n_steps))()
    feas = (C.c_double * max(1, n_steps))()
    done = C.c_int()
    if comm is None:
        check(load().cf_solve_loading_sequence(prob._h, state._h, C.byref(mat), C.byref(reg), C.byref(o),
                                               int(n_steps), its, max_its, n_its, conv, feas, C.byref(done)))
    else:
        check(load().cf_solve_loading_sequence_comm(prob._h, state._h, C.byref(mat), C.byref(reg), C.byref(o),
                                                    comm._h, int(n_steps), its, max_its, n_its, conv, feas,
                                                    C.byref(done)))
    out, off = [], 0
    for s in range(done.value):
        k = n_its[s]
        sub = (type(its[0]) * max(1, k))(*[its[off + i] for i in range(k)])
        out.append(_report(sub, k, conv[s], feas[s]))
        off += k
    return out

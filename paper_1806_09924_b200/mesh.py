"""General (adaptive) meshes: the reference's Mesh / DofMap / adaptivity API
over the C ABI of include/crackfield_b200.h.  Names, argument meaning and error behaviour follow
/root/reference/proj/include/crackfield/{mesh,fem,model,solver,postproc,adapt}.hpp:

    mesh = create_mesh(dim=2, half_width=5.0, n0=10)          # mesh.cpp:18-34
    refine(mesh, [cell ids]); uniform_refine(mesh, 2)         # mesh.cpp:203-223 (2:1 closure)
    cs   = build_constraints(mesh, active_set={dof: value})   # fem.cpp:189-267 (hanging nodes)
    R    = assemble_residual(mesh, cs, mat, reg, x, pt)       # model.cpp:127-202
    st   = make_initial_state(mesh, mat)                      # solver.cpp:24-35
    rep  = newton_active_set_step(st, mat, mesh, reg, opts)   # solver.cpp:49-188
    recs = adaptive_cycle(mesh, st, mat, AdaptiveOptions(cycles=2))   # adapt.cpp:122-190

Everything per vertex / cell / dof runs on the device (DofMap, constraints, assembly plans, Newton
step, estimator, marking, transfer); the forest's refinement bookkeeping is host C++.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import (BlockSystem, FractureState, _ptr, _report)
from ._lib import (AdaptiveOptions, LevelRecordC, Material, Regularization, RefinementPolicy, SolverOptions, check,
                   load)

KUNIT = 1 << 16


class Mesh:
    """Adaptive forest + DofMap (mesh.hpp:52-119, fem.hpp:33-74), device resident."""

    def __init__(self, dim: int = 2, half_width: float = 20.0, n0: int = 8, _handle=None):
        self.dim, self.half_width, self.n0 = dim, float(half_width), n0
        if _handle is None:
            self._h = C.c_void_p()
            check(load().cf_mesh_create(dim, float(half_width), n0, C.byref(self._h)))
        else:
            self._h = _handle
        self._info()

    def _info(self):
        info = np.zeros(4, dtype=np.int64)
        hmin = C.c_double()
        check(load().cf_mesh_info(self._h, _ptr(info), C.byref(hmin)))
        self.n_cells, self.n_active, self.max_level, self.n_vertices = (int(v) for v in info)
        self.min_active_edge = hmin.value
        self.n_u, self.n_phi = self.dim * self.n_vertices, self.n_vertices
        self.n_total = self.n_u + self.n_phi

    def __del__(self):
        try:
            load().cf_mesh_destroy(self._h)
        except Exception:
            pass

    def copy(self) -> "Mesh":
        h = C.c_void_p()
        check(load().cf_mesh_copy(self._h, C.byref(h)))
        return Mesh(self.dim, self.half_width, self.n0, _handle=h)

    def level_edge(self, level: int) -> float:
        return 2.0 * self.half_width / (self.n0 * float(1 << level))

    def active_cells(self) -> np.ndarray:
        out = np.zeros(self.n_active, dtype=np.int32)
        check(load().cf_mesh_active_cells(self._h, _ptr(out)))
        return out

    def cells(self) -> dict:
        n = self.n_cells
        lev, par = np.zeros(n, dtype=np.int32), np.zeros(n, dtype=np.int32)
        act, anc = np.zeros(n, dtype=np.int8), np.zeros((n, 3), dtype=np.int64)
        check(load().cf_mesh_cells(self._h, _ptr(lev), _ptr(par), _ptr(act), _ptr(anc)))
        return dict(level=lev, parent=par, active=act.astype(bool), anchor=anc)

    def vertex_keys(self) -> np.ndarray:
        out = np.zeros(self.n_vertices, dtype=np.int64)
        check(load().cf_mesh_vertex_keys(self._h, _ptr(out)))
        return out

    def vertex_physical(self) -> np.ndarray:
        k = self.vertex_keys()
        c = np.stack([k & ((1 << 21) - 1), (k >> 21) & ((1 << 21) - 1), (k >> 42) & ((1 << 21) - 1)], 1)
        unit = 2.0 * self.half_width / (self.n0 * float(KUNIT))
        x = -self.half_width + c.astype(np.float64) * unit
        if self.dim == 2:
            x[:, 2] = 0.0
        return x

    def cell_vertices(self) -> np.ndarray:
        out = np.zeros((self.n_active, 1 << self.dim), dtype=np.int64)
        check(load().cf_mesh_cell_vertices(self._h, _ptr(out)))
        return out

    def faces(self) -> np.ndarray:
        """active_faces (mesh.cpp:225-259): rows (cell, axis, side, neighbor or -1, rel)."""
        n = C.c_int64()
        check(load().cf_mesh_faces(self._h, C.byref(n), None))
        out = np.zeros((n.value, 5), dtype=np.int32)
        check(load().cf_mesh_faces(self._h, C.byref(n), _ptr(out)))
        return out

    def find_active_cell(self, x) -> int:
        p = np.zeros(3)
        p[:len(x)] = x
        out = C.c_int32()
        check(load().cf_mesh_find_cell(self._h, _ptr(p), C.byref(out)))
        return out.value

    # DofMap accessors (fem.hpp:39-43)
    def u_dof(self, vertex: int, component: int) -> int:
        return vertex * self.dim + component

    def phi_dof(self, vertex: int) -> int:
        return self.n_u + vertex


def create_mesh(dim: int = 2, half_width: float = 20.0, n0: int = 8) -> Mesh:
    return Mesh(dim, half_width, n0)


def refine(mesh: Mesh, marked) -> None:
    ids = np.ascontiguousarray(marked, dtype=np.int32)
    check(load().cf_mesh_refine(mesh._h, _ptr(ids), len(ids)))
    mesh._info()


def uniform_refine(mesh: Mesh, times: int) -> None:
    check(load().cf_mesh_uniform_refine(mesh._h, int(times)))
    mesh._info()


class MeshConstraintSet:
    """ConstraintSet of a general mesh (fem.cpp:189-267): Dirichlet clamp, hanging vertices with
    closed lines, active set; device resident."""

    def __init__(self, mesh: Mesh, clamp: bool = True, active_set: dict | None = None):
        self.mesh = mesh
        active_set = active_set or {}
        dofs = np.fromiter(active_set.keys(), dtype=np.int64, count=len(active_set))
        vals = np.fromiter(active_set.values(), dtype=np.float64, count=len(active_set))
        self._h = C.c_void_p()
        check(load().cf_mesh_constraints_build(mesh._h, int(clamp), len(dofs), _ptr(dofs), _ptr(vals),
                                               C.byref(self._h)))

    def __del__(self):
        try:
            load().cf_constraints_destroy(self._h)
        except Exception:
            pass

    def lines(self):
        """The closed lines with entries: dofs, ptr, masters, weights, inhomogeneities (ascending dof)."""
        nl, ne = C.c_int64(), C.c_int64()
        check(load().cf_constraint_lines(self._h, C.byref(nl), C.byref(ne), None, None, None, None, None))
        dofs, ptr = np.zeros(nl.value, dtype=np.int64), np.zeros(nl.value + 1, dtype=np.int64)
        m, w, inh = np.zeros(ne.value, dtype=np.int64), np.zeros(ne.value), np.zeros(nl.value)
        check(load().cf_constraint_lines(self._h, C.byref(nl), C.byref(ne), _ptr(dofs), _ptr(ptr), _ptr(m), _ptr(w),
                                         _ptr(inh)))
        return dofs, ptr, m, w, inh

    def distribute(self, v):
        check(load().cf_constraints_distribute(self._h, _ptr(v), 0))
        return v

    def distribute_homogeneous(self, v):
        check(load().cf_constraints_distribute(self._h, _ptr(v), 1))
        return v


def build_constraints(mesh: Mesh, clamp_displacement_on_boundary: bool = True, active_set: dict | None = None):
    return MeshConstraintSet(mesh, clamp_displacement_on_boundary, active_set)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64) if not type(a).__module__.startswith("torch") else a


def assemble_residual(mesh: Mesh, cs: MeshConstraintSet, mat: Material, reg: Regularization, solution, phi_tilde):
    x, pt = _f64(solution), _f64(phi_tilde)
    R = np.zeros(mesh.n_total)
    check(load().cf_mesh_assemble_residual(mesh._h, cs._h, C.byref(mat), C.byref(reg), _ptr(x), _ptr(pt), _ptr(R)))
    return R


def assemble_jacobian(mesh: Mesh, cs: MeshConstraintSet, mat: Material, reg: Regularization, solution,
                      phi_tilde) -> BlockSystem:
    x, pt = _f64(solution), _f64(phi_tilde)
    h = C.c_void_p()
    check(load().cf_mesh_assemble_jacobian(mesh._h, cs._h, C.byref(mat), C.byref(reg), _ptr(x), _ptr(pt),
                                           C.byref(h)))
    return BlockSystem(h)


def rigid_body_modes(mesh: Mesh, cs: MeshConstraintSet) -> np.ndarray:
    m = 3 if mesh.dim == 2 else 6
    B = np.zeros((m, mesh.n_u))
    check(load().cf_mesh_rigid_body_modes(mesh._h, cs._h, _ptr(B)))
    return B.T.copy()


def slit_band_edge(mesh: Mesh, mat: Material) -> float:
    out = C.c_double()
    check(load().cf_mesh_slit_band_edge(mesh._h, C.byref(mat), C.byref(out)))
    return out.value


def resolve_regularization(mesh: Mesh, mat: Material, band_edge: float) -> Regularization:
    reg = Regularization()
    check(load().cf_mesh_resolve_regularization(mesh._h, C.byref(mat), float(band_edge), C.byref(reg)))
    return reg


def initial_crack(mesh: Mesh, mat: Material, band_half: float = 0.0):
    phi = np.zeros(mesh.n_vertices)
    be = C.c_double()
    check(load().cf_mesh_initial_crack(mesh._h, C.byref(mat), float(band_half), _ptr(phi), C.byref(be)))
    return phi, be.value


def make_initial_state(mesh: Mesh, mat: Material, seed_band: float = 0.0) -> FractureState:
    h = C.c_void_p()
    check(load().cf_mesh_make_initial_state(mesh._h, C.byref(mat), float(seed_band), C.byref(h)))
    return FractureState(mesh, _handle=h)


def state(mesh: Mesh, solution=None, phi_old=None, phi_prev2=None, step: int = 0) -> FractureState:
    arrs = [None if a is None else _f64(a) for a in (solution, phi_old, phi_prev2)]
    h = C.c_void_p()
    check(load().cf_mesh_state_create(mesh._h, *[_ptr(a) for a in arrs], int(step), C.byref(h)))
    return FractureState(mesh, _handle=h)


def newton_active_set_step(st: FractureState, mat: Material, mesh: Mesh, reg: Regularization,
                           opts: SolverOptions | None = None, max_its: int = 256) -> dict:
    from ._lib import NewtonIterationC, PhaseTimesC
    o = opts or SolverOptions()
    its = (NewtonIterationC * max_its)()
    n, conv, feas, times = C.c_int(), C.c_int(), C.c_double(), PhaseTimesC()
    check(load().cf_mesh_newton_active_set_step(mesh._h, st._h, C.byref(mat), C.byref(reg), C.byref(o), its,
                                                max_its, C.byref(n), C.byref(conv), C.byref(feas), C.byref(times)))
    return _report(its, n.value, conv.value, feas.value, times)


def solve_loading_sequence(st: FractureState, mat: Material, mesh: Mesh, reg: Regularization,
                           opts: SolverOptions | None, n_steps: int, max_its: int = 1024) -> list:
    from ._lib import NewtonIterationC
    o = opts or SolverOptions()
    its = (NewtonIterationC * max_its)()
    n_its = (C.c_int * max(1, n_steps))()
    conv = (C.c_int * max(1, n_steps))()
    feas = (C.c_double * max(1, n_steps))()
    done = C.c_int()
    check(load().cf_mesh_solve_loading_sequence(mesh._h, st._h, C.byref(mat), C.byref(reg), C.byref(o),
                                                int(n_steps), its, max_its, n_its, conv, feas, C.byref(done)))
    out, off = [], 0
    for s in range(done.value):
        k = n_its[s]
        sub = (type(its[0]) * max(1, k))(*[its[off + i] for i in range(k)])
        out.append(_report(sub, k, conv[s], feas[s]))
        off += k
    return out


def compute_tcv(mesh: Mesh, solution) -> float:
    x = _f64(solution)
    out = C.c_double()
    check(load().cf_mesh_compute_tcv(mesh._h, _ptr(x), C.byref(out)))
    return out.value


def compute_cod(mesh: Mesh, solution, stations) -> np.ndarray:
    x = _f64(solution)
    st = np.ascontiguousarray(stations, dtype=np.float64)
    out = np.zeros(len(st))
    check(load().cf_mesh_compute_cod(mesh._h, _ptr(x), _ptr(st), len(st), _ptr(out)))
    return out


def jump_estimator(mesh: Mesh, solution) -> np.ndarray:
    """adapt.cpp:16-55: eta per active cell (mesh.active_cells() order)."""
    x = _f64(solution)
    eta = np.zeros(mesh.n_active)
    check(load().cf_mesh_jump_estimator(mesh._h, _ptr(x), _ptr(eta)))
    return eta


def mark_cells(mesh: Mesh, solution, eta=None, policy: RefinementPolicy | None = None) -> np.ndarray:
    """adapt.cpp:57-97: marked active cell ids, ascending."""
    x = _f64(solution)
    e = None if eta is None else _f64(eta)
    pol = policy or RefinementPolicy()
    out = np.zeros(max(1, mesh.n_active), dtype=np.int32)
    n = C.c_int64()
    check(load().cf_mesh_mark_cells(mesh._h, _ptr(x), _ptr(e), C.byref(pol), _ptr(out), C.byref(n)))
    return out[:n.value].copy()


def transfer(old_mesh: Mesh, old_vec, new_mesh: Mesh) -> np.ndarray:
    """fem.cpp:318-333."""
    x = _f64(old_vec)
    out = np.zeros(new_mesh.n_total)
    check(load().cf_mesh_transfer(old_mesh._h, _ptr(x), new_mesh._h, _ptr(out)))
    return out


def adaptive_cycle(mesh: Mesh, st: FractureState, mat: Material, opts: AdaptiveOptions) -> list:
    """adapt.cpp:122-190: one record per solved level; the mesh is refined in place and the state
    replaced by the final level's."""
    recs = (LevelRecordC * max(1, opts.cycles + 1))()
    n = C.c_int()
    check(load().cf_mesh_adaptive_cycle(mesh._h, st._h, C.byref(mat), C.byref(opts), recs, opts.cycles + 1,
                                        C.byref(n)))
    mesh._info()
    return [dict(level=r.level, dofs=r.dofs, eps=r.eps, h_min=r.h_min, tcv=r.tcv, newton_iters=r.newton_iters,
                 gmres_mean=r.gmres_mean, converged=bool(r.converged)) for r in recs[:n.value]]

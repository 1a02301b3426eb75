"""Loader of libcrackfield_b200.so (the C ABI declared in include/crackfield_b200.h).

The library is built in-tree by __graft_entry__.build() (nvcc, sm_100a).  There is no
fallback: if the shared object is missing or no CUDA device is present, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcrackfield_b200.so")

CF_OK = 0
ERRORS = {1: ValueError, 2: RuntimeError, 3: RuntimeError, 4: RuntimeError, 5: MemoryError, 6: NotImplementedError,
          7: RuntimeError}


class CfError(RuntimeError):
    pass


class Material(C.Structure):
    """model.hpp:14-30 (eps_mode 0 = tied, 1 = fixed; pressure_coupling 0 = extrapolated)."""
    _fields_ = [("E", C.c_double), ("nu", C.c_double), ("G_c", C.c_double), ("pressure", C.c_double),
                ("l0", C.c_double), ("kappa_factor", C.c_double), ("eps_mode", C.c_int),
                ("c_eps", C.c_double), ("eps_fixed", C.c_double), ("pressure_coupling", C.c_int)]

    def __init__(self, **kw):
        d = dict(E=1.0, nu=0.2, G_c=1.0, pressure=1e-3, l0=1.0, kappa_factor=1e-12, eps_mode=0, c_eps=2.0,
                 eps_fixed=0.0625, pressure_coupling=0)
        d.update(kw)
        super().__init__(**d)

    def mu(self):
        return self.E / (2.0 * (1.0 + self.nu))

    def lam(self):
        return self.E * self.nu / ((1.0 + self.nu) * (1.0 - 2.0 * self.nu))


class Regularization(C.Structure):
    """model.hpp:38-41."""
    _fields_ = [("eps", C.c_double), ("kappa", C.c_double)]


class AmgOptions(C.Structure):
    """linsolve.hpp:51-60."""
    _fields_ = [("strength_threshold", C.c_double), ("prolongation_omega", C.c_double),
                ("jacobi_omega", C.c_double), ("smoothing_sweeps", C.c_int), ("coarse_size", C.c_int),
                ("max_levels", C.c_int), ("smoother", C.c_int), ("chebyshev_degree", C.c_int)]

    def __init__(self, **kw):
        # smoother 0: damped Jacobi (the reference); 1: Chebyshev (opt-in, outside the parity contract)
        d = dict(strength_threshold=0.02, prolongation_omega=2.0 / 3.0, jacobi_omega=2.0 / 3.0,
                 smoothing_sweeps=1, coarse_size=64, max_levels=25, smoother=0, chebyshev_degree=3)
        d.update(kw)
        super().__init__(**d)


class GmresOptions(C.Structure):
    """linsolve.hpp:32-36."""
    _fields_ = [("rtol", C.c_double), ("max_iter", C.c_int), ("restart", C.c_int)]

    def __init__(self, **kw):
        d = dict(rtol=1e-8, max_iter=1000, restart=100)
        d.update(kw)
        super().__init__(**d)


class RefinementPolicy(C.Structure):
    """adapt.hpp:12-20."""
    _fields_ = [("phi_threshold", C.c_double), ("h_target", C.c_double), ("theta", C.c_double),
                ("max_level", C.c_int), ("estimator", C.c_int)]

    def __init__(self, **kw):
        d = dict(phi_threshold=0.8, h_target=0.0, theta=0.3, max_level=16, estimator=1)
        d.update(kw)
        super().__init__(**d)


class SolverOptions(C.Structure):
    """solver.hpp:13-26 (prec_kind 0 exact, 1 amg, 2 diagonal)."""
    _fields_ = [("newton_tol", C.c_double), ("newton_abs_floor", C.c_double), ("newton_max_iter", C.c_int),
                ("active_set_c_scale", C.c_double), ("cycle_window", C.c_int), ("cycle_toggles", C.c_int),
                ("damping", C.c_int), ("prec_kind", C.c_int), ("freeze_preconditioner", C.c_int),
                ("log", C.c_int), ("gmres", GmresOptions), ("amg", AmgOptions), ("operator_kind", C.c_int)]

    def __init__(self, **kw):
        # operator_kind 1: matrix-free M_uu in the Krylov operator and the finest smoother (3d uniform,
        # one GPU); 0: the assembled operator, bitwise identical to the CPU oracle
        d = dict(newton_tol=1e-8, newton_abs_floor=1e-11, newton_max_iter=50, active_set_c_scale=100.0,
                 cycle_window=8, cycle_toggles=3, damping=0, prec_kind=1, freeze_preconditioner=0, log=0,
                 gmres=GmresOptions(), amg=AmgOptions(), operator_kind=1)
        d.update(kw)
        super().__init__(**d)


class AdaptiveOptions(C.Structure):
    """adapt.hpp:38-55 (cod_stations: compute_cod per level)."""
    _fields_ = [("policy", RefinementPolicy), ("solver", SolverOptions), ("cycles", C.c_int), ("n_steps", C.c_int),
                ("halve_band_target", C.c_int), ("estimator_rounds", C.c_int), ("seed_band", C.c_double)]

    def __init__(self, **kw):
        d = dict(policy=RefinementPolicy(), solver=SolverOptions(), cycles=0, n_steps=1, halve_band_target=1,
                 estimator_rounds=1, seed_band=0.0)
        d.update(kw)
        super().__init__(**d)


class LevelRecordC(C.Structure):
    _fields_ = [("level", C.c_int), ("dofs", C.c_int64), ("eps", C.c_double), ("h_min", C.c_double),
                ("tcv", C.c_double), ("newton_iters", C.c_int), ("gmres_mean", C.c_double), ("converged", C.c_int)]


_lib = None

# (name, restype, argtypes); the not-gpu test checks every symbol of include/crackfield_b200.h is here
_P = C.c_void_p
_D = C.c_double
_I = C.c_int
_L = C.c_int64
_PD = C.POINTER(C.c_double)
SIGNATURES = [
    ("cf_last_error", C.c_char_p, []),
    ("cf_version", _I, []),
    ("cf_device_info", _I, [C.POINTER(_I), C.POINTER(_I), C.POINTER(_L)]),
    ("cf_set_stream", _I, [_P]),
    ("cf_synchronize", _I, []),
    ("cf_kernel_launches", _L, []),
    ("cf_problem_create_uniform", _I, [_I, _D, _I, _I, C.POINTER(_P)]),
    ("cf_problem_destroy", _I, [_P]),
    ("cf_problem_info", _I, [_P, C.POINTER(_L), C.POINTER(_L), C.POINTER(_D)]),
    ("cf_constraints_build", _I, [_P, _I, _L, _P, _P, C.POINTER(_P)]),
    ("cf_constraints_destroy", _I, [_P]),
    ("cf_constraints_distribute", _I, [_P, _P, _I]),
    ("cf_assemble_residual", _I, [_P, _P, C.POINTER(Material), C.POINTER(Regularization), _P, _P, _P]),
    ("cf_assemble_jacobian", _I, [_P, _P, C.POINTER(Material), C.POINTER(Regularization), _P, _P, C.POINTER(_P)]),
    ("cf_assemble_residual_planes", _I, [_P, _P, C.POINTER(Material), C.POINTER(Regularization), _P, _P, _L, _L,
                                         _P]),
    ("cf_assemble_jacobian_planes", _I, [_P, _P, C.POINTER(Material), C.POINTER(Regularization), _P, _P, _L, _L,
                                         C.POINTER(_P)]),
    ("cf_slab_info", _I, [_P, _I, _I, _P]),
    ("cf_assemble_pattern", _I, [_P, _P, C.POINTER(_P)]),
    ("cf_mf_apply_uu", _I, [_P, _P, C.POINTER(Material), C.POINTER(Regularization), _P, _P, _P]),
    ("cf_fp64_peak", _I, [C.POINTER(_D)]),
    ("cf_sigma", _I, [_P, C.POINTER(Material), _I, _P]),
    ("cf_q1_shape", _I, [_I, _P, _P, _P]),
    ("cf_detect_cycles", _I, [_I, _P, _P, _P, _I, _I, _P, C.POINTER(_I)]),
    ("cf_extrapolate_phi", _I, [_P, _P]),
    ("cf_block_shape", _I, [_P, _P]),
    ("cf_block_format", _I, [_P, _I, C.POINTER(_I)]),
    ("cf_block_info", _I, [_P, C.POINTER(_L), C.POINTER(_L), C.POINTER(_L)]),
    ("cf_block_export", _I, [_P, _I, _P, _P, _P]),
    ("cf_block_apply", _I, [_P, _P, _P]),
    ("cf_block_spmv", _I, [_P, _I, _P, _P]),
    ("cf_block_destroy", _I, [_P]),
    ("cf_tune_spmv", _I, [_P, _I, _I, _I, _P, _P]),
    ("cf_tune_level_spmv", _I, [_P, _I, _I, _I, _I, _P, _P]),
    ("cf_test_div_by", _I, [C.c_double, _P, C.c_int64, _P]),
    ("cf_csr_create", _I, [_L, _L, _P, _P, _P, C.POINTER(_P)]),
    ("cf_block_csr", _I, [_P, _I, C.POINTER(_P)]),
    ("cf_csr_info", _I, [_P, C.POINTER(_L), C.POINTER(_L), C.POINTER(_L)]),
    ("cf_csr_export", _I, [_P, _P, _P, _P]),
    ("cf_csr_spgemm", _I, [_P, _P, _P, C.POINTER(_P)]),
    ("cf_csr_spmv", _I, [_P, _P, _P]),
    ("cf_csr_destroy", _I, [_P]),
    ("cf_amg_build", _I, [_P, _P, _P, _I, C.POINTER(AmgOptions), C.POINTER(_P)]),
    ("cf_amg_vcycle", _I, [_P, _P, _P]),
    ("cf_amg_info", _I, [_P, C.POINTER(_I), C.POINTER(_L)]),
    ("cf_amg_level_info", _I, [_P, _I, _P, C.POINTER(_D), C.POINTER(_D)]),
    ("cf_amg_level_aggregates", _I, [_P, _I, _P]),
    ("cf_amg_level_export", _I, [_P, _I, _I, _P, _P, _P]),
    ("cf_amg_destroy", _I, [_P]),
    ("cf_amg_set_matrix_free", _I, [_P, _P, _P, C.POINTER(Material), C.POINTER(Regularization), _P]),
    ("cf_prec_build", _I, [_P, _I, C.POINTER(AmgOptions), _P, _P, C.POINTER(_P)]),
    ("cf_prec_apply", _I, [_P, _P, _P]),
    ("cf_prec_destroy", _I, [_P]),
    ("cf_rigid_body_modes", _I, [_P, _P, _P]),
    ("cf_gmres", _I, [_P, _P, _P, _P, _P, C.POINTER(GmresOptions), _P, _P, _P, _I]),
    ("cf_compute_tcv", _I, [_P, _P, C.POINTER(_D)]),
    ("cf_compute_cod", _I, [_P, _P, _P, _I, _P]),
    ("cf_slit_band_edge", _I, [_P, C.POINTER(Material), C.POINTER(_D)]),
    ("cf_resolve_regularization", _I, [_P, C.POINTER(Material), _D, C.POINTER(Regularization)]),
    ("cf_initial_crack", _I, [_P, C.POINTER(Material), _D, _P, C.POINTER(_D)]),
    ("cf_make_initial_state", _I, [_P, C.POINTER(Material), _D, C.POINTER(_P)]),
    ("cf_state_create", _I, [_P, _P, _P, _P, _I, C.POINTER(_P)]),
    ("cf_state_get", _I, [_P, _P, _P, _P, C.POINTER(_I)]),
    ("cf_state_destroy", _I, [_P]),
    ("cf_newton_active_set_step", _I, [_P, _P, C.POINTER(Material), C.POINTER(Regularization),
                                       C.POINTER(SolverOptions), _P, _I, C.POINTER(_I), C.POINTER(_I),
                                       C.POINTER(_D), _P]),
    ("cf_solve_loading_sequence", _I, [_P, _P, C.POINTER(Material), C.POINTER(Regularization),
                                       C.POINTER(SolverOptions), _I, _P, _I, _P, _P, _P, C.POINTER(_I)]),
    ("cf_block_write_matrix_market", _I, [_P, _I, C.c_char_p]),
    ("cf_csr_write_matrix_market", _I, [_P, C.c_char_p]),
    ("cf_write_vtk", _I, [_P, _P, _P, C.c_char_p, _I]),
    ("cf_mesh_create", _I, [_I, _D, _I, C.POINTER(_P)]),
    ("cf_mesh_copy", _I, [_P, C.POINTER(_P)]),
    ("cf_mesh_destroy", _I, [_P]),
    ("cf_mesh_refine", _I, [_P, _P, _L]),
    ("cf_mesh_uniform_refine", _I, [_P, _I]),
    ("cf_mesh_info", _I, [_P, _P, C.POINTER(_D)]),
    ("cf_mesh_active_cells", _I, [_P, _P]),
    ("cf_mesh_cells", _I, [_P, _P, _P, _P, _P]),
    ("cf_mesh_vertex_keys", _I, [_P, _P]),
    ("cf_mesh_cell_vertices", _I, [_P, _P]),
    ("cf_mesh_faces", _I, [_P, C.POINTER(_L), _P]),
    ("cf_mesh_find_cell", _I, [_P, _P, C.POINTER(C.c_int32)]),
    ("cf_mesh_constraints_build", _I, [_P, _I, _L, _P, _P, C.POINTER(_P)]),
    ("cf_constraint_lines", _I, [_P, C.POINTER(_L), C.POINTER(_L), _P, _P, _P, _P, _P]),
    ("cf_mesh_assemble_residual", _I, [_P, _P, C.POINTER(Material), C.POINTER(Regularization), _P, _P, _P]),
    ("cf_mesh_assemble_jacobian", _I, [_P, _P, C.POINTER(Material), C.POINTER(Regularization), _P, _P,
                                       C.POINTER(_P)]),
    ("cf_mesh_rigid_body_modes", _I, [_P, _P, _P]),
    ("cf_mesh_slit_band_edge", _I, [_P, C.POINTER(Material), C.POINTER(_D)]),
    ("cf_mesh_resolve_regularization", _I, [_P, C.POINTER(Material), _D, C.POINTER(Regularization)]),
    ("cf_mesh_initial_crack", _I, [_P, C.POINTER(Material), _D, _P, C.POINTER(_D)]),
    ("cf_mesh_make_initial_state", _I, [_P, C.POINTER(Material), _D, C.POINTER(_P)]),
    ("cf_mesh_state_create", _I, [_P, _P, _P, _P, _I, C.POINTER(_P)]),
    ("cf_mesh_newton_active_set_step", _I, [_P, _P, C.POINTER(Material), C.POINTER(Regularization),
                                            C.POINTER(SolverOptions), _P, _I, C.POINTER(_I), C.POINTER(_I),
                                            C.POINTER(_D), _P]),
    ("cf_mesh_solve_loading_sequence", _I, [_P, _P, C.POINTER(Material), C.POINTER(Regularization),
                                            C.POINTER(SolverOptions), _I, _P, _I, _P, _P, _P, C.POINTER(_I)]),
    ("cf_mesh_compute_tcv", _I, [_P, _P, C.POINTER(_D)]),
    ("cf_mesh_compute_cod", _I, [_P, _P, _P, _I, _P]),
    ("cf_mesh_jump_estimator", _I, [_P, _P, _P]),
    ("cf_mesh_mark_cells", _I, [_P, _P, _P, C.POINTER(RefinementPolicy), _P, C.POINTER(_L)]),
    ("cf_mesh_transfer", _I, [_P, _P, _P, _P]),
    ("cf_mesh_adaptive_cycle", _I, [_P, _P, C.POINTER(Material), C.POINTER(AdaptiveOptions), _P, _I,
                                    C.POINTER(_I)]),
    ("cf_comm_unique_id", _I, [_P]),
    ("cf_comm_create", _I, [_P, _I, _I, C.POINTER(_P)]),
    ("cf_comm_create_host", _I, [_I, _I, _P, C.POINTER(_P)]),
    ("cf_comm_info", _I, [_P, C.POINTER(_I), C.POINTER(_I)]),
    ("cf_comm_selftest", _I, [C.POINTER(_I)]),
    ("cf_comm_destroy", _I, [_P]),
    ("cf_newton_active_set_step_comm", _I, [_P, _P, C.POINTER(Material), C.POINTER(Regularization),
                                            C.POINTER(SolverOptions), _P, _P, _I, C.POINTER(_I), C.POINTER(_I),
                                            C.POINTER(_D), _P]),
    ("cf_solve_loading_sequence_comm", _I, [_P, _P, C.POINTER(Material), C.POINTER(Regularization),
                                            C.POINTER(SolverOptions), _P, _I, _P, _I, _P, _P, _P, C.POINTER(_I)]),
]


AllgatherF64 = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int)
AllreduceI64 = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_longlong), C.c_int, C.c_int)
SendRecv = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                       C.POINTER(C.c_size_t), C.POINTER(C.c_int))
Bcast = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int)


class HostTransport(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("allgather_f64", AllgatherF64), ("allreduce_i64", AllreduceI64),
                ("sendrecv", SendRecv), ("bcast", Bcast)]


class GmresResultC(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("breakdown", C.c_int), ("residual", C.c_double)]


class NewtonIterationC(C.Structure):
    _fields_ = [("residual_norm", C.c_double), ("active_size", C.c_int), ("set_changes", C.c_int),
                ("gmres_iterations", C.c_int)]


class PhaseTimesC(C.Structure):
    _fields_ = [("residual_ms", C.c_double), ("active_set_ms", C.c_double), ("jacobian_ms", C.c_double),
                ("amg_setup_ms", C.c_double), ("gmres_ms", C.c_double), ("total_ms", C.c_double)]


def load(path: str | None = None):
    """Load the library and bind the C ABI.  Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("CF_LIB_PATH") or LIB_PATH  # CF_LIB_PATH: A/B builds of the same ABI
    if not os.path.exists(path):
        raise ImportError(f"crackfield_b200: {path} is missing; run __graft_entry__.build() "
                          "(there is no CPU fallback)")
    L = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(rc: int):
    if rc != CF_OK:
        msg = load().cf_last_error().decode()
        raise ERRORS.get(rc, CfError)(msg)

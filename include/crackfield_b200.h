/*
 * crackfield_b200 — C ABI of the B200-native Newton/active-set hot path of the
 * pressurized phase-field fracture solver (arXiv 1806.09924; reference: /root/reference/proj).
 *
 * Every entry point replaces one reference C++ interface on the hot path; the
 * citation on each declaration names it.  Conventions:
 *   - every function returns an int status (CF_OK = 0, else a CF_ERR_* code); a C++
 *     exception never crosses the ABI; cf_last_error() returns the message of the last
 *     failure on the calling thread (the reference's exception text where one exists);
 *   - handles are opaque, owned by the caller and released with the matching *_destroy;
 *   - array arguments are borrowed for the duration of the call and may be HOST or DEVICE
 *     pointers (detected with cudaPointerGetAttributes): host arrays are staged through
 *     device memory and the call is synchronous; with device arrays the call is ordered on
 *     the library stream (cf_set_stream) and returns without a host synchronisation;
 *   - all floating-point data are IEEE double (FP64), matching types.hpp:9-13; row pointers
 *     are int64 (the reference's int32 StorageIndex cannot index config 4), column indices int32;
 *   - calls are serialised per process (not thread-safe per handle), like the reference.
 * There is no CPU fallback: without a usable CUDA device every compute call fails with
 * CF_ERR_CUDA.
 */
#ifndef CRACKFIELD_B200_H
#define CRACKFIELD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CF_OK 0
#define CF_ERR_INVALID_ARGUMENT 1 /* std::invalid_argument in the reference */
#define CF_ERR_NUMERICAL 2        /* std::runtime_error (singular coarse LU, GMRES stagnation) */
#define CF_ERR_LOGIC 3            /* std::logic_error */
#define CF_ERR_CUDA 4             /* CUDA runtime / no device */
#define CF_ERR_OUT_OF_MEMORY 5
#define CF_ERR_UNSUPPORTED 6

/* Material (model.hpp:14-30). eps_mode: 0 tied, 1 fixed; pressure_coupling: 0 extrapolated, 1 current. */
typedef struct {
  double E, nu, G_c, pressure, l0, kappa_factor;
  int eps_mode;
  double c_eps, eps_fixed;
  int pressure_coupling;
} cf_material;

/* Regularization (model.hpp:38-41). */
typedef struct {
  double eps, kappa;
} cf_regularization;

/* AmgOptions (linsolve.hpp:51-60). */
typedef struct {
  double strength_threshold, prolongation_omega, jacobi_omega;
  int smoothing_sweeps, coarse_size, max_levels;
} cf_amg_options;

/* GmresOptions (linsolve.hpp:32-36). */
typedef struct {
  double rtol;
  int max_iter, restart;
} cf_gmres_options;

/* SolverOptions (solver.hpp:13-26). prec_kind: 0 exact, 1 amg, 2 diagonal (linsolve.hpp:100). */
typedef struct {
  double newton_tol, newton_abs_floor;
  int newton_max_iter;
  double active_set_c_scale;
  int cycle_window, cycle_toggles, damping, prec_kind, freeze_preconditioner, log;
  cf_gmres_options gmres;
  cf_amg_options amg;
} cf_solver_options;

typedef struct cf_problem_s* cf_problem;         /* Mesh + DofMap of a uniform grid */
typedef struct cf_constraints_s* cf_constraints; /* ConstraintSet */
typedef struct cf_block_s* cf_block;             /* BlockSystem (three CSR blocks) */

/* ------------------------------------------------------------------ runtime */
const char* cf_last_error(void);
int cf_version(void);
/* Device ordinal, SM count and global memory of the current device. */
int cf_device_info(int* device, int* sm_count, int64_t* total_mem);
/* Stream for all subsequent device work (a cudaStream_t; NULL = legacy default stream). */
int cf_set_stream(void* stream);
int cf_synchronize(void);
/* Number of kernels this library has launched since load (gpu_launches accounting). */
int64_t cf_kernel_launches(void);

/* ------------------------------------------------------------------ problem / dof map */
/* create_mesh(DomainSpec{dim, half_width, n0}) + uniform_refine(refinements) + build_dof_map
 * (mesh.cpp:18-34, 209-215; fem.cpp:98-116).  Vertices are numbered lexicographically
 * (x fastest), u dofs interleaved (v*d+c), phi dofs after all u dofs (fem.hpp:35-43). */
int cf_problem_create_uniform(int dim, double half_width, int n0, int refinements, cf_problem* out);
int cf_problem_destroy(cf_problem p);
int cf_problem_info(cf_problem p, int64_t* n_vertices, int64_t* n_cells, double* h);

/* ------------------------------------------------------------------ constraints */
/* build_constraints(mesh, map, DirichletSpec{clamp_boundary}, active_set) (fem.cpp:205-267):
 * Dirichlet u = 0 on boundary vertices, then phi dof = value for each active entry
 * (Dirichlet wins).  Uniform meshes have no hanging vertices. */
int cf_constraints_build(cf_problem p, int clamp_boundary, int64_t n_active, const int64_t* active_dofs,
                         const double* active_values, cf_constraints* out);
int cf_constraints_destroy(cf_constraints c);
/* ConstraintSet::distribute / distribute_homogeneous (fem.cpp:189-203), in place on v (length n_total). */
int cf_constraints_distribute(cf_constraints c, double* v, int homogeneous);

/* ------------------------------------------------------------------ assembly */
/* assemble_residual (model.hpp:62-64, model.cpp:127-202): R (length n_total), condensed. */
int cf_assemble_residual(cf_problem p, cf_constraints c, const cf_material* mat, const cf_regularization* reg,
                         const double* solution, const double* phi_tilde, double* R);
/* assemble_jacobian (model.hpp:68-70, model.cpp:204-322): new BlockSystem handle. */
int cf_assemble_jacobian(cf_problem p, cf_constraints c, const cf_material* mat, const cf_regularization* reg,
                         const double* solution, const double* phi_tilde, cf_block* out);

/* ------------------------------------------------------------------ block system */
/* Sizes: n_u, n_phi and nnz of M_uu, M_phiu, M_phiphi (linsolve.hpp:17-28). */
int cf_block_info(cf_block b, int64_t* n_u, int64_t* n_phi, int64_t* nnz3);
/* Copy one block out as CSR (which: 0 M_uu, 1 M_phiu, 2 M_phiphi). */
int cf_block_export(cf_block b, int which, int64_t* rowptr, int32_t* col, double* val);
/* BlockSystem::apply (linsolve.cpp:13-19): y = J x. */
int cf_block_apply(cf_block b, const double* x, double* y);
/* One block times a vector (the M_uu operator microbenchmark, config 1). */
int cf_block_spmv(cf_block b, int which, const double* x, double* y);
int cf_block_destroy(cf_block b);

#ifdef __cplusplus
}
#endif

#endif /* CRACKFIELD_B200_H */

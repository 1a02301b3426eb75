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
#define CF_ERR_COMM 7             /* NCCL (multi-GPU communicator) */

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

/* AmgOptions (linsolve.hpp:51-60).  smoother: 0 = damped Jacobi, the reference's smoother
 * (linsolve.cpp:301-311); 1 = Chebyshev of degree chebyshev_degree (3 recommended) on D^-1 A over
 * [g / 10, g], g the Gershgorin bound of D^-1 A (the north star's "Jacobi/Chebyshev smoothing";
 * opt-in, no reference counterpart, so not part of the parity contract; smoothing_sweeps
 * applications per visit; with it the V-cycle is not row-split over ranks but replicated). */
typedef struct {
  double strength_threshold, prolongation_omega, jacobi_omega;
  int smoothing_sweeps, coarse_size, max_levels;
  int smoother, chebyshev_degree;
} cf_amg_options;

/* GmresOptions (linsolve.hpp:32-36). */
typedef struct {
  double rtol;
  int max_iter, restart;
} cf_gmres_options;

/* SolverOptions (solver.hpp:13-26). prec_kind: 0 exact, 1 amg, 2 diagonal (linsolve.hpp:100).
 * operator_kind (no reference counterpart): 1 (default) applies M_uu matrix-free (sum-factorised,
 * 3d uniform grids on one GPU) in the Krylov operator and in the u-hierarchy's finest-level
 * smoother / residual; 0 applies the assembled M_uu everywhere (the reference's operator, and
 * the mode that is bitwise identical to the CPU oracle).  Both agree to rounding (north-star
 * tolerances, tests/test_gpu_mf_solver.py). */
typedef struct {
  double newton_tol, newton_abs_floor;
  int newton_max_iter;
  double active_set_c_scale;
  int cycle_window, cycle_toggles, damping, prec_kind, freeze_preconditioner, log;
  cf_gmres_options gmres;
  cf_amg_options amg;
  int operator_kind;
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

/* Matrix-free M_uu apply (BASELINE config 1's "matrix-free equivalent"): y_u = M_uu x_u computed
 * cell by cell from phi_tilde, without the assembled matrix (the assembled block's Dirichlet
 * condensation included).  Equal to cf_block_spmv(M_uu) to rounding (not bitwise).  x, y: n_u. */
int cf_mf_apply_uu(cf_problem p, cf_constraints c, const cf_material* mat, const cf_regularization* reg,
                   const double* phi_tilde, const double* x, double* y);
/* FP64 FMA throughput of the device (TFLOP/s, a DFMA loop), the roofline of the matrix-free apply. */
int cf_fp64_peak(double* tflops);

/* Host helpers of the model (no device needed): sigma (model.cpp:19-26; grad_u and out row-major
 * 3x3), q1_shape (fem.cpp:76-96; values[2^d], grads[2^d x d] row-major), detect_cycles
 * (solver.cpp:10-22; the histories of n dofs as one byte array with offsets[n+1]; out receives the
 * cycling dofs ascending, *n_out their count). */
int cf_sigma(const double grad_u[9], const cf_material* mat, int d, double out[9]);
int cf_q1_shape(int d, const double xi[3], double* values, double* grads);
int cf_detect_cycles(int n, const int32_t* dofs, const int64_t* offsets, const uint8_t* bits, int window,
                     int toggles, int32_t* out, int* n_out);

/* assemble_pattern (linsolve.hpp:138, linsolve.cpp:417-476): the BlockSparsity after condensation as
 * a block handle whose values are 0 (constrained dofs keep their diagonal, unlike the Jacobian,
 * which drops a constrained diagonal that sums to 0). */
int cf_assemble_pattern(cf_problem p, cf_constraints c, cf_block* out);

/* Slab decomposition (no reference counterpart: the reference is single-threaded).
 * A slab owns vertex planes [p_lo, p_hi) along the slowest axis (z in 3d, y in 2d) = a
 * contiguous vertex range.  Its residual rows come back in the local layout
 * [u_own (d*nv) | phi_own (nv)]; its Jacobian rows are the owned rows with columns numbered
 * over the owned + one ghost plane each side ("ext" layout [u_ext (d*ne) | phi_ext (ne)]).
 * x / phi_tilde are global-length and must be valid on the ext planes.  The full slab
 * [0, n_planes) reproduces cf_assemble_residual / cf_assemble_jacobian exactly. */
int cf_assemble_residual_planes(cf_problem p, cf_constraints c, const cf_material* mat, const cf_regularization* reg,
                                const double* solution, const double* phi_tilde, int64_t p_lo, int64_t p_hi,
                                double* R);
int cf_assemble_jacobian_planes(cf_problem p, cf_constraints c, const cf_material* mat, const cf_regularization* reg,
                                const double* solution, const double* phi_tilde, int64_t p_lo, int64_t p_hi,
                                cf_block* out);
/* The slab of rank `rank` of `size` (planes split evenly): {v_lo, v_hi, ve_lo, ve_hi, c_lo, c_hi,
 * vertices per plane}. */
int cf_slab_info(cf_problem p, int rank, int size, int64_t info[7]);

/* ------------------------------------------------------------------ block system */
/* {n_u rows, n_phi rows, n_u input columns, n_phi input columns} (inputs > rows for a slab). */
int cf_block_shape(cf_block b, int64_t shape[4]);
/* Storage format the SpMV of one block streams (which: 0 M_uu, 1 M_phiu, 2 M_phiphi): 0 CSR
 * (8 B value + 4 B column per entry), 1 stencil-implicit columns (values only; the columns of a
 * row follow from its vertex, verified against the stored CSR columns at assembly). */
int cf_block_format(cf_block b, int which, int* format);
/* Sizes: n_u, n_phi and nnz of M_uu, M_phiu, M_phiphi (linsolve.hpp:17-28). */
int cf_block_info(cf_block b, int64_t* n_u, int64_t* n_phi, int64_t* nnz3);
/* Copy one block out as CSR (which: 0 M_uu, 1 M_phiu, 2 M_phiphi). */
int cf_block_export(cf_block b, int which, int64_t* rowptr, int32_t* col, double* val);
/* BlockSystem::apply (linsolve.cpp:13-19): y = J x. */
int cf_block_apply(cf_block b, const double* x, double* y);
/* One block times a vector (the M_uu operator microbenchmark, config 1). */
int cf_block_spmv(cf_block b, int which, const double* x, double* y);
int cf_block_destroy(cf_block b);
/* Tuning hook (not a reference interface): one block times a vector with an explicit kernel
 * variant (threads per row in {4,8,16,32}; unroll 0 = plain loop, else batched loads). */
int cf_tune_spmv(cf_block b, int which, int threads_per_row, int unroll, const double* x, double* y);
/* Test hook (not a reference interface): q[i] = a[i] / h through the residual kernel's division by
 * the cell size (reciprocal + two Markstein corrections); must equal the IEEE quotient bit for bit. */
int cf_test_div_by(double h, const double* a, int64_t n, double* q);

/* ------------------------------------------------------------------ generic CSR operators */
typedef struct cf_csr_s* cf_csr;   /* CsrMatrix (types.hpp:12) on the device */
typedef struct cf_amg_s* cf_amg;   /* AmgHierarchy (linsolve.hpp:64-85) */
typedef struct cf_prec_s* cf_prec; /* BlockPreconditioner (linsolve.hpp:106-128) */

int cf_csr_create(int64_t rows, int64_t cols, const int64_t* rowptr, const int32_t* col, const double* val,
                  cf_csr* out);
/* A block of a BlockSystem as a shared CSR handle (which: 0 M_uu, 1 M_phiu, 2 M_phiphi). */
int cf_block_csr(cf_block b, int which, cf_csr* out);
int cf_csr_info(cf_csr A, int64_t* rows, int64_t* cols, int64_t* nnz);
int cf_csr_spmv(cf_csr A, const double* x, double* y);
/* The CSR arrays of A (rowptr: rows + 1; col, val: nnz), host or device pointers. */
int cf_csr_export(cf_csr A, int64_t* rowptr, int32_t* col, double* val);
/* C = diag(row_scale) A B (row_scale may be NULL): Eigen's sparse x sparse product as the AMG setup
 * uses it (linsolve.cpp:248-263: D^-1 A T, A P, P^T (A P)); sorted columns, structural zeros kept,
 * every entry the k-ascending sequential sum (any output row length). */
int cf_csr_spgemm(cf_csr A, cf_csr B, const double* row_scale, cf_csr* out);
int cf_csr_destroy(cf_csr A);

/* ------------------------------------------------------------------ AMG */
/* build_amg(A, node_of_dof, near_nullspace) (linsolve.hpp:90-94, linsolve.cpp:170-287).
 * node_of_dof (length rows) and B (rows x m, column-major) may both be NULL: the scalar overload
 * (identity nodes, constant nullspace, linsolve.cpp:289-293). */
int cf_amg_build(cf_csr A, const int32_t* node_of_dof, const double* B, int m, const cf_amg_options* opts,
                 cf_amg* out);
/* AmgHierarchy::v_cycle (linsolve.cpp:314-318): x = V(r). */
int cf_amg_vcycle(cf_amg h, const double* r, double* x);
/* n_levels() and coarse_dim() (linsolve.hpp:67-68). */
int cf_amg_info(cf_amg h, int* n_levels, int64_t* coarse_dim);
/* the hierarchy's finest level applied matrix-free in its V-cycles (residual, smoothing), as in the
 * Newton step with operator_kind 1: h must be a u-block hierarchy of the 3d problem p */
int cf_amg_set_matrix_free(cf_amg h, cf_problem p, cf_constraints c, const cf_material* mat,
                           const cf_regularization* reg, const double* phi_tilde);
/* Diagnostics of one non-coarsest level: info8 = {rows(A), nnz(A), nnz(P), cols(P), n_nodes,
 * n_aggregates, strong edges, LFMIS rounds}; lambda_max and the Jacobi weight. */
int cf_amg_level_info(cf_amg h, int level, int64_t* info8, double* lambda, double* jacobi_weight);
int cf_amg_level_aggregates(cf_amg h, int level, int32_t* agg_of_node);
/* Level operator (which 0: A, 1: P) as CSR. */
int cf_amg_level_export(cf_amg h, int level, int which, int64_t* rowptr, int32_t* col, double* val);
/* Tuning hook (not a reference interface): y = M x for a level operator (which 0: A, 1: P,
 * 2: R = P^T) with an explicit kernel variant as in cf_tune_spmv (unroll 200 + U: the persistent
 * pointer-prefetching kernel); threads_per_row 0 takes the production dispatch. */
int cf_tune_level_spmv(cf_amg h, int level, int which, int threads_per_row, int unroll, const double* x, double* y);
int cf_amg_destroy(cf_amg h);

/* ------------------------------------------------------------------ block preconditioner */
/* BlockPreconditioner::build (linsolve.cpp:352-396).  kind 0 exact (dense LU, small blocks
 * only), 1 amg, 2 diagonal.  With problem/constraints given, the AMG gets the reference's
 * NullspaceInfo (rigid-body modes zeroed on constrained u dofs, phi ones zeroed on constrained
 * phi dofs, vertex nodes; solver.cpp:142-150); with NULL, the scalar overload. */
int cf_prec_build(cf_block J, int kind, const cf_amg_options* opts, cf_problem p, cf_constraints c, cf_prec* out);
int cf_prec_apply(cf_prec P, const double* r, double* z);  /* linsolve.cpp:398-415 */
int cf_prec_destroy(cf_prec P);
/* rigid_body_modes (linsolve.cpp:320-343): B (n_u x m, column-major), m = 3 (2d) / 6 (3d). */
int cf_rigid_body_modes(cf_problem p, cf_constraints c, double* B);

/* ------------------------------------------------------------------ GMRES */
typedef struct {
  int iterations, converged, breakdown;
  double residual;
} cf_gmres_result;
/* gmres(op, prec, rhs) (linsolve.hpp:48-49): op = the block system (J != NULL) or a CSR matrix;
 * prec = a block preconditioner, an AMG hierarchy or none (identity).  history receives the
 * relative residual estimate of every inner iteration (up to history_cap entries). */
int cf_gmres(cf_block J, cf_csr A, cf_prec P, cf_amg M, const double* rhs, const cf_gmres_options* opts, double* x,
             cf_gmres_result* result, double* history, int history_cap);

/* ------------------------------------------------------------------ functionals */
/* compute_tcv (postproc.cpp:12-28): signed TCV of a solution (length n_total). */
int cf_compute_tcv(cf_problem p, const double* solution, double* tcv);
/* compute_cod, CodMethod::line_integral (postproc.cpp:38-99): openings at strictly increasing
 * stations (host arrays). */
int cf_compute_cod(cf_problem p, const double* solution, const double* stations, int n_stations, double* openings);

/* ------------------------------------------------------------------ Newton / active set */
typedef struct cf_state_s* cf_state; /* FractureState (model.hpp:50-55), device resident */
typedef struct {
  double residual_norm;
  int active_size, set_changes, gmres_iterations;
} cf_newton_iteration;             /* NewtonIteration (solver.hpp:28-33) */
typedef struct {
  double residual_ms, active_set_ms, jacobian_ms, amg_setup_ms, gmres_ms, total_ms;
} cf_phase_times;

/* slit_band_edge / resolve_regularization / initial_crack (model.cpp:28-58, 324-349). */
int cf_slit_band_edge(cf_problem p, const cf_material* mat, double* edge);
int cf_resolve_regularization(cf_problem p, const cf_material* mat, double band_edge, cf_regularization* out);
int cf_initial_crack(cf_problem p, const cf_material* mat, double band_half, double* phi, double* band_edge);
/* make_initial_state (solver.cpp:24-35) or an explicit state (any of the arrays may be NULL = zeros). */
int cf_make_initial_state(cf_problem p, const cf_material* mat, double seed_band, cf_state* out);
int cf_state_create(cf_problem p, const double* solution, const double* phi_old, const double* phi_prev2, int step,
                    cf_state* out);
int cf_state_get(cf_state s, double* solution, double* phi_old, double* phi_prev2, int* step);
int cf_state_destroy(cf_state s);
/* extrapolate_phi (model.cpp:60-64): phi_tilde of the state (phi_old for step <= 2, else
 * clip(2 phi_old - phi_prev2, [0, 1])); phi_tilde host or device, n_phi entries. */
int cf_extrapolate_phi(cf_state s, double* phi_tilde);
/* newton_active_set_step (solver.cpp:49-188).  its receives up to max_its iterations. */
int cf_newton_active_set_step(cf_problem p, cf_state s, const cf_material* mat, const cf_regularization* reg,
                              const cf_solver_options* opts, cf_newton_iteration* its, int max_its, int* n_its,
                              int* converged, double* feasibility, cf_phase_times* times);
/* solve_loading_sequence (solver.cpp:190-204): per step shift phi history, step = n, Newton;
 * stops after a non-converged step.  Per-step iteration counts in n_its[n_steps]. */
int cf_solve_loading_sequence(cf_problem p, cf_state s, const cf_material* mat, const cf_regularization* reg,
                              const cf_solver_options* opts, int n_steps, cf_newton_iteration* its, int max_its,
                              int* n_its, int* converged, double* feasibility, int* steps_done);

/* ------------------------------------------------------------------ I/O
 * write_matrix_market (linsolve.cpp:478-490): one block (which: 0 M_uu, 1 M_phiu, 2 M_phiphi)
 * or a CSR handle, byte-identical text.  write_vtk (postproc.cpp:111-167): the solution (and
 * phi_old, may be NULL) on the problem's mesh; binary = 0 is the reference's ASCII file, 1 the
 * same dataset in legacy big-endian BINARY encoding.  Arrays may be host or device. */
int cf_block_write_matrix_market(cf_block b, int which, const char* path);
int cf_csr_write_matrix_market(cf_csr A, const char* path);
int cf_write_vtk(cf_problem p, const double* solution, const double* phi_old, const char* path, int binary);

/* ------------------------------------------------------------------ general (adaptive) meshes
 * A cf_mesh is the reference's Mesh + DofMap (mesh.hpp:52-119, fem.hpp:33-74): a forest of
 * n0^d root cells on (-K, K)^d, refined with the 2:1 face-balance closure; cell ids in creation
 * order; vertices = sorted packed integer corner keys (the DofMap, built on the device).  The
 * constraint / assembly / Newton / post-processing entries below mirror the uniform ones with the
 * mesh in place of the problem; constraint sets of a mesh come from cf_mesh_constraints_build
 * (Dirichlet clamp, hanging vertices with closed lines, active set; fem.cpp:189-267) and are
 * accepted by cf_constraints_distribute.  States of a mesh come from cf_mesh_state_create. */
typedef struct cf_mesh_s* cf_mesh;
/* RefinementPolicy (adapt.hpp:12-20) */
typedef struct {
  double phi_threshold, h_target, theta;
  int max_level, estimator;
} cf_refinement_policy;
/* AdaptiveOptions (adapt.hpp:38-55; cod_stations omitted: use cf_mesh_compute_cod per level) */
typedef struct {
  cf_refinement_policy policy;
  cf_solver_options solver;
  int cycles, n_steps, halve_band_target, estimator_rounds;
  double seed_band;
} cf_adaptive_options;
/* LevelRecord (postproc.hpp:33-43) without the COD profile, plus the last report's convergence */
typedef struct {
  int level;
  int64_t dofs;
  double eps, h_min, tcv;
  int newton_iters;
  double gmres_mean;
  int converged;
} cf_level_record;

int cf_mesh_create(int dim, double half_width, int n0, cf_mesh* out);       /* create_mesh (mesh.cpp:18-34) */
int cf_mesh_copy(cf_mesh m, cf_mesh* out);
int cf_mesh_destroy(cf_mesh m);
int cf_mesh_refine(cf_mesh m, const int32_t* cells, int64_t n);            /* refine (mesh.cpp:203-215) */
int cf_mesh_uniform_refine(cf_mesh m, int times);                          /* uniform_refine (mesh.cpp:217-223) */
/* info4: n_cells, n_active, max_active_level, n_vertices; h_min = min_active_edge */
int cf_mesh_info(cf_mesh m, int64_t info4[4], double* h_min);
int cf_mesh_active_cells(cf_mesh m, int32_t* ids);                         /* active_cells, ascending */
/* per cell (id order): level, parent, active, anchor (3 integer coordinates) */
int cf_mesh_cells(cf_mesh m, int32_t* level, int32_t* parent, int8_t* active, int64_t* anchor);
int cf_mesh_vertex_keys(cf_mesh m, int64_t* keys);                         /* DofMap numbering (fem.cpp:98-116) */
int cf_mesh_cell_vertices(cf_mesh m, int64_t* out);                        /* per active cell, 2^d corners */
/* active_faces (mesh.cpp:225-259): rows of 5 (cell, axis, side, neighbor or -1, rel); out5 NULL counts */
int cf_mesh_faces(cf_mesh m, int64_t* n, int32_t* out5);
int cf_mesh_find_cell(cf_mesh m, const double x[3], int32_t* cell);        /* find_active_cell (mesh.cpp:143-150) */
int cf_mesh_constraints_build(cf_mesh m, int clamp_boundary, int64_t n_active, const int64_t* active_dofs,
                              const double* active_values, cf_constraints* out);
/* the closed lines with entries, ascending dof: counts first (dofs NULL), then CSR export */
int cf_constraint_lines(cf_constraints c, int64_t* n_lines, int64_t* n_entries, int64_t* dofs, int64_t* ptr,
                        int64_t* masters, double* weights, double* inhomogeneities);
int cf_mesh_assemble_residual(cf_mesh m, cf_constraints c, const cf_material* mat, const cf_regularization* reg,
                              const double* solution, const double* phi_tilde, double* residual);
int cf_mesh_assemble_jacobian(cf_mesh m, cf_constraints c, const cf_material* mat, const cf_regularization* reg,
                              const double* solution, const double* phi_tilde, cf_block* out);
int cf_mesh_rigid_body_modes(cf_mesh m, cf_constraints c, double* B);
int cf_mesh_slit_band_edge(cf_mesh m, const cf_material* mat, double* edge);
int cf_mesh_resolve_regularization(cf_mesh m, const cf_material* mat, double band_edge, cf_regularization* out);
int cf_mesh_initial_crack(cf_mesh m, const cf_material* mat, double band_half, double* phi, double* band_edge);
int cf_mesh_make_initial_state(cf_mesh m, const cf_material* mat, double seed_band, cf_state* out);
int cf_mesh_state_create(cf_mesh m, const double* solution, const double* phi_old, const double* phi_prev2, int step,
                         cf_state* out);
int cf_mesh_newton_active_set_step(cf_mesh m, cf_state s, const cf_material* mat, const cf_regularization* reg,
                                   const cf_solver_options* opts, cf_newton_iteration* its, int max_its, int* n_its,
                                   int* converged, double* feasibility, cf_phase_times* times);
int cf_mesh_solve_loading_sequence(cf_mesh m, cf_state s, const cf_material* mat, const cf_regularization* reg,
                                   const cf_solver_options* opts, int n_steps, cf_newton_iteration* its, int max_its,
                                   int* n_its, int* converged, double* feasibility, int* steps_done);
int cf_mesh_compute_tcv(cf_mesh m, const double* solution, double* tcv);
int cf_mesh_compute_cod(cf_mesh m, const double* solution, const double* stations, int n_stations, double* openings);
/* jump_estimator (adapt.cpp:16-55): eta per active cell in active order */
int cf_mesh_jump_estimator(cf_mesh m, const double* solution, double* eta);
/* mark_cells (adapt.cpp:57-97): eta may be NULL (no estimator field); ids ascending */
int cf_mesh_mark_cells(cf_mesh m, const double* solution, const double* eta, const cf_refinement_policy* policy,
                       int32_t* marked, int64_t* n_marked);
/* transfer (fem.cpp:318-333): nodal interpolation of old_vec onto the refined mesh */
int cf_mesh_transfer(cf_mesh old_mesh, const double* old_vec, cf_mesh new_mesh, double* new_vec);
/* adaptive_cycle (adapt.cpp:122-190): the mesh is refined in place and the state replaced by the
 * final level's; records[max_records] */
int cf_mesh_adaptive_cycle(cf_mesh m, cf_state s, cf_material* mat, const cf_adaptive_options* opts,
                           cf_level_record* records, int max_records, int* n_records);

/* ------------------------------------------------------------------ multi-GPU
 * One process per GPU.  Rank 0 makes an id, the launcher broadcasts it (e.g. over
 * torch.distributed), every rank creates its communicator on its current CUDA device.  The _comm
 * variants run the slab-decomposed step: rank r owns the planes of cf_slab_info(r, size); halo
 * planes move by NCCL send/recv, every dot / norm is a rank-ordered sum (bitwise identical on
 * all ranks), the preconditioner is restricted additive Schwarz over the slabs (each rank's block
 * AMG on its planes plus one overlap plane each side; CF_BLOCK_JACOBI=1: block-Jacobi).  The
 * state is global-length on every rank and holds the full solution on return.  size == 1 is the
 * single-GPU step exactly. */
typedef struct cf_comm_s* cf_comm;
/* Host-staged transport (TEST ONLY: lets several ranks share one GPU to exercise the decomposed
 * step's control flow without NCCL; device data is staged through host memory, so it is never
 * used for a measurement).  Callbacks return 0 on success; rank-ordered semantics as NCCL's. */
typedef struct {
  void* ctx;
  int (*allgather_f64)(void* ctx, const double* send, double* recv, int count);  /* recv: size*count */
  int (*allreduce_i64)(void* ctx, long long* vals, int count, int op);           /* in place; op 0 sum, 1 max */
  int (*sendrecv)(void* ctx, int n, const void* const* send, void* const* recv, const size_t* bytes,
                  const int* peer);                                              /* send/recv may be NULL */
  int (*bcast)(void* ctx, void* buf, size_t bytes, int root);
} cf_host_transport;
int cf_comm_create_host(int rank, int size, const cf_host_transport* transport, cf_comm* out);
int cf_comm_unique_id(uint8_t id[128]);
int cf_comm_create(const uint8_t id[128], int rank, int size, cf_comm* out);
int cf_comm_info(cf_comm c, int* rank, int* size);
/* Runs every NCCL entry point the decomposed step uses (id, init, all-gather in and out of place,
 * int64 sum / max all-reduce, broadcast, grouped broadcasts, grouped send / receive, destroy) on a
 * one-rank communicator on the current device and checks the results; *failed_checks = 0 when all
 * hold.  What a single-GPU box can verify of the NCCL transport. */
int cf_comm_selftest(int* failed_checks);
int cf_comm_destroy(cf_comm c);
int cf_newton_active_set_step_comm(cf_problem p, cf_state s, const cf_material* mat, const cf_regularization* reg,
                                   const cf_solver_options* opts, cf_comm comm, cf_newton_iteration* its,
                                   int max_its, int* n_its, int* converged, double* feasibility,
                                   cf_phase_times* times);
int cf_solve_loading_sequence_comm(cf_problem p, cf_state s, const cf_material* mat, const cf_regularization* reg,
                                   const cf_solver_options* opts, cf_comm comm, int n_steps,
                                   cf_newton_iteration* its, int max_its, int* n_its, int* converged,
                                   double* feasibility, int* steps_done);

#ifdef __cplusplus
}
#endif

#endif /* CRACKFIELD_B200_H */

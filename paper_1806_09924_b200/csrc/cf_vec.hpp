// Vector / Krylov primitives (vec.cu), SpGEMM & CSR utilities (spgemm.cu), AMG (amg.cu),
// GMRES (gmres.cu) and the Newton driver (newton.cu).
#pragma once

#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "cf_types.hpp"

namespace cfb {

struct Scratch {
  DevBuf<double> part, scal;
};

// ---- vec.cu
double* scalar_buf(int count);
void vfill(double* x, double a, i64 n);
void vcopy(double* dst, const double* src, i64 n);
void vaxpy(double a, const double* x, double* y, i64 n);                 // y += a x
void vaxpby(double a, const double* x, double b, double* y, i64 n);      // y = a x + b y
void vsub(const double* a, const double* b, double* out, i64 n);         // out = a - b
void vscale(double* x, double a, i64 n);
void vdiv_dev(const double* x, const double* s_dev, double* y, i64 n);   // y = x / *s
void vdiag_mul(const double* d, const double* x, double* y, double a, i64 n);  // y = a (d .* x)
void vdot_dev(const double* x, const double* y, i64 n, double* out, bool do_sqrt);
// w -= (*h_dev) v; *out = w . y (y = nullptr: w . w), bitwise the separate axpy + vdot_dev
void vaxpy_dot_dev(const double* h_dev, const double* v, double* w, const double* y, i64 n, double* out,
                   bool do_sqrt);
double vdot(const double* x, const double* y, i64 n);

// NP-invariant reductions of the Newton step's block vectors [u rows | phi rows].
// The vector is cut into partials that depend only on the grid, never on the rank count: each
// vertex plane's u part and phi part is split into chunks of `chunk` entries, every chunk is
// reduced by one 256-thread block (thread t sums entries t, t+256, ... sequentially, then the
// block tree), and the partials, in global order (u planes, then phi planes), go through the
// fixed final tree.  A rank owns whole planes, so it computes exactly its planes' partials; an
// all-gather places them, and every rank (and a single GPU) adds the same partials in the same
// order: the result is bitwise independent of the number of ranks.
struct SegLayout {
  i64 plane_u = 0, plane_p = 0;  // entries of one vertex plane in the u / phi part
  i64 chunk = 8192;
  int p_lo = 0, p_hi = 0;        // owned planes
  int nplanes = 0;               // planes of the grid
  __host__ __device__ int cu() const { return int((plane_u + chunk - 1) / chunk); }
  __host__ __device__ int cp() const { return int((plane_p + chunk - 1) / chunk); }
  __host__ __device__ i64 nu_local() const { return plane_u * (p_hi - p_lo); }
  __host__ __device__ int nparts() const { return nplanes * (cu() + cp()); }
  __host__ __device__ int nblocks_local() const { return (p_hi - p_lo) * (cu() + cp()); }
};
struct Comm;
// *out = x . y (sqrt optional) over all ranks' rows
void seg_dot_dev(const double* x, const double* y, const SegLayout& L, double* out, bool do_sqrt, const Comm* comm);
// w -= (*h) v, then *out = w . y (y = nullptr: w . w), bitwise the separate axpy + seg_dot_dev
void seg_axpy_dot_dev(const double* h, const double* v, double* w, const double* y, const SegLayout& L, double* out,
                      bool do_sqrt, const Comm* comm);
double vnorm(const double* x, i64 n);
void multidot(const double* V, i64 ld, int k, const double* w, i64 n, double* out_dev);   // out_i = V_i . w
void multi_axpy(double* w, const double* V, i64 ld, int k, const double* coef_dev, i64 n, double alpha);

// ---- spgemm.cu: CSR utilities (deterministic)
std::unique_ptr<Csr> spgemm(const Csr& A, const Csr& B, const double* row_scale = nullptr);  // diag(s) A B
std::unique_ptr<Csr> transpose(const Csr& A);
// row groups of A (runs of equal-pattern rows, <= gmax rows each); null when they would not pay
// (fewer than 4/3 rows per group on average, or short rows)
std::shared_ptr<RowGroups> csr_row_groups(const Csr& A, int gmax);
// P = T - w * DAT (union pattern), entries with |v| <= 1e-300 removed
std::unique_ptr<Csr> csr_axpy_prune(const Csr& T, double w, const Csr& DAT);
void csr_prune(Csr& A);  // in place (Eigen prune(1.0, 1e-300))
void csr_diagonal(const Csr& A, double* diag);  // A(i,i) or 0
std::unique_ptr<Csr> csr_copy(const Csr& A);
// the entries with column in [lo, hi), columns renumbered from lo (a slab's diagonal block)
std::unique_ptr<Csr> csr_extract_cols(const Csr& A, i64 lo, i64 hi);
// rows [lo, hi) (all columns), carrying the lane split of A (mean_hint)
std::unique_ptr<Csr> csr_extract_rows(const Csr& A, i64 lo, i64 hi);

// ---- dense LU (amg.cu): column-major n x n, unblocked partial pivoting (PartialPivLU)
struct DenseLu {
  i64 n = 0;
  DevBuf<double> lu;
  DevBuf<int> piv;
  double min_abs_pivot = 0.0;
  // a diagonal coarsest matrix beyond the dense size (e.g. the all-active phi block of a slab far
  // from the crack, where aggregation stops at once): LU without pivoting is the diagonal itself,
  // so the solve is x_i = b_i / a_ii
  bool diagonal = false;
  void factor_from_csr(const Csr& A);
  void solve(const double* b, double* x) const;  // device vectors
};

// ---- amg.cu (linsolve.hpp:62-94)
struct AmgLevel {
  std::shared_ptr<Csr> A;
  std::unique_ptr<Csr> P, R;
  DevBuf<double> inv_diag;
  double jacobi_weight = 2.0 / 3.0;
  double lambda = 0.0;
  double cheb_hi = 0.0;  // Chebyshev upper bound (smoother 1): Gershgorin bound of D^-1 A
  i64 n_nodes = 0, n_aggregates = 0, strong_edges = 0;
  int lfmis_rounds = 0;
  DevBuf<int> agg_of_node;  // kept for parity checks
  mutable DevBuf<double> tmp_r, tmp_b, tmp_x;  // V-cycle work vectors of this level
  mutable DevBuf<double> tmp_d;                // Chebyshev search direction (smoother 1)
};

struct Comm;
// A level whose rows are split over the ranks (distributed V-cycle): rank r applies
// rows [r c, (r+1) c) of A and P and rows [r cc, (r+1) cc) of R (c, cc: chunks padded so the
// vectors all-gather in place), every row exactly as the undivided operator computes it.
struct DistLevel {
  std::shared_ptr<Csr> A, P, R;
  i64 chunk = 0, cchunk = 0, lo = 0, hi = 0, clo = 0, chi = 0;
  mutable DevBuf<double> x, r, bc;  // padded to size x chunk (size x cchunk for bc)
};

struct Amg {
  std::vector<std::unique_ptr<AmgLevel>> levels;
  std::vector<DistLevel> dist;  // leading levels split over the ranks (empty: single-GPU V-cycle)
  const Comm* comm = nullptr;
  // split the large leading levels over the ranks of cm (the hierarchy itself is replicated)
  void distribute(const Comm* cm, i64 min_rows);
  void vcycle_range(size_t l0, const double* b0, double* x0) const;  // levels l0.. (single GPU)
  void vcycle_dist(const double* r, double* x) const;
  DenseLu coarse;
  cf_amg_options opts{};
  i64 n = 0;
  std::shared_ptr<Csr> coarse_A;
  // the build inputs, kept so an identical rebuild can be recognised bitwise and skipped
  std::shared_ptr<Csr> A0;
  DevBuf<int> nod0;
  DevBuf<double> B0;
  int m0 = 0;
  mutable DevBuf<double> cb, cx;  // coarsest rhs / solution
  // set: the finest level's operator (residual, smoothing sweeps) is applied matrix-free; level 0's A
  // stays the assembled matrix the hierarchy was built from
  std::shared_ptr<MfOp> mf0;
  void vcycle(const double* r, double* x) const;  // x = V(r), zero initial guess
  // true iff build_amg(A, node_of_dof, B, m, opts) would rebuild exactly this hierarchy
  bool same_inputs(const Csr& A, const int* node_of_dof, const double* B, int m, const cf_amg_options& o) const;
};

std::unique_ptr<Amg> build_amg(std::shared_ptr<Csr> A, const int* node_of_dof, const double* B, int m,
                               const cf_amg_options& opts);

// ---- block preconditioner (linsolve.cpp:352-415)
struct BlockPrec {
  int kind = 1;  // 0 exact, 1 amg, 2 diagonal
  bool serial = false;  // V-cycles in sequence on the library stream (distributed hierarchies)
  i64 nu = 0, np = 0;
  std::shared_ptr<Amg> amg_u, amg_p;
  std::shared_ptr<DenseLu> lu_u, lu_p;
  DevBuf<double> inv_u, inv_p;
  void apply(const double* r, double* z) const;
};

struct NullspaceDev {  // NullspaceInfo on the device (linsolve.hpp:108-113)
  const int* u_node = nullptr;
  const double* u_modes = nullptr;  // n_u x m column-major
  int m_u = 0;
  const int* p_node = nullptr;
  const double* p_modes = nullptr;  // n_phi x 1
};

// prev (optional): a previous preconditioner whose hierarchies are reused when their inputs are
// bitwise identical (build_amg is deterministic, so the rebuilt hierarchy would be identical)
std::unique_ptr<BlockPrec> build_block_prec(const BlockSystem& J, int kind, const cf_amg_options& o,
                                            const NullspaceDev* ns, const BlockPrec* prev = nullptr);
bool bitwise_equal(const void* a, const void* b, size_t bytes);  // device arrays

// ---- gmres.cu (linsolve.cpp:21-115)
using DevOp = std::function<void(const double* in, double* out)>;
struct GmresResult {
  int iterations = 0;
  bool converged = false, breakdown = false;
  double residual = 0.0;
  std::vector<double> history;
};
struct Comm;
// comm (optional, distributed): rhs / x are this rank's rows; every dot is summed over the ranks
// seg (optional): the NP-invariant segmented reductions of a slab block vector (required with comm)
GmresResult gmres(const DevOp& op, const DevOp* prec, const double* rhs, i64 n, const cf_gmres_options& o,
                  double* x, const Comm* comm = nullptr, const SegLayout* seg = nullptr);

// ---- postproc.cu (postproc.cpp:12-99)
double compute_tcv(const Problem& P, const double* sol);
void compute_cod(const Problem& P, const double* sol, const double* stations_host, int ns, double* out_host);

// ---- mf.cu: matrix-free M_uu apply (x, y: n_u), FP64 FMA probe
void mf_apply_uu(Problem& P, const Constraints& cs, const cf_material& m, const cf_regularization& reg,
                 const double* pt, const double* x, double* y);
double fp64_peak_tflops();

// ---- io.cu (linsolve.cpp:478-490, postproc.cpp:111-167)
void write_matrix_market(const Csr& A, const std::string& path);
void write_vtk(const Problem& P, const double* sol_dev, const double* phi_old_dev, const std::string& path,
               bool binary);

// ---- newton.cu (solver.cpp:24-204)
struct State {  // FractureState (model.hpp:50-55), device resident
  DevBuf<double> solution, phi_old, phi_prev2;
  int step = 0;
};
struct NewtonIter {
  double residual_norm;
  int active_size, set_changes, gmres_iterations;
};
struct PhaseTimes {  // per-phase device time of the last Newton step (ms)
  double residual = 0, active_set = 0, jacobian = 0, amg_setup = 0, gmres = 0, other = 0;
};
struct NewtonReport {
  std::vector<NewtonIter> its;
  bool converged = false;
  double feasibility = 0.0;
  PhaseTimes times;
};
// comm / slab (optional): the slab-decomposed step of one rank.  The state's vectors
// are global-length on every rank; on return they hold the full solution on every rank.
NewtonReport newton_active_set_step(Problem& P, State& st, const cf_material& mat, const cf_regularization& reg,
                                    const cf_solver_options& opts, const Comm* comm = nullptr,
                                    const Slab* slab = nullptr);
Slab rank_slab(const GridDesc& g, int rank, int size);  // planes split evenly over the ranks
void extrapolate_phi(const State& st, double* pt, i64 V);  // model.cpp:60-64
// n_u x m column-major rigid-body modes (rows of the slab's owned u dofs when slab is given)
void rigid_body_modes(const Problem& P, const Constraints& c, double* B, const Slab* slab = nullptr);
// host helpers (model.cpp:28-64, 324-349)
double slit_band_edge(const Problem& P, const cf_material& mat);
cf_regularization resolve_regularization(const Problem& P, const cf_material& mat, double band_edge);
std::vector<double> initial_crack(const Problem& P, const cf_material& mat, double band_half, double* band_edge);

}  // namespace cfb

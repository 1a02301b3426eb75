// Device-resident data structures of the hot path: the uniform grid + DofMap descriptor
// (mesh.hpp / fem.hpp), the constraint set, CSR matrices and the block system.
#pragma once

#include <cmath>
#include <memory>
#include <vector>

#include "cf_common.hpp"

namespace cfb {

// Uniform grid of (n0 << r)^d cells on (-K, K)^d.  Vertex v = x + nn*(y + nn*z) (fem.cpp:98-116
// numbers vertices by the packed key x | y<<21 | z<<42, i.e. lexicographically with x fastest).
struct GridDesc {
  int d, r, n0;
  i64 nc, nn, V, ncells;
  double K, unit, h, detJ;
  __host__ __device__ i64 n_u() const { return d * V; }
  __host__ __device__ i64 n_total() const { return (d + 1) * V; }
};

// Quadrature / Q1 tables of one problem (fem.cpp:53-96; model.cpp:111-123), computed on the
// host with the reference's expressions (compiled without FMA contraction) so device
// assembly reproduces the reference's element arithmetic bit for bit.
struct Tables {
  double w[8];                 // quad weight * detJ
  double s[8][8];              // shape[q][k]
  double G[8][8][3];           // reference gradients[q][k][a]
  double gp[8][8][3];          // G / h  (gphys, model.cpp:245-247)
  double gg[8][8][8];          // sum_b gphys(k,b) gphys(l,b)
  double val[8][8][8][3][3];   // mu((a==b)gg + gp(l,a)gp(k,b)) + lam gp(l,b)gp(k,a)  (model.cpp:274-275)
};

// Slab decomposition: a rank owns a contiguous run of vertex planes along the slowest
// axis (z in 3d, y in 2d), i.e. a contiguous vertex range in the reference's lexicographic
// numbering.  Its rows need x on one ghost plane each side ("ext" range) and the cells touching
// its planes (a contiguous range of lexicographic cell indices).  Local vectors are laid out
// [u_own (d*nv) | phi_own (nv)], ext vectors [u_ext (d*ne) | phi_ext (ne)]; the full slab of a
// single GPU makes both layouts the global [u | phi].
struct Slab {
  i64 v_lo = 0, v_hi = 0;    // owned vertices
  i64 ve_lo = 0, ve_hi = 0;  // owned + ghost planes (clipped to the grid)
  i64 c_lo = 0, c_hi = 0;    // cells adjacent to owned vertices
  i64 plane = 0;             // vertices per plane
  __host__ __device__ i64 nv() const { return v_hi - v_lo; }
  __host__ __device__ i64 ne() const { return ve_hi - ve_lo; }
  bool full(const GridDesc& g) const { return v_lo == 0 && v_hi == g.V; }
};
// planes [p_lo, p_hi) of the nn vertex planes
Slab make_slab(const GridDesc& g, i64 p_lo, i64 p_hi);
inline Slab full_slab(const GridDesc& g) { return make_slab(g, 0, g.nn); }

struct Problem {
  GridDesc g{};
  Tables host_tab{};
  DevBuf<Tables> tab;
  double mu = 0.0, lam = 0.0;  // cached for the material the tables were built with
  bool val_ready = false;
};

struct Constraints {
  const Problem* prob = nullptr;
  DevBuf<std::uint8_t> flag;  // per dof
  DevBuf<double> inhom;       // per dof (phi_old on the active set, 0 elsewhere)
  i64 count = 0;
  // lines with entries (hanging vertices of a general mesh, closed: every master is unconstrained):
  // dof line_dof[i] = inhom + sum of line_w * x[line_m] over [line_ptr[i], line_ptr[i+1]), in the
  // reference's entry order (fem.cpp:229-247)
  i64 n_lines = 0;
  DevBuf<int> line_dof;
  DevBuf<i64> line_ptr;
  DevBuf<int> line_m;
  DevBuf<double> line_w;
  const void* mesh = nullptr;  // the MeshDisc of a general-mesh set (nullptr: uniform grid)
  std::uint64_t uid = 0;       // identity of a general-mesh set (its assembly plans are cached by it)
};

// Stencil-implicit columns of the uniform-grid blocks M_uu / M_phiu when the Dirichlet clamp is the
// only u constraint: the columns of a row follow from its vertex (the 3^d neighbours whose u dofs
// are free, ascending), so an SpMV can stream the values alone (8 instead of 12 bytes per entry).
// Set by assemble_jacobian only after a device check that every stored column equals the computed
// one; the stored columns stay (AMG setup reads them).
struct StencilCols {
  int kind = 0;  // 0 off, 1 rows are u dofs (row = lv * d + a), 2 rows are phi dofs (row = lv)
  int d = 0;
  i64 nn = 0, v_lo = 0, shift = 0;  // nodes per side, first row vertex, global -> stored column shift
  double inv_nn = 0.0;
};

// Runs of consecutive rows with one column pattern (the dofs of a mesh node, the coarse dofs of an
// aggregate), chunked to <= gmax rows: group g is rows heads[g] .. heads[g] + len[g] - 1, stored
// contiguously with equal lengths.  Set on the AMG level operators (A of levels >= 1, P, R), where
// the SpMV reads each group's column indices and x entries once for all its rows.
struct RowGroups {
  DevBuf<int> heads, len;
  i64 n = 0;
  int gmax = 1;
};

// Rows with at most one entry (constrained dofs: the diagonal) apart from the rest (ascending list):
// set on a level-0 operator most of whose rows are such (the phi block late in a Newton step), where
// the SpMV runs the heavy rows from the list and the light rows one thread each.
struct RowSplit {
  DevBuf<int> heavy;
  DevBuf<std::uint8_t> flag;
  i64 n_heavy = 0;
};

struct Csr {
  i64 rows = 0, cols = 0, nnz = 0;
  std::shared_ptr<RowGroups> grp;  // optional (SpMV only; the pattern must not change while set)
  std::shared_ptr<RowSplit> split;  // optional (SpMV only; the pattern must not change while set)
  StencilCols st;
  DevBuf<i64> ptr;
  DevBuf<int> col;
  DevBuf<double> val;
  // mean row length that picks the SpMV lane split (< 0: nnz / rows).  A slab of a distributed
  // matrix carries the global mean so its rows reduce exactly as the undivided matrix's.
  double mean_hint = -1.0;
};

// Matrix-free stand-in for a uniform 3d grid's M_uu (the block's values are never read): y = M_uu x
// with the assembled block's condensation (constrained columns dropped, constrained rows keep the
// summed element diagonal), optionally with an SpMV row epilogue (modes 0-2 of SpmvEpi).
struct MfOp {
  Problem* P = nullptr;
  const std::uint8_t* flag = nullptr;  // u constraint flags (global dof numbering)
  double mu = 0.0, lam = 0.0, kap = 0.0;
  const double* pt = nullptr;  // phi_tilde (global vertex numbering)
  // rows of the vertices [y_lo, y_hi) (all when y_hi < 0), written at local row (v - y_lo) d + a;
  // x holds the vertices from x_off on (a slab's ext range, or the global vector)
  i64 x_off = 0, y_lo = 0, y_hi = -1;
};

struct BlockSystem {
  i64 nu = 0, np = 0;
  // input layout of block_apply: [u (nu_in) | phi (np_in)]; < 0 means square (nu, np).  A slab's
  // blocks read ext vectors (owned rows, columns over owned + ghost planes).
  i64 nu_in = -1, np_in = -1;
  std::shared_ptr<Csr> uu = std::make_shared<Csr>(), pu = std::make_shared<Csr>(), pp = std::make_shared<Csr>();
  int d = 2;
  std::shared_ptr<MfOp> mf_uu;  // set: M_uu applied matrix-free in block_apply (uu keeps its values)
  i64 in_u() const { return nu_in >= 0 ? nu_in : nu; }
  // phi rows split for block_apply (spmv.cu, built on first use): rows with a non-empty M_phiu row or
  // more than one M_phiphi entry ("heavy", ascending) and the rest (active phi dofs: one diagonal entry)
  mutable DevBuf<int> phi_heavy;
  mutable DevBuf<std::uint8_t> phi_heavy_flag;
  mutable i64 n_phi_heavy = -1;  // -1: not classified yet
};

// ---- host helpers implemented in the .cu files
Problem* make_problem(int d, double K, int n0, int r);
void build_tables(Problem& P, double mu, double lam);
void fill_tables(Tables& T, int d, double h, double detJ, double mu, double lam);
void distribute_lines(const Constraints& c, double* v, bool homogeneous);  // mesh.cu
std::unique_ptr<Constraints> build_constraints(const Problem& P, bool clamp, i64 n_active,
                                               const i64* dofs_dev, const double* vals_dev);
void distribute(const Constraints& c, double* v_dev, bool homogeneous);
// x, pt: global-length vectors (valid on the slab's ext range).  R: local layout of the slab.
// cache (optional): keeps the per-cell element residuals of the call, so that a following
// assemble_residual_moved (same problem, material, phi_tilde and slab) recomputes only the cells
// touching the vertices whose dofs changed; bitwise the full assembly (each element residual is a
// function of its own corners only)
struct ResidualCache {
  DevBuf<double> cellres;
  DevBuf<int> list, count;
  DevBuf<std::uint8_t> moved;
  i64 c_lo = 0, c_hi = 0;
  bool valid = false;
};
void assemble_residual(Problem& P, const Constraints& c, const cf_material& m, const cf_regularization& reg,
                       const double* x, const double* pt, double* R, const Slab* slab = nullptr,
                       ResidualCache* cache = nullptr);
// x_before: x of the cached call (global layout); only the cells with a corner whose dofs differ
// between x_before and x are recomputed, then every owned row is gathered with c's flags
void assemble_residual_moved(Problem& P, const Constraints& c, const cf_material& m, const cf_regularization& reg,
                             const double* x, const double* x_before, const double* pt, double* R,
                             const Slab* slab, ResidualCache& cache);
// rows of the slab's owned vertices; columns in the slab's ext numbering.  reuse_uu: an M_uu of
// the same phi_tilde, slab and Dirichlet set (M_uu depends on nothing else, model.cpp:268-276),
// taken as is instead of being recomputed.
struct Csr;
std::unique_ptr<BlockSystem> assemble_jacobian(Problem& P, const Constraints& c, const cf_material& m,
                                               const cf_regularization& reg, const double* x, const double* pt,
                                               const Slab* slab = nullptr, std::shared_ptr<Csr> reuse_uu = nullptr);
// assemble_pattern (linsolve.cpp:417-476): BlockSparsity as CSR blocks with zero values
std::unique_ptr<BlockSystem> assemble_pattern(const Problem& P, const Constraints& c);
void csr_spmv_add(const Csr& A, const double* x, double* y, const double* add);  // y = A x (+ add)
// row epilogue of a fused SpMV (A square for modes 1 and 2; y must not alias x):
//   0: y = A x (+ b)   1: y = b - A x (residual)   2: y = x + w (d (b - A x)) (one damped Jacobi sweep)
//   3: y = w (d (A x)) (the power iteration's D^-1 A x with w = 1)
// each mode is the same IEEE operation sequence as the SpMV followed by the separate vector kernel
struct SpmvEpi {
  const double* b = nullptr;
  const double* d = nullptr;
  double w = 0.0;
  int mode = 0;
  i64 xoff = 0;  // mode 2 reads x[row + xoff] (a row slice of a square matrix applied to a full x)
};
void csr_spmv_epi(const Csr& A, const double* x, double* y, const SpmvEpi& ep);
void mf_apply(const MfOp& op, const double* x, double* y, const SpmvEpi& ep);  // mf.cu (3d)
void csr_spmv(const Csr& A, const double* x, double* y, double unused = 0.0);
void block_apply(const BlockSystem& J, const double* x, double* y);
bool csr_spmv_variant(const Csr& A, int tpr, int unroll, const double* x, double* y);
bool csr_enable_stencil(Csr& A, const StencilCols& sc);
void csr_enable_row_split(Csr& A);  // sets A.split when at least half of a long matrix's rows hold <= 1 entry
void div_by_h(double h, const double* a, i64 n, double* q);  // test hook of the residual's a / h  // CF_NO_STENCIL_COLS=1 disables

inline double mat_mu(const cf_material& m) { return m.E / (2.0 * (1.0 + m.nu)); }              // model.hpp:26
inline double mat_lambda(const cf_material& m) {                                                  // model.hpp:27
  return m.E * m.nu / ((1.0 + m.nu) * (1.0 - 2.0 * m.nu));
}
void validate_material(const cf_material& m);  // model.cpp:8-17

}  // namespace cfb

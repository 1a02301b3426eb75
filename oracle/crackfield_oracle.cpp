// =====================================================================================
//  crackfield ORACLE — TEST INFRASTRUCTURE ONLY.
//
//  A plain C++17 (no Eigen) CPU restatement of the reference hot path of
//  /root/reference/proj (crackfield, arXiv 1806.09924), restricted to uniformly
//  refined meshes (every BASELINE config is uniform; hanging nodes are SURVEY §8f "next").
//
//  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
//  legs may load this library, and only as the checker / the CPU baseline.  The product
//  (paper_1806_09924_b200/) never links or calls it.
//
//  Pinning: the reference cannot be built here (Eigen3, doctest, CLI11 are absent;
//  SURVEY §8c), so this restatement is pinned against the reference's own known-answer
//  tests (model_test, linsolve_test, solver_test, fem_test, postproc_test,
//  reference_test KATs; see tests/test_oracle_kat.py).  ColPivHouseholderQR,
//  makeHouseholder and applyHouseholderOnTheLeft follow Eigen 3.3's published algorithm
//  step by step; the coarse LU is unblocked (Eigen blocks above 16 rows).
//
//  Two reduction orders (orc_set_order), because Eigen's own order is not pinned by any
//  reference test:
//   * ORDER_PRODUCT (0, default): the product's documented deterministic order.  An SpMV
//     row is split over TPR lanes (lane l sums entries l, l+TPR, ...; xor butterfly), TPR
//     from the mean row length; a dot/norm is a 256-thread block tree over a fixed grid.
//     This is NOT the reference's order: it is the order the B200 kernels use, adopted
//     here so that the device can be checked bit for bit (same algorithm, same order).
//   * ORDER_REFERENCE (1): the reference's arithmetic as written — every CSR row is one
//     left-to-right sum (Eigen's RowMajor sparse x dense, linsolve.cpp:16-17,304-311),
//     every dot/norm one sequential sum (linsolve.cpp:30,38,57,60).  The device is checked
//     against this mode at the north-star tolerances (1e-8 solution, 1e-6 COD/TCV, +-10%
//     Newton/GMRES counts), not bitwise.
//  Everything else (assembly in the reference's cell order, SpGEMM as k-ascending
//  sequential sums, QR, LU, the aggregation greedy) is the same in both modes.
//
//  Threads (orc_set_threads): results are bitwise independent of the thread count.  With
//  one thread the assembly is the literal cell loop of model.cpp; with more, every row is
//  owned by one vertex that sums its cells' contributions in the same reference cell
//  order (tests/test_oracle_kat.py checks the two forms bit for bit).
//
//  Compile with -ffp-contract=off (no FMA contraction) so the element arithmetic is
//  the reference's expression order exactly.
// =====================================================================================
#include <algorithm>
#include <chrono>
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <malloc.h>
#include <functional>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <unordered_map>
#include <vector>

namespace orc {

using i64 = std::int64_t;
using Vec = std::vector<double>;

static thread_local std::string g_err;

// ------------------------------------------------------------------ options (C layout)
extern "C" {
struct orc_material {
  double E, nu, G_c, pressure, l0, kappa_factor;
  int eps_mode;  // 0 tied, 1 fixed            (model.hpp:11)
  double c_eps, eps_fixed;
  int pressure_coupling;  // 0 extrapolated, 1 current (model.hpp:12)
};
struct orc_regularization {
  double eps, kappa;
};
struct orc_amg_options {  // linsolve.hpp:51-60
  double strength_threshold, prolongation_omega, jacobi_omega;
  int smoothing_sweeps, coarse_size, max_levels;
};
struct orc_gmres_options {  // linsolve.hpp:32-36
  double rtol;
  int max_iter, restart;
};
struct orc_solver_options {  // solver.hpp:13-26
  double newton_tol, newton_abs_floor;
  int newton_max_iter;
  double active_set_c_scale;
  int cycle_window, cycle_toggles, damping, prec_kind, freeze_preconditioner, log;
  orc_gmres_options gmres;
  orc_amg_options amg;
};
}

static double mat_mu(const orc_material& m) { return m.E / (2.0 * (1.0 + m.nu)); }        // model.hpp:26
static double mat_lambda(const orc_material& m) {                                            // model.hpp:27
  return m.E * m.nu / ((1.0 + m.nu) * (1.0 - 2.0 * m.nu));
}

// ------------------------------------------------------------------ uniform grid (mesh.cpp / fem.cpp)
struct Grid {
  int d = 2, n0 = 1, r = 0;
  double K = 1.0;
  i64 nc = 1, nn = 2, V = 4, ncells = 1;
  double unit = 0.0, h = 0.0, detJ = 0.0;
  std::vector<i64> cell_order;  // cells in the reference's active-cell order
  std::vector<i64> cell_rank;   // inverse permutation: position of a cell in cell_order

  // mesh.hpp:73 to_physical(c) with c = i * isize, isize = kUnit >> r
  double coord(i64 i) const { return -K + double(i * (i64(1) << (16 - r))) * unit; }
  i64 vid(i64 x, i64 y, i64 z) const { return x + nn * (y + nn * z); }
  void vxyz(i64 v, i64& x, i64& y, i64& z) const {
    x = v % nn;
    y = (v / nn) % nn;
    z = (d == 3) ? v / (nn * nn) : 0;
  }
  i64 cid(i64 x, i64 y, i64 z) const { return x + nc * (y + nc * z); }
  void cxyz(i64 c, i64& x, i64& y, i64& z) const {
    x = c % nc;
    y = (c / nc) % nc;
    z = (d == 3) ? c / (nc * nc) : 0;
  }
  // DofMap::cell_vertices (fem.cpp:139-146): corners in z-order, bit a = high side on axis a
  void cell_vertices(i64 c, i64* out) const {
    i64 x, y, z;
    cxyz(c, x, y, z);
    for (int k = 0; k < (1 << d); ++k)
      out[k] = vid(x + (k & 1), y + ((k >> 1) & 1), z + ((k >> 2) & 1));
  }
  bool on_boundary(i64 v) const {  // fem.cpp:131-137
    i64 c[3];
    vxyz(v, c[0], c[1], c[2]);
    for (int a = 0; a < d; ++a)
      if (c[a] == 0 || c[a] == nc) return true;
    return false;
  }
  i64 n_u() const { return d * V; }
  i64 n_phi() const { return V; }
  i64 n_total() const { return (d + 1) * V; }
};

// Reference active-cell order after uniform_refine (mesh.cpp:18-34, 147-169, 209-215):
// roots lexicographic, then each split appends its 2^d children in z-order, so the
// order is "root lex index, then hierarchical Morton code of the local position".
static void build_cell_order(Grid& g) {
  const int d = g.d, r = g.r;
  const i64 nroot = (d == 3) ? i64(g.n0) * g.n0 * g.n0 : i64(g.n0) * g.n0;
  const i64 nloc = i64(1) << (d * r);
  g.cell_order.resize(g.ncells);
  i64 pos = 0;
  for (i64 root = 0; root < nroot; ++root) {
    const i64 rx = root % g.n0, ry = (root / g.n0) % g.n0, rz = (d == 3) ? root / (i64(g.n0) * g.n0) : 0;
    for (i64 m = 0; m < nloc; ++m) {
      i64 l[3] = {0, 0, 0};
      for (int lev = 1; lev <= r; ++lev) {
        const i64 child = (m >> (d * (r - lev))) & ((i64(1) << d) - 1);
        for (int a = 0; a < d; ++a)
          if (child & (i64(1) << a)) l[a] |= i64(1) << (r - lev);
      }
      g.cell_order[pos++] = g.cid((rx << r) + l[0], (ry << r) + l[1], (rz << r) + l[2]);
    }
  }
  g.cell_rank.resize(g.ncells);
  for (i64 p = 0; p < g.ncells; ++p) g.cell_rank[g.cell_order[p]] = p;
}

static Grid make_grid(int d, double K, int n0, int r) {
  if (d != 2 && d != 3) throw std::invalid_argument("DomainSpec: dimension must be 2 or 3");
  if (!(K > 0.0)) throw std::invalid_argument("DomainSpec: half_width must be positive");
  if (n0 < 1 || n0 > 16) throw std::invalid_argument("DomainSpec: initial_cells_per_side must be in [1,16]");
  if (r < 0 || r > 16) throw std::invalid_argument("uniform_refine: bad refinement count");
  Grid g;
  g.d = d;
  g.K = K;
  g.n0 = n0;
  g.r = r;
  g.nc = i64(n0) << r;
  g.nn = g.nc + 1;
  g.V = (d == 3) ? g.nn * g.nn * g.nn : g.nn * g.nn;
  g.ncells = (d == 3) ? g.nc * g.nc * g.nc : g.nc * g.nc;
  g.unit = 2.0 * K / (n0 * double(i64(1) << 16));                      // mesh.cpp:20
  g.h = 2.0 * K / (n0 * double(i64(1) << r));                          // mesh.hpp:65-67
  g.detJ = std::pow(g.h, d);                                            // model.cpp:148
  build_cell_order(g);
  return g;
}

// ------------------------------------------------------------------ quadrature + Q1 (fem.cpp:17-96)
struct QpData {
  int nq = 0, nv = 0, d = 0;
  double pts[8][3];
  double wts[8];
  double shape[8][8];    // [q][k]
  double grads[8][8][3]; // [q][k][a]
};

static void q1_shape(int d, const double xi[3], double* values, double (*grads)[3]) {
  const int n = 1 << d;
  for (int k = 0; k < n; ++k) {
    double v = 1.0;
    for (int a = 0; a < d; ++a) v *= (k & (1 << a)) ? xi[a] : 1.0 - xi[a];
    values[k] = v;
    for (int a = 0; a < d; ++a) {
      double g = (k & (1 << a)) ? 1.0 : -1.0;
      for (int b = 0; b < d; ++b) {
        if (b == a) continue;
        g *= (k & (1 << b)) ? xi[b] : 1.0 - xi[b];
      }
      grads[k][a] = g;
    }
  }
}

static void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w) {
  switch (n) {
    case 1: x = {0.0}; w = {2.0}; break;
    case 2: { const double a = 1.0 / std::sqrt(3.0); x = {-a, a}; w = {1.0, 1.0}; break; }
    case 3: { const double a = std::sqrt(3.0 / 5.0); x = {-a, 0.0, a}; w = {5.0 / 9.0, 8.0 / 9.0, 5.0 / 9.0}; break; }
    case 4: {
      const double a = std::sqrt(3.0 / 7.0 - 2.0 / 7.0 * std::sqrt(6.0 / 5.0));
      const double b = std::sqrt(3.0 / 7.0 + 2.0 / 7.0 * std::sqrt(6.0 / 5.0));
      const double wa = (18.0 + std::sqrt(30.0)) / 36.0;
      const double wb = (18.0 - std::sqrt(30.0)) / 36.0;
      x = {-b, -a, a, b}; w = {wb, wa, wa, wb};
      break;
    }
    default: throw std::invalid_argument("gauss_legendre: up to 4 points supported here");
  }
}

struct Rule {  // Quadrature::cell_rule (fem.cpp:53-74)
  int nq = 0;
  std::vector<double> pts;  // nq x d
  std::vector<double> w;
};
static Rule cell_rule(int d, int n1) {
  std::vector<double> x, w;
  gauss_legendre(n1, x, w);
  int nq = 1;
  for (int a = 0; a < d; ++a) nq *= n1;
  Rule q;
  q.nq = nq;
  q.pts.assign(size_t(nq) * d, 0.0);
  q.w.assign(nq, 0.0);
  for (int k = 0; k < nq; ++k) {
    int rem = k;
    double wt = 1.0;
    for (int a = 0; a < d; ++a) {
      int i = rem % n1;
      rem /= n1;
      q.pts[size_t(k) * d + a] = 0.5 * (x[i] + 1.0);
      wt *= 0.5 * w[i];
    }
    q.w[k] = wt;
  }
  return q;
}

static QpData make_qp_data(int d) {  // model.cpp:111-123
  QpData qp;
  Rule q = cell_rule(d, 2);
  qp.nq = q.nq;
  qp.nv = 1 << d;
  qp.d = d;
  for (int iq = 0; iq < q.nq; ++iq) {
    double xi[3] = {0, 0, 0};
    for (int a = 0; a < d; ++a) xi[a] = q.pts[size_t(iq) * d + a];
    for (int a = 0; a < 3; ++a) qp.pts[iq][a] = xi[a];
    qp.wts[iq] = q.w[iq];
    q1_shape(d, xi, qp.shape[iq], qp.grads[iq]);
  }
  return qp;
}

// ------------------------------------------------------------------ constraints (fem.cpp:148-267)
// On a uniform mesh every line is entry-free: Dirichlet (u = 0 on the boundary) and the
// active set (phi = phi_old).  close() is then the identity.
struct Constraints {
  std::vector<unsigned char> flag;  // per dof
  std::vector<double> inhom;        // per dof
  i64 count = 0;
  bool is(i64 dof) const { return flag[dof] != 0; }
  void distribute(Vec& v) const {
    for (size_t i = 0; i < flag.size(); ++i)
      if (flag[i]) v[i] = inhom[i];
  }
  void distribute_homogeneous(Vec& v) const {
    for (size_t i = 0; i < flag.size(); ++i)
      if (flag[i]) v[i] = 0.0;
  }
};

static Constraints build_constraints(const Grid& g, bool clamp, const std::vector<i64>& active_dofs,
                                     const std::vector<double>& active_vals) {
  Constraints cs;
  cs.flag.assign(g.n_total(), 0);
  cs.inhom.assign(g.n_total(), 0.0);
  if (clamp)
    for (i64 v = 0; v < g.V; ++v)
      if (g.on_boundary(v))
        for (int c = 0; c < g.d; ++c) cs.flag[v * g.d + c] = 1;
  for (size_t k = 0; k < active_dofs.size(); ++k) {  // fem.cpp:258-263
    const i64 dof = active_dofs[k];
    if (dof < 0 || dof >= g.n_total()) throw std::invalid_argument("build_constraints: dof out of range");
    if (cs.flag[dof]) continue;
    cs.flag[dof] = 1;
    cs.inhom[dof] = active_vals[k];
  }
  for (auto f : cs.flag) cs.count += f;
  return cs;
}

// ------------------------------------------------------------------ CSR
// Large arrays are allocated without value-initialisation (resize() leaves them untouched), so
// the first touch happens in the parallel loops that fill them.
template <class T>
struct UninitAlloc : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = UninitAlloc<U>;
  };
  UninitAlloc() = default;
  template <class U>
  UninitAlloc(const UninitAlloc<U>&) noexcept {}
  template <class U>
  void construct(U* p) noexcept {
    ::new (static_cast<void*>(p)) U;
  }
  template <class U, class... Args>
  void construct(U* p, Args&&... args) {
    ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...);
  }
};
template <class T>
using uvec = std::vector<T, UninitAlloc<T>>;

struct Csr {
  i64 rows = 0, cols = 0;
  uvec<i64> ptr{0};
  uvec<int> col;
  uvec<double> val;
  i64 nnz() const { return i64(col.size()); }
  double coeff(i64 i, i64 j) const {
    for (i64 k = ptr[i]; k < ptr[i + 1]; ++k)
      if (col[k] == j) return val[k];
    return 0.0;
  }
};

// ---- Reduction order (see the header): ORDER_PRODUCT = the device's documented order,
// ORDER_REFERENCE = the reference's sequential sums.
enum { ORDER_PRODUCT = 0, ORDER_REFERENCE = 1 };
static int g_order = ORDER_PRODUCT;

// ORC_TIMING=1: phase times on stderr (profiling of the CPU baseline only)
static bool timing_on() {
  static const bool on = std::getenv("ORC_TIMING") != nullptr;
  return on;
}
struct PhaseTimer {
  const char* name;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  explicit PhaseTimer(const char* n) : name(n) {}
  ~PhaseTimer() {
    if (timing_on())
      std::fprintf(stderr, "[orc] %-18s %9.1f ms\n", name,
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
};

static int spmv_tpr(const Csr& A) {
  if (g_order == ORDER_REFERENCE) return 1;
  const double mean = A.rows ? double(A.nnz()) / double(A.rows) : 0.0;
  return mean > 64 ? 16 : (mean > 24 ? 8 : 4);
}
static double row_sum_lanes(const Csr& A, i64 i, const double* x, int tpr) {
  if (tpr == 1) {  // Eigen RowMajor sparse x dense: tmp = 0; tmp += v * x[c] in storage order
    double s = 0.0;
    for (i64 k = A.ptr[i]; k < A.ptr[i + 1]; ++k) s += A.val[k] * x[A.col[k]];
    return s;
  }
  double lane[32];
  for (int l = 0; l < tpr; ++l) {
    double s = 0.0;
    for (i64 k = A.ptr[i] + l; k < A.ptr[i + 1]; k += tpr) s += A.val[k] * x[A.col[k]];
    lane[l] = s;
  }
  double tmp[32];
  for (int o = tpr / 2; o > 0; o >>= 1) {
    for (int l = 0; l < tpr; ++l) tmp[l] = lane[l] + lane[l ^ o];
    for (int l = 0; l < tpr; ++l) lane[l] = tmp[l];
  }
  return lane[0];
}
// Persistent host thread pool (orc_set_threads; 1 = the single-threaded reference).  Work is
// split into chunks whose results never depend on the split: every floating-point sum keeps
// its sequential order, so results are bitwise independent of the thread count.
class RowPool {
 public:
  void resize(int n) {
    stop_all();
    n_ = std::max(1, n);
    const int g0 = gen_;  // new workers wait for the next dispatch, not the ones already done
    for (int t = 1; t < n_; ++t) th_.emplace_back([this, t, g0] { loop(t, g0); });
  }
  int size() const { return n_; }
  template <class F>
  void run(i64 rows, F&& f) {  // f(lo, hi) over n_ static chunks, chunk 0 on the caller
    if (n_ == 1 || rows < 4096) {
      f(i64(0), rows);
      return;
    }
    dispatch([&](int t) {
      const i64 chunk = (rows + n_ - 1) / n_;
      f(std::min(rows, t * chunk), std::min(rows, (t + 1) * chunk));
    });
  }
  // f(tid, lo, hi) over dynamically claimed chunks of `grain` items
  template <class F>
  void run_dyn(i64 n, i64 grain, F&& f) {
    grain = std::max<i64>(1, grain);
    if (n_ == 1 || n <= grain) {
      for (i64 lo = 0; lo < n; lo += grain) f(0, lo, std::min(n, lo + grain));
      return;
    }
    std::atomic<i64> next{0};
    dispatch([&](int t) {
      for (;;) {
        const i64 lo = next.fetch_add(grain);
        if (lo >= n) break;
        f(t, lo, std::min(n, lo + grain));
      }
    });
  }
  ~RowPool() { stop_all(); }

 private:
  void dispatch(const std::function<void(int)>& job) {
    {
      std::unique_lock<std::mutex> lk(m_);
      job_ = &job;
      pending_ = n_ - 1;
      ++gen_;
    }
    cv_.notify_all();
    job(0);
    std::unique_lock<std::mutex> lk(m_);
    done_.wait(lk, [&] { return pending_ == 0; });
    job_ = nullptr;
  }
  void loop(int t, int seen) {
    for (;;) {
      const std::function<void(int)>* job;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        job = job_;
      }
      (*job)(t);
      std::lock_guard<std::mutex> lk(m_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  void stop_all() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& x : th_) x.join();
    th_.clear();
    stop_ = false;
  }
  int n_ = 1, gen_ = 0, pending_ = 0;
  bool stop_ = false;
  const std::function<void(int)>* job_ = nullptr;
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_;
};
static RowPool& row_pool() {
  static RowPool p;
  return p;
}
// Multi-GB vectors are allocated and freed many times per Newton iteration (GMRES, V-cycles, AMG
// products).  glibc serves blocks above 32 MB with fresh mmaps, so each allocation page-faults
// its whole size again; keep them in the heap instead (performance only).
static const int g_malloc_tuned = [] {
  mallopt(M_MMAP_MAX, 0);
  mallopt(M_TRIM_THRESHOLD, -1);
  return 1;
}();
// elementwise loop i in [0, n): f(i), split over the pool (no reductions)
template <class F>
static void par_for(i64 n, F&& f) {
  row_pool().run(n, [&](i64 lo, i64 hi) {
    for (i64 i = lo; i < hi; ++i) f(i);
  });
}

static void spmv(const Csr& A, const double* x, double* y) {  // y = A x
  const int tpr = spmv_tpr(A);
  row_pool().run(A.rows, [&](i64 lo, i64 hi) {
    for (i64 i = lo; i < hi; ++i) y[i] = row_sum_lanes(A, i, x, tpr);
  });
}
static void spmv_add(const Csr& A, const double* x, double* y) {  // y += A x
  const int tpr = spmv_tpr(A);
  row_pool().run(A.rows, [&](i64 lo, i64 hi) {
    for (i64 i = lo; i < hi; ++i) y[i] = y[i] + row_sum_lanes(A, i, x, tpr);
  });
}

// Row-chunked CSR construction: rows [0, n) are produced by `emit(i, cols, vals)` (appending
// row i's entries) over dynamically claimed chunks, then concatenated in row order.
template <class Emit>
static Csr build_rows(i64 rows, i64 cols, i64 grain, Emit&& emit) {
  Csr C;
  C.rows = rows;
  C.cols = cols;
  C.ptr.assign(rows + 1, 0);
  const i64 nch = (rows + grain - 1) / grain;
  std::vector<std::vector<int>> ccol(nch);
  std::vector<std::vector<double>> cval(nch);
  row_pool().run_dyn(nch, 1, [&](int tid, i64 c0, i64 c1) {
    for (i64 c = c0; c < c1; ++c) {
      const i64 lo = c * grain, hi = std::min(rows, lo + grain);
      for (i64 i = lo; i < hi; ++i) {
        emit(tid, i, ccol[c], cval[c]);
        C.ptr[i + 1] = i64(ccol[c].size());  // chunk-local end, fixed below
      }
    }
  });
  std::vector<i64> base(nch + 1, 0);
  for (i64 c = 0; c < nch; ++c) base[c + 1] = base[c] + i64(ccol[c].size());
  par_for(rows, [&](i64 i) { C.ptr[i + 1] += base[i / grain]; });
  C.col.resize(base[nch]);
  C.val.resize(base[nch]);
  row_pool().run_dyn(nch, 1, [&](int, i64 c0, i64 c1) {
    for (i64 c = c0; c < c1; ++c) {
      std::copy(ccol[c].begin(), ccol[c].end(), C.col.begin() + base[c]);
      std::copy(cval[c].begin(), cval[c].end(), C.val.begin() + base[c]);
      std::vector<int>().swap(ccol[c]);
      std::vector<double>().swap(cval[c]);
    }
  });
  return C;
}

static Csr transpose(const Csr& A) {
  Csr T;
  T.rows = A.cols;
  T.cols = A.rows;
  T.ptr.assign(T.rows + 1, 0);
  T.col.resize(A.nnz());
  T.val.resize(A.nnz());
  const int nt = row_pool().size();
  if (nt == 1 || A.rows < 4096 || double(A.cols) * nt > 4e8) {
    for (i64 k = 0; k < A.nnz(); ++k) T.ptr[A.col[k] + 1]++;
    for (i64 i = 0; i < T.rows; ++i) T.ptr[i + 1] += T.ptr[i];
    std::vector<i64> pos(T.ptr.begin(), T.ptr.end() - 1);
    for (i64 i = 0; i < A.rows; ++i)
      for (i64 k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
        const i64 p = pos[A.col[k]]++;
        T.col[p] = int(i);
        T.val[p] = A.val[k];
      }
    return T;
  }
  // row chunks c = 0..nt-1; output row j lists chunk 0's entries, then chunk 1's, ... (each in
  // row order), i.e. ascending source row exactly as the serial counting sort
  const i64 chunk = (A.rows + nt - 1) / nt;
  std::vector<std::vector<i64>> cnt(nt, std::vector<i64>(A.cols, 0));
  row_pool().run_dyn(nt, 1, [&](int, i64 c0, i64) {
    auto& cc = cnt[c0];
    for (i64 i = c0 * chunk; i < std::min(A.rows, (c0 + 1) * chunk); ++i)
      for (i64 k = A.ptr[i]; k < A.ptr[i + 1]; ++k) cc[A.col[k]]++;
  });
  for (i64 j = 0; j < A.cols; ++j) {
    i64 run = T.ptr[j];
    for (int c = 0; c < nt; ++c) {
      const i64 n = cnt[c][j];
      cnt[c][j] = run;
      run += n;
    }
    T.ptr[j + 1] = run;
  }
  row_pool().run_dyn(nt, 1, [&](int, i64 c0, i64) {
    auto& pos = cnt[c0];
    for (i64 i = c0 * chunk; i < std::min(A.rows, (c0 + 1) * chunk); ++i)
      for (i64 k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
        const i64 p = pos[A.col[k]]++;
        T.col[p] = int(i);
        T.val[p] = A.val[k];
      }
  });
  return T;
}

// C = A * B, Gustavson: for each row i, for k in A.row(i) ascending, for j in B.row(k):
// C(i,j) += A(i,k) B(k,j).  Structural nonzeros are kept (no numeric pruning), columns sorted.
// Rows are independent, so the row-chunked parallel form is bitwise the serial one.
static Csr spgemm(const Csr& A, const Csr& B, const double* row_scale = nullptr) {
  const int nt = row_pool().size();
  std::vector<std::vector<i64>> marker(nt);
  std::vector<std::vector<double>> acc(nt);
  std::vector<std::vector<int>> cols(nt);
  return build_rows(A.rows, B.cols, 2048, [&](int t, i64 i, std::vector<int>& oc, std::vector<double>& ov) {
    auto& mk = marker[t];
    auto& ac = acc[t];
    auto& cl = cols[t];
    if (mk.empty()) {
      mk.assign(B.cols, -1);
      ac.assign(B.cols, 0.0);
    }
    cl.clear();
    for (i64 ka = A.ptr[i]; ka < A.ptr[i + 1]; ++ka) {
      const i64 k = A.col[ka];
      const double a = row_scale ? row_scale[i] * A.val[ka] : A.val[ka];  // (D^-1 A)(i,k) when scaled
      for (i64 kb = B.ptr[k]; kb < B.ptr[k + 1]; ++kb) {
        const int j = B.col[kb];
        if (mk[j] != i) {
          mk[j] = i;
          ac[j] = a * B.val[kb];
          cl.push_back(j);
        } else {
          ac[j] += a * B.val[kb];
        }
      }
    }
    std::sort(cl.begin(), cl.end());
    for (int j : cl) {
      oc.push_back(j);
      ov.push_back(ac[j]);
    }
  });
}

// Eigen SparseMatrix::prune(1.0, 1e-300): keep |v| > 1e-300
static void prune(Csr& A) {
  uvec<i64> cnt(A.rows + 1);
  cnt[0] = 0;
  par_for(A.rows, [&](i64 i) {
    i64 c = 0;
    for (i64 k = A.ptr[i]; k < A.ptr[i + 1]; ++k) c += std::abs(A.val[k]) > 1e-300;
    cnt[i + 1] = c;
  });
  for (i64 i = 0; i < A.rows; ++i) cnt[i + 1] += cnt[i];
  if (cnt[A.rows] == A.nnz()) return;
  Csr B;
  B.rows = A.rows;
  B.cols = A.cols;
  B.col.resize(cnt[A.rows]);
  B.val.resize(cnt[A.rows]);
  par_for(A.rows, [&](i64 i) {
    i64 w = cnt[i];
    for (i64 k = A.ptr[i]; k < A.ptr[i + 1]; ++k)
      if (std::abs(A.val[k]) > 1e-300) {
        B.col[w] = A.col[k];
        B.val[w] = A.val[k];
        ++w;
      }
  });
  B.ptr = std::move(cnt);
  A = std::move(B);
}

// ------------------------------------------------------------------ block system (linsolve.hpp:17-28)
struct BlockSystem {
  Csr uu, pu, pp;
  i64 n_u() const { return uu.rows; }
  i64 n_phi() const { return pp.rows; }
  Vec apply(const Vec& x) const {  // linsolve.cpp:13-19
    const i64 nu = n_u(), np = n_phi();
    Vec y(nu + np);
    spmv(uu, x.data(), y.data());
    // phi rows: one lane group per row over both blocks; the group size follows M_phiu's mean
    const int tpr = spmv_tpr(pu);
    row_pool().run(np, [&](i64 lo, i64 hi) {
      for (i64 i = lo; i < hi; ++i)
        y[nu + i] = row_sum_lanes(pu, i, x.data(), tpr) + row_sum_lanes(pp, i, x.data() + nu, tpr);
    });
    return y;
  }
};

// ------------------------------------------------------------------ assembly (model.cpp:127-322)
static void check_material(const orc_material& m) {  // model.cpp:8-17
  if (!(m.E > 0.0)) throw std::invalid_argument("Material: E must be positive");
  if (!(m.nu >= 0.0 && m.nu < 0.5)) throw std::invalid_argument("Material: nu must be in [0, 0.5)");
  if (!(m.G_c > 0.0)) throw std::invalid_argument("Material: G_c must be positive");
}

// Element residual from the corner values of one cell of edge h (the body of the cell loop,
// model.cpp:136-196): ru[k*d+a], rphi[k].  Shared by the uniform grid and the general meshes.
static void elem_residual(int d, const QpData& qp, const orc_material& mat, const orc_regularization& reg, double h,
                          double detJ, const double (*uloc)[3], const double* philoc, const double* ptloc, double* ru,
                          double* rphi) {
  const int nv = 1 << d;
  const double kap = reg.kappa, eps = reg.eps, p = mat.pressure, Gc = mat.G_c;
  const double mu = mat_mu(mat), lam = mat_lambda(mat);
  for (int i = 0; i < nv * d; ++i) ru[i] = 0.0;
  for (int i = 0; i < nv; ++i) rphi[i] = 0.0;
  for (int q = 0; q < qp.nq; ++q) {
    const double* s = qp.shape[q];
    double gu[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    double gphi[3] = {0, 0, 0};
    double phi = 0.0, pt = 0.0;
    for (int k = 0; k < nv; ++k) {
      phi += s[k] * philoc[k];
      pt += s[k] * ptloc[k];
      for (int b = 0; b < d; ++b) {
        gphi[b] += philoc[k] * qp.grads[q][k][b] / h;
        for (int a = 0; a < d; ++a) gu[a][b] += uloc[k][a] * qp.grads[q][k][b] / h;
      }
    }
    double e[3][3], sig[3][3];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) e[a][b] = 0.5 * (gu[a][b] + gu[b][a]);
    double tre = 0.0;
    for (int a = 0; a < d; ++a) tre += e[a][a];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) sig[a][b] = 2.0 * mu * e[a][b];
    for (int a = 0; a < d; ++a) sig[a][a] += lam * tre;
    double sig_ee = 0.0;
    for (int a = 0; a < d; ++a)
      for (int b = 0; b < d; ++b) sig_ee += sig[a][b] * e[a][b];
    const double gcoef = (1.0 - kap) * pt * pt + kap;
    const double pphi = (mat.pressure_coupling == 0) ? pt * pt : phi * phi;
    const double w = qp.wts[q] * detJ;
    for (int k = 0; k < nv; ++k) {
      for (int a = 0; a < d; ++a) {
        double val = 0.0;
        for (int b = 0; b < d; ++b) val += gcoef * sig[a][b] * qp.grads[q][k][b] / h;
        val += pphi * p * qp.grads[q][k][a] / h;
        ru[k * d + a] += w * val;
      }
      double vphi = ((1.0 - kap) * phi * sig_ee + 2.0 * phi * p * tre - Gc / eps * (1.0 - phi)) * s[k];
      for (int b = 0; b < d; ++b) vphi += Gc * eps * gphi[b] * qp.grads[q][k][b] / h;
      rphi[k] += w * vphi;
    }
  }
}

// Element residual of one cell of the uniform grid
static void cell_residual(const Grid& g, const QpData& qp, const orc_material& mat, const orc_regularization& reg,
                          const double* solution, const double* phi_tilde, i64 id, double* ru, double* rphi) {
  const int d = g.d, nv = 1 << d;
  const i64 nu = g.n_u();
  double uloc[8][3], philoc[8], ptloc[8];
  i64 verts[8];
  g.cell_vertices(id, verts);
  for (int k = 0; k < nv; ++k) {
    for (int a = 0; a < d; ++a) uloc[k][a] = solution[verts[k] * d + a];
    philoc[k] = solution[nu + verts[k]];
    ptloc[k] = phi_tilde[verts[k]];
  }
  elem_residual(d, qp, mat, reg, g.h, g.detJ, uloc, philoc, ptloc, ru, rphi);
}

static const QpData& qp_data(int d) {
  static const QpData q2 = make_qp_data(2), q3 = make_qp_data(3);
  return d == 2 ? q2 : q3;
}

// Cells incident to a vertex, in the reference cell order, with the vertex's corner index
struct CellRef {
  i64 rank, id;
  int k;
};
static int incident_cells(const Grid& g, i64 v, CellRef* out) {
  i64 x, y, z;
  g.vxyz(v, x, y, z);
  int n = 0;
  for (int k = 0; k < (1 << g.d); ++k) {
    const i64 cx = x - (k & 1), cy = y - ((k >> 1) & 1), cz = z - ((k >> 2) & 1);
    if (cx < 0 || cy < 0 || cz < 0 || cx >= g.nc || cy >= g.nc || (g.d == 3 && cz >= g.nc)) continue;
    const i64 id = g.cid(cx, cy, cz);
    out[n++] = CellRef{g.cell_rank[id], id, k};
  }
  for (int i = 1; i < n; ++i)
    for (int j = i; j > 0 && out[j].rank < out[j - 1].rank; --j) std::swap(out[j], out[j - 1]);
  return n;
}

// assemble_residual (model.cpp:127-202): the cell loop in the reference's cell order.
static Vec assemble_residual_seq(const Grid& g, const Constraints& cs, const orc_material& mat,
                                 const orc_regularization& reg, const double* solution, const double* phi_tilde) {
  const int d = g.d, nv = 1 << d;
  const QpData& qp = qp_data(d);
  const i64 nu = g.n_u();
  Vec R(g.n_total(), 0.0);
  double ru[24], rphi[8];
  i64 verts[8];
  for (i64 id : g.cell_order) {
    cell_residual(g, qp, mat, reg, solution, phi_tilde, id, ru, rphi);
    g.cell_vertices(id, verts);
    for (int k = 0; k < nv; ++k) {  // Scatter::vector_add (model.cpp:74-80); entry-free lines drop
      for (int a = 0; a < d; ++a) {
        const i64 dof = verts[k] * d + a;
        if (!cs.is(dof)) R[dof] += ru[k * d + a];
      }
      const i64 pd = nu + verts[k];
      if (!cs.is(pd)) R[pd] += rphi[k];
    }
  }
  return R;
}

// The same sums, thread-parallel: element residuals of every cell, then each dof adds its
// cells' contributions in the reference cell order (bitwise the cell loop).
static Vec assemble_residual_par(const Grid& g, const Constraints& cs, const orc_material& mat,
                                 const orc_regularization& reg, const double* solution, const double* phi_tilde) {
  const int d = g.d, nv = 1 << d, st = nv * (d + 1);
  const QpData& qp = qp_data(d);
  const i64 nu = g.n_u();
  std::vector<double> el(size_t(g.ncells) * st);
  row_pool().run_dyn(g.ncells, 1024, [&](int, i64 lo, i64 hi) {
    for (i64 id = lo; id < hi; ++id) {
      double* e = el.data() + size_t(id) * st;
      cell_residual(g, qp, mat, reg, solution, phi_tilde, id, e, e + nv * d);
    }
  });
  Vec R(g.n_total(), 0.0);
  row_pool().run_dyn(g.V, 4096, [&](int, i64 lo, i64 hi) {
    CellRef cells[8];
    for (i64 v = lo; v < hi; ++v) {
      const int n = incident_cells(g, v, cells);
      for (int a = 0; a <= d; ++a) {
        const i64 dof = (a < d) ? v * d + a : nu + v;
        if (cs.is(dof)) continue;
        double s = 0.0;
        for (int c = 0; c < n; ++c) {
          const double* e = el.data() + size_t(cells[c].id) * st;
          s += (a < d) ? e[cells[c].k * d + a] : e[nv * d + cells[c].k];
        }
        R[dof] = s;
      }
    }
  });
  return R;
}

static Vec assemble_residual(const Grid& g, const Constraints& cs, const orc_material& mat,
                             const orc_regularization& reg, const double* solution, const double* phi_tilde) {
  return row_pool().size() > 1 ? assemble_residual_par(g, cs, mat, reg, solution, phi_tilde)
                               : assemble_residual_seq(g, cs, mat, reg, solution, phi_tilde);
}

// Vertex neighbourhood (3^d, lexicographic = ascending vertex index)
static int vertex_neighbours(const Grid& g, i64 v, i64* out) {
  i64 x, y, z;
  g.vxyz(v, x, y, z);
  int n = 0;
  const int zlo = (g.d == 3) ? -1 : 0, zhi = (g.d == 3) ? 1 : 0;
  for (int dz = zlo; dz <= zhi; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const i64 X = x + dx, Y = y + dy, Z = z + dz;
        if (X < 0 || Y < 0 || Z < 0 || X >= g.nn || Y >= g.nn || (g.d == 3 && Z >= g.nn)) continue;
        out[n++] = g.vid(X, Y, Z);
      }
  return n;
}

// Pattern of the condensed element sparsity (the setFromTriplets pattern, model.cpp:294-319;
// equals assemble_pattern, linsolve.cpp:417-476, on entry-free constraint lines).  Constrained
// rows get a diagonal slot; it is removed afterwards when the summed diagonal is exactly 0
// (model.cpp:308-311 emits it only if != 0).
static void build_pattern(const Grid& g, const Constraints& cs, BlockSystem& J) {
  const int d = g.d;
  const i64 nu = g.n_u(), np = g.n_phi();
  J.uu.rows = J.uu.cols = nu;
  J.pu.rows = np;
  J.pu.cols = nu;
  J.pp.rows = J.pp.cols = np;
  J.uu.ptr.assign(nu + 1, 0);
  J.pu.ptr.assign(np + 1, 0);
  J.pp.ptr.assign(np + 1, 0);
  J.uu.col.clear(); J.pu.col.clear(); J.pp.col.clear();
  i64 nb[27];
  for (i64 v = 0; v < g.V; ++v) {
    const int n = vertex_neighbours(g, v, nb);
    for (int a = 0; a < d; ++a) {
      const i64 row = v * d + a;
      if (cs.is(row)) {
        J.uu.col.push_back(int(row));
      } else {
        for (int t = 0; t < n; ++t)
          for (int b = 0; b < d; ++b)
            if (!cs.is(nb[t] * d + b)) J.uu.col.push_back(int(nb[t] * d + b));
      }
      J.uu.ptr[row + 1] = i64(J.uu.col.size());
    }
    const i64 prow = nu + v;
    if (!cs.is(prow)) {
      for (int t = 0; t < n; ++t)
        for (int b = 0; b < d; ++b)
          if (!cs.is(nb[t] * d + b)) J.pu.col.push_back(int(nb[t] * d + b));
      for (int t = 0; t < n; ++t)
        if (!cs.is(nu + nb[t])) J.pp.col.push_back(int(nb[t]));
    } else {
      J.pp.col.push_back(int(v));
    }
    J.pu.ptr[v + 1] = i64(J.pu.col.size());
    J.pp.ptr[v + 1] = i64(J.pp.col.size());
  }
  J.uu.val.assign(J.uu.col.size(), 0.0);
  J.pu.val.assign(J.pu.col.size(), 0.0);
  J.pp.val.assign(J.pp.col.size(), 0.0);
}

static inline i64 find_slot(const Csr& A, i64 row, i64 col) {
  const int* b = A.col.data() + A.ptr[row];
  const int* e = A.col.data() + A.ptr[row + 1];
  const int* it = std::lower_bound(b, e, int(col));
  if (it == e || *it != col) throw std::logic_error("oracle: pattern slot missing");
  return i64(it - A.col.data());
}

static void drop_zero_constrained_diag(Csr& A, const Constraints& cs, i64 off) {
  bool any = false;
  for (i64 i = 0; i < A.rows; ++i)
    if (cs.is(off + i) && A.ptr[i + 1] - A.ptr[i] == 1 && A.val[A.ptr[i]] == 0.0) any = true;
  if (!any) return;
  Csr B;
  B.rows = A.rows;
  B.cols = A.cols;
  B.ptr.assign(A.rows + 1, 0);
  for (i64 i = 0; i < A.rows; ++i) {
    const bool drop = cs.is(off + i) && A.ptr[i + 1] - A.ptr[i] == 1 && A.val[A.ptr[i]] == 0.0;
    if (!drop)
      for (i64 k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
        B.col.push_back(A.col[k]);
        B.val.push_back(A.val[k]);
      }
    B.ptr[i + 1] = i64(B.col.size());
  }
  A = std::move(B);
}

// Element matrices of one cell of edge h (model.cpp:226-289): kuu, kpu, kpp (zeroed here).
static void elem_jacobian(int d, const QpData& qp, const orc_material& mat, const orc_regularization& reg, double h,
                          double detJ, const double (*uloc)[3], const double* philoc, const double* ptloc,
                          double (*kuu)[24], double (*kpu)[24], double (*kpp)[8]) {
  const int nv = 1 << d;
  const double kap = reg.kappa, eps = reg.eps, p = mat.pressure, Gc = mat.G_c;
  const double mu = mat_mu(mat), lam = mat_lambda(mat);
  double gphys[8][3];
  for (int i = 0; i < 24; ++i)
    for (int j = 0; j < 24; ++j) kuu[i][j] = 0.0;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 24; ++j) kpu[i][j] = 0.0;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) kpp[i][j] = 0.0;
  for (int q = 0; q < qp.nq; ++q) {
    const double* s = qp.shape[q];
    for (int k = 0; k < nv; ++k)
      for (int b = 0; b < 3; ++b) gphys[k][b] = (b < d) ? qp.grads[q][k][b] / h : 0.0;
    double gu[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    double phi = 0.0, pt = 0.0;
    for (int k = 0; k < nv; ++k) {
      phi += s[k] * philoc[k];
      pt += s[k] * ptloc[k];
      for (int b = 0; b < d; ++b)
        for (int a = 0; a < d; ++a) gu[a][b] += uloc[k][a] * gphys[k][b];
    }
    double e[3][3], sig[3][3];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) e[a][b] = 0.5 * (gu[a][b] + gu[b][a]);
    double tre = 0.0;
    for (int a = 0; a < d; ++a) tre += e[a][a];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) sig[a][b] = 2.0 * mu * e[a][b];
    for (int a = 0; a < d; ++a) sig[a][a] += lam * tre;
    double sig_ee = 0.0;
    for (int a = 0; a < d; ++a)
      for (int b = 0; b < d; ++b) sig_ee += sig[a][b] * e[a][b];
    const double gcoef = (1.0 - kap) * pt * pt + kap;
    const double w = qp.wts[q] * detJ;
    for (int k = 0; k < nv; ++k) {
      for (int l = 0; l < nv; ++l) {
        double gg = 0.0;
        for (int b = 0; b < d; ++b) gg += gphys[k][b] * gphys[l][b];
        for (int a = 0; a < d; ++a)
          for (int b = 0; b < d; ++b) {
            double val = mu * ((a == b ? gg : 0.0) + gphys[l][a] * gphys[k][b]) + lam * gphys[l][b] * gphys[k][a];
            kuu[k * d + a][l * d + b] += w * gcoef * val;
          }
        for (int b = 0; b < d; ++b) {
          double sgl = 0.0;
          for (int c = 0; c < d; ++c) sgl += sig[b][c] * gphys[l][c];
          kpu[k][l * d + b] += w * (2.0 * (1.0 - kap) * phi * sgl + 2.0 * p * phi * gphys[l][b]) * s[k];
        }
        kpp[k][l] += w * (((1.0 - kap) * sig_ee + 2.0 * p * tre + Gc / eps) * s[l] * s[k] + Gc * eps * gg);
      }
    }
  }
}

static BlockSystem assemble_jacobian_seq(const Grid& g, const Constraints& cs, const orc_material& mat,
                                         const orc_regularization& reg, const double* solution,
                                         const double* phi_tilde) {
  const int d = g.d, nv = 1 << d;
  static thread_local QpData qp2, qp3;
  QpData& qp = (d == 2) ? qp2 : qp3;
  if (qp.nq == 0) qp = make_qp_data(d);
  const i64 nu = g.n_u();
  BlockSystem J;
  build_pattern(g, cs, J);
  double uloc[8][3], philoc[8], ptloc[8];
  double kuu[24][24], kpu[8][24], kpp[8][8];
  i64 verts[8], udofs[24], pdofs[8];
  for (i64 id : g.cell_order) {
    g.cell_vertices(id, verts);
    for (int k = 0; k < nv; ++k) {
      for (int a = 0; a < d; ++a) uloc[k][a] = solution[verts[k] * d + a];
      philoc[k] = solution[nu + verts[k]];
      ptloc[k] = phi_tilde[verts[k]];
    }
    elem_jacobian(d, qp, mat, reg, g.h, g.detJ, uloc, philoc, ptloc, kuu, kpu, kpp);
    for (int k = 0; k < nv; ++k) {
      for (int a = 0; a < d; ++a) udofs[k * d + a] = verts[k] * d + a;
      pdofs[k] = nu + verts[k];
    }
    // Scatter::matrix_add with entry-free lines: constrained rows/cols drop, constrained
    // diagonals accumulate separately (model.cpp:294-305).  Accumulating straight into the
    // pattern in cell order == setFromTriplets' duplicate summation in insertion order.
    for (int i = 0; i < nv * d; ++i) {
      const i64 ri = udofs[i];
      if (cs.is(ri)) {
        J.uu.val[J.uu.ptr[ri]] += kuu[i][i];
        continue;
      }
      for (int j = 0; j < nv * d; ++j) {
        if (cs.is(udofs[j])) continue;
        J.uu.val[find_slot(J.uu, ri, udofs[j])] += kuu[i][j];
      }
    }
    for (int i = 0; i < nv; ++i) {
      const i64 ri = pdofs[i];
      if (cs.is(ri)) {
        J.pp.val[J.pp.ptr[ri - nu]] += kpp[i][i];
        continue;
      }
      for (int j = 0; j < nv * d; ++j) {
        if (cs.is(udofs[j])) continue;
        J.pu.val[find_slot(J.pu, ri - nu, udofs[j])] += kpu[i][j];
      }
      for (int j = 0; j < nv; ++j) {
        if (cs.is(pdofs[j])) continue;
        J.pp.val[find_slot(J.pp, ri - nu, pdofs[j] - nu)] += kpp[i][j];
      }
    }
  }
  drop_zero_constrained_diag(J.uu, cs, 0);
  drop_zero_constrained_diag(J.pp, cs, nu);
  return J;
}

// Pattern rows of one vertex (the serial build_pattern's rule): uu rows v*d+a, the pu and pp rows
// of the phi dof; returns the entries written (cols may be null to count only).
static void pattern_rows(const Grid& g, const Constraints& cs, i64 v, int* uu_cols, i64* uu_len, int* pu_cols,
                         i64* pu_len, int* pp_cols, i64* pp_len) {
  const int d = g.d;
  const i64 nu = g.n_u();
  i64 nb[27];
  const int n = vertex_neighbours(g, v, nb);
  for (int a = 0; a < d; ++a) {
    const i64 row = v * d + a;
    i64 c = 0;
    if (cs.is(row)) {
      if (uu_cols) uu_cols[c] = int(row);
      ++c;
    } else {
      for (int t = 0; t < n; ++t)
        for (int b = 0; b < d; ++b)
          if (!cs.is(nb[t] * d + b)) {
            if (uu_cols) uu_cols[c] = int(nb[t] * d + b);
            ++c;
          }
    }
    uu_len[a] = c;
    if (uu_cols) uu_cols += c;
  }
  i64 cp = 0, cq = 0;
  if (!cs.is(nu + v)) {
    for (int t = 0; t < n; ++t)
      for (int b = 0; b < d; ++b)
        if (!cs.is(nb[t] * d + b)) {
          if (pu_cols) pu_cols[cp] = int(nb[t] * d + b);
          ++cp;
        }
    for (int t = 0; t < n; ++t)
      if (!cs.is(nu + nb[t])) {
        if (pp_cols) pp_cols[cq] = int(nb[t]);
        ++cq;
      }
  } else {
    if (pp_cols) pp_cols[0] = int(v);
    cq = 1;
  }
  *pu_len = cp;
  *pp_len = cq;
}

static void build_pattern_par(const Grid& g, const Constraints& cs, BlockSystem& J) {
  const int d = g.d;
  const i64 nu = g.n_u(), np = g.n_phi();
  J.uu.rows = J.uu.cols = nu;
  J.pu.rows = np;
  J.pu.cols = nu;
  J.pp.rows = J.pp.cols = np;
  J.uu.ptr.assign(nu + 1, 0);
  J.pu.ptr.assign(np + 1, 0);
  J.pp.ptr.assign(np + 1, 0);
  par_for(g.V, [&](i64 v) {
    i64 ul[3], pl, ql;
    pattern_rows(g, cs, v, nullptr, ul, nullptr, &pl, nullptr, &ql);
    for (int a = 0; a < d; ++a) J.uu.ptr[v * d + a + 1] = ul[a];
    J.pu.ptr[v + 1] = pl;
    J.pp.ptr[v + 1] = ql;
  });
  for (i64 i = 0; i < nu; ++i) J.uu.ptr[i + 1] += J.uu.ptr[i];
  for (i64 i = 0; i < np; ++i) {
    J.pu.ptr[i + 1] += J.pu.ptr[i];
    J.pp.ptr[i + 1] += J.pp.ptr[i];
  }
  J.uu.col.resize(J.uu.ptr[nu]);
  J.pu.col.resize(J.pu.ptr[np]);
  J.pp.col.resize(J.pp.ptr[np]);
  J.uu.val.resize(J.uu.col.size());
  J.pu.val.resize(J.pu.col.size());
  J.pp.val.resize(J.pp.col.size());
  par_for(g.V, [&](i64 v) {  // columns and zeroed values, first-touched by the owning thread
    i64 ul[3], pl, ql;
    pattern_rows(g, cs, v, J.uu.col.data() + J.uu.ptr[v * d], ul, J.pu.col.data() + J.pu.ptr[v], &pl,
                 J.pp.col.data() + J.pp.ptr[v], &ql);
    std::fill(J.uu.val.begin() + J.uu.ptr[v * d], J.uu.val.begin() + J.uu.ptr[(v + 1) * d], 0.0);
    std::fill(J.pu.val.begin() + J.pu.ptr[v], J.pu.val.begin() + J.pu.ptr[v + 1], 0.0);
    std::fill(J.pp.val.begin() + J.pp.ptr[v], J.pp.val.begin() + J.pp.ptr[v + 1], 0.0);
  });
}

// assemble_jacobian, thread-parallel: each vertex owns its u and phi rows and adds, cell by cell in
// the reference cell order, its corner's rows of the element matrices (the same expressions as the
// cell loop, so every entry is the same sequence of IEEE additions).
static BlockSystem assemble_jacobian_par(const Grid& g, const Constraints& cs, const orc_material& mat,
                                         const orc_regularization& reg, const double* solution,
                                         const double* phi_tilde) {
  const int d = g.d, nv = 1 << d;
  const double kap = reg.kappa, eps = reg.eps, p = mat.pressure, Gc = mat.G_c;
  const double mu = mat_mu(mat), lam = mat_lambda(mat);
  const QpData& qp = qp_data(d);
  const i64 nu = g.n_u();
  BlockSystem J;
  build_pattern_par(g, cs, J);
  const double h = g.h, detJ = g.detJ;
  row_pool().run_dyn(g.V, 512, [&](int, i64 lo, i64 hi) {
    CellRef cells[8];
    double uloc[8][3], philoc[8], ptloc[8];
    double kuu[3][24], kpu[24], kpp[8], gphys[8][3];
    i64 verts[8], udofs[24], pdofs[8];
    for (i64 v = lo; v < hi; ++v) {
      const int nc = incident_cells(g, v, cells);
      for (int ci = 0; ci < nc; ++ci) {
        const i64 id = cells[ci].id;
        const int k = cells[ci].k;
        g.cell_vertices(id, verts);
        for (int kk = 0; kk < nv; ++kk) {
          for (int a = 0; a < d; ++a) uloc[kk][a] = solution[verts[kk] * d + a];
          philoc[kk] = solution[nu + verts[kk]];
          ptloc[kk] = phi_tilde[verts[kk]];
        }
        std::memset(kuu, 0, sizeof(kuu));
        std::memset(kpu, 0, sizeof(kpu));
        std::memset(kpp, 0, sizeof(kpp));
        for (int q = 0; q < qp.nq; ++q) {
          const double* s = qp.shape[q];
          for (int kk = 0; kk < nv; ++kk)
            for (int b = 0; b < 3; ++b) gphys[kk][b] = (b < d) ? qp.grads[q][kk][b] / h : 0.0;
          double gu[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
          double phi = 0.0, pt = 0.0;
          for (int kk = 0; kk < nv; ++kk) {
            phi += s[kk] * philoc[kk];
            pt += s[kk] * ptloc[kk];
            for (int b = 0; b < d; ++b)
              for (int a = 0; a < d; ++a) gu[a][b] += uloc[kk][a] * gphys[kk][b];
          }
          double e[3][3], sig[3][3];
          for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) e[a][b] = 0.5 * (gu[a][b] + gu[b][a]);
          double tre = 0.0;
          for (int a = 0; a < d; ++a) tre += e[a][a];
          for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) sig[a][b] = 2.0 * mu * e[a][b];
          for (int a = 0; a < d; ++a) sig[a][a] += lam * tre;
          double sig_ee = 0.0;
          for (int a = 0; a < d; ++a)
            for (int b = 0; b < d; ++b) sig_ee += sig[a][b] * e[a][b];
          const double gcoef = (1.0 - kap) * pt * pt + kap;
          const double w = qp.wts[q] * detJ;
          for (int l = 0; l < nv; ++l) {
            double gg = 0.0;
            for (int b = 0; b < d; ++b) gg += gphys[k][b] * gphys[l][b];
            for (int a = 0; a < d; ++a)
              for (int b = 0; b < d; ++b) {
                double val = mu * ((a == b ? gg : 0.0) + gphys[l][a] * gphys[k][b]) + lam * gphys[l][b] * gphys[k][a];
                kuu[a][l * d + b] += w * gcoef * val;
              }
            for (int b = 0; b < d; ++b) {
              double sgl = 0.0;
              for (int c = 0; c < d; ++c) sgl += sig[b][c] * gphys[l][c];
              kpu[l * d + b] += w * (2.0 * (1.0 - kap) * phi * sgl + 2.0 * p * phi * gphys[l][b]) * s[k];
            }
            kpp[l] += w * (((1.0 - kap) * sig_ee + 2.0 * p * tre + Gc / eps) * s[l] * s[k] + Gc * eps * gg);
          }
        }
        for (int kk = 0; kk < nv; ++kk) {
          for (int a = 0; a < d; ++a) udofs[kk * d + a] = verts[kk] * d + a;
          pdofs[kk] = nu + verts[kk];
        }
        for (int a = 0; a < d; ++a) {
          const i64 ri = udofs[k * d + a];
          if (cs.is(ri)) {
            J.uu.val[J.uu.ptr[ri]] += kuu[a][k * d + a];
            continue;
          }
          for (int j = 0; j < nv * d; ++j) {
            if (cs.is(udofs[j])) continue;
            J.uu.val[find_slot(J.uu, ri, udofs[j])] += kuu[a][j];
          }
        }
        const i64 ri = pdofs[k];
        if (cs.is(ri)) {
          J.pp.val[J.pp.ptr[ri - nu]] += kpp[k];
          continue;
        }
        for (int j = 0; j < nv * d; ++j) {
          if (cs.is(udofs[j])) continue;
          J.pu.val[find_slot(J.pu, ri - nu, udofs[j])] += kpu[j];
        }
        for (int j = 0; j < nv; ++j) {
          if (cs.is(pdofs[j])) continue;
          J.pp.val[find_slot(J.pp, ri - nu, pdofs[j] - nu)] += kpp[j];
        }
      }
    }
  });
  drop_zero_constrained_diag(J.uu, cs, 0);
  drop_zero_constrained_diag(J.pp, cs, nu);
  return J;
}

static BlockSystem assemble_jacobian(const Grid& g, const Constraints& cs, const orc_material& mat,
                                     const orc_regularization& reg, const double* solution,
                                     const double* phi_tilde) {
  return row_pool().size() > 1 ? assemble_jacobian_par(g, cs, mat, reg, solution, phi_tilde)
                               : assemble_jacobian_seq(g, cs, mat, reg, solution, phi_tilde);
}

// ------------------------------------------------------------------ GMRES (linsolve.cpp:21-115)
using Op = std::function<Vec(const Vec&)>;
struct GmresResult {
  Vec x;
  int iterations = 0;
  bool converged = false, breakdown = false;
  double residual = 0.0;
  std::vector<double> history;
};
static double tree256(double* sh) {  // in-place block tree of 256 values
  for (int s = 128; s > 0; s >>= 1)
    for (int t = 0; t < s; ++t) sh[t] += sh[t + s];
  return sh[0];
}
// The Newton step's dots and norms in the product order (the device's SegLayout, cf_vec.hpp):
// each vertex plane's u part and phi part is cut into chunks of 8192 entries, a chunk is reduced
// by 256 lanes (lane t: entries t, t+256, ... sequentially, then the block tree), and the chunk
// partials, u planes then phi planes, go through the fixed final tree.  This order does not depend
// on how the planes are split over ranks, which makes the multi-GPU step bitwise the 1-GPU step.
struct SegDot {
  bool on = false;
  i64 plane_u = 0, plane_p = 0, chunk = 8192, n = 0;
  int nplanes = 0;
};
static SegDot g_seg;
struct SegScope {  // segmented dots for block vectors of the grid while in scope
  SegDot prev;
  SegScope(const Grid& g) : prev(g_seg) {
    const i64 plane = (g.d == 3) ? g.nn * g.nn : g.nn;
    g_seg.on = true;
    g_seg.plane_u = g.d * plane;
    g_seg.plane_p = plane;
    g_seg.nplanes = int(g.nn);
    g_seg.n = g.n_total();
  }
  ~SegScope() { g_seg = prev; }
};
static double seg_dot(const Vec& a, const Vec& b) {
  const SegDot& L = g_seg;
  const int cu = int((L.plane_u + L.chunk - 1) / L.chunk), cp = int((L.plane_p + L.chunk - 1) / L.chunk);
  const i64 np = i64(L.nplanes) * (cu + cp);
  std::vector<double> G(np);
  row_pool().run_dyn(np, 16, [&](int, i64 lo, i64 hi) {
    double sh[256];
    for (i64 gi = lo; gi < hi; ++gi) {
      i64 start, len;
      if (gi < i64(L.nplanes) * cu) {
        const i64 p = gi / cu, c = gi % cu;
        start = p * L.plane_u + c * L.chunk;
        len = std::min(L.chunk, L.plane_u - c * L.chunk);
      } else {
        const i64 q = gi - i64(L.nplanes) * cu, p = q / cp, c = q % cp;
        start = i64(L.nplanes) * L.plane_u + p * L.plane_p + c * L.chunk;
        len = std::min(L.chunk, L.plane_p - c * L.chunk);
      }
      for (int t = 0; t < 256; ++t) {
        double s = 0.0;
        for (i64 i = t; i < len; i += 256) s += a[start + i] * b[start + i];
        sh[t] = s;
      }
      G[gi] = tree256(sh);
    }
  });
  double sh[256];
  for (int t = 0; t < 256; ++t) {
    double s = 0.0;
    for (i64 bk = t; bk < np; bk += 256) s += G[bk];
    sh[t] = s;
  }
  return tree256(sh);
}

static double dot(const Vec& a, const Vec& b) {
  const i64 n = i64(a.size());
  if (g_order == ORDER_REFERENCE) {  // a.dot(b): one sequential sum
    double s = 0.0;
    for (i64 i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
  }
  if (g_seg.on && n == g_seg.n) return seg_dot(a, b);
  // fixed block-tree order (the device's k_dot_partial / k_final)
  const i64 nb = std::min<i64>(1024, std::max<i64>(1, (n + 4 * 256 - 1) / (4 * 256)));
  std::vector<double> part(nb);
  row_pool().run_dyn(nb, 8, [&](int, i64 b0, i64 b1) {
    double sh[256];
    for (i64 bk = b0; bk < b1; ++bk) {
      for (int t = 0; t < 256; ++t) {
        double s = 0.0;
        for (i64 i = bk * 256 + t; i < n; i += nb * 256) s += a[i] * b[i];
        sh[t] = s;
      }
      part[bk] = tree256(sh);
    }
  });
  double sh[256];
  for (int t = 0; t < 256; ++t) {
    double s = 0.0;
    for (i64 bk = t; bk < nb; bk += 256) s += part[bk];
    sh[t] = s;
  }
  return tree256(sh);
}
static double norm(const Vec& a) { return std::sqrt(dot(a, a)); }

static GmresResult gmres(const Op& op, const Op& prec, const Vec& rhs, const orc_gmres_options& o) {
  if (!(o.rtol > 0.0 && o.rtol < 1.0)) throw std::invalid_argument("gmres: rtol must be in (0,1)");
  const size_t n = rhs.size();
  Op M = prec ? prec : Op([](const Vec& v) { return v; });
  GmresResult res;
  res.x.assign(n, 0.0);
  const double bnorm = norm(rhs);
  if (bnorm == 0.0) {
    res.converged = true;
    return res;
  }
  Vec r = rhs;
  while (res.iterations < o.max_iter) {
    const double beta = norm(r);
    if (beta <= o.rtol * bnorm) {
      res.converged = true;
      res.residual = beta / bnorm;
      return res;
    }
    const int m = std::min(o.restart, o.max_iter - res.iterations);
    std::vector<Vec> V(m + 1);
    std::vector<double> H(size_t(m + 1) * m, 0.0);
    auto Hij = [&](int i, int j) -> double& { return H[size_t(i) * m + j]; };
    Vec cs(m, 0.0), sn(m, 0.0), gv(m + 1, 0.0);
    gv[0] = beta;
    V[0].resize(n);
    par_for(i64(n), [&](i64 i) { V[0][i] = r[i] / beta; });
    int j = 0;
    bool inner_done = false;
    for (; j < m && !inner_done; ++j) {
      Vec w = op(M(V[j]));
      for (int i = 0; i <= j; ++i) {  // MGS
        Hij(i, j) = dot(w, V[i]);
        const double hij = Hij(i, j);
        const Vec& Vi = V[i];
        par_for(i64(n), [&](i64 t) { w[t] -= hij * Vi[t]; });
      }
      Hij(j + 1, j) = norm(w);
      const bool happy = Hij(j + 1, j) <= 1e-14 * bnorm;
      if (!happy) {
        V[j + 1].resize(n);
        const double hn = Hij(j + 1, j);
        Vec& Vn = V[j + 1];
        par_for(i64(n), [&](i64 t) { Vn[t] = w[t] / hn; });
      }
      for (int i = 0; i < j; ++i) {
        double t = cs[i] * Hij(i, j) + sn[i] * Hij(i + 1, j);
        Hij(i + 1, j) = -sn[i] * Hij(i, j) + cs[i] * Hij(i + 1, j);
        Hij(i, j) = t;
      }
      const double denom = std::hypot(Hij(j, j), Hij(j + 1, j));
      if (denom == 0.0) {
        res.breakdown = true;
        inner_done = true;
        --j;
        break;
      }
      cs[j] = Hij(j, j) / denom;
      sn[j] = Hij(j + 1, j) / denom;
      Hij(j, j) = denom;
      Hij(j + 1, j) = 0.0;
      gv[j + 1] = -sn[j] * gv[j];
      gv[j] = cs[j] * gv[j];
      ++res.iterations;
      const double rel = std::abs(gv[j + 1]) / bnorm;
      res.history.push_back(rel);
      if (rel <= o.rtol || happy || res.iterations >= o.max_iter) inner_done = true;
    }
    const int k = j;
    if (k > 0) {
      Vec y(k);
      for (int i = k - 1; i >= 0; --i) {
        double s = gv[i];
        for (int l = i + 1; l < k; ++l) s -= Hij(i, l) * y[l];
        if (Hij(i, i) == 0.0) {
          res.breakdown = true;
          y[i] = 0.0;
        } else {
          y[i] = s / Hij(i, i);
        }
      }
      Vec z(n, 0.0);
      par_for(i64(n), [&](i64 t) {  // V.leftCols(k) * y
        double s = 0.0;
        for (int l = 0; l < k; ++l) s += V[l][t] * y[l];
        z[t] = s;
      });
      Vec mz = M(z);
      par_for(i64(n), [&](i64 t) { res.x[t] += mz[t]; });
    }
    Vec ax = op(res.x);
    par_for(i64(n), [&](i64 t) { r[t] = rhs[t] - ax[t]; });
    res.residual = norm(r) / bnorm;
    if (res.residual <= o.rtol) {
      res.converged = true;
      return res;
    }
    if (res.breakdown) return res;
  }
  res.residual = norm(r) / bnorm;
  return res;
}

// ------------------------------------------------------------------ dense helpers
struct Dense {  // column-major
  i64 rows = 0, cols = 0;
  std::vector<double> a;
  Dense() = default;
  Dense(i64 r, i64 c) : rows(r), cols(c), a(size_t(r * c), 0.0) {}
  double& operator()(i64 i, i64 j) { return a[size_t(j * rows + i)]; }
  double operator()(i64 i, i64 j) const { return a[size_t(j * rows + i)]; }
};

// Eigen PartialPivLU, unblocked right-looking variant (Eigen's blocked variant for >16
// rows reorders the same updates; not reproduced bit-for-bit).
struct Lu {
  Dense lu;
  std::vector<i64> piv;  // row transpositions
  void factor(const Dense& A) {
    lu = A;
    const i64 n = A.rows;
    piv.assign(n, 0);
    for (i64 k = 0; k < n; ++k) {
      i64 p = k;
      double big = std::abs(lu(k, k));
      for (i64 i = k + 1; i < n; ++i)
        if (std::abs(lu(i, k)) > big) {
          big = std::abs(lu(i, k));
          p = i;
        }
      piv[k] = p;
      if (big != 0.0) {
        if (p != k)
          for (i64 j = 0; j < n; ++j) std::swap(lu(k, j), lu(p, j));
        for (i64 i = k + 1; i < n; ++i) lu(i, k) /= lu(k, k);
      }
      for (i64 j = k + 1; j < n; ++j)
        for (i64 i = k + 1; i < n; ++i) lu(i, j) -= lu(i, k) * lu(k, j);
    }
  }
  double min_abs_pivot() const {
    double m = INFINITY;
    for (i64 i = 0; i < lu.rows; ++i) m = std::min(m, std::abs(lu(i, i)));
    return m;
  }
  Vec solve(const Vec& b) const {
    const i64 n = lu.rows;
    Vec x = b;
    for (i64 k = 0; k < n; ++k)
      if (piv[k] != k) std::swap(x[k], x[piv[k]]);
    for (i64 i = 0; i < n; ++i)
      for (i64 j = 0; j < i; ++j) x[i] -= lu(i, j) * x[j];
    for (i64 i = n - 1; i >= 0; --i) {
      for (i64 j = i + 1; j < n; ++j) x[i] -= lu(i, j) * x[j];
      x[i] /= lu(i, i);
    }
    return x;
  }
};

// Eigen ColPivHouseholderQR (3.3 computeInPlace), threshold set via setThreshold().
struct ColPivQR {
  Dense qr;
  std::vector<double> hc;
  std::vector<i64> perm;  // colsPermutation indices: AP(:,k) = A(:,perm[k])
  i64 nonzero_pivots = 0;
  double maxpivot = 0.0;

  static double colnorm(const Dense& M, i64 j, i64 r0) {
    double s = 0.0;
    for (i64 i = r0; i < M.rows; ++i) s += M(i, j) * M(i, j);
    return std::sqrt(s);
  }

  void compute(const Dense& A) {
    qr = A;
    const i64 rows = A.rows, cols = A.cols, size = std::min(rows, cols);
    hc.assign(size, 0.0);
    std::vector<i64> transp(cols, 0);
    std::vector<double> upd(cols), dir(cols), temp(cols, 0.0);
    for (i64 k = 0; k < cols; ++k) {
      dir[k] = colnorm(qr, k, 0);
      upd[k] = dir[k];
    }
    double mx = 0.0;
    for (i64 k = 0; k < cols; ++k) mx = (k == 0 || upd[k] > mx) ? upd[k] : mx;
    const double th_helper = (mx * DBL_EPSILON) * (mx * DBL_EPSILON) / double(rows);
    const double ndt = std::sqrt(DBL_EPSILON);
    nonzero_pivots = size;
    maxpivot = 0.0;
    for (i64 k = 0; k < size; ++k) {
      i64 bi = k;
      double bv = upd[k];
      for (i64 j = k + 1; j < cols; ++j)
        if (upd[j] > bv) {
          bv = upd[j];
          bi = j;
        }
      const double bsq = bv * bv;
      if (nonzero_pivots == size && bsq < th_helper * double(rows - k)) nonzero_pivots = k;
      transp[k] = bi;
      if (k != bi) {
        for (i64 i = 0; i < rows; ++i) std::swap(qr(i, k), qr(i, bi));
        std::swap(upd[k], upd[bi]);
        std::swap(dir[k], dir[bi]);
      }
      // makeHouseholderInPlace on qr(k:rows, k)
      double beta, tau;
      {
        const double c0 = qr(k, k);
        double tsq = 0.0;
        for (i64 i = k + 1; i < rows; ++i) tsq += qr(i, k) * qr(i, k);
        if (tsq <= DBL_MIN) {
          tau = 0.0;
          beta = c0;
          for (i64 i = k + 1; i < rows; ++i) qr(i, k) = 0.0;
        } else {
          beta = std::sqrt(c0 * c0 + tsq);
          if (c0 >= 0.0) beta = -beta;
          for (i64 i = k + 1; i < rows; ++i) qr(i, k) = qr(i, k) / (c0 - beta);
          tau = (beta - c0) / beta;
        }
      }
      hc[k] = tau;
      qr(k, k) = beta;
      if (std::abs(beta) > maxpivot) maxpivot = std::abs(beta);
      // applyHouseholderOnTheLeft to qr(k:rows, k+1:cols)
      for (i64 j = k + 1; j < cols; ++j) {
        if (rows - k == 1) {
          qr(k, j) *= (1.0 - tau);
        } else if (tau != 0.0) {
          double t = 0.0;
          for (i64 i = k + 1; i < rows; ++i) t += qr(i, k) * qr(i, j);
          t += qr(k, j);
          qr(k, j) -= tau * t;
          for (i64 i = k + 1; i < rows; ++i) qr(i, j) -= (tau * qr(i, k)) * t;
        }
      }
      for (i64 j = k + 1; j < cols; ++j) {
        if (upd[j] != 0.0) {
          double tmp = std::abs(qr(k, j)) / upd[j];
          tmp = (1.0 + tmp) * (1.0 - tmp);
          tmp = tmp < 0.0 ? 0.0 : tmp;
          const double ratio = upd[j] / dir[j];
          const double tmp2 = tmp * (ratio * ratio);
          if (tmp2 <= ndt) {
            dir[j] = colnorm(qr, j, k + 1);
            upd[j] = dir[j];
          } else {
            upd[j] *= std::sqrt(tmp);
          }
        }
      }
    }
    perm.resize(cols);
    for (i64 k = 0; k < cols; ++k) perm[k] = k;
    for (i64 k = 0; k < size; ++k) std::swap(perm[k], perm[transp[k]]);
  }

  i64 rank(double threshold) const {
    const double pt = std::abs(maxpivot) * threshold;
    i64 r = 0;
    for (i64 i = 0; i < nonzero_pivots; ++i) r += (std::abs(qr(i, i)) > pt);
    return r;
  }

  // Column c of householderQ(): H_0 ... H_{size-1} e_c, applied in reverse (HouseholderSequence::evalTo)
  void q_column(i64 c, double* out) const {
    const i64 rows = qr.rows, size = std::min(qr.rows, qr.cols);
    for (i64 i = 0; i < rows; ++i) out[i] = (i == c) ? 1.0 : 0.0;
    for (i64 k = size - 1; k >= 0; --k) {
      const double tau = hc[k];
      if (rows - k == 1) {
        out[k] *= (1.0 - tau);
      } else if (tau != 0.0) {
        double t = 0.0;
        for (i64 i = k + 1; i < rows; ++i) t += qr(i, k) * out[i];
        t += out[k];
        out[k] -= tau * t;
        for (i64 i = k + 1; i < rows; ++i) out[i] -= (tau * qr(i, k)) * t;
      }
    }
  }
};

// ------------------------------------------------------------------ AMG (linsolve.cpp:117-318)
struct AmgLevel {
  Csr A, P, Pt;
  Vec inv_diag;
  double jacobi_weight = 2.0 / 3.0;
  // diagnostics for parity
  i64 n_nodes = 0, n_aggregates = 0;
  std::vector<int> agg_of_node;
  double lambda = 0.0;
};
struct Amg {
  std::vector<AmgLevel> levels;
  Lu coarse;
  i64 coarse_n = 0;
  orc_amg_options opts;
  std::vector<i64> stop_info;  // per-level strong edges (diagnostic)
  void cycle(size_t lev, const Vec& b, Vec& x) const {  // linsolve.cpp:295-312
    if (lev == levels.size()) {
      x = coarse_n > 0 ? coarse.solve(b) : Vec();
      return;
    }
    const AmgLevel& L = levels[lev];
    const double w = L.jacobi_weight;
    const i64 n = L.A.rows;
    x.assign(n, 0.0);
    par_for(n, [&](i64 i) { x[i] = w * (L.inv_diag[i] * b[i]); });
    Vec ax(n);
    for (int s = 1; s < opts.smoothing_sweeps; ++s) {
      spmv(L.A, x.data(), ax.data());
      par_for(n, [&](i64 i) { x[i] += w * (L.inv_diag[i] * (b[i] - ax[i])); });
    }
    spmv(L.A, x.data(), ax.data());
    Vec r(n);
    par_for(n, [&](i64 i) { r[i] = b[i] - ax[i]; });
    Vec bc(L.P.cols);
    spmv(L.Pt, r.data(), bc.data());
    Vec xc;
    cycle(lev + 1, bc, xc);
    spmv_add(L.P, xc.data(), x.data());
    for (int s = 0; s < opts.smoothing_sweeps; ++s) {
      spmv(L.A, x.data(), ax.data());
      par_for(n, [&](i64 i) { x[i] += w * (L.inv_diag[i] * (b[i] - ax[i])); });
    }
  }
  Vec vcycle(const Vec& r) const {
    Vec x;
    cycle(0, r, x);
    return x;
  }
};

static double estimate_lambda_max(const Csr& A, const Vec& inv_diag) {  // linsolve.cpp:120-134
  const i64 n = A.rows;
  Vec v(n), w(n);
  for (i64 i = 0; i < n; ++i) v[i] = 1.0 + 0.5 * std::sin(1.0 + double(i));
  const double nv = norm(v);
  for (auto& t : v) t /= nv;
  double lambda = 1.0;
  for (int it = 0; it < 15; ++it) {
    spmv(A, v.data(), w.data());
    par_for(n, [&](i64 i) { w[i] = inv_diag[i] * w[i]; });
    const double nw = norm(w);
    if (nw == 0.0) return 1.0;
    lambda = nw;
    par_for(n, [&](i64 i) { v[i] = w[i] / nw; });
  }
  return std::max(lambda, 1e-12);
}

struct Aggregation {
  std::vector<int> agg_of_node;
  int n_aggregates = 0;
};
static Aggregation aggregate_nodes(int n_nodes, const std::vector<std::vector<int>>& strong) {  // linsolve.cpp:142-166
  Aggregation agg;
  agg.agg_of_node.assign(n_nodes, -1);
  for (int i = 0; i < n_nodes; ++i) {
    if (agg.agg_of_node[i] >= 0) continue;
    bool fr = true;
    for (int j : strong[i])
      if (agg.agg_of_node[j] >= 0) { fr = false; break; }
    if (!fr) continue;
    const int a = agg.n_aggregates++;
    agg.agg_of_node[i] = a;
    for (int j : strong[i]) agg.agg_of_node[j] = a;
  }
  for (int i = 0; i < n_nodes; ++i) {
    if (agg.agg_of_node[i] >= 0) continue;
    for (int j : strong[i])
      if (agg.agg_of_node[j] >= 0) { agg.agg_of_node[i] = agg.agg_of_node[j]; break; }
  }
  for (int i = 0; i < n_nodes; ++i)
    if (agg.agg_of_node[i] < 0) agg.agg_of_node[i] = agg.n_aggregates++;
  return agg;
}

static Amg build_amg(const Csr& A_in, const std::vector<int>& node_in, const Dense& B_in,
                     const orc_amg_options& opts) {  // linsolve.cpp:170-287
  Amg h;
  h.opts = opts;
  Csr A = A_in;
  std::vector<int> node_of_dof = node_in;
  Dense B = B_in;
  for (int lev = 0; lev < opts.max_levels; ++lev) {
    const i64 n = A.rows;
    if (n <= opts.coarse_size) break;
    const int n_nodes = node_of_dof.empty() ? 0 : *std::max_element(node_of_dof.begin(), node_of_dof.end()) + 1;
    // node-block strength (linsolve.cpp:185-203); blk[ni] is an ordered map ni -> sum a^2
    // (std::map semantics), accumulated over the node's dofs in ascending order
    PhaseTimer t_st("amg strength");
    std::vector<std::vector<std::pair<int, double>>> blk(n_nodes);
    auto add_row = [&](i64 i) {
      auto& row = blk[node_of_dof[i]];
      for (i64 k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
        const int nj = node_of_dof[A.col[k]];
        const double a2 = A.val[k] * A.val[k];
        auto it = std::lower_bound(row.begin(), row.end(), nj,
                                   [](const std::pair<int, double>& e, int key) { return e.first < key; });
        if (it != row.end() && it->first == nj)
          it->second += a2;
        else
          row.insert(it, {nj, a2});
      }
    };
    bool monotone = true;  // every node's dofs contiguous: nodes can be filled in parallel
    for (i64 i = 1; i < n && monotone; ++i) monotone = node_of_dof[i] >= node_of_dof[i - 1];
    if (monotone) {
      std::vector<i64> first(n_nodes + 1, n);
      for (i64 i = n - 1; i >= 0; --i) first[node_of_dof[i]] = i;
      for (int ni = n_nodes - 1; ni >= 0; --ni) first[ni] = std::min(first[ni], first[ni + 1]);
      row_pool().run_dyn(n_nodes, 4096, [&](int, i64 lo, i64 hi) {
        for (i64 ni = lo; ni < hi; ++ni)
          for (i64 i = first[ni]; i < first[ni + 1]; ++i) add_row(i);
      });
    } else {
      for (i64 i = 0; i < n; ++i) add_row(i);
    }
    std::vector<double> dsq(n_nodes, 0.0);
    par_for(n_nodes, [&](i64 i) {
      for (auto& e : blk[i])
        if (e.first == i) { dsq[i] = e.second; break; }
    });
    std::vector<std::vector<int>> strong(n_nodes);
    par_for(n_nodes, [&](i64 i) {
      const double dii = std::sqrt(dsq[i]);
      for (auto& [j, s2] : blk[i]) {
        if (j == i) continue;
        const double djj = std::sqrt(dsq[j]);
        if (std::sqrt(s2) > opts.strength_threshold * std::sqrt(dii * djj)) strong[i].push_back(j);
      }
    });
    std::vector<std::vector<std::pair<int, double>>>().swap(blk);
    Aggregation agg;
    { PhaseTimer t("amg aggregate"); agg = aggregate_nodes(n_nodes, strong); }
    std::vector<std::vector<int>>().swap(strong);
    if (agg.n_aggregates >= n_nodes && n_nodes > 1) break;

    // tentative prolongator: ColPivHouseholderQR of each aggregate's nullspace rows
    // (linsolve.cpp:205-239); aggregates are independent
    const i64 m = B.cols;
    const int na = agg.n_aggregates;
    std::vector<i64> dptr(na + 1, 0), dofs_sorted(n), pos_in_agg(n);
    for (i64 i = 0; i < n; ++i) dptr[agg.agg_of_node[node_of_dof[i]] + 1]++;
    for (int a2 = 0; a2 < na; ++a2) dptr[a2 + 1] += dptr[a2];
    {
      std::vector<i64> fill(dptr.begin(), dptr.end() - 1);
      for (i64 i = 0; i < n; ++i) {
        const int a2 = agg.agg_of_node[node_of_dof[i]];
        pos_in_agg[i] = fill[a2] - dptr[a2];
        dofs_sorted[fill[a2]++] = i;
      }
    }
    std::vector<std::vector<double>> agg_Q(na);   // dofs x rank, column-major
    std::vector<Dense> agg_R(na);
    std::vector<i64> agg_rank(na, 0);
    row_pool().run_dyn(na, 256, [&](int, i64 lo, i64 hi) {
      for (i64 a2 = lo; a2 < hi; ++a2) {
        const i64* dofs = dofs_sorted.data() + dptr[a2];
        const i64 rws = dptr[a2 + 1] - dptr[a2];
        Dense Bg(rws, m);
        for (i64 r = 0; r < rws; ++r)
          for (i64 c = 0; c < m; ++c) Bg(r, c) = B(dofs[r], c);
        ColPivQR qr;
        qr.compute(Bg);
        i64 rank = qr.rank(1e-10);
        rank = std::max<i64>(0, std::min<i64>(rank, std::min<i64>(m, rws)));
        agg_Q[a2].assign(size_t(rws * rank), 0.0);
        for (i64 c = 0; c < rank; ++c) qr.q_column(c, agg_Q[a2].data() + size_t(c * rws));
        Dense R(rank, m);
        for (i64 i = 0; i < rank; ++i)
          for (i64 k = i; k < m; ++k) R(i, qr.perm[k]) = qr.qr(i, k);  // (triu R) * Perm^T
        agg_R[a2] = R;
        agg_rank[a2] = rank;
      }
    });
    std::vector<i64> agg_offset(na + 1, 0);
    for (int a2 = 0; a2 < na; ++a2) agg_offset[a2 + 1] = agg_offset[a2] + agg_rank[a2];
    const i64 nc = agg_offset.back();
    if (nc == 0 || nc >= n) break;

    // T (setFromTriplets of one entry per (dof, coarse column)): a dof lies in one aggregate,
    // so its row holds that aggregate's Q row, columns ascending
    Csr T = build_rows(n, nc, 8192, [&](int, i64 i, std::vector<int>& oc, std::vector<double>& ov) {
      const int a2 = agg.agg_of_node[node_of_dof[i]];
      const i64 rws = dptr[a2 + 1] - dptr[a2], r = pos_in_agg[i];
      for (i64 c = 0; c < agg_rank[a2]; ++c) {
        const double q = agg_Q[a2][size_t(c * rws + r)];
        if (std::abs(q) > 1e-300) {
          oc.push_back(int(agg_offset[a2] + c));
          ov.push_back(q);
        }
      }
    });
    std::vector<std::vector<double>>().swap(agg_Q);
    Vec inv_diag(n);
    par_for(n, [&](i64 i) {
      const double dv = A.coeff(i, i);
      inv_diag[i] = (dv != 0.0) ? 1.0 / dv : 0.0;
    });
    double lambda;
    { PhaseTimer t("amg lambda"); lambda = estimate_lambda_max(A, inv_diag); }
    const double wp = opts.prolongation_omega * 2.0 / lambda;
    PhaseTimer t_p("amg P");
    Csr DAT;
    { PhaseTimer t("  DAT"); DAT = spgemm(A, T, inv_diag.data()); }  // (D^-1 A) T
    // P = T - (wp * DAT), union pattern, then prune
    Csr P = build_rows(n, nc, 8192, [&](int, i64 i, std::vector<int>& oc, std::vector<double>& ov) {
      i64 a = T.ptr[i], b = DAT.ptr[i];
      while (a < T.ptr[i + 1] || b < DAT.ptr[i + 1]) {
        if (b >= DAT.ptr[i + 1] || (a < T.ptr[i + 1] && T.col[a] < DAT.col[b])) {
          oc.push_back(T.col[a]);
          ov.push_back(T.val[a]);
          ++a;
        } else if (a >= T.ptr[i + 1] || DAT.col[b] < T.col[a]) {
          oc.push_back(DAT.col[b]);
          ov.push_back(0.0 - wp * DAT.val[b]);
          ++b;
        } else {
          oc.push_back(T.col[a]);
          ov.push_back(T.val[a] - wp * DAT.val[b]);
          ++a;
          ++b;
        }
      }
    });
    DAT = Csr();
    T = Csr();
    { PhaseTimer t("  prune"); prune(P); }

    AmgLevel level;
    { PhaseTimer t("  transpose"); level.Pt = transpose(P); }
    level.inv_diag = inv_diag;
    level.jacobi_weight = opts.jacobi_omega * 2.0 / lambda;
    level.n_nodes = n_nodes;
    level.n_aggregates = agg.n_aggregates;
    level.agg_of_node = agg.agg_of_node;
    level.lambda = lambda;

    Csr Ac;
    {
      PhaseTimer t("amg RAP");
      Csr AP;
      { PhaseTimer t("  AP"); AP = spgemm(A, P); }
      { PhaseTimer t("  PtAP"); Ac = spgemm(level.Pt, AP); }
    }
    prune(Ac);
    level.A = std::move(A);
    level.P = std::move(P);
    Dense Bc(nc, m);
    for (int a2 = 0; a2 < na; ++a2)
      for (i64 i = 0; i < agg_R[a2].rows; ++i)
        for (i64 c = 0; c < m; ++c) Bc(agg_offset[a2] + i, c) = agg_R[a2](i, c);
    std::vector<int> coarse_node(nc);
    for (int a2 = 0; a2 < na; ++a2)
      for (i64 c = agg_offset[a2]; c < agg_offset[a2 + 1]; ++c) coarse_node[c] = a2;
    h.levels.push_back(std::move(level));
    A = std::move(Ac);
    B = std::move(Bc);
    node_of_dof = std::move(coarse_node);
  }
  Dense Ad(A.rows, A.rows);
  for (i64 i = 0; i < A.rows; ++i)
    for (i64 k = A.ptr[i]; k < A.ptr[i + 1]; ++k) Ad(i, A.col[k]) = A.val[k];
  h.coarse_n = A.rows;
  h.coarse.factor(Ad);
  if (Ad.rows > 0 && h.coarse.min_abs_pivot() == 0.0)
    throw std::runtime_error("build_amg: coarsest-level matrix is singular");
  return h;
}

// ------------------------------------------------------------------ block preconditioner (linsolve.cpp:352-415)
struct BlockPrec {
  int kind = 1;  // 0 exact, 1 amg, 2 diagonal   (linsolve.hpp:100)
  i64 nu = 0, np = 0;
  std::shared_ptr<Amg> amg_u, amg_p;
  std::shared_ptr<Lu> lu_u, lu_p;
  Vec inv_u, inv_p;
  Vec apply(const Vec& r) const {
    Vec z(nu + np);
    Vec ru(r.begin(), r.begin() + nu), rp(r.begin() + nu, r.end());
    Vec zu, zp;
    if (kind == 0) {
      zu = lu_u->solve(ru);
      zp = lu_p->solve(rp);
    } else if (kind == 1) {
      zu = amg_u->vcycle(ru);
      zp = amg_p->vcycle(rp);
    } else {
      zu.resize(nu);
      zp.resize(np);
      for (i64 i = 0; i < nu; ++i) zu[i] = inv_u[i] * ru[i];
      for (i64 i = 0; i < np; ++i) zp[i] = inv_p[i] * rp[i];
    }
    std::copy(zu.begin(), zu.end(), z.begin());
    std::copy(zp.begin(), zp.end(), z.begin() + nu);
    return z;
  }
};

struct Nullspace {
  std::vector<int> u_node, p_node;
  Dense u_modes, p_modes;
};

static Lu dense_lu_of(const Csr& A) {
  if (A.rows > 20000) throw std::invalid_argument("oracle exact preconditioner: block too large");
  Dense D(A.rows, A.rows);
  for (i64 i = 0; i < A.rows; ++i)
    for (i64 k = A.ptr[i]; k < A.ptr[i + 1]; ++k) D(i, A.col[k]) = A.val[k];
  Lu lu;
  lu.factor(D);
  if (A.rows > 0 && lu.min_abs_pivot() == 0.0) throw std::runtime_error("BlockPreconditioner: block factorization failed");
  return lu;
}

static std::vector<int> identity_nodes(i64 n) {
  std::vector<int> v(n);
  for (i64 i = 0; i < n; ++i) v[i] = int(i);
  return v;
}
static Dense ones(i64 n) {
  Dense D(n, 1);
  for (i64 i = 0; i < n; ++i) D(i, 0) = 1.0;
  return D;
}

static BlockPrec build_prec(const BlockSystem& sys, int kind, const orc_amg_options& ao, const Nullspace* ns) {
  BlockPrec p;
  p.kind = kind;
  p.nu = sys.n_u();
  p.np = sys.n_phi();
  if (kind == 0) {
    p.lu_u = std::make_shared<Lu>(dense_lu_of(sys.uu));
    p.lu_p = std::make_shared<Lu>(dense_lu_of(sys.pp));
  } else if (kind == 1) {
    if (ns) {
      p.amg_u = std::make_shared<Amg>(build_amg(sys.uu, ns->u_node, ns->u_modes, ao));
      p.amg_p = std::make_shared<Amg>(build_amg(sys.pp, ns->p_node, ns->p_modes, ao));
    } else {
      p.amg_u = std::make_shared<Amg>(build_amg(sys.uu, identity_nodes(p.nu), ones(p.nu), ao));
      p.amg_p = std::make_shared<Amg>(build_amg(sys.pp, identity_nodes(p.np), ones(p.np), ao));
    }
  } else if (kind == 2) {
    p.inv_u.assign(p.nu, 1.0);
    p.inv_p.assign(p.np, 1.0);
    for (i64 i = 0; i < p.nu; ++i) {
      const double dv = sys.uu.coeff(i, i);
      if (dv != 0.0) p.inv_u[i] = 1.0 / dv;
    }
    for (i64 i = 0; i < p.np; ++i) {
      const double dv = sys.pp.coeff(i, i);
      if (dv != 0.0) p.inv_p[i] = 1.0 / dv;
    }
  } else {
    throw std::invalid_argument("unknown preconditioner kind");
  }
  return p;
}

static Dense rigid_body_modes(const Grid& g, const Constraints& cs) {  // linsolve.cpp:320-343
  const int d = g.d;
  const i64 n = g.n_u();
  const i64 m = (d == 2) ? 3 : 6;
  Dense B(n, m);
  for (i64 v = 0; v < g.V; ++v) {
    i64 c[3];
    g.vxyz(v, c[0], c[1], c[2]);
    const double x0 = g.coord(c[0]), x1 = g.coord(c[1]), x2 = (d == 3) ? g.coord(c[2]) : 0.0;
    for (int a = 0; a < d; ++a) B(v * d + a, a) = 1.0;
    if (d == 2) {
      B(v * d + 0, 2) = -x1;
      B(v * d + 1, 2) = x0;
    } else {
      B(v * d + 1, 3) = -x2;
      B(v * d + 2, 3) = x1;
      B(v * d + 0, 4) = x2;
      B(v * d + 2, 4) = -x0;
      B(v * d + 0, 5) = -x1;
      B(v * d + 1, 5) = x0;
    }
  }
  for (i64 i = 0; i < n; ++i)
    if (cs.is(i))
      for (i64 c = 0; c < m; ++c) B(i, c) = 0.0;
  return B;
}

// ------------------------------------------------------------------ model helpers (model.cpp:28-64, 324-349)
static double slit_band_edge(const Grid& g, const orc_material& mat) {
  double edge = -1.0;
  const int d = g.d;
  for (i64 id : g.cell_order) {
    i64 c[3];
    g.cxyz(id, c[0], c[1], c[2]);
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int a = 0; a < d; ++a) {
      lo[a] = g.coord(c[a]);
      hi[a] = g.coord(c[a] + 1);
    }
    bool meets;
    if (d == 2) {
      meets = lo[1] <= 0.0 && hi[1] >= 0.0 && lo[0] <= mat.l0 && hi[0] >= -mat.l0;
    } else {
      if (!(lo[2] <= 0.0 && hi[2] >= 0.0)) continue;
      const double dx = std::max({lo[0], 0.0, -hi[0]});
      const double dy = std::max({lo[1], 0.0, -hi[1]});
      meets = std::hypot(dx, dy) <= mat.l0;
    }
    if (meets) {
      if (edge < 0.0 || g.h < edge) edge = g.h;
    }
  }
  if (edge < 0.0) throw std::runtime_error("slit_band_edge: no active cell meets the slit");
  return edge;
}

static orc_regularization resolve_regularization(const Grid& g, const orc_material& mat, double band_edge) {
  orc_regularization reg;
  const double diam = band_edge * std::sqrt(double(g.d));
  reg.eps = (mat.eps_mode == 0) ? mat.c_eps * diam : mat.eps_fixed;
  reg.kappa = mat.kappa_factor * g.h;
  return reg;
}

static Vec initial_crack(const Grid& g, const orc_material& mat, double band_half, double* band_edge_out) {
  const int d = g.d;
  const double be = band_half > 0.0 ? band_half : slit_band_edge(g, mat);
  Vec phi(g.V, 1.0);
  const double tol = 1e-9 * be;
  i64 n_zero = 0, n_plane = 0;
  for (i64 v = 0; v < g.V; ++v) {
    i64 c[3];
    g.vxyz(v, c[0], c[1], c[2]);
    const double x0 = g.coord(c[0]), x1 = g.coord(c[1]), x2 = (d == 3) ? g.coord(c[2]) : 0.0;
    bool in;
    if (d == 2)
      in = std::abs(x0) <= mat.l0 + tol && std::abs(x1) <= be + tol;
    else
      in = std::hypot(x0, x1) <= mat.l0 + tol && std::abs(x2) <= be + tol;
    if (in) {
      phi[v] = 0.0;
      ++n_zero;
      if (std::abs(d == 2 ? x1 : x2) <= tol) ++n_plane;
    }
  }
  if (n_zero == 0 || n_plane == 0)
    throw std::runtime_error("initial_crack: slit is not resolved by the mesh (no vertex layer inside the band)");
  if (band_edge_out) *band_edge_out = be;
  return phi;
}

// ------------------------------------------------------------------ Newton / active set (solver.cpp)
struct State {
  Vec solution, phi_old, phi_prev2;
  int step = 0;
};
struct NewtonIter {
  double residual_norm;
  int active_size, set_changes, gmres_iterations;
};
struct NewtonReport {
  std::vector<NewtonIter> its;
  bool converged = false;
  double feasibility = 0.0;
};

static Vec extrapolate_phi(const State& st) {  // model.cpp:60-64
  if (st.step <= 2) return st.phi_old;
  Vec t(st.phi_old.size());
  for (size_t i = 0; i < t.size(); ++i) {
    const double v = 2.0 * st.phi_old[i] - st.phi_prev2[i];
    t[i] = std::min(std::max(v, 0.0), 1.0);
  }
  return t;
}

static std::set<i64> detect_cycles(const std::map<i64, std::vector<char>>& history, int window, int toggles) {
  std::set<i64> out;  // solver.cpp:10-22
  for (const auto& [dof, bits] : history) {
    const int n = int(bits.size());
    const int start = std::max(0, n - window);
    int changes = 0;
    for (int i = start + 1; i < n; ++i)
      if (bits[i] != bits[i - 1]) ++changes;
    if (changes >= toggles) out.insert(dof);
  }
  return out;
}

// newton_active_set_step (solver.cpp:49-188).  The active set A and the toggle history are kept
// as flat per-vertex arrays instead of std::set / std::map: a dof's history is tracked from the
// iteration it first enters A, backfilled with zeros to the current history length (so every
// tracked history has the global length, and its entries before tracking are 0 = "not active"),
// which is exactly the reference's map semantics (solver.cpp:88-102).
static NewtonReport newton_step(State& state, const orc_material& mat, const Grid& g,
                                const orc_regularization& reg, const orc_solver_options& opts) {
  NewtonReport report;
  const i64 nu = g.n_u(), np = g.n_phi();
  Constraints base = build_constraints(g, true, {}, {});
  Vec& x = state.solution;
  base.distribute(x);
  const Vec phi_tilde = extrapolate_phi(state);  // conforming_phi: base has no phi lines on uniform meshes
  const double c = opts.active_set_c_scale * mat.G_c / reg.eps;
  std::vector<char> fixed(np, 0), active(np, 0), prev_active(np, 0), tracked(np, 0), candidate(np, 0);
  std::vector<std::vector<char>> hist;  // hist[t][v]: iteration t of the history (global length)
  for (i64 v = 0; v < np; ++v) candidate[v] = !base.is(nu + v);
  double res0 = -1.0;
  BlockPrec prec;
  bool have_prec = false;
  for (int it = 1; it <= opts.newton_max_iter; ++it) {
    Vec R;
    { PhaseTimer t("residual"); R = assemble_residual(g, base, mat, reg, x.data(), phi_tilde.data()); }
    PhaseTimer t_as("active set");
    const double active_tol = 1e-14 * c;
    par_for(np, [&](i64 v) {
      char a = fixed[v];
      if (!a && candidate[v]) {
        const i64 dof = nu + v;
        const double lambda = -R[dof];
        a = (c * (x[dof] - state.phi_old[v]) + lambda > active_tol) ? 1 : 0;
      }
      active[v] = a;
    });
    // history: a newly tracked dof starts at the current length (zeros before), all push 1/0
    bool any_tracked = !hist.empty();
    for (i64 v = 0; v < np && !any_tracked; ++v) any_tracked = active[v] != 0;
    if (any_tracked) {
      par_for(np, [&](i64 v) {
        if (active[v]) tracked[v] = 1;
      });
      hist.emplace_back(active.begin(), active.end());
      const int L = int(hist.size()), start = std::max(0, L - opts.cycle_window);
      par_for(np, [&](i64 v) {  // detect_cycles (solver.cpp:10-22) over the tracked dofs
        if (!tracked[v]) return;
        int changes = 0;
        for (int t = start + 1; t < L; ++t)
          if (hist[t][v] != hist[t - 1][v]) ++changes;
        if (changes >= opts.cycle_toggles) {
          fixed[v] = 1;
          active[v] = 1;
        }
      });
    }
    i64 n_active = 0, changes = 0;
    for (i64 v = 0; v < np; ++v) {
      n_active += active[v];
      changes += (active[v] != prev_active[v]);
    }
    std::vector<i64> adofs;
    std::vector<double> avals;
    adofs.reserve(n_active);
    avals.reserve(n_active);
    for (i64 v = 0; v < np; ++v)
      if (active[v]) {
        adofs.push_back(nu + v);
        avals.push_back(state.phi_old[v]);
      }
    Constraints full = build_constraints(g, true, adofs, avals);
    Vec x_before = x;
    full.distribute(x);
    double moved = 0.0;
    for (size_t i = 0; i < x.size(); ++i) moved = std::max(moved, std::abs(x[i] - x_before[i]));
    if (moved > 0.0) {
      R = assemble_residual(g, full, mat, reg, x.data(), phi_tilde.data());
    } else {
      for (i64 dof : adofs) R[dof] = 0.0;
    }
    double res;
    {
      SegScope seg(g);
      res = norm(R);
    }
    if (res0 < 0.0) res0 = res;
    NewtonIter rec{res, int(n_active), int(changes), 0};
    const bool small = res <= std::max(opts.newton_tol * res0, opts.newton_abs_floor);
    if (changes == 0 && small) {
      report.its.push_back(rec);
      if (opts.log)
        std::printf("newton step=%d it=%d res=%.6e active=%d changed=%d gmres=0\n", state.step, it, res,
                    rec.active_size, int(changes));
      report.converged = true;
      break;
    }
    BlockSystem J;
    { PhaseTimer t("jacobian"); J = assemble_jacobian(g, full, mat, reg, x.data(), phi_tilde.data()); }
    if (!have_prec || !opts.freeze_preconditioner) {
      Nullspace ns;
      ns.u_modes = rigid_body_modes(g, full);
      ns.u_node.resize(nu);
      for (i64 i = 0; i < nu; ++i) ns.u_node[i] = int(i / g.d);
      ns.p_modes = ones(np);
      for (i64 v = 0; v < np; ++v)
        if (full.is(nu + v)) ns.p_modes(v, 0) = 0.0;
      ns.p_node = identity_nodes(np);
      PhaseTimer t("prec build");
      prec = BlockPrec();  // release the previous hierarchies before building the new ones
      prec = build_prec(J, opts.prec_kind, opts.amg, &ns);
      have_prec = true;
    }
    Vec mR(R.size());
    par_for(i64(R.size()), [&](i64 i) { mR[i] = -R[i]; });
    PhaseTimer t_gm("gmres");
    SegScope seg(g);
    GmresResult lin = gmres([&J](const Vec& v) { return J.apply(v); },
                            [&prec](const Vec& v) { return prec.apply(v); }, mR, opts.gmres);
    if (!lin.converged && !lin.breakdown)
      throw std::runtime_error("newton_active_set_step: GMRES stagnated at max_iter");
    rec.gmres_iterations = lin.iterations;
    report.its.push_back(rec);
    if (opts.log)
      std::printf("newton step=%d it=%d res=%.6e active=%d changed=%d gmres=%d\n", state.step, it, res,
                  rec.active_size, int(changes), lin.iterations);
    Vec delta = lin.x;
    full.distribute_homogeneous(delta);
    par_for(i64(x.size()), [&](i64 i) { x[i] += delta[i]; });
    if (opts.damping) {
      double scale = 1.0;
      for (int half = 0; half < 4; ++half) {
        Vec Rn = assemble_residual(g, full, mat, reg, x.data(), phi_tilde.data());
        SegScope seg2(g);
        if (norm(Rn) <= 10.0 * res) break;
        scale *= 0.5;
        for (size_t i = 0; i < x.size(); ++i) x[i] -= scale * delta[i];
      }
    }
    prev_active = active;
  }
  double viol = 0.0;
  for (i64 v = 0; v < np; ++v) viol = std::max(viol, x[nu + v] - state.phi_old[v]);
  report.feasibility = viol;
  return report;
}

// ------------------------------------------------------------------ post-processing (postproc.cpp:12-99)
struct PointVal {
  double u[3] = {0, 0, 0}, phi = 0.0, gphi[3] = {0, 0, 0};
};
static PointVal evaluate_on_cell(const Grid& g, const double* sol, i64 cell, const double x[3]) {
  const int d = g.d;
  i64 c[3];
  g.cxyz(cell, c[0], c[1], c[2]);
  double xi[3] = {0, 0, 0};
  for (int a = 0; a < d; ++a) {
    const double lo = g.coord(c[a]);
    xi[a] = std::clamp((x[a] - lo) / g.h, 0.0, 1.0);
  }
  double shape[8], grads[8][3];
  q1_shape(d, xi, shape, grads);
  i64 verts[8];
  g.cell_vertices(cell, verts);
  PointVal pv;
  const i64 nu = g.n_u();
  for (int k = 0; k < (1 << d); ++k) {
    const double phi = sol[nu + verts[k]];
    pv.phi += shape[k] * phi;
    for (int a = 0; a < d; ++a) {
      pv.gphi[a] += grads[k][a] / g.h * phi;
      pv.u[a] += shape[k] * sol[verts[k] * d + a];
    }
  }
  return pv;
}

static double compute_tcv(const Grid& g, const double* sol) {
  const int d = g.d;
  Rule q = cell_rule(d, 2);
  double tcv = 0.0;
  for (i64 id : g.cell_order) {
    i64 c[3];
    g.cxyz(id, c[0], c[1], c[2]);
    double lo[3] = {0, 0, 0};
    for (int a = 0; a < d; ++a) lo[a] = g.coord(c[a]);
    for (int iq = 0; iq < q.nq; ++iq) {
      double x[3] = {lo[0], lo[1], lo[2]};
      for (int a = 0; a < d; ++a) x[a] += q.pts[size_t(iq) * d + a] * g.h;
      PointVal pv = evaluate_on_cell(g, sol, id, x);
      double dotp = 0.0;
      for (int a = 0; a < 3; ++a) dotp += pv.u[a] * pv.gphi[a];
      tcv += q.w[iq] * g.detJ * dotp;
    }
  }
  return tcv;
}

static void compute_cod(const Grid& g, const double* sol, const double* stations, int ns, double* out) {
  const int d = g.d, axis = d - 1;
  const double K = g.K;
  for (int i = 1; i < ns; ++i)
    if (!(stations[i] > stations[i - 1])) throw std::invalid_argument("compute_cod: stations must be strictly increasing");
  Rule line = cell_rule(1, 4);
  auto owns = [K](double lo, double hi, double s) { return (s < K) ? (lo <= s && s < hi) : (lo < s && s <= hi); };
  for (int si = 0; si < ns; ++si) {
    const double s = stations[si];
    if (std::abs(s) > K) throw std::invalid_argument("compute_cod: station outside domain");
    double total = 0.0;
    for (i64 id : g.cell_order) {
      i64 c[3];
      g.cxyz(id, c[0], c[1], c[2]);
      double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
      for (int a = 0; a < d; ++a) {
        lo[a] = g.coord(c[a]);
        hi[a] = g.coord(c[a] + 1);
      }
      if (!owns(lo[0], hi[0], s)) continue;
      if (d == 3 && !owns(lo[1], hi[1], 0.0)) continue;
      for (int iq = 0; iq < line.nq; ++iq) {
        double x[3] = {s, 0.0, 0.0};
        x[axis] = lo[axis] + line.pts[iq] * g.h;
        PointVal pv = evaluate_on_cell(g, sol, id, x);
        double dotp = 0.0;
        for (int a = 0; a < 3; ++a) dotp += pv.u[a] * pv.gphi[a];
        total += line.w[iq] * g.h * dotp;
      }
    }
    out[si] = 0.5 * std::abs(total);
  }
}

#include "oracle_mesh.inc"

}  // namespace orc

// =====================================================================================
//  C ABI for the Python tests (ctypes).  Every function returns 0 on success, -1 on a
//  C++ exception (message via orc_last_error()).
// =====================================================================================
using namespace orc;

struct orc_problem {
  Grid g;
};
struct orc_constraints {
  Constraints cs;
};
struct orc_block {
  BlockSystem J;
};
struct orc_csr {
  Csr A;
};
struct orc_amg {
  Amg h;
};
struct orc_prec {
  BlockPrec p;
};

#define ORC_TRY try {
#define ORC_CATCH                 \
  }                               \
  catch (const std::exception& e) { \
    g_err = e.what();             \
    return -1;                    \
  }                               \
  return 0;

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

int orc_problem_create(int d, double K, int n0, int r, orc_problem** out) {
  ORC_TRY
  *out = new orc_problem{make_grid(d, K, n0, r)};
  ORC_CATCH
}
void orc_problem_destroy(orc_problem* p) { delete p; }
int orc_problem_info(orc_problem* p, int64_t* V, int64_t* ncells, double* h, double* detJ) {
  *V = p->g.V;
  *ncells = p->g.ncells;
  *h = p->g.h;
  *detJ = p->g.detJ;
  return 0;
}
int orc_vertex_coords(orc_problem* p, double* xyz) {  // V x 3
  const Grid& g = p->g;
  for (i64 v = 0; v < g.V; ++v) {
    i64 c[3];
    g.vxyz(v, c[0], c[1], c[2]);
    xyz[3 * v] = g.coord(c[0]);
    xyz[3 * v + 1] = g.coord(c[1]);
    xyz[3 * v + 2] = g.d == 3 ? g.coord(c[2]) : 0.0;
  }
  return 0;
}
int orc_cell_order(orc_problem* p, int64_t* out) {
  std::copy(p->g.cell_order.begin(), p->g.cell_order.end(), out);
  return 0;
}
int orc_initial_crack(orc_problem* p, const orc_material* m, double band_half, double* phi, double* band_edge) {
  ORC_TRY
  Vec v = initial_crack(p->g, *m, band_half, band_edge);
  std::copy(v.begin(), v.end(), phi);
  ORC_CATCH
}
int orc_slit_band_edge(orc_problem* p, const orc_material* m, double* out) {
  ORC_TRY
  *out = slit_band_edge(p->g, *m);
  ORC_CATCH
}
int orc_resolve_regularization(orc_problem* p, const orc_material* m, double band_edge, orc_regularization* out) {
  ORC_TRY
  *out = resolve_regularization(p->g, *m, band_edge);
  ORC_CATCH
}
int orc_constraints_build(orc_problem* p, int clamp, int64_t n_active, const int64_t* dofs, const double* vals,
                          orc_constraints** out) {
  ORC_TRY
  std::vector<i64> ad(dofs, dofs + n_active);
  std::vector<double> av(vals, vals + n_active);
  *out = new orc_constraints{build_constraints(p->g, clamp != 0, ad, av)};
  ORC_CATCH
}
void orc_constraints_destroy(orc_constraints* c) { delete c; }
int orc_constraints_flags(orc_constraints* c, uint8_t* flags, double* inhom) {
  std::copy(c->cs.flag.begin(), c->cs.flag.end(), flags);
  std::copy(c->cs.inhom.begin(), c->cs.inhom.end(), inhom);
  return 0;
}
int orc_distribute(orc_constraints* c, double* v, int homogeneous) {
  Vec x(v, v + c->cs.flag.size());
  if (homogeneous) c->cs.distribute_homogeneous(x); else c->cs.distribute(x);
  std::copy(x.begin(), x.end(), v);
  return 0;
}

int orc_assemble_residual(orc_problem* p, orc_constraints* c, const orc_material* m, const orc_regularization* r,
                          const double* x, const double* pt, double* R) {
  ORC_TRY
  check_material(*m);
  Vec v = assemble_residual(p->g, c->cs, *m, *r, x, pt);
  std::copy(v.begin(), v.end(), R);
  ORC_CATCH
}
int orc_assemble_jacobian(orc_problem* p, orc_constraints* c, const orc_material* m, const orc_regularization* r,
                          const double* x, const double* pt, orc_block** out) {
  ORC_TRY
  check_material(*m);
  *out = new orc_block{assemble_jacobian(p->g, c->cs, *m, *r, x, pt)};
  ORC_CATCH
}
void orc_block_destroy(orc_block* b) { delete b; }
static const Csr& blk_of(orc_block* b, int which) { return which == 0 ? b->J.uu : (which == 1 ? b->J.pu : b->J.pp); }
int orc_block_nnz(orc_block* b, int which, int64_t* rows, int64_t* cols, int64_t* nnz) {
  const Csr& A = blk_of(b, which);
  *rows = A.rows;
  *cols = A.cols;
  *nnz = A.nnz();
  return 0;
}
int orc_block_export(orc_block* b, int which, int64_t* ptr, int32_t* col, double* val) {
  const Csr& A = blk_of(b, which);
  std::copy(A.ptr.begin(), A.ptr.end(), ptr);
  std::copy(A.col.begin(), A.col.end(), col);
  std::copy(A.val.begin(), A.val.end(), val);
  return 0;
}
int orc_block_apply(orc_block* b, const double* x, double* y) {
  Vec xv(x, x + b->J.n_u() + b->J.n_phi());
  Vec yv = b->J.apply(xv);
  std::copy(yv.begin(), yv.end(), y);
  return 0;
}
// host threads of the row-parallel SpMV (1 = the single-threaded reference)
int orc_set_threads(int threads) {
  row_pool().resize(threads);
  return 0;
}
int orc_get_threads(void) { return row_pool().size(); }
// reduction order: 0 = the product's documented order (bitwise checks), 1 = the reference's
// sequential row sums and dots (tolerance checks); see the file header
int orc_set_order(int order) {
  if (order != ORDER_PRODUCT && order != ORDER_REFERENCE) return -1;
  g_order = order;
  return 0;
}
int orc_get_order(void) { return g_order; }

// SpMV of one block with `threads` OpenMP threads (row-parallel; each row summed sequentially,
// so the result is independent of the thread count).  Used for the bounded CPU baseline.
int orc_block_spmv_threads(orc_block* b, int which, const double* x, double* y, int threads) {
  const Csr& A = blk_of(b, which);
  threads = std::max(1, threads);
  auto work = [&](i64 lo, i64 hi) {
    for (i64 i = lo; i < hi; ++i) {
      double s = 0.0;
      for (i64 k = A.ptr[i]; k < A.ptr[i + 1]; ++k) s += A.val[k] * x[A.col[k]];
      y[i] = s;
    }
  };
  std::vector<std::thread> pool;
  const i64 chunk = (A.rows + threads - 1) / threads;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back(work, std::min(A.rows, t * chunk), std::min(A.rows, (t + 1) * chunk));
  for (auto& th : pool) th.join();
  return 0;
}
// SpMV of one block (used for the bounded CPU-baseline sample)
int orc_block_spmv(orc_block* b, int which, const double* x, double* y) {
  spmv(blk_of(b, which), x, y);
  return 0;
}

int orc_csr_create(int64_t rows, int64_t cols, const int64_t* ptr, const int32_t* col, const double* val,
                   orc_csr** out) {
  ORC_TRY
  auto* c = new orc_csr;
  c->A.rows = rows;
  c->A.cols = cols;
  c->A.ptr.assign(ptr, ptr + rows + 1);
  c->A.col.assign(col, col + ptr[rows]);
  c->A.val.assign(val, val + ptr[rows]);
  *out = c;
  ORC_CATCH
}
void orc_csr_destroy(orc_csr* c) { delete c; }
// C = diag(rs) A B (rs may be null): the AMG setup's sparse product (k-ascending Gustavson)
int orc_csr_spgemm(orc_csr* A, orc_csr* B, const double* rs, orc_csr** out) {
  ORC_TRY
  if (A->A.cols != B->A.rows) throw std::invalid_argument("spgemm: inner dimensions differ");
  *out = new orc_csr{spgemm(A->A, B->A, rs)};
  ORC_CATCH
}
int orc_csr_info(orc_csr* A, int64_t* rows, int64_t* cols, int64_t* nnz) {
  *rows = A->A.rows;
  *cols = A->A.cols;
  *nnz = A->A.nnz();
  return 0;
}
int orc_csr_export(orc_csr* A, int64_t* ptr, int32_t* col, double* val) {
  std::copy(A->A.ptr.begin(), A->A.ptr.end(), ptr);
  std::copy(A->A.col.begin(), A->A.col.end(), col);
  std::copy(A->A.val.begin(), A->A.val.end(), val);
  return 0;
}

int orc_amg_build(orc_csr* A, const int32_t* node_of_dof, const double* B_colmajor, int m, const orc_amg_options* o,
                  orc_amg** out) {
  ORC_TRY
  const i64 n = A->A.rows;
  std::vector<int> nod(n);
  Dense B(n, m);
  if (node_of_dof) {
    for (i64 i = 0; i < n; ++i) nod[i] = node_of_dof[i];
    std::copy(B_colmajor, B_colmajor + n * m, B.a.begin());
  } else {
    nod = identity_nodes(n);
    B = ones(n);
  }
  *out = new orc_amg{build_amg(A->A, nod, B, *o)};
  ORC_CATCH
}
void orc_amg_destroy(orc_amg* a) { delete a; }
int orc_amg_info(orc_amg* a, int* n_levels, int64_t* coarse_dim) {
  *n_levels = int(a->h.levels.size()) + 1;
  *coarse_dim = a->h.coarse_n;
  return 0;
}
// per level: rows(A), nnz(A), nnz(P), cols(P), n_nodes, n_aggregates ; lambda
int orc_amg_level(orc_amg* a, int lev, int64_t* info6, double* lambda, double* jacobi_weight) {
  const AmgLevel& L = a->h.levels.at(lev);
  info6[0] = L.A.rows;
  info6[1] = L.A.nnz();
  info6[2] = L.P.nnz();
  info6[3] = L.P.cols;
  info6[4] = L.n_nodes;
  info6[5] = L.n_aggregates;
  *lambda = L.lambda;
  *jacobi_weight = L.jacobi_weight;
  return 0;
}
int orc_amg_level_aggregates(orc_amg* a, int lev, int32_t* agg) {
  const AmgLevel& L = a->h.levels.at(lev);
  std::copy(L.agg_of_node.begin(), L.agg_of_node.end(), agg);
  return 0;
}
int orc_amg_level_export(orc_amg* a, int lev, int which, int64_t* ptr, int32_t* col, double* val) {
  const AmgLevel& L = a->h.levels.at(lev);
  const Csr& M = which == 0 ? L.A : L.P;
  std::copy(M.ptr.begin(), M.ptr.end(), ptr);
  std::copy(M.col.begin(), M.col.end(), col);
  std::copy(M.val.begin(), M.val.end(), val);
  return 0;
}
int orc_amg_vcycle(orc_amg* a, const double* r, double* x) {
  ORC_TRY
  const i64 n = a->h.levels.empty() ? a->h.coarse_n : a->h.levels[0].A.rows;
  Vec rv(r, r + n);
  Vec xv = a->h.vcycle(rv);
  std::copy(xv.begin(), xv.end(), x);
  ORC_CATCH
}

int orc_prec_build(orc_block* b, int kind, const orc_amg_options* o, int with_nullspace, orc_problem* p,
                   orc_constraints* c, orc_prec** out) {
  ORC_TRY
  Nullspace ns;
  if (with_nullspace) {
    const Grid& g = p->g;
    const i64 nu = g.n_u(), np = g.n_phi();
    ns.u_modes = rigid_body_modes(g, c->cs);
    ns.u_node.resize(nu);
    for (i64 i = 0; i < nu; ++i) ns.u_node[i] = int(i / g.d);
    ns.p_modes = ones(np);
    for (i64 v = 0; v < np; ++v)
      if (c->cs.is(nu + v)) ns.p_modes(v, 0) = 0.0;
    ns.p_node = identity_nodes(np);
  }
  *out = new orc_prec{build_prec(b->J, kind, *o, with_nullspace ? &ns : nullptr)};
  ORC_CATCH
}
void orc_prec_destroy(orc_prec* p) { delete p; }
int orc_prec_apply(orc_prec* p, const double* r, double* z) {
  ORC_TRY
  Vec rv(r, r + p->p.nu + p->p.np);
  Vec zv = p->p.apply(rv);
  std::copy(zv.begin(), zv.end(), z);
  ORC_CATCH
}
int orc_rigid_body_modes(orc_problem* p, orc_constraints* c, double* B_colmajor) {
  Dense B = rigid_body_modes(p->g, c->cs);
  std::copy(B.a.begin(), B.a.end(), B_colmajor);
  return 0;
}

// GMRES on a block system (op = J.apply) or a CSR matrix (op = A x); prec: block prec, amg
// (CSR only) or none.  history must hold max_iter doubles.
int orc_gmres(orc_block* b, orc_csr* A, orc_prec* pb, orc_amg* pa, const double* rhs, const orc_gmres_options* o,
              double* x, int* iterations, int* converged, int* breakdown, double* residual, double* history) {
  ORC_TRY
  Op op, prec;
  i64 n;
  if (b) {
    n = b->J.n_u() + b->J.n_phi();
    op = [b](const Vec& v) { return b->J.apply(v); };
  } else {
    n = A->A.rows;
    op = [A](const Vec& v) {
      Vec y(A->A.rows);
      spmv(A->A, v.data(), y.data());
      return y;
    };
  }
  if (pb) prec = [pb](const Vec& v) { return pb->p.apply(v); };
  if (pa) prec = [pa](const Vec& v) { return pa->h.vcycle(v); };
  Vec r(rhs, rhs + n);
  GmresResult res = gmres(op, prec, r, *o);
  std::copy(res.x.begin(), res.x.end(), x);
  *iterations = res.iterations;
  *converged = res.converged;
  *breakdown = res.breakdown;
  *residual = res.residual;
  if (history) std::copy(res.history.begin(), res.history.end(), history);
  ORC_CATCH
}

// One loading step (solve_loading_sequence body, solver.cpp:196-201) or a bare Newton step
// (shift == 0).  State arrays are updated in place.  its_out: max_its x 4 (res, active, changes, gmres).
int orc_newton_step(orc_problem* p, const orc_material* m, const orc_regularization* r, const orc_solver_options* o,
                    double* solution, double* phi_old, double* phi_prev2, int step, int shift, int max_its,
                    double* its_out, int* n_its, int* converged, double* feasibility) {
  ORC_TRY
  const Grid& g = p->g;
  State st;
  st.solution.assign(solution, solution + g.n_total());
  st.phi_old.assign(phi_old, phi_old + g.V);
  st.phi_prev2.assign(phi_prev2, phi_prev2 + g.V);
  st.step = step;
  if (shift) {
    st.phi_prev2 = st.phi_old;
    st.phi_old.assign(st.solution.begin() + g.n_u(), st.solution.end());
  }
  NewtonReport rep = newton_step(st, *m, g, *r, *o);
  std::copy(st.solution.begin(), st.solution.end(), solution);
  std::copy(st.phi_old.begin(), st.phi_old.end(), phi_old);
  std::copy(st.phi_prev2.begin(), st.phi_prev2.end(), phi_prev2);
  *n_its = int(rep.its.size());
  for (int i = 0; i < int(rep.its.size()) && i < max_its; ++i) {
    its_out[4 * i] = rep.its[i].residual_norm;
    its_out[4 * i + 1] = rep.its[i].active_size;
    its_out[4 * i + 2] = rep.its[i].set_changes;
    its_out[4 * i + 3] = rep.its[i].gmres_iterations;
  }
  *converged = rep.converged;
  *feasibility = rep.feasibility;
  ORC_CATCH
}

int orc_tcv(orc_problem* p, const double* sol, double* out) {
  ORC_TRY
  *out = compute_tcv(p->g, sol);
  ORC_CATCH
}
int orc_cod(orc_problem* p, const double* sol, const double* stations, int ns, double* out) {
  ORC_TRY
  compute_cod(p->g, sol, stations, ns, out);
  ORC_CATCH
}
int orc_detect_cycles(int n_dofs, const int32_t* lens, const int8_t* bits, int window, int toggles, int32_t* out_flags) {
  std::map<i64, std::vector<char>> h;
  i64 off = 0;
  for (int i = 0; i < n_dofs; ++i) {
    h[i] = std::vector<char>(bits + off, bits + off + lens[i]);
    off += lens[i];
  }
  auto s = detect_cycles(h, window, toggles);
  for (int i = 0; i < n_dofs; ++i) out_flags[i] = s.count(i) ? 1 : 0;
  return 0;
}
// Quadrature tables (KAT checks)
int orc_qp_tables(int d, double* pts, double* wts, double* shape, double* grads) {
  QpData q = make_qp_data(d);
  for (int i = 0; i < q.nq; ++i) {
    wts[i] = q.wts[i];
    for (int a = 0; a < 3; ++a) pts[i * 3 + a] = q.pts[i][a];
    for (int k = 0; k < q.nv; ++k) {
      shape[i * q.nv + k] = q.shape[i][k];
      for (int a = 0; a < 3; ++a) grads[(i * q.nv + k) * 3 + a] = q.grads[i][k][a];
    }
  }
  return 0;
}
// Dense column-pivoting QR (exported for the QR parity test)
int orc_colpiv_qr(int rows, int cols, const double* A_colmajor, double threshold, int* rank, double* Q_colmajor,
                  double* R_colmajor, int32_t* perm) {
  Dense A(rows, cols);
  std::copy(A_colmajor, A_colmajor + rows * cols, A.a.begin());
  ColPivQR qr;
  qr.compute(A);
  i64 rk = qr.rank(threshold);
  rk = std::max<i64>(0, std::min<i64>(rk, std::min(rows, cols)));
  *rank = int(rk);
  for (i64 c = 0; c < rk; ++c) qr.q_column(c, Q_colmajor + c * rows);
  for (i64 i = 0; i < rk; ++i)
    for (i64 j = 0; j < cols; ++j) R_colmajor[j * rk + i] = 0.0;
  for (i64 i = 0; i < rk; ++i)
    for (i64 k = i; k < cols; ++k) R_colmajor[qr.perm[k] * rk + i] = qr.qr(i, k);
  for (int k = 0; k < cols; ++k) perm[k] = int(qr.perm[k]);
  return 0;
}


int orc_lame(const orc_material* m, double* mu, double* lam) {
  *mu = mat_mu(*m);
  *lam = mat_lambda(*m);
  return 0;
}
// sigma(grad_u) (model.cpp:19-26); grad and out are 3x3 row-major
int orc_sigma(const double* grad, const orc_material* m, int d, double* out) {
  const double mu = mat_mu(*m), lam = mat_lambda(*m);
  double e[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) e[a][b] = 0.5 * (grad[3 * a + b] + grad[3 * b + a]);
  double tr = 0.0;
  for (int a = 0; a < d; ++a) tr += e[a][a];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) out[3 * a + b] = 2.0 * mu * e[a][b];
  for (int a = 0; a < d; ++a) out[3 * a + a] += lam * tr;
  return 0;
}


// ---- general (adaptive) meshes (oracle_mesh.inc)
struct orc_mesh {
  gm::Mesh m;
  gm::DofMap map;
  void remap() { map = gm::build_dof_map(m); }
};
struct orc_mcs {
  gm::CSet cs;
};
int orc_mesh_create(int d, double K, int n0, orc_mesh** out) {
  ORC_TRY
  auto* o = new orc_mesh{gm::Mesh(d, K, n0), {}};
  o->remap();
  *out = o;
  ORC_CATCH
}
int orc_mesh_copy(orc_mesh* src, orc_mesh** out) {
  ORC_TRY
  *out = new orc_mesh(*src);
  ORC_CATCH
}
void orc_mesh_destroy(orc_mesh* m) { delete m; }
int orc_mesh_refine(orc_mesh* m, const int32_t* ids, int64_t n) {
  ORC_TRY
  m->m.refine(std::vector<int>(ids, ids + n));
  m->remap();
  ORC_CATCH
}
int orc_mesh_uniform_refine(orc_mesh* m, int times) {
  ORC_TRY
  m->m.uniform_refine(times);
  m->remap();
  ORC_CATCH
}
// n_cells, n_active, max_level, V
int orc_mesh_info(orc_mesh* m, int64_t* info4, double* h_min) {
  info4[0] = int64_t(m->m.cells.size());
  info4[1] = int64_t(m->m.active.size());
  info4[2] = m->m.max_active_level();
  info4[3] = m->map.V;
  *h_min = m->m.min_active_edge();
  return 0;
}
// per cell: level, parent, active, anchor x/y/z (cells in id order)
int orc_mesh_cells(orc_mesh* m, int32_t* level, int32_t* parent, int8_t* active, int64_t* anchor) {
  for (size_t i = 0; i < m->m.cells.size(); ++i) {
    const gm::Cell& c = m->m.cells[i];
    level[i] = c.level;
    parent[i] = c.parent;
    active[i] = c.active;
    for (int a = 0; a < 3; ++a) anchor[3 * i + a] = c.anchor[a];
  }
  return 0;
}
int orc_mesh_active(orc_mesh* m, int32_t* ids) {
  std::copy(m->m.active.begin(), m->m.active.end(), ids);
  return 0;
}
int orc_mesh_vertex_keys(orc_mesh* m, int64_t* keys) {
  std::copy(m->map.keys.begin(), m->map.keys.end(), keys);
  return 0;
}
int orc_mesh_cell_vertices(orc_mesh* m, int64_t* out) {
  ORC_TRY
  const int nv = 1 << m->m.d;
  for (size_t i = 0; i < m->m.active.size(); ++i) m->map.cell_vertices(m->m, m->m.active[i], out + i * nv);
  ORC_CATCH
}
int orc_mesh_faces(orc_mesh* m, int64_t* n, int32_t* out5) {  // out5 may be null (count only)
  std::vector<gm::FaceEntry> f = gm::active_faces(m->m);
  *n = int64_t(f.size());
  if (out5)
    for (size_t i = 0; i < f.size(); ++i) {
      out5[5 * i] = f[i].cell;
      out5[5 * i + 1] = f[i].axis;
      out5[5 * i + 2] = f[i].side;
      out5[5 * i + 3] = f[i].neighbor;
      out5[5 * i + 4] = f[i].rel;
    }
  return 0;
}
int orc_mesh_find_cell(orc_mesh* m, const double* x, int32_t* out) {
  *out = m->m.find_active_cell_x(x);
  return 0;
}
int orc_mesh_constraints(orc_mesh* m, int clamp, int64_t n_active, const int64_t* dofs, const double* vals,
                         orc_mcs** out) {
  ORC_TRY
  *out = new orc_mcs{gm::build_constraints(m->m, m->map, clamp != 0, std::vector<i64>(dofs, dofs + n_active),
                                           std::vector<double>(vals, vals + n_active))};
  ORC_CATCH
}
void orc_mcs_destroy(orc_mcs* c) { delete c; }
// lines in ascending dof order: n_lines, total entries
int orc_mcs_info(orc_mcs* c, int64_t* n_lines, int64_t* n_entries) {
  *n_lines = int64_t(c->cs.lines.size());
  int64_t e = 0;
  for (const auto& kv : c->cs.lines) e += int64_t(kv.second.e.size());
  *n_entries = e;
  return 0;
}
int orc_mcs_export(orc_mcs* c, int64_t* dofs, int64_t* ptr, int64_t* masters, double* weights, double* inhom) {
  int64_t i = 0, k = 0;
  ptr[0] = 0;
  for (const auto& [dof, l] : c->cs.lines) {
    dofs[i] = dof;
    inhom[i] = l.inhom;
    for (const auto& [mm, w] : l.e) {
      masters[k] = mm;
      weights[k] = w;
      ++k;
    }
    ptr[++i] = k;
  }
  return 0;
}
int orc_mcs_distribute(orc_mcs* c, double* v, int64_t n, int homogeneous) {
  Vec x(v, v + n);
  if (homogeneous) c->cs.distribute_homogeneous(x); else c->cs.distribute(x);
  std::copy(x.begin(), x.end(), v);
  return 0;
}
int orc_mesh_residual(orc_mesh* m, orc_mcs* c, const orc_material* mat, const orc_regularization* r, const double* x,
                      const double* pt, double* R) {
  ORC_TRY
  check_material(*mat);
  Vec out = gm::assemble_residual(m->m, m->map, c->cs, *mat, *r, x, pt);
  std::copy(out.begin(), out.end(), R);
  ORC_CATCH
}
int orc_mesh_jacobian(orc_mesh* m, orc_mcs* c, const orc_material* mat, const orc_regularization* r, const double* x,
                      const double* pt, orc_block** out) {
  ORC_TRY
  check_material(*mat);
  *out = new orc_block{gm::assemble_jacobian(m->m, m->map, c->cs, *mat, *r, x, pt)};
  ORC_CATCH
}
int orc_mesh_rigid_body_modes(orc_mesh* m, orc_mcs* c, double* B_colmajor) {
  Dense B = gm::rigid_body_modes(m->m, m->map, c->cs);
  std::copy(B.a.begin(), B.a.end(), B_colmajor);
  return 0;
}
int orc_mesh_slit_band_edge(orc_mesh* m, const orc_material* mat, double* out) {
  ORC_TRY
  *out = gm::slit_band_edge(m->m, *mat);
  ORC_CATCH
}
int orc_mesh_resolve_regularization(orc_mesh* m, const orc_material* mat, double band_edge, orc_regularization* out) {
  ORC_TRY
  *out = gm::resolve_regularization(m->m, *mat, band_edge);
  ORC_CATCH
}
int orc_mesh_initial_crack(orc_mesh* m, const orc_material* mat, double band_half, double* phi, double* band_edge) {
  ORC_TRY
  Vec v = gm::initial_crack(m->m, m->map, *mat, band_half, band_edge);
  std::copy(v.begin(), v.end(), phi);
  ORC_CATCH
}
int orc_mesh_newton_step(orc_mesh* m, const orc_material* mat, const orc_regularization* r,
                         const orc_solver_options* o, double* solution, double* phi_old, double* phi_prev2, int step,
                         int shift, int max_its, double* its_out, int* n_its, int* converged, double* feasibility) {
  ORC_TRY
  const gm::DofMap& map = m->map;
  State st;
  st.solution.assign(solution, solution + map.n_total());
  st.phi_old.assign(phi_old, phi_old + map.V);
  st.phi_prev2.assign(phi_prev2, phi_prev2 + map.V);
  st.step = step;
  if (shift) {
    st.phi_prev2 = st.phi_old;
    st.phi_old.assign(st.solution.begin() + map.n_u(), st.solution.end());
  }
  NewtonReport rep = gm::newton_step(st, *mat, m->m, map, *r, *o);
  std::copy(st.solution.begin(), st.solution.end(), solution);
  std::copy(st.phi_old.begin(), st.phi_old.end(), phi_old);
  std::copy(st.phi_prev2.begin(), st.phi_prev2.end(), phi_prev2);
  *n_its = int(rep.its.size());
  for (int i = 0; i < int(rep.its.size()) && i < max_its; ++i) {
    its_out[4 * i] = rep.its[i].residual_norm;
    its_out[4 * i + 1] = rep.its[i].active_size;
    its_out[4 * i + 2] = rep.its[i].set_changes;
    its_out[4 * i + 3] = rep.its[i].gmres_iterations;
  }
  *converged = rep.converged;
  *feasibility = rep.feasibility;
  ORC_CATCH
}
int orc_mesh_tcv(orc_mesh* m, const double* sol, double* out) {
  ORC_TRY
  *out = gm::compute_tcv(m->m, m->map, sol);
  ORC_CATCH
}
int orc_mesh_cod(orc_mesh* m, const double* sol, const double* stations, int ns, double* out) {
  ORC_TRY
  gm::compute_cod(m->m, m->map, sol, stations, ns, out);
  ORC_CATCH
}
int orc_mesh_estimator(orc_mesh* m, const double* sol, double* eta) {
  ORC_TRY
  Vec e = gm::jump_estimator(m->m, m->map, sol);
  std::copy(e.begin(), e.end(), eta);
  ORC_CATCH
}
// policy5: phi_threshold, h_target, theta, max_level, estimator; eta may be null
int orc_mesh_mark(orc_mesh* m, const double* sol, const double* eta, const double* policy5, int32_t* out,
                  int64_t* n_out) {
  ORC_TRY
  gm::Policy pol{policy5[0], policy5[1], policy5[2], int(policy5[3]), policy5[4] != 0.0};
  Vec e;
  if (eta) e.assign(eta, eta + m->m.active.size());
  std::vector<int> ids = gm::mark_cells(m->m, m->map, sol, e, pol);
  std::copy(ids.begin(), ids.end(), out);
  *n_out = int64_t(ids.size());
  ORC_CATCH
}
int orc_mesh_transfer(orc_mesh* om, const double* ov, orc_mesh* nm, double* nv) {
  ORC_TRY
  Vec o(ov, ov + om->map.n_total());
  Vec out = gm::transfer(om->m, om->map, o, nm->m, nm->map);
  std::copy(out.begin(), out.end(), nv);
  ORC_CATCH
}
// adaptive_cycle: the mesh is refined in place; the final state is returned through the
// caller's buffers (sized by the caller after reading orc_mesh_info), records as 8 doubles each
int orc_mesh_adaptive_cycle(orc_mesh* m, const orc_material* mat, const orc_solver_options* so,
                            const double* policy5, int cycles, int n_steps, int estimator_rounds,
                            int halve_band_target, double seed_band, int max_rec, double* rec_out, int* n_rec,
                            double* solution, int64_t sol_cap) {
  ORC_TRY
  gm::AdaptOpts o;
  o.policy = gm::Policy{policy5[0], policy5[1], policy5[2], int(policy5[3]), policy5[4] != 0.0};
  o.solver = *so;
  o.cycles = cycles;
  o.n_steps = n_steps;
  o.estimator_rounds = estimator_rounds;
  o.halve_band_target = halve_band_target != 0;
  o.seed_band = seed_band;
  State st = gm::initial_state(m->m, m->map, *mat, seed_band);
  std::vector<gm::LevelRec> recs = gm::adaptive_cycle(m->m, m->map, st, *mat, o);
  *n_rec = int(recs.size());
  for (int i = 0; i < int(recs.size()) && i < max_rec; ++i) {
    double* r = rec_out + 8 * i;
    r[0] = recs[i].level;
    r[1] = double(recs[i].dofs);
    r[2] = recs[i].eps;
    r[3] = recs[i].h_min;
    r[4] = recs[i].tcv;
    r[5] = recs[i].newton_iters;
    r[6] = recs[i].gmres_mean;
    r[7] = recs[i].converged;
  }
  if (solution && sol_cap >= int64_t(st.solution.size())) std::copy(st.solution.begin(), st.solution.end(), solution);
  ORC_CATCH
}

}  // extern "C"

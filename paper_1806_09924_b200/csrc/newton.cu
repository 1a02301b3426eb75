// K9/K10 and the Newton / primal-dual active-set driver (solver.cpp:24-204).
//
// Control flow stays on the host exactly as in newton_active_set_step; every per-dof
// operation is a device kernel: the active-set test, the membership history (a 64-bit shift
// register per phi dof: all tracked histories have the same length, so the reference's
// zero-backfill is implicit), cycle detection (popcount of toggles in the last W bits), the
// change count, the constraint arrays, distribute, the rigid-body near-nullspace.  Only
// scalars (norms, counts) cross to the host per iteration.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "cf_comm.hpp"
#include "cf_mesh.hpp"
#include "cf_vec.hpp"

namespace cfb {

namespace {

template <class T>
T read_dev(const T* p) {
  T h{};
  read_small(&h, p, sizeof(T));
  return h;
}

// phi_tilde = phi_old (step <= 2) else clip(2 phi_old - phi_prev2, [0, 1]) (model.cpp:60-64)
__global__ void k_extrapolate(i64 V, int step, const double* __restrict__ po, const double* __restrict__ pp,
                              double* __restrict__ pt) {
  const i64 v = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= V) return;
  if (step <= 2) {
    pt[v] = po[v];
  } else {
    const double t = 2.0 * po[v] - pp[v];
    pt[v] = fmin(fmax(t, 0.0), 1.0);
  }
}

// Kernels below run over the slab's owned vertices lv in [0, nv) (v = v_lo + lv; the full slab of
// one GPU is v = lv).  Global-layout arrays (x, phi_old, constraint flags) are indexed by v,
// local-layout ones (R, delta, active-set state) by lv.

// active-set test + history push (solver.cpp:81-96).  tracked dofs push their bit.
__global__ void k_active1(Slab sl, i64 nu, double c, double tol, const double* __restrict__ x,
                          const double* __restrict__ po, const double* __restrict__ R,
                          const std::uint8_t* __restrict__ base_flag, const std::uint8_t* __restrict__ fixed,
                          std::uint8_t* __restrict__ active, std::uint8_t* __restrict__ tracked,
                          unsigned long long* __restrict__ hist, int nw, int* __restrict__ any_tracked, int d) {
  const i64 lv = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (lv >= sl.nv()) return;
  const i64 v = sl.v_lo + lv;
  const i64 dof = nu + v;
  bool a = fixed[lv] != 0;
  if (!base_flag[dof]) {  // candidates: phi dofs not constrained by the base set
    const double lambda = -R[d * sl.nv() + lv];
    if (c * (x[dof] - po[v]) + lambda > tol) a = true;
  }
  active[lv] = a ? 1 : 0;
  bool tr = tracked[lv] != 0 || a;
  if (tr) {  // the history is an nw-word shift register per dof, newest entry in bit 0 of word 0
    tracked[lv] = 1;
    unsigned long long* h = hist + lv * nw;
    for (int k = nw - 1; k > 0; --k) h[k] = (h[k] << 1) | (h[k - 1] >> 63);
    h[0] = (h[0] << 1) | (a ? 1ull : 0ull);
    *any_tracked = 1;
  }
}

// cycle detection on the last min(len, W) entries (solver.cpp:10-22, 97-100), set changes and |A|
__global__ void k_active2(i64 V, int len, int window, int toggles, const std::uint8_t* __restrict__ tracked,
                          const unsigned long long* __restrict__ hist, int nw, std::uint8_t* __restrict__ fixed,
                          std::uint8_t* __restrict__ active, const std::uint8_t* __restrict__ prev,
                          int* __restrict__ counts) {
  const i64 v = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= V) return;
  if (tracked[v]) {
    const int w = len < window ? len : window;
    int ch = 0;
    if (w > 1) {  // changes between entries i and i+1, i = 0 .. w-2 (bits of h ^ (h >> 1))
      const unsigned long long* h = hist + v * nw;
      for (int k = 0; k < nw && 64 * k < w - 1; ++k) {
        const unsigned long long nxt = (k + 1 < nw) ? (h[k + 1] << 63) : 0ull;
        const unsigned long long t = h[k] ^ ((h[k] >> 1) | nxt);
        const int bits = w - 1 - 64 * k;
        const unsigned long long mask = bits >= 64 ? ~0ull : ((1ull << bits) - 1ull);
        ch += __popcll(t & mask);
      }
    }
    if (ch >= toggles) {
      fixed[v] = 1;
      active[v] = 1;
    }
  }
  const int a = active[v];
  if (a) atomicAdd(&counts[0], 1);
  if (a != prev[v]) atomicAdd(&counts[1], 1);
}

// full constraint set on the owned phi dofs: base + active phi = phi_old (solver.cpp:109-111,
// fem.cpp:258-263); the u dofs keep the base (Dirichlet) lines
__global__ void k_full_constraints(Slab sl, i64 nu, const std::uint8_t* __restrict__ bflag,
                                   const double* __restrict__ binh, const std::uint8_t* __restrict__ active,
                                   const double* __restrict__ po, std::uint8_t* __restrict__ flag,
                                   double* __restrict__ inh) {
  const i64 lv = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (lv >= sl.nv()) return;
  const i64 v = sl.v_lo + lv, i = nu + v;
  std::uint8_t f = bflag[i];
  double g = binh[i];
  if (!f && active[lv]) {
    f = 1;
    g = po[v];
  }
  flag[i] = f;
  inh[i] = g;
}

// local dof i of the slab -> global dof
__device__ __forceinline__ i64 global_dof(const Slab& sl, int d, i64 nu, i64 i) {
  const i64 nul = d * sl.nv();
  return i < nul ? d * sl.v_lo + i : nu + sl.v_lo + (i - nul);
}

// distribute on the owned dofs of the global-layout x + "moved" flag (solver.cpp:114-116)
__global__ void k_distribute_moved(Slab sl, int d, i64 nu, const std::uint8_t* __restrict__ flag,
                                   const double* __restrict__ inh, double* __restrict__ x, int* __restrict__ moved) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= (d + 1) * sl.nv()) return;
  const i64 gi = global_dof(sl, d, nu, i);
  if (!flag[gi]) return;
  const double old = x[gi];
  x[gi] = inh[gi];
  if (fabs(x[gi] - old) > 0.0) *moved = 1;
}

// distribute on a local-layout vector (fem.cpp:229-247 on uniform meshes)
__global__ void k_distribute_local(Slab sl, int d, i64 nu, const std::uint8_t* __restrict__ flag,
                                   const double* __restrict__ inh, double* __restrict__ v, int homogeneous) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= (d + 1) * sl.nv()) return;
  const i64 gi = global_dof(sl, d, nu, i);
  if (flag[gi]) v[i] = homogeneous ? 0.0 : inh[gi];
}

// x(owned, global layout) += a * delta(local layout)
__global__ void k_axpy_owned(Slab sl, int d, i64 nu, double a, const double* __restrict__ delta,
                             double* __restrict__ x) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= (d + 1) * sl.nv()) return;
  x[global_dof(sl, d, nu, i)] += a * delta[i];
}

__global__ void k_zero_active(i64 V, i64 nu, const std::uint8_t* __restrict__ active, double* __restrict__ R) {
  const i64 v = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v < V && active[v]) R[nu + v] = 0.0;
}

__global__ void k_neg(i64 n, const double* __restrict__ a, double* __restrict__ b) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) b[i] = -a[i];
}

// rigid body modes (linsolve.cpp:320-343) of the owned vertices, zero rows on constrained u dofs
__global__ void k_rigid(GridDesc g, Slab sl, const std::uint8_t* __restrict__ flag, double* __restrict__ B) {
  const i64 lv = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (lv >= sl.nv()) return;
  const i64 v = sl.v_lo + lv;
  const int d = g.d;
  const i64 n = d * sl.nv();
  const i64 ix = v % g.nn, iy = (v / g.nn) % g.nn, iz = (d == 3) ? v / (g.nn * g.nn) : 0;
  const double x0 = -g.K + double(ix * (i64(1) << (16 - g.r))) * g.unit;
  const double x1 = -g.K + double(iy * (i64(1) << (16 - g.r))) * g.unit;
  const double x2 = (d == 3) ? -g.K + double(iz * (i64(1) << (16 - g.r))) * g.unit : 0.0;
  const int m = (d == 2) ? 3 : 6;
  double row[3][6];
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 6; ++c) row[a][c] = 0.0;
  for (int a = 0; a < d; ++a) row[a][a] = 1.0;
  if (d == 2) {
    row[0][2] = -x1;
    row[1][2] = x0;
  } else {
    row[1][3] = -x2;
    row[2][3] = x1;
    row[0][4] = x2;
    row[2][4] = -x0;
    row[0][5] = -x1;
    row[1][5] = x0;
  }
  for (int a = 0; a < d; ++a) {
    const bool con = flag[v * d + a] != 0;
    for (int c = 0; c < m; ++c) B[i64(c) * n + lv * d + a] = con ? 0.0 : row[a][c];
  }
}

__global__ void k_phi_modes(Slab sl, i64 nu, const std::uint8_t* __restrict__ flag, double* __restrict__ B,
                            int* __restrict__ pnode, int* __restrict__ unode, int d) {
  const i64 lv = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (lv >= sl.nv()) return;
  B[lv] = flag[nu + sl.v_lo + lv] ? 0.0 : 1.0;
  pnode[lv] = int(lv);
  for (int a = 0; a < d; ++a) unode[lv * d + a] = int(lv);
}

__global__ void k_feas(Slab sl, i64 nu, const double* __restrict__ x, const double* __restrict__ po, double* out) {
  const i64 lv = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  // max via the ordered-int trick for doubles (handles negatives); a warp maximum first, one
  // atomic per warp (the maximum is exact in any order)
  long long bits = LLONG_MIN;
  if (lv < sl.nv()) {
    const i64 v = sl.v_lo + lv;
    const double d = x[nu + v] - po[v];
    bits = __double_as_longlong(d);
    bits = bits >= 0 ? bits : (bits ^ 0x7fffffffffffffffLL);
  }
  for (int o = 16; o > 0; o >>= 1) bits = max(bits, __shfl_xor_sync(0xffffffffu, bits, o));
  if ((threadIdx.x & 31) == 0 && bits != LLONG_MIN) atomicMax(reinterpret_cast<long long*>(out), bits);
}

struct Timer {
  cudaEvent_t a, b;
  double* acc;
  Timer(double* slot) : acc(slot) {
    CF_CUDA(cudaEventCreate(&a));
    CF_CUDA(cudaEventCreate(&b));
    CF_CUDA(cudaEventRecord(a, stream()));
  }
  ~Timer() {
    cudaEventRecord(b, stream());
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    *acc += ms;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
};

}  // namespace

void rigid_body_modes(const Problem& P, const Constraints& c, double* B, const Slab* slab) {
  const Slab sl = slab ? *slab : full_slab(P.g);
  k_rigid<<<grid_for(sl.nv(), 256), 256, 0, stream()>>>(P.g, sl, c.flag.p, B);
  CF_LAUNCHED();
}

void extrapolate_phi(const State& st, double* pt, i64 V) {
  k_extrapolate<<<grid_for(V, 256), 256, 0, stream()>>>(V, st.step, st.phi_old.p, st.phi_prev2.p, pt);
  CF_LAUNCHED();
}

Slab rank_slab(const GridDesc& g, int rank, int size) {
  if (size < 1 || rank < 0 || rank >= size) fail(CF_ERR_INVALID_ARGUMENT, "rank_slab: bad rank / size");
  if (g.nn < size) fail(CF_ERR_UNSUPPORTED, "rank_slab: fewer vertex planes than ranks");
  return make_slab(g, g.nn * rank / size, g.nn * (rank + 1) / size);
}

namespace {

// Ghost-plane exchange of a global-layout vector [u (d V) | phi (V)] of element size es: the
// owned boundary planes go to the neighbours, their planes land in this rank's ghost planes.
void halo_global(const Comm& cm, const GridDesc& g, const Slab& sl, void* vec, size_t es, bool u_part, bool p_part) {
  if (!cm.distributed()) return;
  auto* b = static_cast<unsigned char*>(vec);
  const i64 d = g.d, pl = sl.plane;
  std::vector<HaloOp> ops;
  auto add = [&](i64 send_off, i64 recv_off, i64 count, int peer) {
    ops.push_back({b + size_t(send_off) * es, b + size_t(recv_off) * es, size_t(count) * es, peer});
  };
  if (cm.rank > 0) {
    if (u_part) add(d * sl.v_lo, d * (sl.v_lo - pl), d * pl, cm.rank - 1);
    if (p_part) add(g.n_u() + sl.v_lo, g.n_u() + sl.v_lo - pl, pl, cm.rank - 1);
  }
  if (cm.rank + 1 < cm.size) {
    if (u_part) add(d * (sl.v_hi - pl), d * sl.v_hi, d * pl, cm.rank + 1);
    if (p_part) add(g.n_u() + sl.v_hi - pl, g.n_u() + sl.v_hi, pl, cm.rank + 1);
  }
  cm.sendrecv(ops);
}

// local-layout z [u_own | phi_own] -> ext-layout e [u_ext | phi_ext] (interior copy + ghost planes)
void to_ext(const Comm& cm, const GridDesc& g, const Slab& sl, const double* z, double* e) {
  const i64 d = g.d, nv = sl.nv(), ne = sl.ne(), pl = sl.plane, lo = sl.v_lo - sl.ve_lo;
  const i64 nul = d * nv, nue = d * ne;
  CF_CUDA(cudaMemcpyAsync(e + d * lo, z, size_t(nul) * sizeof(double), cudaMemcpyDeviceToDevice, stream()));
  CF_CUDA(cudaMemcpyAsync(e + nue + lo, z + nul, size_t(nv) * sizeof(double), cudaMemcpyDeviceToDevice, stream()));
  std::vector<HaloOp> ops;
  const size_t ub = size_t(d * pl) * sizeof(double), pb = size_t(pl) * sizeof(double);
  if (cm.rank > 0) {
    ops.push_back({z, e, ub, cm.rank - 1});
    ops.push_back({z + nul, e + nue, pb, cm.rank - 1});
  }
  if (cm.rank + 1 < cm.size) {
    ops.push_back({z + nul - d * pl, e + d * (ne - pl), ub, cm.rank + 1});
    ops.push_back({z + nul + nv - pl, e + nue + ne - pl, pb, cm.rank + 1});
  }
  cm.sendrecv(ops);
}

// every rank's owned part of a global-layout vector to every rank
void allgather_owned(const Comm& cm, const GridDesc& g, double* x) {
  if (!cm.distributed()) return;
  std::vector<HaloOp> ops;
  for (int r = 0; r < cm.size; ++r) {
    const Slab s = rank_slab(g, r, cm.size);
    ops.push_back({nullptr, x + g.d * s.v_lo, size_t(g.d * s.nv()) * sizeof(double), r});
    ops.push_back({nullptr, x + g.n_u() + s.v_lo, size_t(s.nv()) * sizeof(double), r});
  }
  cm.bcast_many(ops);
}

// every rank's owned part of a global-layout array of element size es (bytes) to every rank
void allgather_owned_bytes(const Comm& cm, const GridDesc& g, void* vec, size_t es) {
  if (!cm.distributed()) return;
  auto* b = static_cast<unsigned char*>(vec);
  std::vector<HaloOp> ops;
  for (int r = 0; r < cm.size; ++r) {
    const Slab s = rank_slab(g, r, cm.size);
    ops.push_back({nullptr, b + size_t(g.d * s.v_lo) * es, size_t(g.d * s.nv()) * es, r});
    ops.push_back({nullptr, b + size_t(g.n_u() + s.v_lo) * es, size_t(s.nv()) * es, r});
  }
  cm.bcast_many(ops);
}

__global__ void k_shift_i64(const i64* __restrict__ a, i64 n, i64 add, i64* __restrict__ out) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i] + add;
}
__global__ void k_shift_i32(const int* __restrict__ a, i64 n, i64 add, int* __restrict__ out) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = int(a[i] + add);
}

// The undivided CSR block on every rank: rank r holds the rows of its owned vertices
// (rows_per_vertex each) with columns in its ext numbering (global column = column + cols_per_vertex
// * ve_lo); the row pointers, columns and values of every rank are broadcast into one global
// matrix, bitwise the single-GPU block.
std::shared_ptr<Csr> gather_block(const Comm& cm, const GridDesc& g, const Csr& loc, int rows_per_vertex,
                                  int cols_per_vertex) {
  const int P = cm.size;
  std::vector<long long> nnz(P, 0);
  nnz[cm.rank] = loc.nnz;
  cm.sum_i64(nnz.data(), P);
  auto G = std::make_shared<Csr>();
  G->rows = G->cols = rows_per_vertex * g.V;
  i64 tot = 0;
  for (int r = 0; r < P; ++r) tot += nnz[r];
  G->nnz = tot;
  G->ptr.alloc(G->rows + 1);
  G->col.alloc(std::max<i64>(tot, 1));
  G->val.alloc(std::max<i64>(tot, 1));
  std::vector<HaloOp> ops;
  i64 off = 0;
  for (int r = 0; r < P; ++r) {
    const Slab s = rank_slab(g, r, P);
    const i64 row0 = rows_per_vertex * s.v_lo, nr = rows_per_vertex * s.nv();
    if (r == cm.rank) {
      if (nr > 0) {
        k_shift_i64<<<grid_for(nr, 256), 256, 0, stream()>>>(loc.ptr.p, nr, off, G->ptr.p + row0);
        CF_LAUNCHED();
      }
      if (loc.nnz > 0) {
        k_shift_i32<<<grid_for(loc.nnz, 256), 256, 0, stream()>>>(loc.col.p, loc.nnz, cols_per_vertex * s.ve_lo,
                                                                  G->col.p + off);
        CF_LAUNCHED();
        CF_CUDA(cudaMemcpyAsync(G->val.p + off, loc.val.p, size_t(loc.nnz) * sizeof(double), cudaMemcpyDeviceToDevice,
                                stream()));
      }
    }
    ops.push_back({nullptr, G->ptr.p + row0, size_t(nr) * sizeof(i64), r});
    ops.push_back({nullptr, G->col.p + off, size_t(nnz[r]) * sizeof(int), r});
    ops.push_back({nullptr, G->val.p + off, size_t(nnz[r]) * sizeof(double), r});
    off += nnz[r];
  }
  cm.bcast_many(ops);
  const i64 end = tot;
  CF_CUDA(cudaMemcpyAsync(G->ptr.p + G->rows, &end, sizeof(i64), cudaMemcpyHostToDevice, stream()));
  CF_CUDA(cudaStreamSynchronize(stream()));
  return G;
}

// ||v|| of a slab block vector in the NP-invariant segmented order (SegLayout)
double gnorm(const Comm* cm, const double* v, const SegLayout& L) {
  double* s = scalar_buf(1);
  seg_dot_dev(v, v, L, s, true, cm);
  double h = 0.0;
  read_small(&h, s, sizeof(double));
  return h;
}

SegLayout seg_layout(const GridDesc& g, const Slab& sl) {
  SegLayout L;
  L.plane_u = g.d * sl.plane;
  L.plane_p = sl.plane;
  L.p_lo = int(sl.v_lo / sl.plane);
  L.p_hi = int(sl.v_hi / sl.plane);
  L.nplanes = int(g.nn);
  return L;
}

}  // namespace

double slit_band_edge(const Problem& P, const cf_material& mat) {  // model.cpp:28-50 (uniform cells)
  const GridDesc& g = P.g;
  auto coord = [&](i64 i) { return -g.K + double(i * (i64(1) << (16 - g.r))) * g.unit; };
  const i64 nz = (g.d == 3) ? g.nc : 1;
  for (i64 cz = 0; cz < nz; ++cz) {
    if (g.d == 3 && !(coord(cz) <= 0.0 && coord(cz + 1) >= 0.0)) continue;
    for (i64 cy = 0; cy < g.nc; ++cy)
      for (i64 cx = 0; cx < g.nc; ++cx) {
        const double lo0 = coord(cx), hi0 = coord(cx + 1), lo1 = coord(cy), hi1 = coord(cy + 1);
        bool meets;
        if (g.d == 2) {
          meets = lo1 <= 0.0 && hi1 >= 0.0 && lo0 <= mat.l0 && hi0 >= -mat.l0;
        } else {
          const double dx = std::max({lo0, 0.0, -hi0});
          const double dy = std::max({lo1, 0.0, -hi1});
          meets = std::hypot(dx, dy) <= mat.l0;
        }
        if (meets) return g.h;  // all active cells share the edge h on a uniform mesh
      }
  }
  fail(CF_ERR_NUMERICAL, "slit_band_edge: no active cell meets the slit");
}

cf_regularization resolve_regularization(const Problem& P, const cf_material& mat, double band_edge) {
  cf_regularization reg;  // model.cpp:52-58
  const double diam = band_edge * std::sqrt(double(P.g.d));
  reg.eps = (mat.eps_mode == 0) ? mat.c_eps * diam : mat.eps_fixed;
  reg.kappa = mat.kappa_factor * P.g.h;
  return reg;
}

std::vector<double> initial_crack(const Problem& P, const cf_material& mat, double band_half, double* band_edge) {
  const GridDesc& g = P.g;  // model.cpp:324-349
  const double be = band_half > 0.0 ? band_half : slit_band_edge(P, mat);
  std::vector<double> phi(g.V, 1.0);
  const double tol = 1e-9 * be;
  auto coord = [&](i64 i) { return -g.K + double(i * (i64(1) << (16 - g.r))) * g.unit; };
  i64 n_zero = 0, n_plane = 0;
  for (i64 v = 0; v < g.V; ++v) {
    const i64 ix = v % g.nn, iy = (v / g.nn) % g.nn, iz = (g.d == 3) ? v / (g.nn * g.nn) : 0;
    const double x0 = coord(ix), x1 = coord(iy), x2 = (g.d == 3) ? coord(iz) : 0.0;
    bool in;
    if (g.d == 2)
      in = std::abs(x0) <= mat.l0 + tol && std::abs(x1) <= be + tol;
    else
      in = std::hypot(x0, x1) <= mat.l0 + tol && std::abs(x2) <= be + tol;
    if (in) {
      phi[v] = 0.0;
      ++n_zero;
      if (std::abs(g.d == 2 ? x1 : x2) <= tol) ++n_plane;
    }
  }
  if (n_zero == 0 || n_plane == 0)
    fail(CF_ERR_NUMERICAL, "initial_crack: slit is not resolved by the mesh (no vertex layer inside the band)");
  if (band_edge) *band_edge = be;
  return phi;
}

NewtonReport newton_active_set_step(Problem& P, State& st, const cf_material& mat, const cf_regularization& reg,
                                    const cf_solver_options& opts, const Comm* comm, const Slab* slab) {
  const GridDesc& g = P.g;
  const Comm solo;
  const Comm& cm = comm ? *comm : solo;
  const bool dist = cm.distributed();
  const Slab sl = slab ? *slab : (dist ? rank_slab(g, cm.rank, cm.size) : full_slab(g));
  if (!dist && !sl.full(g)) fail(CF_ERR_INVALID_ARGUMENT, "newton_active_set_step: a partial slab needs a communicator");
  const int d = g.d;
  const i64 nu = g.n_u(), V = g.V, nt = g.n_total();
  const i64 nv = sl.nv(), nul = d * nv, ntl = (d + 1) * nv;  // this rank's rows
  // history words per dof: the last `window` entries (any window, as detect_cycles, solver.cpp:10-22;
  // window <= 1 sees no change)
  const int nw = std::max(1, (opts.cycle_window + 63) / 64);
  NewtonReport report;
  PhaseTimes& T = report.times;
  auto base = build_constraints(P, true, 0, nullptr, nullptr);  // solver.cpp:55
  double* x = st.solution.p;
  distribute(*base, x, false);
  DevBuf<double> pt(V);
  extrapolate_phi(st, pt.p, V);
  const double c = opts.active_set_c_scale * mat.G_c / reg.eps;
  DevBuf<std::uint8_t> fixed(nv), active(nv), prev(nv), tracked(nv);
  DevBuf<unsigned long long> hist(nv * nw);
  fixed.zero();
  prev.zero();
  tracked.zero();
  hist.zero();
  DevBuf<int> flags(4);
  DevBuf<double> R(ntl), rhs(ntl), delta(ntl);
  DevBuf<double> xb(nt);    // x before the active-set distribute (the moved cells)
  ResidualCache rcache;     // element residuals of the iteration's first assembly
  DevBuf<double> ext(dist ? (d + 1) * sl.ne() : 0);  // GMRES operator input with ghost planes
  int hist_len = 0;
  double res0 = -1.0;
  std::unique_ptr<BlockPrec> prec;
  Constraints full;
  full.prob = &P;
  full.flag.alloc(nt);
  full.inhom.alloc(nt);
  CF_CUDA(cudaMemcpyAsync(full.flag.p, base->flag.p, size_t(nt), cudaMemcpyDeviceToDevice, stream()));
  CF_CUDA(cudaMemcpyAsync(full.inhom.p, base->inhom.p, size_t(nt) * sizeof(double), cudaMemcpyDeviceToDevice,
                          stream()));
  DevBuf<double> Bu(nul * (d == 2 ? 3 : 6)), Bp(nv);
  std::shared_ptr<Csr> uu_step;  // this load step's M_uu
  std::shared_ptr<Csr> uu_loc;   // its diagonal slab block (distributed preconditioner)
  const Csr* uu_loc_src = nullptr;
  // distributed preconditioner: restricted additive Schwarz with one plane of overlap (default), or
  // block-Jacobi over the slabs (CF_BLOCK_JACOBI=1)
  // distributed preconditioner (N > 1):
  //  * default: the reference's block AMG on the undivided blocks (gathered on every rank once per
  //    build; the global hierarchy is identical to the single-GPU one), applied to the all-gathered
  //    residual: together with the segmented dots the N-rank step is bitwise the 1-GPU step;
  //  * CF_RAS=1: restricted additive Schwarz, per-slab block AMG with one plane of overlap;
  //  * CF_BLOCK_JACOBI=1: block-Jacobi over the slabs.
  // The two local variants scale the setup but change the preconditioner (and GMRES counts) with N.
  static const bool bj_env = std::getenv("CF_BLOCK_JACOBI") != nullptr;
  static const bool ras_env = std::getenv("CF_RAS") != nullptr;
  const bool ras = dist && ras_env && !bj_env;
  const bool glob = dist && !ras_env && !bj_env;
  std::shared_ptr<Csr> uu_glob;  // the gathered M_uu of this load step
  const Csr* uu_glob_src = nullptr;
  Constraints fullg;  // every rank's constraint flags (global preconditioner)
  if (glob) {
    fullg.prob = &P;
    fullg.flag.alloc(nt);
  }
  DevBuf<double> Bug(glob ? nu * (d == 2 ? 3 : 6) : 0), Bpg(glob ? V : 0);
  DevBuf<int> unodeg(glob ? nu : 0), pnodeg(glob ? V : 0);
  DevBuf<double> gin(glob ? nt : 0), gout(glob ? nt : 0);
  const Slab sx = ras ? make_slab(g, sl.ve_lo / sl.plane, sl.ve_hi / sl.plane) : sl;
  std::shared_ptr<Csr> uu_x_step;
  DevBuf<double> Bux(ras ? d * sx.nv() * (d == 2 ? 3 : 6) : 0), Bpx(ras ? sx.nv() : 0);
  DevBuf<int> unodex(ras ? d * sx.nv() : 0), pnodex(ras ? sx.nv() : 0);
  DevBuf<double> pin(ras ? (d + 1) * sx.nv() : 0), pout(ras ? (d + 1) * sx.nv() : 0);
  DevBuf<int> unode(nul), pnode(nv);
  const unsigned gv = grid_for(nv, 256), gl = grid_for(ntl, 256);
  const SegLayout seg = seg_layout(g, sl);  // every norm / dot of the step: NP-invariant order
  // operator_kind 1 (3d, one GPU): M_uu applied matrix-free in the Krylov operator and on the
  // u-hierarchy's finest level (mf.cu); M_uu is still assembled once per step for the AMG setup
  // N > 1 (the gathered global AMG): each rank applies its slab's rows (x on the ext planes) and its
  // V-cycle row chunk of level 0 matrix-free, bitwise the rows of the 1-GPU apply
  std::shared_ptr<MfOp> mf, mf_slab;
  if (opts.operator_kind == 1 && d == 3 && (!dist || glob)) {
    mf = std::make_shared<MfOp>();
    mf->P = &P;
    mf->flag = base->flag.p;  // the u constraints of every set of the step
    mf->mu = mat_mu(mat);
    mf->lam = mat_lambda(mat);
    mf->kap = reg.kappa;
    mf->pt = pt.p;
    mf_slab = std::make_shared<MfOp>(*mf);
    mf_slab->x_off = sl.ve_lo;
    mf_slab->y_lo = sl.v_lo;
    mf_slab->y_hi = sl.v_hi;
  }
  for (int it = 1; it <= opts.newton_max_iter; ++it) {
    {
      Timer t(&T.residual);
      assemble_residual(P, *base, mat, reg, x, pt.p, R.p, &sl, &rcache);
    }
    int changes = 0, asize = 0;
    {
      Timer t(&T.active_set);
      flags.zero();
      k_active1<<<gv, 256, 0, stream()>>>(sl, nu, c, 1e-14 * c, x, st.phi_old.p, R.p, base->flag.p, fixed.p,
                                          active.p, tracked.p, hist.p, nw, flags.p + 2, d);
      CF_LAUNCHED();
      long long any = read_dev(flags.p + 2);
      cm.max_i64(&any, 1);
      if (any) ++hist_len;
      k_active2<<<gv, 256, 0, stream()>>>(nv, hist_len, opts.cycle_window, opts.cycle_toggles, tracked.p, hist.p, nw,
                                          fixed.p, active.p, prev.p, flags.p);
      CF_LAUNCHED();
      int hc[2];
      read_small(hc, flags.p, 2 * sizeof(int));
      long long counts[2] = {hc[0], hc[1]};
      cm.sum_i64(counts, 2);
      asize = int(counts[0]);
      changes = int(counts[1]);
      k_full_constraints<<<gv, 256, 0, stream()>>>(sl, nu, base->flag.p, base->inhom.p, active.p, st.phi_old.p,
                                                   full.flag.p, full.inhom.p);
      CF_LAUNCHED();
      halo_global(cm, g, sl, full.flag.p, 1, false, true);  // neighbours' active phi columns
      CF_CUDA(cudaMemcpyAsync(xb.p, x, size_t(nt) * sizeof(double), cudaMemcpyDeviceToDevice, stream()));
      CF_CUDA(cudaMemsetAsync(flags.p + 3, 0, sizeof(int), stream()));
      k_distribute_moved<<<gl, 256, 0, stream()>>>(sl, d, nu, full.flag.p, full.inhom.p, x, flags.p + 3);
      CF_LAUNCHED();
      halo_global(cm, g, sl, x, sizeof(double), false, true);
    }
    long long moved = read_dev(flags.p + 3);
    cm.max_i64(&moved, 1);
    {
      Timer t(&T.residual);
      if (moved) {  // only the cells touching moved dofs are recomputed (bitwise the full assembly)
        assemble_residual_moved(P, full, mat, reg, x, xb.p, pt.p, R.p, &sl, rcache);
      } else {
        k_zero_active<<<gv, 256, 0, stream()>>>(nv, nul, active.p, R.p);
        CF_LAUNCHED();
      }
    }
    const double res = gnorm(comm, R.p, seg);
    if (res0 < 0.0) res0 = res;
    NewtonIter rec{res, asize, changes, 0};
    const bool small = res <= std::max(opts.newton_tol * res0, opts.newton_abs_floor);
    if (changes == 0 && small) {
      report.its.push_back(rec);
      if (opts.log && cm.rank == 0)
        std::printf("newton step=%d it=%d res=%.6e active=%d changed=%d gmres=0\n", st.step, it, res, asize,
                    changes);
      report.converged = true;
      break;
    }
    std::unique_ptr<BlockSystem> J;
    {
      Timer t(&T.jacobian);
      // M_uu depends only on phi_tilde (fixed for the load step) and the Dirichlet set
      // (model.cpp:268-276): it is assembled once per step and shared by the later iterations.
      // CF_VERIFY_UU_REUSE=1 re-assembles it every iteration and checks it bitwise.
      static const bool verify = std::getenv("CF_VERIFY_UU_REUSE") != nullptr;
      static const bool no_reuse = std::getenv("CF_NO_UU_REUSE") != nullptr;
      J = assemble_jacobian(P, full, mat, reg, x, pt.p, &sl, (verify || no_reuse) ? nullptr : uu_step);
      if (verify && uu_step) {
        const Csr &a = *J->uu, &b = *uu_step;
        if (a.nnz != b.nnz || !bitwise_equal(a.ptr.p, b.ptr.p, size_t(a.rows + 1) * sizeof(i64)) ||
            !bitwise_equal(a.col.p, b.col.p, size_t(a.nnz) * sizeof(int)) ||
            !bitwise_equal(a.val.p, b.val.p, size_t(a.nnz) * sizeof(double)))
          fail(CF_ERR_LOGIC, "newton_active_set_step: M_uu changed within a load step");
        J->uu = uu_step;
      }
      if (!uu_step) uu_step = J->uu;
      if (dist) {  // lane split of the undivided matrix, so every row reduces as on one GPU
        long long tot[4] = {J->uu->nnz, J->uu->rows, J->pu->nnz, J->pu->rows};
        cm.sum_i64(tot, 4);
        J->uu->mean_hint = tot[1] ? double(tot[0]) / double(tot[1]) : 0.0;
        J->pu->mean_hint = tot[3] ? double(tot[2]) / double(tot[3]) : 0.0;
      }
    }
    if (mf) J->mf_uu = mf_slab;
    if (!prec || !opts.freeze_preconditioner) {
      Timer t(&T.amg_setup);
      NullspaceDev ns;
      rigid_body_modes(P, full, Bu.p, &sl);
      k_phi_modes<<<gv, 256, 0, stream()>>>(sl, nu, full.flag.p, Bp.p, pnode.p, unode.p, d);
      CF_LAUNCHED();
      ns.u_node = unode.p;
      ns.u_modes = Bu.p;
      ns.m_u = d == 2 ? 3 : 6;
      ns.p_node = pnode.p;
      ns.p_modes = Bp.p;
      // hierarchies whose inputs are bitwise unchanged (M_uu within a load step: it depends only
      // on phi_tilde and the Dirichlet set) are reused; a rebuild would be bit-identical
      if (glob) {
        CF_CUDA(cudaMemcpyAsync(fullg.flag.p, full.flag.p, size_t(nt), cudaMemcpyDeviceToDevice, stream()));
        allgather_owned_bytes(cm, g, fullg.flag.p, 1);
        BlockSystem Jg;
        Jg.d = d;
        Jg.nu = nu;
        Jg.np = V;
        if (uu_glob_src != J->uu.get()) {  // the M_uu of a load step is gathered once
          uu_glob = gather_block(cm, g, *J->uu, d, d);
          csr_enable_stencil(*uu_glob, StencilCols{1, d, g.nn, 0, 0, 1.0 / double(g.nn)});
          uu_glob_src = J->uu.get();
        }
        Jg.uu = uu_glob;
        Jg.pp = gather_block(cm, g, *J->pp, 1, 1);
        rigid_body_modes(P, fullg, Bug.p, nullptr);
        const Slab fs = full_slab(g);
        k_phi_modes<<<grid_for(V, 256), 256, 0, stream()>>>(fs, nu, fullg.flag.p, Bpg.p, pnodeg.p, unodeg.p, d);
        CF_LAUNCHED();
        NullspaceDev nsg{unodeg.p, Bug.p, d == 2 ? 3 : 6, pnodeg.p, Bpg.p};
        prec = build_block_prec(Jg, opts.prec_kind, opts.amg, &nsg, prec.get());
        // the large leading levels apply by rows split over the ranks (a reused hierarchy keeps
        // its split); the V-cycles then run in sequence on the library stream (collectives)
        static const bool no_split = std::getenv("CF_VCYCLE_REPLICATED") != nullptr;
        if (!no_split) {
          // CF_VCYCLE_SPLIT_MIN (test switch): the smallest level split over the ranks
          static const char* smin = std::getenv("CF_VCYCLE_SPLIT_MIN");
          const i64 min_rows = smin ? std::atoll(smin) : std::max<i64>(65536, 1024 * i64(cm.size));
          for (Amg* h : {prec->amg_u.get(), prec->amg_p.get()})
            if (h && h->comm != &cm) h->distribute(&cm, min_rows);
          prec->serial = true;
        }
      } else if (dist) {
        // block-Jacobi over the slabs: the preconditioner of each rank is built on the diagonal
        // block of its rows (owned columns only); one GPU is the undivided block
        BlockSystem Jl;
        Jl.d = d;
        if (ras) {
          // restricted additive Schwarz: the block of the owned planes plus one plane of overlap
          // on each side (rows assembled for the extended slab, columns cut to it).  The overlap
          // rows read x and the constraint flags two planes beyond the owned ones, where the
          // one-plane halo is not current: every rank's owned planes are all-gathered first.
          allgather_owned(cm, g, x);
          allgather_owned_bytes(cm, g, full.flag.p, 1);
          auto Jx = assemble_jacobian(P, full, mat, reg, x, pt.p, &sx, uu_x_step);
          if (!uu_x_step) uu_x_step = Jx->uu;
          const i64 lo = sx.v_lo - sx.ve_lo, nx = sx.nv();
          if (uu_loc_src != Jx->uu.get()) {
            uu_loc = csr_extract_cols(*Jx->uu, d * lo, d * (lo + nx));
            uu_loc_src = Jx->uu.get();
          }
          Jl.nu = d * nx;
          Jl.np = nx;
          Jl.uu = uu_loc;
          Jl.pp = csr_extract_cols(*Jx->pp, lo, lo + nx);
          rigid_body_modes(P, full, Bux.p, &sx);
          k_phi_modes<<<grid_for(nx, 256), 256, 0, stream()>>>(sx, nu, full.flag.p, Bpx.p, pnodex.p, unodex.p, d);
          CF_LAUNCHED();
          NullspaceDev nsx{unodex.p, Bux.p, d == 2 ? 3 : 6, pnodex.p, Bpx.p};
          prec = build_block_prec(Jl, opts.prec_kind, opts.amg, &nsx, prec.get());
        } else {
          // block-Jacobi over the slabs: each rank's preconditioner on its diagonal block
          Jl.nu = nul;
          Jl.np = nv;
          const i64 lo = sl.v_lo - sl.ve_lo;
          if (uu_loc_src != J->uu.get()) {  // the diagonal block of a reused M_uu is reused too
            uu_loc = csr_extract_cols(*J->uu, d * lo, d * (lo + nv));
            uu_loc_src = J->uu.get();
          }
          Jl.uu = uu_loc;
          Jl.pp = csr_extract_cols(*J->pp, lo, lo + nv);
          prec = build_block_prec(Jl, opts.prec_kind, opts.amg, &ns, prec.get());
        }
      } else {
        prec = build_block_prec(*J, opts.prec_kind, opts.amg, &ns, prec.get());
      }
    }
    if (mf && prec->amg_u && prec->amg_u->n == nu) prec->amg_u->mf0 = mf;
    GmresResult lin;
    {
      Timer t(&T.gmres);
      k_neg<<<gl, 256, 0, stream()>>>(ntl, R.p, rhs.p);
      CF_LAUNCHED();
      const BlockSystem& Jr = *J;
      DevOp op;
      if (dist) {
        double* e = ext.p;
        op = [&Jr, &cm, &g, &sl, e](const double* in, double* out) {
          to_ext(cm, g, sl, in, e);
          block_apply(Jr, e, out);
        };
      } else {
        op = [&Jr](const double* in, double* out) { block_apply(Jr, in, out); };
      }
      const BlockPrec& Pr = *prec;
      DevOp pop = [&Pr](const double* in, double* out) { Pr.apply(in, out); };
      if (glob) {  // the whole residual on every rank, the global V-cycles, the owned rows kept
        double *gi = gin.p, *go = gout.p;
        pop = [&Pr, &cm, &g, &sl, gi, go, d, nv, nul, nu](const double* in, double* out) {
          CF_CUDA(cudaMemcpyAsync(gi + d * sl.v_lo, in, size_t(nul) * sizeof(double), cudaMemcpyDeviceToDevice,
                                  stream()));
          CF_CUDA(cudaMemcpyAsync(gi + nu + sl.v_lo, in + nul, size_t(nv) * sizeof(double), cudaMemcpyDeviceToDevice,
                                  stream()));
          allgather_owned(cm, g, gi);
          Pr.apply(gi, go);
          CF_CUDA(cudaMemcpyAsync(out, go + d * sl.v_lo, size_t(nul) * sizeof(double), cudaMemcpyDeviceToDevice,
                                  stream()));
          CF_CUDA(cudaMemcpyAsync(out + nul, go + nu + sl.v_lo, size_t(nv) * sizeof(double), cudaMemcpyDeviceToDevice,
                                  stream()));
        };
      }
      if (ras) {  // residual on the extended slab (halo planes), local solve, keep the owned rows
        double *pi = pin.p, *po = pout.p;
        pop = [&Pr, &cm, &g, &sl, &sx, pi, po, d, nv, nul](const double* in, double* out) {
          to_ext(cm, g, sl, in, pi);
          Pr.apply(pi, po);
          const i64 lo = sl.v_lo - sl.ve_lo, nx = sx.nv();
          CF_CUDA(cudaMemcpyAsync(out, po + d * lo, size_t(nul) * sizeof(double), cudaMemcpyDeviceToDevice, stream()));
          CF_CUDA(cudaMemcpyAsync(out + nul, po + d * nx + lo, size_t(nv) * sizeof(double), cudaMemcpyDeviceToDevice,
                                  stream()));
        };
      }
      lin = gmres(op, &pop, rhs.p, ntl, opts.gmres, delta.p, comm, &seg);
    }
    if (!lin.converged && !lin.breakdown) fail(CF_ERR_NUMERICAL, "newton_active_set_step: GMRES stagnated at max_iter");
    rec.gmres_iterations = lin.iterations;
    report.its.push_back(rec);
    if (opts.log && cm.rank == 0)
      std::printf("newton step=%d it=%d res=%.6e active=%d changed=%d gmres=%d\n", st.step, it, res, asize, changes,
                  lin.iterations);
    auto update_x = [&](double a) {
      if (sl.full(g)) {
        vaxpy(a, delta.p, x, nt);
      } else {
        k_axpy_owned<<<gl, 256, 0, stream()>>>(sl, d, nu, a, delta.p, x);
        CF_LAUNCHED();
        halo_global(cm, g, sl, x, sizeof(double), true, true);
      }
    };
    if (sl.full(g)) {
      distribute(full, delta.p, true);
    } else {
      k_distribute_local<<<gl, 256, 0, stream()>>>(sl, d, nu, full.flag.p, full.inhom.p, delta.p, 1);
      CF_LAUNCHED();
    }
    update_x(1.0);
    if (opts.damping) {
      double scale = 1.0;
      for (int half = 0; half < 4; ++half) {
        assemble_residual(P, full, mat, reg, x, pt.p, R.p, &sl);
        if (gnorm(comm, R.p, seg) <= 10.0 * res) break;
        scale *= 0.5;
        update_x(-scale);
      }
    }
    CF_CUDA(cudaMemcpyAsync(prev.p, active.p, size_t(nv), cudaMemcpyDeviceToDevice, stream()));
  }
  DevBuf<double> mx(1);
  {
    const long long lowest = 0x8000000000000000LL;  // below every mapped double
    CF_CUDA(cudaMemcpyAsync(mx.p, &lowest, sizeof(lowest), cudaMemcpyHostToDevice, stream()));
  }
  k_feas<<<gv, 256, 0, stream()>>>(sl, nu, x, st.phi_old.p, mx.p);
  CF_LAUNCHED();
  long long bits = 0;
  read_small(&bits, mx.p, sizeof(bits));
  cm.max_i64(&bits, 1);
  bits = bits >= 0 ? bits : (bits ^ 0x7fffffffffffffffLL);
  double viol;
  std::memcpy(&viol, &bits, sizeof(viol));
  report.feasibility = std::max(0.0, viol);  // solver.cpp:183-186 starts from viol = 0
  allgather_owned(cm, g, x);  // every rank leaves with the full solution
  return report;
}

// ------------------------------------------------------------------ general meshes
namespace {
__global__ void k_any_diff(i64 n, const double* __restrict__ a, const double* __restrict__ b, int* flag) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n && fabs(a[i] - b[i]) > 0.0) *flag = 1;
}
}  // namespace

// newton_active_set_step (solver.cpp:49-188) on a general mesh, single GPU.  Same control flow
// and device kernels as the uniform step; the mesh pieces are the plan-based assembly (base
// plans, masked by the full set), the constraint lines (conforming phi_tilde, distribute) and the
// flat segmented reduction order (each block cut into 8192-entry chunks, oracle_mesh.inc SegFlat).
NewtonReport mesh_newton_step(MeshDisc& m, State& st, const cf_material& mat, const cf_regularization& reg,
                              const cf_solver_options& opts) {
  const int d = m.d;
  const i64 nu = m.n_u(), V = m.V, nt = m.n_total();
  Slab sl;
  sl.v_lo = 0;
  sl.v_hi = V;
  sl.ve_lo = 0;
  sl.ve_hi = V;
  sl.c_lo = 0;
  sl.c_hi = m.nact;
  sl.plane = V;
  const int nw = std::max(1, (opts.cycle_window + 63) / 64);
  NewtonReport report;
  PhaseTimes& T = report.times;
  if (!m.base_cache) m.base_cache = mesh_build_constraints(m, true, 0, nullptr, nullptr);  // solver.cpp:55
  const Constraints* base = m.base_cache.get();
  double* x = st.solution.p;
  distribute(*base, x, false);
  DevBuf<double> ptfull(nt);  // conforming_phi (solver.cpp:40-47): phi_tilde distributed by the base set
  ptfull.zero();
  extrapolate_phi(st, ptfull.p + nu, V);
  distribute(*base, ptfull.p, false);
  const double* pt = ptfull.p + nu;
  const double c = opts.active_set_c_scale * mat.G_c / reg.eps;
  DevBuf<std::uint8_t> fixed(V), active(V), prev(V), tracked(V);
  DevBuf<unsigned long long> hist(V * nw);
  fixed.zero();
  prev.zero();
  tracked.zero();
  hist.zero();
  DevBuf<int> flags(4);
  DevBuf<double> R(nt), rhs(nt), delta(nt), xb(nt);
  int hist_len = 0;
  double res0 = -1.0;
  std::unique_ptr<BlockPrec> prec;
  Constraints full;
  full.mesh = &m;
  full.flag.alloc(nt);
  full.inhom.alloc(nt);
  CF_CUDA(cudaMemcpyAsync(full.flag.p, base->flag.p, size_t(nt), cudaMemcpyDeviceToDevice, stream()));
  CF_CUDA(cudaMemcpyAsync(full.inhom.p, base->inhom.p, size_t(nt) * sizeof(double), cudaMemcpyDeviceToDevice,
                          stream()));
  DevBuf<double> Bu(nu * (d == 2 ? 3 : 6)), Bp(V);
  DevBuf<int> unode(nu), pnode(V);
  const unsigned gv = grid_for(V, 256), gl = grid_for(nt, 256);
  SegLayout seg;
  seg.plane_u = nu;
  seg.plane_p = V;
  seg.p_lo = 0;
  seg.p_hi = 1;
  seg.nplanes = 1;
  for (int it = 1; it <= opts.newton_max_iter; ++it) {
    {
      Timer t(&T.residual);
      mesh_assemble_residual(m, *base, *base, mat, reg, x, pt, R.p);
    }
    int changes = 0, asize = 0;
    {
      Timer t(&T.active_set);
      flags.zero();
      k_active1<<<gv, 256, 0, stream()>>>(sl, nu, c, 1e-14 * c, x, st.phi_old.p, R.p, base->flag.p, fixed.p,
                                          active.p, tracked.p, hist.p, nw, flags.p + 2, d);
      CF_LAUNCHED();
      if (read_dev(flags.p + 2)) ++hist_len;
      k_active2<<<gv, 256, 0, stream()>>>(V, hist_len, opts.cycle_window, opts.cycle_toggles, tracked.p, hist.p, nw,
                                          fixed.p, active.p, prev.p, flags.p);
      CF_LAUNCHED();
      int hc[2];
      read_small(hc, flags.p, 2 * sizeof(int));
      asize = hc[0];
      changes = hc[1];
      k_full_constraints<<<gv, 256, 0, stream()>>>(sl, nu, base->flag.p, base->inhom.p, active.p, st.phi_old.p,
                                                   full.flag.p, full.inhom.p);
      CF_LAUNCHED();
      mesh_full_lines(*base, full);
      CF_CUDA(cudaMemcpyAsync(xb.p, x, size_t(nt) * sizeof(double), cudaMemcpyDeviceToDevice, stream()));
      distribute(full, x, false);
      CF_CUDA(cudaMemsetAsync(flags.p + 3, 0, sizeof(int), stream()));
      k_any_diff<<<gl, 256, 0, stream()>>>(nt, x, xb.p, flags.p + 3);
      CF_LAUNCHED();
    }
    const int moved = read_dev(flags.p + 3);
    {
      Timer t(&T.residual);
      if (moved) {
        mesh_assemble_residual(m, *base, full, mat, reg, x, pt, R.p);
      } else {
        k_zero_active<<<gv, 256, 0, stream()>>>(V, nu, active.p, R.p);
        CF_LAUNCHED();
      }
    }
    const double res = gnorm(nullptr, R.p, seg);
    if (res0 < 0.0) res0 = res;
    NewtonIter rec{res, asize, changes, 0};
    const bool small = res <= std::max(opts.newton_tol * res0, opts.newton_abs_floor);
    if (changes == 0 && small) {
      report.its.push_back(rec);
      if (opts.log)
        std::printf("newton step=%d it=%d res=%.6e active=%d changed=%d gmres=0\n", st.step, it, res, asize,
                    changes);
      report.converged = true;
      break;
    }
    std::unique_ptr<BlockSystem> J;
    {
      Timer t(&T.jacobian);
      J = mesh_assemble_jacobian(m, *base, full, mat, reg, x, pt);
    }
    if (!prec || !opts.freeze_preconditioner) {
      Timer t(&T.amg_setup);
      NullspaceDev ns;
      mesh_rigid_body_modes(m, full, Bu.p);
      k_phi_modes<<<gv, 256, 0, stream()>>>(sl, nu, full.flag.p, Bp.p, pnode.p, unode.p, d);
      CF_LAUNCHED();
      ns.u_node = unode.p;
      ns.u_modes = Bu.p;
      ns.m_u = d == 2 ? 3 : 6;
      ns.p_node = pnode.p;
      ns.p_modes = Bp.p;
      prec = build_block_prec(*J, opts.prec_kind, opts.amg, &ns, prec.get());
    }
    GmresResult lin;
    {
      Timer t(&T.gmres);
      k_neg<<<gl, 256, 0, stream()>>>(nt, R.p, rhs.p);
      CF_LAUNCHED();
      const BlockSystem& Jr = *J;
      DevOp op = [&Jr](const double* in, double* out) { block_apply(Jr, in, out); };
      const BlockPrec& Pr = *prec;
      DevOp pop = [&Pr](const double* in, double* out) { Pr.apply(in, out); };
      lin = gmres(op, &pop, rhs.p, nt, opts.gmres, delta.p, nullptr, &seg);
    }
    if (!lin.converged && !lin.breakdown) fail(CF_ERR_NUMERICAL, "newton_active_set_step: GMRES stagnated at max_iter");
    rec.gmres_iterations = lin.iterations;
    report.its.push_back(rec);
    if (opts.log)
      std::printf("newton step=%d it=%d res=%.6e active=%d changed=%d gmres=%d\n", st.step, it, res, asize, changes,
                  lin.iterations);
    distribute(full, delta.p, true);
    vaxpy(1.0, delta.p, x, nt);
    if (opts.damping) {
      double scale = 1.0;
      for (int half = 0; half < 4; ++half) {
        mesh_assemble_residual(m, *base, full, mat, reg, x, pt, R.p);
        if (gnorm(nullptr, R.p, seg) <= 10.0 * res) break;
        scale *= 0.5;
        vaxpy(-scale, delta.p, x, nt);
      }
    }
    CF_CUDA(cudaMemcpyAsync(prev.p, active.p, size_t(V), cudaMemcpyDeviceToDevice, stream()));
  }
  DevBuf<double> mx(1);
  {
    const long long lowest = 0x8000000000000000LL;
    CF_CUDA(cudaMemcpyAsync(mx.p, &lowest, sizeof(lowest), cudaMemcpyHostToDevice, stream()));
  }
  k_feas<<<gv, 256, 0, stream()>>>(sl, nu, x, st.phi_old.p, mx.p);
  CF_LAUNCHED();
  long long bits = 0;
  read_small(&bits, mx.p, sizeof(bits));
  bits = bits >= 0 ? bits : (bits ^ 0x7fffffffffffffffLL);
  double viol;
  std::memcpy(&viol, &bits, sizeof(viol));
  report.feasibility = std::max(0.0, viol);
  return report;
}

}  // namespace cfb

// K1 residual and K2 Jacobian assembly on a uniform Q1 grid.
//
// Reference: assemble_residual / assemble_jacobian (proj/src/model.cpp:127-322).  The
// reference loops cells, builds element vectors/matrices, and scatters them through the
// constraint set into triplets summed by setFromTriplets (duplicates summed in insertion =
// cell order).  The B200 design is atomic-free and deterministic:
//   * a cell-centric pass computes the per-cell quadrature-point state (or, for the residual,
//     the element vector) once per cell and writes it to an HBM scratch array;
//   * a vertex-centric pass owns its rows and gathers the contributions of its 2^d cells in
//     the reference's cell order (root-lexicographic, then hierarchical z-order), so every
//     entry is the same sequence of IEEE operations as the reference's: this file is compiled
//     with -fmad=false and mirrors the reference's expression order term by term;
//   * the CSR pattern is the geometric 3^d stencil minus constrained rows/columns, with a
//     diagonal kept on constrained rows iff its summed value is non-zero (model.cpp:308-311);
//     row pointers come from a count pass + device scan, so no triplets are materialised
//     (the reference's triplet path would need ~65 GB at config 1).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "cf_types.hpp"

namespace cfb {

namespace {

// ------------------------------------------------------------------ cell order
// Reference active-cell order after uniform_refine (mesh.cpp:147-169, 209-215).
__host__ __device__ inline i64 cell_key(const GridDesc& g, i64 cx, i64 cy, i64 cz) {
  const i64 mask = (i64(1) << g.r) - 1;
  const i64 rx = cx >> g.r, ry = cy >> g.r, rz = cz >> g.r;
  const i64 lx = cx & mask, ly = cy & mask, lz = cz & mask;
  i64 m = 0;
  for (int j = 0; j < g.r; ++j) {
    m |= ((lx >> j) & 1) << (g.d * j);
    m |= ((ly >> j) & 1) << (g.d * j + 1);
    if (g.d == 3) m |= ((lz >> j) & 1) << (g.d * j + 2);
  }
  const i64 root = rx + i64(g.n0) * (ry + i64(g.n0) * rz);
  return (root << (g.d * g.r)) | m;
}

template <int D>
struct CellList {
  int n;
  i64 cell[1 << D];
  int kv[1 << D];  // local index of the row vertex in the cell
  int kw[1 << D];  // local index of the column vertex (pair lists)
};

// Cells containing both v=(x,y,z) and w=v+delta, in reference order.
template <int D>
__device__ inline void common_cells(const GridDesc& g, i64 x, i64 y, i64 z, int dx, int dy, int dz,
                                    CellList<D>& L) {
  L.n = 0;
  i64 key[1 << D];
  const int del[3] = {dx, dy, dz};
  const i64 vc[3] = {x, y, z};
  for (int t = 0; t < (1 << D); ++t) {
    bool ok = true;
    i64 anc[3] = {0, 0, 0};
    int kv = 0, kw = 0;
    for (int a = 0; a < D; ++a) {
      const int ta = (t >> a) & 1;  // 1: v is the high corner of the cell along axis a
      const int la = ta + del[a];
      anc[a] = vc[a] - ta;
      if (la < 0 || la > 1 || anc[a] < 0 || anc[a] >= g.nc) ok = false;
      kv |= ta << a;
      kw |= la << a;
    }
    if (!ok) continue;
    const i64 c = anc[0] + g.nc * (anc[1] + g.nc * anc[2]);
    const i64 k = cell_key(g, anc[0], anc[1], anc[2]);
    int p = L.n++;
    while (p > 0 && key[p - 1] > k) {  // insertion sort by reference order
      key[p] = key[p - 1];
      L.cell[p] = L.cell[p - 1];
      L.kv[p] = L.kv[p - 1];
      L.kw[p] = L.kw[p - 1];
      --p;
    }
    key[p] = k;
    L.cell[p] = c;
    L.kv[p] = kv;
    L.kw[p] = kw;
  }
}

template <int D>
__device__ inline void vxyz(const GridDesc& g, i64 v, i64& x, i64& y, i64& z) {
  x = v % g.nn;
  y = (v / g.nn) % g.nn;
  z = (D == 3) ? v / (g.nn * g.nn) : 0;
}

struct Coef {
  double kap, eps, p, Gc, mu, lam;
  int coupling;
};

// ------------------------------------------------------------------ K1a: element residuals
// K1a (fast form): one thread per (cell, quadrature point), the 2^d lanes of a cell adjacent in
// the warp.  Lane q loads corner q's values and the cell's corner data is exchanged with
// shuffles; each lane evaluates its point's state and its contribution to every (k, a); the
// contributions are then folded in q order (0.0 + c_0 + c_1 + ...) — exactly the reference's
// `ru[k*d+a] += w * val` sequence over q — and lane k keeps corner k's sums.
// a / h for the fixed cell size h > 0 (the reference divides every shape-gradient product by h,
// model.cpp; the oracle and this kernel keep that IEEE operation).  y = RN(1/h) once per thread,
// then q = RN(a y) refined by two Markstein corrections q += (a - q h) y (exact remainders by FMA):
// the first leaves q faithful, the second, with y the correctly rounded reciprocal, gives the
// correctly rounded quotient RN(a / h) (Markstein's theorem).  Zero, tiny and huge dividends
// take the IEEE division (0 / h = 0 with a's sign).  Five dependent FP64 operations instead of the
// division's reciprocal refinement per quotient; bitwise a / h (tests/test_gpu_assembly.py,
// test_div_by_h_is_ieee_division).
struct DivBy {
  double h, y;
  __device__ explicit DivBy(double h_) : h(h_), y(1.0 / h_) {}
  __device__ __forceinline__ double div(double a) const {
#ifdef CF_PLAIN_DIV
    return a / h;
#else
    const double m = fabs(a);
    if (m == 0.0) return a;
    if (!(m >= 0x1p-900 && m <= 0x1p900)) return a / h;
    double q = a * y;
    double r = __fma_rn(-q, h, a);
    q = __fma_rn(r, y, q);
    r = __fma_rn(-q, h, a);
    return __fma_rn(r, y, q);
#endif
  }
};

__global__ void k_div_by(double h, const double* __restrict__ a, i64 n, double* __restrict__ q) {
  const DivBy dv(h);
  for (i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += i64(gridDim.x) * blockDim.x) q[i] = dv.div(a[i]);
}

#ifndef CF_RES_MINB
#define CF_RES_MINB 4  // 64 registers, 32 warps per SM: 5.35 -> 4.2-4.9 ms on config 3 (A/B, bitwise the same)
#endif
template <int D, bool SMX = true>
__global__ void __launch_bounds__(256, CF_RES_MINB) k_cell_residual_q(GridDesc g, const Tables* __restrict__ T, Coef cf,
                                                         const double* __restrict__ sol,
                                                         const double* __restrict__ ptil,
                                                         double* __restrict__ out, i64 c_lo, i64 c_hi,
                                                         const int* __restrict__ list, int nlist) {
  constexpr int NV = 1 << D, NQ = 1 << D;
  __shared__ double sG[NQ][NV][D], sS[NQ][NV], sW[NQ];
  for (int i = threadIdx.x; i < NQ * NV; i += blockDim.x) {
    const int qq = i / NV, k = i % NV;
    sS[qq][k] = T->s[qq][k];
    for (int b = 0; b < D; ++b) sG[qq][k][b] = T->G[qq][k][b];
  }
  if (threadIdx.x < NQ) sW[threadIdx.x] = T->w[threadIdx.x];
  // 3d: per-cell exchange buffer (corner values first, then the fold of the contributions)
  constexpr bool SM3 = D == 3 && SMX;
  constexpr int XC = 4 * 4 * 9 + 8;  // doubles per cell: [corner of the half][component][q (+1)] (+8: banks)
  __shared__ double sXf[SM3 ? (256 / 8) * XC : 1];
  double* sXc = sXf + (SM3 ? (int(threadIdx.x) >> 3) * XC : 0);
  __syncthreads();
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  // list: only the listed cells (offsets from c_lo) are recomputed (assemble_residual_moved)
  const bool valid = list ? t / NQ < nlist : c_lo + t / NQ < c_hi;
  const i64 c = list ? (valid ? c_lo + list[t / NQ] : c_lo) : c_lo + t / NQ;
  const int q = int(t % NQ);
  const i64 cc = valid ? c : c_lo;
  const i64 cx = cc % g.nc, cy = (cc / g.nc) % g.nc, cz = (D == 3) ? cc / (g.nc * g.nc) : 0;
  const i64 nu = g.n_u();
  double my_u[D], my_phi, my_pt;
  {
    const int k = q;
    const i64 v = (cx + (k & 1)) + g.nn * ((cy + ((k >> 1) & 1)) + g.nn * (cz + ((k >> 2) & 1)));
#pragma unroll
    for (int a = 0; a < D; ++a) my_u[a] = sol[v * D + a];
    my_phi = sol[nu + v];
    my_pt = ptil[v];
  }
  const DivBy dv(g.h);
  double gu[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  double gphi[3] = {0, 0, 0};
  double phi = 0.0, pt = 0.0;
  if constexpr (SM3) {  // corner q's values, read back by the cell's lanes as broadcasts
#pragma unroll
    for (int a = 0; a < D; ++a) sXc[q * (D + 2) + a] = my_u[a];
    sXc[q * (D + 2) + D] = my_phi;
    sXc[q * (D + 2) + D + 1] = my_pt;
    __syncwarp();
  }
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double uk[D], phik, ptk;
    if constexpr (SM3) {
#pragma unroll
      for (int a = 0; a < D; ++a) uk[a] = sXc[k * (D + 2) + a];
      phik = sXc[k * (D + 2) + D];
      ptk = sXc[k * (D + 2) + D + 1];
    } else {
#pragma unroll
      for (int a = 0; a < D; ++a) uk[a] = __shfl_sync(0xffffffffu, my_u[a], k, NQ);
      phik = __shfl_sync(0xffffffffu, my_phi, k, NQ);
      ptk = __shfl_sync(0xffffffffu, my_pt, k, NQ);
    }
    const double sk = sS[q][k];
    phi += sk * phik;
    pt += sk * ptk;
#pragma unroll
    for (int b = 0; b < D; ++b) {
      const double Gkb = sG[q][k][b];
      gphi[b] += dv.div(phik * Gkb);
#pragma unroll
      for (int a = 0; a < D; ++a) gu[a][b] += dv.div(uk[a] * Gkb);
    }
  }
  double e[3][3], sig[3][3];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) e[a][b] = 0.5 * (gu[a][b] + gu[b][a]);
  double tre = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) tre += e[a][a];
  const double two_mu = 2.0 * cf.mu;
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) sig[a][b] = two_mu * e[a][b];
#pragma unroll
  for (int a = 0; a < D; ++a) sig[a][a] += cf.lam * tre;
  double sig_ee = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) sig_ee += sig[a][b] * e[a][b];
  const double gcoef = (1.0 - cf.kap) * pt * pt + cf.kap;
  const double pphi = (cf.coupling == 0) ? pt * pt : phi * phi;
  const double w = sW[q];
  auto contribs = [&](int k, double (&contrib)[D + 1]) {
#pragma unroll
    for (int a = 0; a < D; ++a) {
      double val = 0.0;
#pragma unroll
      for (int b = 0; b < D; ++b) val += dv.div(gcoef * sig[a][b] * sG[q][k][b]);
      val += dv.div(pphi * cf.p * sG[q][k][a]);
      contrib[a] = w * val;
    }
    double vphi = ((1.0 - cf.kap) * phi * sig_ee + 2.0 * phi * cf.p * tre - cf.Gc / cf.eps * (1.0 - phi)) * sS[q][k];
#pragma unroll
    for (int b = 0; b < D; ++b) vphi += dv.div(cf.Gc * cf.eps * gphi[b] * sG[q][k][b]);
    contrib[D] = w * vphi;
  };
  if constexpr (D == 3 && SMX) {
    // 3d: the q-ordered fold through shared memory instead of 8 x 4 x 8 double shuffles per thread
    // (the shuffle pipe cost as much as the FP64 pipe): the corners go in two halves of four; lane q
    // stores its contributions [k][a][q], then lane (k', h) of the cell sums components 2h, 2h + 1
    // of corner k' over q = 0..7 in order (0.0 + c_0 + c_1 + ...: the same sums) and writes them
    __syncwarp();  // the corner values above have been read
    auto X = [&](int kk, int a, int qq) -> double& { return sXc[(kk * 4 + a) * 9 + qq]; };
#pragma unroll
    for (int half = 0; half < 2; ++half) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        double contrib[D + 1];
        contribs(half * 4 + kk, contrib);
#pragma unroll
        for (int a = 0; a <= D; ++a) X(kk, a, q) = contrib[a];
      }
      __syncwarp();
      const int kq = q & 3, h = q >> 2;
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int qq = 0; qq < NQ; ++qq) {
        s0 += X(kq, 2 * h, qq);
        s1 += X(kq, 2 * h + 1, qq);
      }
      if (valid) {
        double* o = out + (c - c_lo) * (NV * (D + 1)) + (half * 4 + kq) * (D + 1) + 2 * h;
        o[0] = s0;
        o[1] = s1;
      }
      __syncwarp();
    }
  } else {
    double keep[D + 1];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double contrib[D + 1];
      contribs(k, contrib);
#pragma unroll
      for (int a = 0; a <= D; ++a) {
        double s = 0.0;
#pragma unroll
        for (int qq = 0; qq < NQ; ++qq) s += __shfl_sync(0xffffffffu, contrib[a], qq, NQ);
        if (q == k) keep[a] = s;
      }
    }
    if (valid) {
      double* o = out + (c - c_lo) * (NV * (D + 1)) + q * (D + 1);
#pragma unroll
      for (int a = 0; a <= D; ++a) o[a] = keep[a];
    }
  }
}

// cells of [c_lo, c_hi) with a corner whose dofs changed (x vs x_before): their offsets, any order
template <int D>
__global__ void k_moved_cells(GridDesc g, i64 c_lo, i64 c_hi, const double* __restrict__ x,
                              const double* __restrict__ xb, int* __restrict__ list, int* __restrict__ count) {
  const i64 c = c_lo + i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= c_hi) return;
  const i64 cx = c % g.nc, cy = (c / g.nc) % g.nc, cz = (D == 3) ? c / (g.nc * g.nc) : 0;
  const i64 nu = g.n_u();
  bool moved = false;
  for (int k = 0; k < (1 << D) && !moved; ++k) {
    const i64 v = (cx + (k & 1)) + g.nn * ((cy + ((k >> 1) & 1)) + g.nn * (cz + ((k >> 2) & 1)));
    for (int a = 0; a < D; ++a) moved = moved || x[v * D + a] != xb[v * D + a];
    moved = moved || x[nu + v] != xb[nu + v];
  }
  if (moved) list[atomicAdd(count, 1)] = int(c - c_lo);
}

// K1b: vertex gather with condensation (Scatter::vector_add, model.cpp:74-80; entry-free lines drop).
template <int D>
__global__ void k_vertex_residual(GridDesc g, const double* __restrict__ cellres,
                                  const std::uint8_t* __restrict__ flag, double* __restrict__ R, Slab sl) {
  constexpr int NV = 1 << D;
  const i64 lv = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (lv >= sl.nv()) return;
  const i64 v = sl.v_lo + lv;
  i64 x, y, z;
  vxyz<D>(g, v, x, y, z);
  CellList<D> L;
  common_cells<D>(g, x, y, z, 0, 0, 0, L);
  double acc[D + 1];
#pragma unroll
  for (int a = 0; a <= D; ++a) acc[a] = 0.0;
  for (int i = 0; i < L.n; ++i) {
    const double* o = cellres + (L.cell[i] - sl.c_lo) * (NV * (D + 1)) + L.kv[i] * (D + 1);
#pragma unroll
    for (int a = 0; a <= D; ++a) acc[a] += o[a];
  }
  const i64 nu = g.n_u(), nul = D * sl.nv();
#pragma unroll
  for (int a = 0; a < D; ++a) R[lv * D + a] = flag[v * D + a] ? 0.0 : acc[a];
  R[nul + lv] = flag[nu + v] ? 0.0 : acc[D];
}

// ------------------------------------------------------------------ K2a: quadrature-point state
// model.cpp:242-266 per (cell, q): wg = w*gcoef, phi, tre, sig:e, sigma.
template <int D>
struct QS {
  static constexpr int NS = 4 + D * D;
};

template <int D>
__global__ void __launch_bounds__(128) k_cell_qpstate(GridDesc g, const Tables* __restrict__ T, Coef cf,
                                                      const double* __restrict__ sol,
                                                      const double* __restrict__ ptil,
                                                      double* __restrict__ out, i64 c_lo, i64 c_hi) {
  constexpr int NV = 1 << D, NQ = 1 << D, NS = QS<D>::NS;
  const i64 c = c_lo + i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= c_hi) return;
  const i64 cx = c % g.nc, cy = (c / g.nc) % g.nc, cz = (D == 3) ? c / (g.nc * g.nc) : 0;
  const i64 nu = g.n_u();
  double uloc[NV][D], philoc[NV], ptloc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const i64 v = (cx + (k & 1)) + g.nn * ((cy + ((k >> 1) & 1)) + g.nn * (cz + ((k >> 2) & 1)));
#pragma unroll
    for (int a = 0; a < D; ++a) uloc[k][a] = sol[v * D + a];
    philoc[k] = sol[nu + v];
    ptloc[k] = ptil[v];
  }
  for (int q = 0; q < NQ; ++q) {
    double gu[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    double phi = 0.0, pt = 0.0;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const double sk = T->s[q][k];
      phi += sk * philoc[k];
      pt += sk * ptloc[k];
#pragma unroll
      for (int b = 0; b < D; ++b)
#pragma unroll
        for (int a = 0; a < D; ++a) gu[a][b] += uloc[k][a] * T->gp[q][k][b];
    }
    double e[3][3], sig[3][3];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) e[a][b] = 0.5 * (gu[a][b] + gu[b][a]);
    double tre = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) tre += e[a][a];
    const double two_mu = 2.0 * cf.mu;
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) sig[a][b] = two_mu * e[a][b];
#pragma unroll
    for (int a = 0; a < D; ++a) sig[a][a] += cf.lam * tre;
    double sig_ee = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) sig_ee += sig[a][b] * e[a][b];
    const double gcoef = (1.0 - cf.kap) * pt * pt + cf.kap;
    const double w = T->w[q];
    // AoS layout: the NQ x NS states of a cell are contiguous (one coalesced 832-byte read per cell)
    auto put = [&](int f, double val) { out[(c - c_lo) * (NQ * NS) + q * NS + f] = val; };
    put(0, w * gcoef);
    put(1, phi);
    put(2, tre);
    put(3, sig_ee);
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) put(4 + a * D + b, sig[a][b]);
  }
}

// the same states, one thread per (cell, point): the 2^d lanes of a cell load one corner each and
// exchange them with shuffles (as K1a); every state is the serial kernel's expression sequence
template <int D>
__global__ void __launch_bounds__(256) k_cell_qpstate_q(GridDesc g, const Tables* __restrict__ T, Coef cf,
                                                        const double* __restrict__ sol,
                                                        const double* __restrict__ ptil, double* __restrict__ out,
                                                        i64 c_lo, i64 c_hi) {
  constexpr int NV = 1 << D, NQ = 1 << D, NS = QS<D>::NS;
  // element tables and the cell's corner values through shared memory: the kernel is bound by the
  // memory-instruction pipe (table loads, 2 x 5 x 2^d shuffles and the state stores per thread), not
  // by arithmetic; a corner value is stored once and read by the cell's lanes as a broadcast
  __shared__ double sS[NQ][NV], sG[NQ][NV][D], sW[NQ];
  __shared__ double sC[256 / NQ][NV][D + 2];
  for (int i = threadIdx.x; i < NQ * NV; i += blockDim.x) {
    const int qq = i / NV, k = i % NV;
    sS[qq][k] = T->s[qq][k];
    for (int b = 0; b < D; ++b) sG[qq][k][b] = T->gp[qq][k][b];
  }
  if (threadIdx.x < NQ) sW[threadIdx.x] = T->w[threadIdx.x];
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  const i64 c = c_lo + t / NQ;
  const int q = int(t % NQ);
  const bool valid = c < c_hi;
  const i64 cc = valid ? c : c_lo;
  const i64 cx = cc % g.nc, cy = (cc / g.nc) % g.nc, cz = (D == 3) ? cc / (g.nc * g.nc) : 0;
  const i64 nu = g.n_u();
  double my_u[D], my_phi, my_pt;
  {
    const int k = q;
    const i64 v = (cx + (k & 1)) + g.nn * ((cy + ((k >> 1) & 1)) + g.nn * (cz + ((k >> 2) & 1)));
#pragma unroll
    for (int a = 0; a < D; ++a) my_u[a] = sol[v * D + a];
    my_phi = sol[nu + v];
    my_pt = ptil[v];
  }
  {
    double* mine = sC[threadIdx.x / NQ][q];
#pragma unroll
    for (int a = 0; a < D; ++a) mine[a] = my_u[a];
    mine[D] = my_phi;
    mine[D + 1] = my_pt;
  }
  __syncthreads();  // tables and corner values
  double gu[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  double phi = 0.0, pt = 0.0;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const double* ck = sC[threadIdx.x / NQ][k];
    const double sk = sS[q][k];
    phi += sk * ck[D];
    pt += sk * ck[D + 1];
    double uk[D];
#pragma unroll
    for (int a = 0; a < D; ++a) uk[a] = ck[a];
#pragma unroll
    for (int b = 0; b < D; ++b)
#pragma unroll
      for (int a = 0; a < D; ++a) gu[a][b] += uk[a] * sG[q][k][b];
  }
  double e[3][3], sig[3][3];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) e[a][b] = 0.5 * (gu[a][b] + gu[b][a]);
  double tre = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) tre += e[a][a];
  const double two_mu = 2.0 * cf.mu;
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) sig[a][b] = two_mu * e[a][b];
#pragma unroll
  for (int a = 0; a < D; ++a) sig[a][a] += cf.lam * tre;
  double sig_ee = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) sig_ee += sig[a][b] * e[a][b];
  const double gcoef = (1.0 - cf.kap) * pt * pt + cf.kap;
  const double w = sW[q];
  if (!valid) return;
  double* o = out + (c - c_lo) * (NQ * NS) + q * NS;
  o[0] = w * gcoef;
  o[1] = phi;
  o[2] = tre;
  o[3] = sig_ee;
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) o[4 + a * D + b] = sig[a][b];
}

// Element-matrix entries coupling row vertex v (local k) and column vertex w (local l),
// summed over their common cells in reference order (kuu/kpu/kpp of model.cpp:268-285).
template <int D>
struct PairBlocks {
  double uu[D][D];
  double pu[D];
  double pp;
};

template <int D>
__device__ inline void pair_blocks(const Tables* __restrict__ T, const Coef& cf, const double* __restrict__ qs,
                                   const CellList<D>& L, bool need_u, bool need_p, PairBlocks<D>& out) {
  constexpr int NQ = 1 << D, NS = QS<D>::NS;
#pragma unroll
  for (int a = 0; a < D; ++a) {
#pragma unroll
    for (int b = 0; b < D; ++b) out.uu[a][b] = 0.0;
    out.pu[a] = 0.0;
  }
  out.pp = 0.0;
  const double c2k = 2.0 * (1.0 - cf.kap);
  const double c2p = 2.0 * cf.p;
  const double omk = 1.0 - cf.kap;
  const double gce = cf.Gc / cf.eps;
  const double gcx = cf.Gc * cf.eps;
  for (int i = 0; i < L.n; ++i) {
    const int k = L.kv[i], l = L.kw[i];
    const double* cs = qs + L.cell[i] * (NQ * NS);
    double bu[D][D], bp[D], bpp = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
#pragma unroll
      for (int b = 0; b < D; ++b) bu[a][b] = 0.0;
      bp[a] = 0.0;
    }
    for (int q = 0; q < NQ; ++q) {
      const double* st = cs + q * NS;
      if (need_u) {
        const double wg = st[0];
        const double* vl = &T->val[q][k][l][0][0];
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int b = 0; b < D; ++b) bu[a][b] += wg * vl[a * 3 + b];
      }
      if (need_p) {
        const double w = T->w[q];
        const double phi = st[1], tre = st[2], see = st[3];
        const double sk = T->s[q][k], sl = T->s[q][l];
#pragma unroll
        for (int b = 0; b < D; ++b) {
          double sgl = 0.0;
#pragma unroll
          for (int c = 0; c < D; ++c) sgl += st[4 + b * D + c] * T->gp[q][l][c];
          bp[b] += w * (c2k * phi * sgl + c2p * phi * T->gp[q][l][b]) * sk;
        }
        bpp += w * ((omk * see + c2p * tre + gce) * sl * sk + gcx * T->gg[q][k][l]);
      }
    }
#pragma unroll
    for (int a = 0; a < D; ++a) {
#pragma unroll
      for (int b = 0; b < D; ++b) out.uu[a][b] += bu[a][b];
      out.pu[a] += bp[a];
    }
    out.pp += bpp;
  }
}

// K2 count pass: row lengths of the three blocks; constrained rows keep a diagonal iff its
// summed value is non-zero (model.cpp:295,300,308-311).
template <int D, bool UU>
__global__ void k_jac_count(GridDesc g, const Tables* __restrict__ T, Coef cf, const double* __restrict__ qs,
                            const std::uint8_t* __restrict__ flag, i64* __restrict__ cnt_uu,
                            i64* __restrict__ cnt_pu, i64* __restrict__ cnt_pp, Slab sl) {
  const i64 lv = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (lv >= sl.nv()) return;
  const i64 v = sl.v_lo + lv;
  qs -= sl.c_lo * ((1 << D) * QS<D>::NS);  // cell states are stored from the slab's first cell
  i64 x, y, z;
  vxyz<D>(g, v, x, y, z);
  const i64 nu = g.n_u();
  i64 nfu = 0, nfp = 0;
  const int zl = (D == 3) ? -1 : 0, zh = (D == 3) ? 1 : 0;
  for (int dz = zl; dz <= zh; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const i64 X = x + dx, Y = y + dy, Z = z + dz;
        if (X < 0 || Y < 0 || Z < 0 || X >= g.nn || Y >= g.nn || Z >= ((D == 3) ? g.nn : 1)) continue;
        const i64 w = X + g.nn * (Y + g.nn * Z);
#pragma unroll
        for (int b = 0; b < D; ++b) nfu += flag[w * D + b] ? 0 : 1;
        nfp += flag[nu + w] ? 0 : 1;
      }
  const bool con_p = flag[nu + v] != 0;
  bool con_u = false;
#pragma unroll
  for (int a = 0; a < D; ++a) con_u |= flag[v * D + a] != 0;
  PairBlocks<D> pb;
  pb.pp = 0.0;
  if (con_p || (UU && con_u)) {  // a constrained row keeps its diagonal iff the summed value is != 0
    CellList<D> L;
    common_cells<D>(g, x, y, z, 0, 0, 0, L);
    pair_blocks<D>(T, cf, qs, L, UU && con_u, con_p, pb);
  }
  if (UU) {
#pragma unroll
    for (int a = 0; a < D; ++a) cnt_uu[lv * D + a] = flag[v * D + a] ? (pb.uu[a][a] != 0.0 ? 1 : 0) : nfu;
  }
  const bool pf = flag[nu + v] == 0;
  cnt_pu[lv] = pf ? nfu : 0;
  cnt_pp[lv] = pf ? nfp : (pb.pp != 0.0 ? 1 : 0);
}

// Pair-parallel fill pass (persistent grid, one warp per row vertex v).  The work of a row
// vertex is 2^d cells x 2^d corners: unit (i, l) = the element block of v's i-th adjacent cell (in
// reference order) for v's corner k and column corner l, summed over q exactly as the reference
// does.  The 32 lanes take 32 units per round (3d: cells 0-3, then 4-7), so every lane does useful
// FP64 work (a slot-per-lane form leaves ~3/4 of the lanes idle on a cell that does not hold
// their column vertex).  After each round lane s adds, for stencil slot s, the round's units of
// the cells holding w in reference order, so every value is the reference's sum.  The cell list
// lives in registers (lane t < 2^d owns candidate cell t, ranks by shuffles) and the integrand
// table in shared memory.
template <int D>
constexpr int pair_wpb() { return 4; }

template <int D, bool UU>
struct PairSmem {  // the M_uu integrand table only when M_uu is filled (smaller footprint, more blocks)
  static constexpr int NQ = 1 << D, NV = 1 << D, NR = D * D + D + 1;
  static constexpr int TQ = UU ? NQ : 1, TV = UU ? NV : 1, TD = UU ? D * D : 1;
  double val[TQ][TV][TV][TD];
  double s[NQ][NV], gp[NQ][NV][D], gg[NQ][NV][NV], w[NQ];
  double res[pair_wpb<D>()][32][NR];
};

template <int D, bool UU>
__global__ void __launch_bounds__(pair_wpb<D>() * 32) k_jac_fill_pair(
    GridDesc g, const Tables* __restrict__ T, Coef cf, const double* __restrict__ qs,
    const std::uint8_t* __restrict__ flag, const i64* __restrict__ ptr_uu, int* __restrict__ col_uu,
    double* __restrict__ val_uu, const i64* __restrict__ ptr_pu, int* __restrict__ col_pu,
    double* __restrict__ val_pu, const i64* __restrict__ ptr_pp, int* __restrict__ col_pp,
    double* __restrict__ val_pp, Slab sl) {
  constexpr int S = (D == 3) ? 27 : 9, NQ = 1 << D, NV = 1 << D, NC = 1 << D, NS = QS<D>::NS, CS = NQ * NS;
  constexpr int NR = D * D + D + 1, CPR = 32 / NV, ROUNDS = (NC + CPR - 1) / CPR;
  extern __shared__ __align__(16) unsigned char smraw[];
  PairSmem<D, UU>& sm = *reinterpret_cast<PairSmem<D, UU>*>(smraw);
  if constexpr (UU) {
    for (int i = threadIdx.x; i < NQ * NV * NV * D * D; i += blockDim.x) {
      const int ab = i % (D * D), l = (i / (D * D)) % NV, k = (i / (D * D * NV)) % NV, q = i / (D * D * NV * NV);
      sm.val[q][k][l][ab] = T->val[q][k][l][ab / D][ab % D];
    }
  }
  for (int i = threadIdx.x; i < NQ * NV; i += blockDim.x) {
    const int q = i / NV, k = i % NV;
    sm.s[q][k] = T->s[q][k];
    for (int b = 0; b < D; ++b) sm.gp[q][k][b] = T->gp[q][k][b];
    for (int l = 0; l < NV; ++l) sm.gg[q][k][l] = T->gg[q][k][l];
  }
  if (threadIdx.x < NQ) sm.w[threadIdx.x] = T->w[threadIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31, wv = threadIdx.x >> 5;
  const unsigned FULL = 0xffffffffu;
  const double c2k = 2.0 * (1.0 - cf.kap), c2p = 2.0 * cf.p, omk = 1.0 - cf.kap;
  const double gce = cf.Gc / cf.eps, gcx = cf.Gc * cf.eps;
  const i64 nu = g.n_u();
  const i64 ushift = D * sl.ve_lo, pshift = sl.ve_lo;
  qs -= sl.c_lo * CS;
  double(*res)[NR] = sm.res[wv];
  for (i64 lv = i64(blockIdx.x) * pair_wpb<D>() + wv; lv < sl.nv(); lv += i64(gridDim.x) * pair_wpb<D>()) {
    const i64 v = sl.v_lo + lv;
    i64 x, y, z;
    vxyz<D>(g, v, x, y, z);
    // ---- candidate cell t = lane (t < 2^d): v is its corner t; rank = reference order position
    bool cvalid = false;
    i64 ccell = 0, ckey = 0;
    if (lane < NC) {
      const i64 vc[3] = {x, y, z};
      i64 anc[3] = {0, 0, 0};
      cvalid = true;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        anc[a] = vc[a] - ((lane >> a) & 1);
        cvalid = cvalid && anc[a] >= 0 && anc[a] < g.nc;
      }
      if (cvalid) {
        ccell = anc[0] + g.nc * (anc[1] + g.nc * anc[2]);
        ckey = cell_key(g, anc[0], anc[1], anc[2]);
      }
    }
    int crank = 0;
#pragma unroll
    for (int t = 0; t < NC; ++t) {
      const i64 kt = __shfl_sync(FULL, ckey, t);
      const bool vt = __shfl_sync(FULL, cvalid, t);
      crank += (vt && kt < ckey) ? 1 : 0;
    }
    if constexpr (!UU) {
      // constrained phi row (the active set: most phi rows once the crack has formed): no M_phiu
      // entries and only the diagonal of M_phiphi, i.e. the units (cell, l = k).  Lane t < 2^d
      // computes its cell's unit with the fill's expression, then the units are added in
      // reference cell order, as the center slot does below.
      if (flag[nu + v] != 0) {
        double u = 0.0;
        if (cvalid) {
          const int k = lane;
          const double* cst = qs + ccell * CS;
          for (int q = 0; q < NQ; ++q) {
            const double* st = cst + q * NS;
            const double see = __ldg(st + 3), tre = __ldg(st + 2);
            const double sk = sm.s[q][k], slv = sm.s[q][k];
            u += sm.w[q] * ((omk * see + c2p * tre + gce) * slv * sk + gcx * sm.gg[q][k][k]);
          }
        }
        double acc = 0.0;
        const unsigned vm = __ballot_sync(FULL, cvalid) & ((1u << NC) - 1u);
        const int ncl = __popc(vm);
        for (int ii = 0; ii < ncl; ++ii) {
          const int src = __ffs(__ballot_sync(FULL, cvalid && crank == ii)) - 1;
          acc += __shfl_sync(FULL, u, src);
        }
        if (lane == 0 && ptr_pp[lv + 1] > ptr_pp[lv]) {
          col_pp[ptr_pp[lv]] = int(v - pshift);
          val_pp[ptr_pp[lv]] = acc;
        }
        continue;
      }
    }
    const unsigned vmask = __ballot_sync(FULL, cvalid) & ((1u << NC) - 1u);
    const int ncell = __popc(vmask);
    auto src_of = [&](int i) {  // lane holding the i-th cell in reference order (uniform i)
      return __ffs(__ballot_sync(FULL, cvalid && crank == i)) - 1;
    };
    // ---- slot lane setup
    const int s = lane;
    const int dx = s % 3 - 1, dy = (s / 3) % 3 - 1, dz = (D == 3) ? s / 9 - 1 : 0;
    const i64 X = x + dx, Y = y + dy, Z = z + dz;
    const bool slot_ok = s < S && X >= 0 && Y >= 0 && Z >= 0 && X < g.nn && Y < g.nn &&
                         Z < ((D == 3) ? g.nn : 1);
    const int del[3] = {dx, dy, dz};
    PairBlocks<D> pb;
#pragma unroll
    for (int a = 0; a < D; ++a) {
#pragma unroll
      for (int b = 0; b < D; ++b) pb.uu[a][b] = 0.0;
      pb.pu[a] = 0.0;
    }
    pb.pp = 0.0;
#pragma unroll
    for (int rd = 0; rd < ROUNDS; ++rd) {
      // my unit: cell rank i = rd * CPR + lane / NV, column corner l = lane % NV
      const int i = rd * CPR + lane / NV, l = lane % NV;
      int src = -1;
#pragma unroll
      for (int t = 0; t < NC; ++t) {
        const int rt = __shfl_sync(FULL, crank, t);
        const bool vt = __shfl_sync(FULL, cvalid, t);
        if (vt && rt == i) src = t;
      }
      const i64 mycell = __shfl_sync(FULL, ccell, src < 0 ? 0 : src);
      if (lane < CPR * NV && src >= 0) {
        const int k = src;  // v is corner t of candidate cell t
        const double* cst = qs + mycell * CS;
        double bu[D][D], bp[D], bpp = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) {
#pragma unroll
          for (int b = 0; b < D; ++b) bu[a][b] = 0.0;
          bp[a] = 0.0;
        }
#pragma unroll 2
        for (int q = 0; q < NQ; ++q) {
          const double* st = cst + q * NS;
          double gl[D];
#pragma unroll
          for (int b = 0; b < D; ++b) gl[b] = sm.gp[q][l][b];
          if constexpr (UU) {
            const double wg = __ldg(st);
            const double* vl = sm.val[q][k][l];
#pragma unroll
            for (int a = 0; a < D; ++a)
#pragma unroll
              for (int b = 0; b < D; ++b) bu[a][b] += wg * vl[a * D + b];
          }
          const double wq = sm.w[q];
          const double phi = __ldg(st + 1), tre = __ldg(st + 2), see = __ldg(st + 3);
          const double sk = sm.s[q][k], slv = sm.s[q][l];
#pragma unroll
          for (int b = 0; b < D; ++b) {
            double sgl = 0.0;
#pragma unroll
            for (int c = 0; c < D; ++c) sgl += __ldg(st + 4 + b * D + c) * gl[c];
            bp[b] += wq * (c2k * phi * sgl + c2p * phi * gl[b]) * sk;
          }
          bpp += wq * ((omk * see + c2p * tre + gce) * slv * sk + gcx * sm.gg[q][k][l]);
        }
        double* o = res[lane];
#pragma unroll
        for (int a = 0; a < D; ++a) {
#pragma unroll
          for (int b = 0; b < D; ++b) o[a * D + b] = bu[a][b];
          o[D * D + a] = bp[a];
        }
        o[D * D + D] = bpp;
      }
      __syncwarp();
      // slot lanes add this round's cells in reference order
      const int i_end = min(ncell, (rd + 1) * CPR);
      for (int ii = rd * CPR; ii < i_end; ++ii) {
        const int k = src_of(ii);
        if (!slot_ok) continue;
        int lw = 0;
        bool in = true;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const int la = ((k >> a) & 1) + del[a];
          in = in && la >= 0 && la <= 1;
          lw |= (la & 1) << a;
        }
        if (!in) continue;
        const double* o = res[(ii - rd * CPR) * NV + lw];
#pragma unroll
        for (int a = 0; a < D; ++a) {
#pragma unroll
          for (int b = 0; b < D; ++b) pb.uu[a][b] += o[a * D + b];
          pb.pu[a] += o[D * D + a];
        }
        pb.pp += o[D * D + D];
      }
      __syncwarp();
    }
    (void)vmask;
    // CSR offsets of this slot's entries: free u / phi dofs of the in-range slots before it, by a
    // warp prefix sum over the slot lanes (lanes >= 3^d and out-of-range slots count 0)
    int myfu = 0, myfp = 0;
    if (slot_ok) {
      const i64 ws = X + g.nn * (Y + g.nn * Z);
#pragma unroll
      for (int b = 0; b < D; ++b) myfu += flag[ws * D + b] ? 0 : 1;
      myfp = flag[nu + ws] ? 0 : 1;
    }
    int incu = myfu, incp = myfp;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int tu = __shfl_up_sync(FULL, incu, o), tp = __shfl_up_sync(FULL, incp, o);
      if (lane >= o) {
        incu += tu;
        incp += tp;
      }
    }
    if (!slot_ok) continue;
    const i64 w = X + g.nn * (Y + g.nn * Z);
    bool rowfree_u[D], colfree_u[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      rowfree_u[a] = flag[v * D + a] == 0;
      colfree_u[a] = flag[w * D + a] == 0;
    }
    const bool rowfree_p = flag[nu + v] == 0, colfree_p = flag[nu + w] == 0;
    const bool center = w == v;
    const i64 off_u = incu - myfu, off_p = incp - myfp;
#pragma unroll
    for (int a = 0; a < D && UU; ++a) {
      const i64 row = lv * D + a;
      if (rowfree_u[a]) {
        i64 pos = ptr_uu[row] + off_u;
#pragma unroll
        for (int b = 0; b < D; ++b)
          if (colfree_u[b]) {
            col_uu[pos] = int(w * D + b - ushift);
            val_uu[pos] = pb.uu[a][b];
            ++pos;
          }
      } else if (center && ptr_uu[row + 1] > ptr_uu[row]) {
        col_uu[ptr_uu[row]] = int(v * D + a - ushift);
        val_uu[ptr_uu[row]] = pb.uu[a][a];
      }
    }
    if (rowfree_p) {
      i64 pos = ptr_pu[lv] + off_u;
#pragma unroll
      for (int b = 0; b < D; ++b)
        if (colfree_u[b]) {
          col_pu[pos] = int(w * D + b - ushift);
          val_pu[pos] = pb.pu[b];
          ++pos;
        }
      if (colfree_p) {
        col_pp[ptr_pp[lv] + off_p] = int(w - pshift);
        val_pp[ptr_pp[lv] + off_p] = pb.pp;
      }
    } else if (center && ptr_pp[lv + 1] > ptr_pp[lv]) {
      col_pp[ptr_pp[lv]] = int(v - pshift);
      val_pp[ptr_pp[lv]] = pb.pp;
    }
  }
}

// assemble_pattern (linsolve.cpp:417-476): the sparsity after condensation on a uniform grid.
// Rows and columns of constrained dofs are dropped (Dirichlet / active lines have no masters),
// every constrained dof keeps its diagonal; free dofs couple with the free dofs of the 3^d
// vertices sharing a cell.  fill = false counts, fill = true writes ascending columns.
template <int D>
__global__ void k_pattern(GridDesc g, const std::uint8_t* __restrict__ flag, i64* __restrict__ ptr_uu,
                          int* __restrict__ col_uu, i64* __restrict__ ptr_pu, int* __restrict__ col_pu,
                          i64* __restrict__ ptr_pp, int* __restrict__ col_pp, bool fill) {
  const i64 v = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= g.V) return;
  i64 x, y, z;
  vxyz<D>(g, v, x, y, z);
  const i64 nu = g.n_u();
  const bool pfree = flag[nu + v] == 0;
  i64 pos_u[D], pos_pu = fill ? ptr_pu[v] : 0, pos_pp = fill ? ptr_pp[v] : 0;
  bool ufree[D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    ufree[a] = flag[v * D + a] == 0;
    pos_u[a] = fill ? ptr_uu[v * D + a] : 0;
  }
  const int zl = (D == 3) ? -1 : 0, zh = (D == 3) ? 1 : 0;
  for (int dz = zl; dz <= zh; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const i64 X = x + dx, Y = y + dy, Z = z + dz;
        if (X < 0 || Y < 0 || Z < 0 || X >= g.nn || Y >= g.nn || Z >= ((D == 3) ? g.nn : 1)) continue;
        const i64 w = X + g.nn * (Y + g.nn * Z);
        for (int b = 0; b < D; ++b) {
          if (flag[w * D + b]) continue;
#pragma unroll
          for (int a = 0; a < D; ++a)
            if (ufree[a]) {
              if (fill) col_uu[pos_u[a]] = int(w * D + b);
              ++pos_u[a];
            }
          if (pfree) {
            if (fill) col_pu[pos_pu] = int(w * D + b);
            ++pos_pu;
          }
        }
        if (pfree && !flag[nu + w]) {
          if (fill) col_pp[pos_pp] = int(w);
          ++pos_pp;
        }
      }
#pragma unroll
  for (int a = 0; a < D; ++a)
    if (!ufree[a]) {  // constrained: its diagonal only
      if (fill) col_uu[pos_u[a]] = int(v * D + a);
      ++pos_u[a];
    }
  if (!pfree) {
    if (fill) col_pp[pos_pp] = int(v);
    ++pos_pp;
  }
  if (!fill) {
#pragma unroll
    for (int a = 0; a < D; ++a) ptr_uu[v * D + a] = pos_u[a];
    ptr_pu[v] = pos_pu;
    ptr_pp[v] = pos_pp;
  }
}

__global__ void k_build_flags(GridDesc g, int clamp, std::uint8_t* flag) {
  const i64 v = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= g.V) return;
  const i64 x = v % g.nn, y = (v / g.nn) % g.nn, z = (g.d == 3) ? v / (g.nn * g.nn) : 0;
  bool b = x == 0 || x == g.nc || y == 0 || y == g.nc;
  if (g.d == 3) b = b || z == 0 || z == g.nc;
  for (int a = 0; a < g.d; ++a) flag[v * g.d + a] = (clamp && b) ? 1 : 0;
  flag[g.n_u() + v] = 0;
}

// fem.cpp:258-263: active entries on unconstrained dofs (Dirichlet wins)
__global__ void k_apply_active(i64 n, const i64* __restrict__ dofs, const double* __restrict__ vals, i64 ntot,
                               std::uint8_t* flag, double* inhom, int* bad) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const i64 dof = dofs[i];
  if (dof < 0 || dof >= ntot) {
    *bad = 1;
    return;
  }
  if (flag[dof] == 1) return;  // Dirichlet (or a duplicate entry with the same value)
  flag[dof] = 2;
  inhom[dof] = vals[i];
}

__global__ void k_normalise_flags(i64 n, std::uint8_t* flag) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n && flag[i]) flag[i] = 1;
}

__global__ void k_distribute(i64 n, const std::uint8_t* __restrict__ flag, const double* __restrict__ inhom,
                             double* v, int homogeneous) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n && flag[i]) v[i] = homogeneous ? 0.0 : inhom[i];
}

Coef make_coef(const Problem& P, const cf_material& m, const cf_regularization& reg) {
  Coef c;
  c.kap = reg.kappa;
  c.eps = reg.eps;
  c.p = m.pressure;
  c.Gc = m.G_c;
  c.mu = mat_mu(m);
  c.lam = mat_lambda(m);
  c.coupling = m.pressure_coupling;
  (void)P;
  return c;
}

template <class T>
void exclusive_scan_inplace(T* data, i64 n) {  // n entries + 1 trailing zero -> offsets
  size_t bytes = 0;
  CF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, data, data, n + 1, stream()));
  DevBuf<unsigned char> tmp{static_cast<i64>(bytes)};
  CF_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, data, data, n + 1, stream()));
  count_launch();
}

}  // namespace

// ------------------------------------------------------------------ host side
void validate_material(const cf_material& m) {
  if (!(m.E > 0.0)) fail(CF_ERR_INVALID_ARGUMENT, "Material: E must be positive");
  if (!(m.nu >= 0.0 && m.nu < 0.5)) fail(CF_ERR_INVALID_ARGUMENT, "Material: nu must be in [0, 0.5)");
  if (!(m.G_c > 0.0)) fail(CF_ERR_INVALID_ARGUMENT, "Material: G_c must be positive");
}

Problem* make_problem(int d, double K, int n0, int r) {
  if (d != 2 && d != 3) fail(CF_ERR_INVALID_ARGUMENT, "DomainSpec: dimension must be 2 or 3");
  if (!(K > 0.0)) fail(CF_ERR_INVALID_ARGUMENT, "DomainSpec: half_width must be positive");
  if (n0 < 1 || n0 > 16) fail(CF_ERR_INVALID_ARGUMENT, "DomainSpec: initial_cells_per_side must be in [1,16]");
  if (r < 0) fail(CF_ERR_INVALID_ARGUMENT, "uniform_refine: times must be >= 0");
  if (r > 16) fail(CF_ERR_NUMERICAL, "Mesh: refinement depth exceeds integer coordinate resolution");
  ensure_device();
  auto* P = new Problem;
  GridDesc& g = P->g;
  g.d = d;
  g.r = r;
  g.n0 = n0;
  g.K = K;
  g.nc = i64(n0) << r;
  g.nn = g.nc + 1;
  g.V = (d == 3) ? g.nn * g.nn * g.nn : g.nn * g.nn;
  g.ncells = (d == 3) ? g.nc * g.nc * g.nc : g.nc * g.nc;
  if (g.V * (d + 1) >= (i64(1) << 31)) fail(CF_ERR_UNSUPPORTED, "problem exceeds int32 column indices");
  g.unit = 2.0 * K / (n0 * double(i64(1) << 16));  // mesh.cpp:20
  g.h = 2.0 * K / (n0 * double(i64(1) << r));      // mesh.hpp:65-67
  g.detJ = std::pow(g.h, d);                        // model.cpp:148
  P->tab.alloc(1);
  return P;
}

// q1_shape / cell_rule (fem.cpp:53-96) and the elasticity integrand table (model.cpp:270-276).
// Quadrature / Q1 tables of a cell of edge h (fem.cpp:53-96; model.cpp:111-123, 245-247, 274-275),
// computed with the reference's expressions (no FMA contraction in this file)
void fill_tables(Tables& T, int d, double h, double detJ, double mu, double lam) {
  const int nv = 1 << d, nq = 1 << d;
  std::memset(&T, 0, sizeof(T));
  const double a1 = 1.0 / std::sqrt(3.0);
  const double x1[2] = {-a1, a1}, w1[2] = {1.0, 1.0};
  for (int q = 0; q < nq; ++q) {
    int rem = q;
    double wt = 1.0;
    double xi[3] = {0, 0, 0};
    for (int a = 0; a < d; ++a) {
      const int i = rem % 2;
      rem /= 2;
      xi[a] = 0.5 * (x1[i] + 1.0);
      wt *= 0.5 * w1[i];
    }
    T.w[q] = wt * detJ;
    for (int k = 0; k < nv; ++k) {
      double v = 1.0;
      for (int a = 0; a < d; ++a) v *= (k & (1 << a)) ? xi[a] : 1.0 - xi[a];
      T.s[q][k] = v;
      for (int a = 0; a < d; ++a) {
        double gr = (k & (1 << a)) ? 1.0 : -1.0;
        for (int b = 0; b < d; ++b) {
          if (b == a) continue;
          gr *= (k & (1 << b)) ? xi[b] : 1.0 - xi[b];
        }
        T.G[q][k][a] = gr;
        T.gp[q][k][a] = gr / h;
      }
    }
    for (int k = 0; k < nv; ++k)
      for (int l = 0; l < nv; ++l) {
        double gg = 0.0;
        for (int b = 0; b < d; ++b) gg += T.gp[q][k][b] * T.gp[q][l][b];
        T.gg[q][k][l] = gg;
        for (int a = 0; a < d; ++a)
          for (int b = 0; b < d; ++b)
            T.val[q][k][l][a][b] =
                mu * ((a == b ? gg : 0.0) + T.gp[q][l][a] * T.gp[q][k][b]) + lam * T.gp[q][l][b] * T.gp[q][k][a];
      }
  }
}

void build_tables(Problem& P, double mu, double lam) {
  if (P.val_ready && P.mu == mu && P.lam == lam) return;
  fill_tables(P.host_tab, P.g.d, P.g.h, P.g.detJ, mu, lam);
  CF_CUDA(cudaMemcpyAsync(P.tab.p, &P.host_tab, sizeof(Tables), cudaMemcpyHostToDevice, stream()));
  P.mu = mu;
  P.lam = lam;
  P.val_ready = true;
}

std::unique_ptr<Constraints> build_constraints(const Problem& P, bool clamp, i64 n_active, const i64* dofs_dev,
                                               const double* vals_dev) {
  auto c = std::make_unique<Constraints>();
  c->prob = &P;
  const i64 nt = P.g.n_total();
  c->flag.alloc(nt);
  c->inhom.alloc(nt);
  c->inhom.zero();
  k_build_flags<<<grid_for(P.g.V, 256), 256, 0, stream()>>>(P.g, clamp ? 1 : 0, c->flag.p);
  CF_LAUNCHED();
  if (n_active > 0) {
    DevBuf<int> bad(1);
    bad.zero();
    k_apply_active<<<grid_for(n_active, 256), 256, 0, stream()>>>(n_active, dofs_dev, vals_dev, nt, c->flag.p,
                                                                   c->inhom.p, bad.p);
    CF_LAUNCHED();
    k_normalise_flags<<<grid_for(nt, 256), 256, 0, stream()>>>(nt, c->flag.p);
    CF_LAUNCHED();
    int hb = 0;
    read_small(&hb, bad.p, sizeof(int));
    if (hb) fail(CF_ERR_INVALID_ARGUMENT, "build_constraints: active dof out of range");
  }
  return c;
}

void distribute(const Constraints& c, double* v, bool homogeneous) {
  const i64 nt = c.flag.n;
  k_distribute<<<grid_for(nt, 256), 256, 0, stream()>>>(nt, c.flag.p, c.inhom.p, v, homogeneous ? 1 : 0);
  CF_LAUNCHED();
  distribute_lines(c, v, homogeneous);  // general meshes: the hanging lines (masters are unconstrained)
}

Slab make_slab(const GridDesc& g, i64 p_lo, i64 p_hi) {
  if (p_lo < 0 || p_hi > g.nn || p_lo >= p_hi) fail(CF_ERR_INVALID_ARGUMENT, "make_slab: empty or out-of-range planes");
  Slab s;
  s.plane = (g.d == 3) ? g.nn * g.nn : g.nn;
  const i64 cplane = (g.d == 3) ? g.nc * g.nc : g.nc;
  s.v_lo = p_lo * s.plane;
  s.v_hi = p_hi * s.plane;
  s.ve_lo = std::max<i64>(p_lo - 1, 0) * s.plane;
  s.ve_hi = std::min<i64>(p_hi + 1, g.nn) * s.plane;
  s.c_lo = std::max<i64>(p_lo - 1, 0) * cplane;  // cells of planes [p_lo - 1, p_hi) touch owned vertices
  s.c_hi = std::min<i64>(p_hi, g.nc) * cplane;
  return s;
}

void assemble_residual(Problem& P, const Constraints& cs, const cf_material& m, const cf_regularization& reg,
                       const double* x, const double* pt, double* R, const Slab* slab, ResidualCache* cache) {
  build_tables(P, mat_mu(m), mat_lambda(m));
  const Coef cf = make_coef(P, m, reg);
  const GridDesc& g = P.g;
  const Slab sl = slab ? *slab : full_slab(g);
  const int nv = 1 << g.d;
  const i64 nc = sl.c_hi - sl.c_lo;
  DevBuf<double> local;
  DevBuf<double>& cellres = cache ? cache->cellres : local;
  if (cellres.n != nc * nv * (g.d + 1)) cellres.alloc(nc * nv * (g.d + 1));
  if (g.d == 2) {
    k_cell_residual_q<2><<<grid_for(nc * 4, 256), 256, 0, stream()>>>(g, P.tab.p, cf, x, pt, cellres.p, sl.c_lo,
                                                                      sl.c_hi, nullptr, 0);
    CF_LAUNCHED();
    k_vertex_residual<2><<<grid_for(sl.nv(), 256), 256, 0, stream()>>>(g, cellres.p, cs.flag.p, R, sl);
    CF_LAUNCHED();
  } else {
    k_cell_residual_q<3><<<grid_for(nc * 8, 256), 256, 0, stream()>>>(g, P.tab.p, cf, x, pt, cellres.p, sl.c_lo,
                                                                      sl.c_hi, nullptr, 0);
    CF_LAUNCHED();
    k_vertex_residual<3><<<grid_for(sl.nv(), 256), 256, 0, stream()>>>(g, cellres.p, cs.flag.p, R, sl);
    CF_LAUNCHED();
  }
  if (cache) {
    cache->c_lo = sl.c_lo;
    cache->c_hi = sl.c_hi;
    cache->valid = true;
  }
}

void assemble_residual_moved(Problem& P, const Constraints& cs, const cf_material& m, const cf_regularization& reg,
                             const double* x, const double* x_before, const double* pt, double* R,
                             const Slab* slab, ResidualCache& cache) {
  const GridDesc& g = P.g;
  const Slab sl = slab ? *slab : full_slab(g);
  if (!cache.valid || cache.c_lo != sl.c_lo || cache.c_hi != sl.c_hi) {
    assemble_residual(P, cs, m, reg, x, pt, R, slab, &cache);
    return;
  }
  build_tables(P, mat_mu(m), mat_lambda(m));
  const Coef cf = make_coef(P, m, reg);
  const i64 nc = sl.c_hi - sl.c_lo;
  if (cache.list.n < nc) cache.list.alloc(nc);
  if (!cache.count.n) cache.count.alloc(1);
  cache.count.zero();
  int n = 0;
  if (g.d == 2) {
    k_moved_cells<2><<<grid_for(nc, 256), 256, 0, stream()>>>(g, sl.c_lo, sl.c_hi, x, x_before, cache.list.p,
                                                              cache.count.p);
  } else {
    k_moved_cells<3><<<grid_for(nc, 256), 256, 0, stream()>>>(g, sl.c_lo, sl.c_hi, x, x_before, cache.list.p,
                                                              cache.count.p);
  }
  CF_LAUNCHED();
  read_small(&n, cache.count.p, sizeof(int));
  if (g.d == 2) {
    if (n)
      k_cell_residual_q<2><<<grid_for(i64(n) * 4, 256), 256, 0, stream()>>>(g, P.tab.p, cf, x, pt, cache.cellres.p,
                                                                            sl.c_lo, sl.c_hi, cache.list.p, n);
    k_vertex_residual<2><<<grid_for(sl.nv(), 256), 256, 0, stream()>>>(g, cache.cellres.p, cs.flag.p, R, sl);
  } else {
    if (n)
      k_cell_residual_q<3><<<grid_for(i64(n) * 8, 256), 256, 0, stream()>>>(g, P.tab.p, cf, x, pt, cache.cellres.p,
                                                                            sl.c_lo, sl.c_hi, cache.list.p, n);
    k_vertex_residual<3><<<grid_for(sl.nv(), 256), 256, 0, stream()>>>(g, cache.cellres.p, cs.flag.p, R, sl);
  }
  CF_LAUNCHED();
}

template <int D>
static void jacobian_impl(Problem& P, const Constraints& cs, const Coef& cf, const double* x, const double* pt,
                          const Slab& sl, BlockSystem& J, bool with_uu) {
  const GridDesc& g = P.g;
  constexpr int NQ = 1 << D, NS = QS<D>::NS;
  const i64 ncl = sl.c_hi - sl.c_lo;
  DevBuf<double> qs(ncl * NQ * NS);
  static const bool serial_qs = std::getenv("CF_QPSTATE_SERIAL") != nullptr;  // A/B: one thread per cell
  if (serial_qs)
    k_cell_qpstate<D><<<grid_for(ncl, 128), 128, 0, stream()>>>(g, P.tab.p, cf, x, pt, qs.p, sl.c_lo, sl.c_hi);
  else
    k_cell_qpstate_q<D><<<grid_for(ncl * (1 << D), 256), 256, 0, stream()>>>(g, P.tab.p, cf, x, pt, qs.p, sl.c_lo,
                                                                              sl.c_hi);
  CF_LAUNCHED();
  const i64 nu = D * sl.nv(), np = sl.nv();
  J.pu->rows = np;
  J.pu->cols = D * sl.ne();
  J.pp->rows = np;
  J.pp->cols = sl.ne();
  if (with_uu) {
    J.uu->rows = nu;
    J.uu->cols = D * sl.ne();
    J.uu->ptr.alloc(nu + 1);
    CF_CUDA(cudaMemsetAsync(J.uu->ptr.p + nu, 0, sizeof(i64), stream()));
  }
  J.pu->ptr.alloc(np + 1);
  J.pp->ptr.alloc(np + 1);
  CF_CUDA(cudaMemsetAsync(J.pu->ptr.p + np, 0, sizeof(i64), stream()));
  CF_CUDA(cudaMemsetAsync(J.pp->ptr.p + np, 0, sizeof(i64), stream()));
  if (with_uu)
    k_jac_count<D, true><<<grid_for(sl.nv(), 128), 128, 0, stream()>>>(g, P.tab.p, cf, qs.p, cs.flag.p, J.uu->ptr.p,
                                                                       J.pu->ptr.p, J.pp->ptr.p, sl);
  else
    k_jac_count<D, false><<<grid_for(sl.nv(), 128), 128, 0, stream()>>>(g, P.tab.p, cf, qs.p, cs.flag.p, nullptr,
                                                                        J.pu->ptr.p, J.pp->ptr.p, sl);
  CF_LAUNCHED();
  if (with_uu) exclusive_scan_inplace(J.uu->ptr.p, nu);
  exclusive_scan_inplace(J.pu->ptr.p, np);
  exclusive_scan_inplace(J.pp->ptr.p, np);
  i64 nnz[3] = {0, 0, 0};
  if (with_uu) CF_CUDA(cudaMemcpyAsync(&nnz[0], J.uu->ptr.p + nu, sizeof(i64), cudaMemcpyDeviceToHost, stream()));
  CF_CUDA(cudaMemcpyAsync(&nnz[1], J.pu->ptr.p + np, sizeof(i64), cudaMemcpyDeviceToHost, stream()));
  read_small(&nnz[2], J.pp->ptr.p + np, sizeof(i64));
  if (with_uu) {
    J.uu->nnz = nnz[0];
    J.uu->col.alloc(nnz[0]);
    J.uu->val.alloc(nnz[0]);
  }
  J.pu->nnz = nnz[1];
  J.pp->nnz = nnz[2];
  J.pu->col.alloc(nnz[1]);
  J.pu->val.alloc(nnz[1]);
  J.pp->col.alloc(nnz[2]);
  J.pp->val.alloc(nnz[2]);
  int bps = 0;
  constexpr int FT = pair_wpb<D>() * 32;
  const int smem = with_uu ? int(sizeof(PairSmem<D, true>)) : int(sizeof(PairSmem<D, false>));
  auto kern = with_uu ? k_jac_fill_pair<D, true> : k_jac_fill_pair<D, false>;
  CF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, FT, smem));
  const int grid = std::max(1, bps) * rt().sm_count;
  i64* uptr = with_uu ? J.uu->ptr.p : nullptr;
  int* ucol = with_uu ? J.uu->col.p : nullptr;
  double* uval = with_uu ? J.uu->val.p : nullptr;
  kern<<<grid, FT, smem, stream()>>>(g, P.tab.p, cf, qs.p, cs.flag.p, uptr, ucol, uval, J.pu->ptr.p, J.pu->col.p,
                                     J.pu->val.p, J.pp->ptr.p, J.pp->col.p, J.pp->val.p, sl);
  CF_LAUNCHED();
  // value-only SpMV streams for the blocks whose pattern is the clamped stencil
  if (with_uu) csr_enable_stencil(*J.uu, StencilCols{1, D, g.nn, sl.v_lo, D * sl.ve_lo, 1.0 / double(g.nn)});
  csr_enable_stencil(*J.pu, StencilCols{2, D, g.nn, sl.v_lo, D * sl.ve_lo, 1.0 / double(g.nn)});
}

std::unique_ptr<BlockSystem> assemble_jacobian(Problem& P, const Constraints& cs, const cf_material& m,
                                               const cf_regularization& reg, const double* x, const double* pt,
                                               const Slab* slab, std::shared_ptr<Csr> reuse_uu) {
  build_tables(P, mat_mu(m), mat_lambda(m));
  const Coef cf = make_coef(P, m, reg);
  const Slab sl = slab ? *slab : full_slab(P.g);
  auto J = std::make_unique<BlockSystem>();
  J->d = P.g.d;
  J->nu = P.g.d * sl.nv();
  J->np = sl.nv();
  if (!sl.full(P.g)) {
    J->nu_in = P.g.d * sl.ne();
    J->np_in = sl.ne();
  }
  if (reuse_uu) J->uu = std::move(reuse_uu);  // M_uu depends only on phi_tilde and the Dirichlet set
  if (P.g.d == 2)
    jacobian_impl<2>(P, cs, cf, x, pt, sl, *J, !J->uu->ptr.p);
  else
    jacobian_impl<3>(P, cs, cf, x, pt, sl, *J, !J->uu->ptr.p);
  return J;
}

template <int D>
static void pattern_impl(const Problem& P, const Constraints& cs, BlockSystem& J) {
  const GridDesc& g = P.g;
  const i64 nu = g.n_u(), np = g.V;
  Csr* B[3] = {J.uu.get(), J.pu.get(), J.pp.get()};
  const i64 rows[3] = {nu, np, np}, cols[3] = {nu, nu, np};
  for (int b = 0; b < 3; ++b) {
    B[b]->rows = rows[b];
    B[b]->cols = cols[b];
    B[b]->ptr.alloc(rows[b] + 1);
    CF_CUDA(cudaMemsetAsync(B[b]->ptr.p + rows[b], 0, sizeof(i64), stream()));
  }
  k_pattern<D><<<grid_for(g.V, 128), 128, 0, stream()>>>(g, cs.flag.p, J.uu->ptr.p, nullptr, J.pu->ptr.p, nullptr,
                                                          J.pp->ptr.p, nullptr, false);
  CF_LAUNCHED();
  for (int b = 0; b < 3; ++b) {
    exclusive_scan_inplace(B[b]->ptr.p, rows[b]);
    CF_CUDA(cudaMemcpyAsync(&B[b]->nnz, B[b]->ptr.p + rows[b], sizeof(i64), cudaMemcpyDeviceToHost, stream()));
  }
  CF_CUDA(cudaStreamSynchronize(stream()));
  ++host_sync_count();
  for (int b = 0; b < 3; ++b) {
    B[b]->col.alloc(B[b]->nnz);
    B[b]->val.alloc(B[b]->nnz);
    B[b]->val.zero();  // a pattern: explicit zeros
  }
  k_pattern<D><<<grid_for(g.V, 128), 128, 0, stream()>>>(g, cs.flag.p, J.uu->ptr.p, J.uu->col.p, J.pu->ptr.p,
                                                          J.pu->col.p, J.pp->ptr.p, J.pp->col.p, true);
  CF_LAUNCHED();
}

std::unique_ptr<BlockSystem> assemble_pattern(const Problem& P, const Constraints& cs) {
  auto J = std::make_unique<BlockSystem>();
  J->d = P.g.d;
  J->nu = P.g.n_u();
  J->np = P.g.V;
  if (P.g.d == 2)
    pattern_impl<2>(P, cs, *J);
  else
    pattern_impl<3>(P, cs, *J);
  return J;
}

// test hook: q = a / h through the residual kernel's division (DivBy)
void div_by_h(double h, const double* a, i64 n, double* q) {
  if (n <= 0) return;
  k_div_by<<<int(std::min<i64>(grid_for(n, 256), 148 * 16)), 256, 0, stream()>>>(h, a, n, q);
  CF_LAUNCHED();
}

}  // namespace cfb

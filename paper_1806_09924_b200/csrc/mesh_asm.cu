// Assembly on general meshes: element kernels with each cell's own edge h and
// the condensation / setFromTriplets plans (see mesh.cu's header for the design).
//
// Element arithmetic follows the uniform kernels (assembly.cu) expression by expression:
//  * residual (model.cpp:127-202): one thread per (cell, quadrature point), every a / h an
//    IEEE-exact quotient (DivBy), the per-point contributions folded in q order;
//  * Jacobian (model.cpp:206-289): per-(cell, q) states (w g, phi, tr e, sig:e, sig), then one
//    thread per (cell, k, l) sums its kuu / kpu / kpp blocks over q from the level's tables.
// Plan slot values are 0.0 + the weighted entries in the reference's insertion order, so every
// residual entry and matrix value equals the reference's (oracle_mesh.inc) bit for bit.
#include <algorithm>
#include <cmath>

#include <cub/cub.cuh>

#include "cf_mesh.hpp"

namespace cfb {

namespace {

template <class T>
T read1(const T* p) {
  T h{};
  read_small(&h, p, sizeof(T));
  return h;
}

template <class T>
void scan_ex(T* data, i64 n1) {
  size_t bytes = 0;
  CF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, data, data, n1, stream()));
  DevBuf<unsigned char> tmp{i64(bytes)};
  CF_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, data, data, n1, stream()));
  count_launch();
}

struct MCoef {
  double kap, eps, p, Gc, mu, lam;
  int coupling;
};

MCoef mcoef(const cf_material& m, const cf_regularization& reg) {
  return MCoef{reg.kappa, reg.eps, m.pressure, m.G_c, mat_mu(m), mat_lambda(m), m.pressure_coupling};
}

// a / h as the IEEE quotient (assembly.cu DivBy, Markstein's correctly rounded reciprocal scheme)
struct MDiv {
  double h, y;
  __device__ explicit MDiv(double h_) : h(h_), y(1.0 / h_) {}
  __device__ __forceinline__ double div(double a) const {
    const double m = fabs(a);
    if (m == 0.0) return a;
    if (!(m >= 0x1p-900 && m <= 0x1p900)) return a / h;
    double q = a * y;
    double r = __fma_rn(-q, h, a);
    q = __fma_rn(r, y, q);
    r = __fma_rn(-q, h, a);
    return __fma_rn(r, y, q);
  }
};

// ---- residual element kernel: out[c][k][comp] (comp < D: u_comp, D: phi)
template <int D>
__global__ void __launch_bounds__(256) k_mesh_residual(i64 nact, const int* __restrict__ cvert,
                                                       const int* __restrict__ clevel, const double* __restrict__ hlev,
                                                       const Tables* __restrict__ tabs, MCoef cf, i64 V,
                                                       const double* __restrict__ sol, const double* __restrict__ ptil,
                                                       double* __restrict__ out) {
  constexpr int NV = 1 << D, NQ = 1 << D;
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  const i64 c = t / NQ;
  const int q = int(t % NQ);
  const bool valid = c < nact;
  const i64 cc = valid ? c : 0;
  const int lev = clevel[cc];
  const Tables* T = tabs + lev;
  const i64 nu = i64(D) * V;
  double my_u[D], my_phi, my_pt;
  {
    const i64 v = cvert[cc * NV + q];
#pragma unroll
    for (int a = 0; a < D; ++a) my_u[a] = sol[v * D + a];
    my_phi = sol[nu + v];
    my_pt = ptil[v];
  }
  const MDiv dv(hlev[lev]);
  double gu[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  double gphi[3] = {0, 0, 0};
  double phi = 0.0, pt = 0.0;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double uk[D];
#pragma unroll
    for (int a = 0; a < D; ++a) uk[a] = __shfl_sync(0xffffffffu, my_u[a], k, NQ);
    const double phik = __shfl_sync(0xffffffffu, my_phi, k, NQ);
    const double ptk = __shfl_sync(0xffffffffu, my_pt, k, NQ);
    const double sk = T->s[q][k];
    phi += sk * phik;
    pt += sk * ptk;
#pragma unroll
    for (int b = 0; b < D; ++b) {
      const double Gkb = T->G[q][k][b];
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
  const double w = T->w[q];
  double keep[D + 1];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double contrib[D + 1];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      double val = 0.0;
#pragma unroll
      for (int b = 0; b < D; ++b) val += dv.div(gcoef * sig[a][b] * T->G[q][k][b]);
      val += dv.div(pphi * cf.p * T->G[q][k][a]);
      contrib[a] = w * val;
    }
    double vphi = ((1.0 - cf.kap) * phi * sig_ee + 2.0 * phi * cf.p * tre - cf.Gc / cf.eps * (1.0 - phi)) * T->s[q][k];
#pragma unroll
    for (int b = 0; b < D; ++b) vphi += dv.div(cf.Gc * cf.eps * gphi[b] * T->G[q][k][b]);
    contrib[D] = w * vphi;
#pragma unroll
    for (int a = 0; a <= D; ++a) {
      double s = 0.0;
#pragma unroll
      for (int qq = 0; qq < NQ; ++qq) s += __shfl_sync(0xffffffffu, contrib[a], qq, NQ);
      if (q == k) keep[a] = s;
    }
  }
  if (valid) {
    double* o = out + c * (NV * (D + 1)) + q * (D + 1);
#pragma unroll
    for (int a = 0; a <= D; ++a) o[a] = keep[a];
  }
}

// ---- Jacobian: per-(cell, q) states (model.cpp:242-266): w g, phi, tr e, sig:e, sig
template <int D>
__global__ void k_mesh_qpstate(i64 nact, const int* __restrict__ cvert, const int* __restrict__ clevel,
                               const Tables* __restrict__ tabs, MCoef cf, i64 V, const double* __restrict__ sol,
                               const double* __restrict__ ptil, double* __restrict__ out) {
  constexpr int NV = 1 << D, NQ = 1 << D, NS = 4 + D * D;
  const i64 c = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= nact) return;
  const Tables* T = tabs + clevel[c];
  const i64 nu = i64(D) * V;
  double uloc[NV][D], philoc[NV], ptloc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const i64 v = cvert[c * NV + k];
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
    double* o = out + (c * NQ + q) * NS;
    o[0] = T->w[q] * gcoef;
    o[1] = phi;
    o[2] = tre;
    o[3] = sig_ee;
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) o[4 + a * D + b] = sig[a][b];
  }
}

// element matrices: one thread per (cell, k, l).  Kuu[c][k*D+a][l*D+b], Kpu[c][k][l*D+b], Kpp[c][k][l]
template <int D>
__global__ void k_mesh_elem(i64 nact, const int* __restrict__ clevel, const Tables* __restrict__ tabs, MCoef cf,
                            const double* __restrict__ qs, double* __restrict__ Kuu, double* __restrict__ Kpu,
                            double* __restrict__ Kpp) {
  constexpr int NV = 1 << D, NQ = 1 << D, NS = 4 + D * D, ND = NV * D;
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nact * NV * NV) return;
  const i64 c = t / (NV * NV);
  const int k = int((t / NV) % NV), l = int(t % NV);
  const Tables* T = tabs + clevel[c];
  const double c2k = 2.0 * (1.0 - cf.kap), c2p = 2.0 * cf.p, omk = 1.0 - cf.kap;
  const double gce = cf.Gc / cf.eps, gcx = cf.Gc * cf.eps;
  double bu[D][D], bp[D], bpp = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
#pragma unroll
    for (int b = 0; b < D; ++b) bu[a][b] = 0.0;
    bp[a] = 0.0;
  }
  for (int q = 0; q < NQ; ++q) {
    const double* st = qs + (c * NQ + q) * NS;
    const double wg = st[0];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) bu[a][b] += wg * T->val[q][k][l][a][b];
    const double w = T->w[q];
    const double phi = st[1], tre = st[2], see = st[3];
    const double sk = T->s[q][k], sl = T->s[q][l];
#pragma unroll
    for (int b = 0; b < D; ++b) {
      double sgl = 0.0;
#pragma unroll
      for (int cc = 0; cc < D; ++cc) sgl += st[4 + b * D + cc] * T->gp[q][l][cc];
      bp[b] += w * (c2k * phi * sgl + c2p * phi * T->gp[q][l][b]) * sk;
    }
    bpp += w * ((omk * see + c2p * tre + gce) * sl * sk + gcx * T->gg[q][k][l]);
  }
#pragma unroll
  for (int a = 0; a < D; ++a) {
#pragma unroll
    for (int b = 0; b < D; ++b) Kuu[c * ND * ND + (k * D + a) * ND + l * D + b] = bu[a][b];
    Kpu[c * NV * ND + k * ND + l * D + a] = bp[a];
  }
  Kpp[c * NV * NV + k * NV + l] = bpp;
}

// ---- plans
// targets of a dof under the base constraints: itself (weight 1) when free, its line entries
// when it has a line, nothing when it is entry-free constrained
struct Targets {
  const std::uint8_t* flag;
  const int* line_of;  // dof -> line index or -1
  const i64* lptr;
  const int* lm;
  const double* lw;
  __device__ int count(i64 dof) const {
    if (!flag[dof]) return 1;
    const int li = line_of[dof];
    return li < 0 ? 0 : int(lptr[li + 1] - lptr[li]);
  }
  __device__ void get(i64 dof, int j, i64& t, double& w) const {
    if (!flag[dof]) {
      t = dof;
      w = 1.0;
      return;
    }
    const i64 e = lptr[line_of[dof]] + j;
    t = lm[e];
    w = lw[e];
  }
};

__global__ void k_line_of(i64 nl, const int* __restrict__ ldof, int* __restrict__ line_of) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < nl) line_of[ldof[i]] = int(i);
}

// residual plan emission: one thread per (cell, corner, component) slot
template <bool FILL>
__global__ void k_res_emit(i64 nact, int d, i64 V, const int* __restrict__ cvert, Targets tg, i64* __restrict__ cnt,
                           const i64* __restrict__ off, i64* __restrict__ key, i64* __restrict__ src,
                           double* __restrict__ w) {
  const int nv = 1 << d, ns = nv * (d + 1);
  const i64 s = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= nact * ns) return;
  const i64 c = s / ns;
  const int k = int((s % ns) / (d + 1)), comp = int(s % (d + 1));
  const i64 v = cvert[c * nv + k];
  const i64 dof = comp < d ? v * d + comp : i64(d) * V + v;
  const int n = tg.count(dof);
  if (!FILL) {
    cnt[s] = n;
    return;
  }
  i64 o = off[s];
  for (int j = 0; j < n; ++j) {
    i64 t;
    double ww;
    tg.get(dof, j, t, ww);
    key[o] = t;
    src[o] = s;
    w[o] = ww;
    ++o;
  }
}

// self incidences: every (cell, corner, component) slot keyed by its own dof
__global__ void k_self_emit(i64 nact, int d, i64 V, const int* __restrict__ cvert, i64* __restrict__ key,
                            i64* __restrict__ src) {
  const int nv = 1 << d, ns = nv * (d + 1);
  const i64 s = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= nact * ns) return;
  const i64 c = s / ns;
  const int k = int((s % ns) / (d + 1)), comp = int(s % (d + 1));
  const i64 v = cvert[c * nv + k];
  key[s] = comp < d ? v * d + comp : i64(d) * V + v;
  src[s] = s;
}

// Jacobian plan emission, one thread per (cell, row-local i): for j, for row target, for column
// target (Scatter::matrix_add's loop order).  blk 0: uu (i, j < NV*D), 1: pu (i < NV, j < NV*D),
// 2: pp (i, j < NV).  Keys row * ncols + col over the block's local numbering.
template <bool FILL>
__global__ void k_jac_emit(int blk, i64 nact, int d, i64 V, const int* __restrict__ cvert, Targets tg,
                           i64* __restrict__ cnt, const i64* __restrict__ off, i64* __restrict__ key,
                           i64* __restrict__ src, double* __restrict__ w) {
  const int nv = 1 << d, nd = nv * d;
  const int ni = blk == 0 ? nd : nv, nj = blk == 2 ? nv : nd;
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nact * ni) return;
  const i64 c = t / ni;
  const int i = int(t % ni);
  const i64 nu = i64(d) * V;
  auto dof_of = [&](int loc, bool u) -> i64 {
    if (u) return i64(cvert[c * nv + loc / d]) * d + loc % d;
    return nu + cvert[c * nv + loc];
  };
  const bool row_u = blk == 0, col_u = blk != 2;
  const i64 rdof = dof_of(i, row_u);
  const int nr = tg.count(rdof);
  if (!FILL) {
    i64 sc = 0;
    for (int j = 0; j < nj; ++j) sc += tg.count(dof_of(j, col_u));
    cnt[t] = i64(nr) * sc;
    return;
  }
  const i64 roff = row_u ? 0 : nu, coff = col_u ? 0 : nu, ncols = col_u ? nu : V;
  const i64 ebase = c * i64(ni) * nj + i64(i) * nj;
  i64 o = off[t];
  for (int j = 0; j < nj; ++j) {
    const i64 cdof = dof_of(j, col_u);
    const int nc = tg.count(cdof);
    for (int r = 0; r < nr; ++r) {
      i64 rt;
      double rw;
      tg.get(rdof, r, rt, rw);
      for (int q = 0; q < nc; ++q) {
        i64 ct;
        double cw;
        tg.get(cdof, q, ct, cw);
        key[o] = (rt - roff) * ncols + (ct - coff);
        src[o] = ebase + j;
        w[o] = rw * cw;
        ++o;
      }
    }
  }
}

__global__ void k_gather_i64(i64 n, const i64* __restrict__ idx, const i64* __restrict__ in, i64* __restrict__ out) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[idx[i]];
}
__global__ void k_gather_f64(i64 n, const i64* __restrict__ idx, const double* __restrict__ in,
                             double* __restrict__ out) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[idx[i]];
}
__global__ void k_iota64(i64 n, i64* out) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = i;
}
// segment heads of sorted keys: head[i] = 1 if i == 0 or key[i] != key[i-1]
__global__ void k_heads(i64 n, const i64* __restrict__ key, i64* __restrict__ head) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) head[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}
// slot pointers / (row, col) of each slot from the scanned heads
__global__ void k_slots(i64 n, const i64* __restrict__ key, const i64* __restrict__ hscan, i64 ncols, int keyed_rows,
                        i64* __restrict__ ptr, int* __restrict__ row, int* __restrict__ col) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i == 0 || key[i] != key[i - 1]) {
    const i64 s = hscan[i];
    ptr[s] = i;
    if (keyed_rows) {
      row[s] = int(key[i] / ncols);
      col[s] = int(key[i] % ncols);
    }
  }
}

__global__ void k_lower_bound(i64 n, const i64* __restrict__ key, i64 nq, i64* __restrict__ out) {
  const i64 q = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  i64 lo = 0, hi = n;
  while (lo < hi) {
    const i64 mid = (lo + hi) >> 1;
    if (key[mid] < q) lo = mid + 1; else hi = mid;
  }
  out[q] = lo;
}

// Build a plan from emitted (key, src, w) triples: stable radix sort by key (the emission order is
// the reference's insertion order, so equal keys keep it), then one slot per key.  dense: slots
// are the keys 0 .. keyspace - 1 (vector plans; empty slots allowed); otherwise one slot per
// distinct key with its (row, col) = (key / ncols, key % ncols).
void build_plan(Plan& P, DevBuf<i64>& key, DevBuf<i64>& src, DevBuf<double>& w, i64 ne, i64 keyspace, bool dense,
                i64 ncols) {
  DevBuf<i64> idx(std::max<i64>(ne, 1)), idx_s(std::max<i64>(ne, 1)), key_s(std::max<i64>(ne, 1));
  if (ne > 0) {
    k_iota64<<<grid_for(ne, 256), 256, 0, stream()>>>(ne, idx.p);
    CF_LAUNCHED();
    int bits = 1;
    while (bits < 63 && (i64(1) << bits) < keyspace) ++bits;
    size_t bytes = 0;
    CF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key.p, key_s.p, idx.p, idx_s.p, ne, 0, bits, stream()));
    DevBuf<unsigned char> tmp{i64(bytes)};
    CF_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, key.p, key_s.p, idx.p, idx_s.p, ne, 0, bits, stream()));
    count_launch();
  }
  P.src.alloc(std::max<i64>(ne, 1));
  P.w.alloc(std::max<i64>(ne, 1));
  if (ne > 0) {
    k_gather_i64<<<grid_for(ne, 256), 256, 0, stream()>>>(ne, idx_s.p, src.p, P.src.p);
    CF_LAUNCHED();
    k_gather_f64<<<grid_for(ne, 256), 256, 0, stream()>>>(ne, idx_s.p, w.p, P.w.p);
    CF_LAUNCHED();
  }
  if (dense) {
    P.n = keyspace;
    P.ptr.alloc(keyspace + 1);
    k_lower_bound<<<grid_for(keyspace + 1, 256), 256, 0, stream()>>>(ne, key_s.p, keyspace + 1, P.ptr.p);
    CF_LAUNCHED();
    return;
  }
  DevBuf<i64> head(ne + 1);
  if (ne > 0) {
    k_heads<<<grid_for(ne, 256), 256, 0, stream()>>>(ne, key_s.p, head.p);
    CF_LAUNCHED();
  }
  CF_CUDA(cudaMemsetAsync(head.p + ne, 0, sizeof(i64), stream()));
  scan_ex(head.p, ne + 1);
  const i64 ns = read1(head.p + ne);
  P.n = ns;
  P.ptr.alloc(ns + 1);
  P.row.alloc(std::max<i64>(ns, 1));
  P.col.alloc(std::max<i64>(ns, 1));
  if (ne > 0) {
    k_slots<<<grid_for(ne, 256), 256, 0, stream()>>>(ne, key_s.p, head.p, ncols, 1, P.ptr.p, P.row.p, P.col.p);
    CF_LAUNCHED();
  }
  CF_CUDA(cudaMemcpyAsync(P.ptr.p + ns, &ne, sizeof(i64), cudaMemcpyHostToDevice, stream()));
  CF_CUDA(cudaStreamSynchronize(stream()));
}

}  // namespace
}  // namespace cfb

namespace cfb {

namespace {

__global__ void k_res_apply(i64 n, const i64* __restrict__ ptr, const i64* __restrict__ src,
                            const double* __restrict__ w, const double* __restrict__ el,
                            const std::uint8_t* __restrict__ mask, double* __restrict__ R) {
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  double s = 0.0;
  if (!mask[t])
    for (i64 e = ptr[t]; e < ptr[t + 1]; ++e) s += w[e] * el[src[e]];
  R[t] = s;
}

__global__ void k_plan_vals(i64 n, const i64* __restrict__ ptr, const i64* __restrict__ src,
                            const double* __restrict__ w, const double* __restrict__ el, double* __restrict__ out) {
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  double s = 0.0;
  for (i64 e = ptr[t]; e < ptr[t + 1]; ++e) s += w[e] * el[src[e]];
  out[t] = s;
}

__global__ void k_row_lb(i64 n, const int* __restrict__ row, i64 nq, i64* __restrict__ out) {
  const i64 q = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  i64 lo = 0, hi = n;
  while (lo < hi) {
    const i64 mid = (lo + hi) >> 1;
    if (row[mid] < q) lo = mid + 1; else hi = mid;
  }
  out[q] = lo;
}

// constrained diagonals: 0.0 + the element diagonals of the row dof's own incidences in cell order
// (model.cpp:294-311); blk 0 uu, 2 pp.  rows: block-local row count, roff: first dof of the block
__global__ void k_diag(int blk, i64 rows, i64 roff, int d, const i64* __restrict__ sptr,
                       const i64* __restrict__ ssrc, const std::uint8_t* __restrict__ mask,
                       const double* __restrict__ K, double* __restrict__ diag) {
  const i64 r = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const i64 dof = roff + r;
  if (!mask[dof]) {
    diag[r] = 0.0;
    return;
  }
  const int nv = 1 << d, ns = nv * (d + 1), nd = nv * d;
  double s = 0.0;
  for (i64 e = sptr[dof]; e < sptr[dof + 1]; ++e) {
    const i64 sl = ssrc[e], c = sl / ns;
    const int k = int((sl % ns) / (d + 1)), comp = int(sl % (d + 1));
    if (blk == 0) {
      const int i = k * d + comp;
      s += K[c * i64(nd) * nd + i64(i) * nd + i];
    } else {
      s += K[c * i64(nv) * nv + k * nv + k];
    }
  }
  diag[r] = s;
}

// CSR of a block from its plan: free rows keep their slots whose column is free, constrained rows
// (in the assembly's set) keep only a nonzero diagonal (uu, pp)
template <bool FILL>
__global__ void k_block_rows(i64 rows, i64 roff, i64 coff, int has_diag, const i64* __restrict__ rptr,
                             const int* __restrict__ scol, const double* __restrict__ svals,
                             const std::uint8_t* __restrict__ mask, const double* __restrict__ diag,
                             i64* __restrict__ cnt, const i64* __restrict__ optr, int* __restrict__ ocol,
                             double* __restrict__ oval) {
  const i64 r = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  if (mask[roff + r]) {
    const bool keep = has_diag && diag[r] != 0.0;
    if (!FILL) {
      cnt[r] = keep ? 1 : 0;
    } else if (keep) {
      ocol[optr[r]] = int(r);
      oval[optr[r]] = diag[r];
    }
    return;
  }
  i64 o = FILL ? optr[r] : 0, n = 0;
  for (i64 s = rptr[r]; s < rptr[r + 1]; ++s) {
    if (mask[coff + scol[s]]) continue;
    if (FILL) {
      ocol[o] = scol[s];
      oval[o] = svals[s];
      ++o;
    }
    ++n;
  }
  if (!FILL) cnt[r] = n;
}

void ensure_plans(MeshDisc& m, const Constraints& pc) {
  if (m.plans_ready && m.plan_uid == pc.uid && pc.uid != 0) return;
  const int d = m.d, nv = 1 << d, ns = nv * (d + 1), nd = nv * d;
  const i64 V = m.V, nu = m.n_u(), nt = m.n_total(), nact = m.nact;
  DevBuf<int> line_of(nt);
  CF_CUDA(cudaMemsetAsync(line_of.p, 0xff, size_t(nt) * sizeof(int), stream()));
  if (pc.n_lines) {
    k_line_of<<<grid_for(pc.n_lines, 256), 256, 0, stream()>>>(pc.n_lines, pc.line_dof.p, line_of.p);
    CF_LAUNCHED();
  }
  Targets tg{pc.flag.p, line_of.p, pc.line_ptr.p, pc.line_m.p, pc.line_w.p};
  auto emit = [&](auto&& count_launch_fn, auto&& fill_launch_fn, i64 nthreads, Plan& P, i64 keyspace, bool dense,
                  i64 ncols) {
    DevBuf<i64> off(nthreads + 1);
    count_launch_fn(off.p);
    CF_CUDA(cudaMemsetAsync(off.p + nthreads, 0, sizeof(i64), stream()));
    scan_ex(off.p, nthreads + 1);
    const i64 ne = read1(off.p + nthreads);
    DevBuf<i64> key(std::max<i64>(ne, 1)), src(std::max<i64>(ne, 1));
    DevBuf<double> w(std::max<i64>(ne, 1));
    fill_launch_fn(off.p, key.p, src.p, w.p);
    build_plan(P, key, src, w, ne, keyspace, dense, ncols);
  };
  const i64 nslots = nact * ns;
  emit([&](i64* cnt) {
         k_res_emit<false><<<grid_for(nslots, 256), 256, 0, stream()>>>(nact, d, V, m.cvert.p, tg, cnt, nullptr,
                                                                          nullptr, nullptr, nullptr);
         CF_LAUNCHED();
       },
       [&](const i64* off, i64* key, i64* src, double* w) {
         k_res_emit<true><<<grid_for(nslots, 256), 256, 0, stream()>>>(nact, d, V, m.cvert.p, tg, nullptr, off, key,
                                                                         src, w);
         CF_LAUNCHED();
       },
       nslots, m.res, nt, true, 0);
  {  // self incidences (every slot once, keyed by its dof)
    DevBuf<i64> key(std::max<i64>(nslots, 1)), src(std::max<i64>(nslots, 1));
    DevBuf<double> w(std::max<i64>(nslots, 1));
    k_self_emit<<<grid_for(nslots, 256), 256, 0, stream()>>>(nact, d, V, m.cvert.p, key.p, src.p);
    CF_LAUNCHED();
    build_plan(m.self, key, src, w, nslots, nt, true, 0);
  }
  Plan* plans[3] = {&m.uu, &m.pu, &m.pp};
  for (int blk = 0; blk < 3; ++blk) {
    const i64 ni = blk == 0 ? nd : nv;
    const i64 nth = nact * ni;
    const i64 rows = blk == 0 ? nu : V, cols = blk == 2 ? V : nu;
    emit([&](i64* cnt) {
           k_jac_emit<false><<<grid_for(nth, 128), 128, 0, stream()>>>(blk, nact, d, V, m.cvert.p, tg, cnt, nullptr,
                                                                         nullptr, nullptr, nullptr);
           CF_LAUNCHED();
         },
         [&](const i64* off, i64* key, i64* src, double* w) {
           k_jac_emit<true><<<grid_for(nth, 128), 128, 0, stream()>>>(blk, nact, d, V, m.cvert.p, tg, nullptr, off,
                                                                        key, src, w);
           CF_LAUNCHED();
         },
         nth, *plans[blk], rows * cols, false, cols);
    Plan& P = *plans[blk];
    P.rows = rows;
    P.cols = cols;
    P.rptr.alloc(rows + 1);
    k_row_lb<<<grid_for(rows + 1, 256), 256, 0, stream()>>>(P.n, P.row.p, rows + 1, P.rptr.p);
    CF_LAUNCHED();
  }
  m.plans_ready = true;
  m.plan_uid = pc.uid;
}

std::shared_ptr<Csr> block_from_plan(const Plan& P, i64 roff, i64 coff, bool has_diag, const std::uint8_t* mask,
                                     const double* svals, const double* diag) {
  auto A = std::make_shared<Csr>();
  A->rows = P.rows;
  A->cols = P.cols;
  A->ptr.alloc(P.rows + 1);
  k_block_rows<false><<<grid_for(P.rows, 256), 256, 0, stream()>>>(P.rows, roff, coff, has_diag ? 1 : 0, P.rptr.p,
                                                                    P.col.p, svals, mask, diag, A->ptr.p, nullptr,
                                                                    nullptr, nullptr);
  CF_LAUNCHED();
  CF_CUDA(cudaMemsetAsync(A->ptr.p + P.rows, 0, sizeof(i64), stream()));
  scan_ex(A->ptr.p, P.rows + 1);
  A->nnz = read1(A->ptr.p + P.rows);
  A->col.alloc(std::max<i64>(A->nnz, 1));
  A->val.alloc(std::max<i64>(A->nnz, 1));
  k_block_rows<true><<<grid_for(P.rows, 256), 256, 0, stream()>>>(P.rows, roff, coff, has_diag ? 1 : 0, P.rptr.p,
                                                                   P.col.p, svals, mask, diag, nullptr, A->ptr.p,
                                                                   A->col.p, A->val.p);
  CF_LAUNCHED();
  return A;
}

void check_mesh_cs(const MeshDisc& m, const Constraints& c, const char* who) {
  if (c.mesh != &m) fail(CF_ERR_INVALID_ARGUMENT, std::string(who) + ": constraint set of another mesh");
}

}  // namespace

void mesh_assemble_residual(MeshDisc& m, const Constraints& pc, const Constraints& c, const cf_material& mat,
                            const cf_regularization& reg, const double* x, const double* pt, double* R) {
  check_mesh_cs(m, pc, "assemble_residual");
  check_mesh_cs(m, c, "assemble_residual");
  validate_material(mat);
  mesh_tables(m, mat_mu(mat), mat_lambda(mat));
  ensure_plans(m, pc);
  const int d = m.d, nv = 1 << d;
  std::vector<double> hl(size_t(m.max_level + 1));
  for (int l = 0; l <= m.max_level; ++l) hl[size_t(l)] = m.level_edge(l);
  DevBuf<double> hlev(m.max_level + 1);
  CF_CUDA(cudaMemcpyAsync(hlev.p, hl.data(), hl.size() * sizeof(double), cudaMemcpyHostToDevice, stream()));
  DevBuf<double> el(m.nact * nv * (d + 1));
  const MCoef cf = mcoef(mat, reg);
  if (d == 2)
    k_mesh_residual<2><<<grid_for(m.nact * 4, 256), 256, 0, stream()>>>(m.nact, m.cvert.p, m.clevel.p, hlev.p,
                                                                       m.tabs.p, cf, m.V, x, pt, el.p);
  else
    k_mesh_residual<3><<<grid_for(m.nact * 8, 256), 256, 0, stream()>>>(m.nact, m.cvert.p, m.clevel.p, hlev.p,
                                                                       m.tabs.p, cf, m.V, x, pt, el.p);
  CF_LAUNCHED();
  k_res_apply<<<grid_for(m.n_total(), 256), 256, 0, stream()>>>(m.n_total(), m.res.ptr.p, m.res.src.p, m.res.w.p,
                                                                el.p, c.flag.p, R);
  CF_LAUNCHED();
  CF_CUDA(cudaStreamSynchronize(stream()));  // hl (host) is read by the async copy
}

std::unique_ptr<BlockSystem> mesh_assemble_jacobian(MeshDisc& m, const Constraints& pc, const Constraints& c,
                                                    const cf_material& mat, const cf_regularization& reg,
                                                    const double* x, const double* pt) {
  check_mesh_cs(m, pc, "assemble_jacobian");
  check_mesh_cs(m, c, "assemble_jacobian");
  validate_material(mat);
  mesh_tables(m, mat_mu(mat), mat_lambda(mat));
  ensure_plans(m, pc);
  const int d = m.d, nv = 1 << d, nd = nv * d, ns = 4 + d * d;
  const i64 nact = m.nact, nu = m.n_u(), V = m.V;
  DevBuf<double> qs(nact * nv * ns), Kuu(nact * nd * nd), Kpu(nact * nv * nd), Kpp(nact * nv * nv);
  const MCoef cf = mcoef(mat, reg);
  if (d == 2) {
    k_mesh_qpstate<2><<<grid_for(nact, 128), 128, 0, stream()>>>(nact, m.cvert.p, m.clevel.p, m.tabs.p, cf, V, x, pt,
                                                                 qs.p);
    CF_LAUNCHED();
    k_mesh_elem<2><<<grid_for(nact * 16, 128), 128, 0, stream()>>>(nact, m.clevel.p, m.tabs.p, cf, qs.p, Kuu.p,
                                                                   Kpu.p, Kpp.p);
  } else {
    k_mesh_qpstate<3><<<grid_for(nact, 128), 128, 0, stream()>>>(nact, m.cvert.p, m.clevel.p, m.tabs.p, cf, V, x, pt,
                                                                 qs.p);
    CF_LAUNCHED();
    k_mesh_elem<3><<<grid_for(nact * 64, 128), 128, 0, stream()>>>(nact, m.clevel.p, m.tabs.p, cf, qs.p, Kuu.p,
                                                                   Kpu.p, Kpp.p);
  }
  CF_LAUNCHED();
  auto J = std::make_unique<BlockSystem>();
  J->d = d;
  J->nu = nu;
  J->np = V;
  const double* K[3] = {Kuu.p, Kpu.p, Kpp.p};
  const Plan* plans[3] = {&m.uu, &m.pu, &m.pp};
  std::shared_ptr<Csr>* outs[3] = {&J->uu, &J->pu, &J->pp};
  for (int blk = 0; blk < 3; ++blk) {
    const Plan& P = *plans[blk];
    DevBuf<double> sv(std::max<i64>(P.n, 1)), diag(std::max<i64>(P.rows, 1));
    k_plan_vals<<<grid_for(P.n, 256), 256, 0, stream()>>>(P.n, P.ptr.p, P.src.p, P.w.p, K[blk], sv.p);
    CF_LAUNCHED();
    const i64 roff = blk == 0 ? 0 : nu, coff = blk == 2 ? nu : 0;
    if (blk != 1) {
      k_diag<<<grid_for(P.rows, 256), 256, 0, stream()>>>(blk, P.rows, roff, d, m.self.ptr.p, m.self.src.p, c.flag.p,
                                                          K[blk], diag.p);
      CF_LAUNCHED();
    }
    *outs[blk] = block_from_plan(P, roff, coff, blk != 1, c.flag.p, sv.p, diag.p);
  }
  return J;
}

}  // namespace cfb

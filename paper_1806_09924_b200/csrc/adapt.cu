// Device adaptivity: active faces, the gradient-jump estimator, marking and
// transfer (adapt.cpp:16-118, fem.cpp:318-333, mesh.cpp:225-259), plus the predictor-corrector
// adaptive loop (adapt.cpp:122-190) orchestrated on the host around device steps.
//
// Bitwise contract with the reference (oracle_mesh.inc): faces in the reference's list order
// (active cell, axis, side) by a scan-compaction; per-face integrals with the reference's point
// evaluation; every cell's eta^2 is 0.0 + its faces' halves in face-list order (a stable sort of
// the (cell, face) contributions); the fixed-fraction marking sorts (-eta^2, id) with a stable
// radix sort and accumulates the cut sequentially, as std::sort + the loop of adapt.cpp:75-91.
#include <algorithm>
#include <cmath>

#include <cub/cub.cuh>

#include "cf_mesh.hpp"

namespace cfb {

namespace {

template <class T>
std::vector<T> dl(const T* p, i64 n) {
  std::vector<T> h(size_t(std::max<i64>(n, 0)));
  if (n > 0) {
    read_small(h.data(), p, size_t(n) * sizeof(T));
  }
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

__device__ __forceinline__ void vcoord(i64 key, i64* c) {
  const i64 msk = (i64(1) << 21) - 1;
  c[0] = key & msk;
  c[1] = (key >> 21) & msk;
  c[2] = (key >> 42) & msk;
}

__device__ __forceinline__ bool f_contains(const DevForest& F, const i64* p) {
  const i64 ext = i64(F.n0) * kUnit;
  for (int a = 0; a < F.d; ++a)
    if (p[a] < 0 || p[a] > ext) return false;
  return true;
}

// as mesh.cu's d_locate: the smallest id (coarsest: among the coarsest) active cell holding p
__device__ int f_locate(const DevForest& F, const i64* p, bool coarsest) {
  if (!f_contains(F, p)) return -1;
  const int n0 = F.n0, d = F.d;
  int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  for (int a = 0; a < d; ++a) {
    const i64 i = p[a] / kUnit;
    lo[a] = int(max(i64(0), (p[a] % kUnit == 0) ? i - 1 : i));
    hi[a] = int(min(i64(n0 - 1), i));
    lo[a] = min(lo[a], n0 - 1);
  }
  int st[136];
  int sp = 0;
  for (int k = lo[2]; k <= (d == 3 ? hi[2] : 0); ++k)
    for (int j = lo[1]; j <= hi[1]; ++j)
      for (int i = lo[0]; i <= hi[0]; ++i) st[sp++] = F.roots[i + n0 * j + (d == 3 ? n0 * n0 * k : 0)];
  int best = -1, blev = 1 << 30;
  while (sp > 0) {
    const int id = st[--sp];
    const i64 sz = kUnit >> F.level[id];
    bool in = true;
    for (int a = 0; a < d; ++a) in = in && p[a] >= F.anchor[3 * id + a] && p[a] <= F.anchor[3 * id + a] + sz;
    if (!in) continue;
    if (F.active[id]) {
      const int lv = coarsest ? F.level[id] : 0;
      if (best < 0 || lv < blev || (lv == blev && id < best)) {
        best = id;
        blev = lv;
      }
      continue;
    }
    for (int c = 0; c < (1 << d) && sp < 136; ++c)
      if (F.child[8 * id + c] >= 0) st[sp++] = F.child[8 * id + c];
  }
  return best;
}

// face slots (cell position, axis, side): neighbour id (-1 boundary), rel, reported flag
__global__ void k_faces(i64 nact, DevForest F, const int* __restrict__ cid, int* __restrict__ nb,
                        int* __restrict__ rel, i64* __restrict__ rep) {
  const int d = F.d;
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nact * d * 2) return;
  const i64 c = t / (2 * d);
  const int a = int((t / 2) % d), s = int(t % 2);
  const int id = cid[c];
  const int lev = F.level[id];
  const i64 sz = kUnit >> lev;
  i64 ctr[3] = {F.anchor[3 * id], F.anchor[3 * id + 1], F.anchor[3 * id + 2]};
  for (int b = 0; b < d; ++b) ctr[b] += sz / 2;
  ctr[a] = (s == 0) ? F.anchor[3 * id + a] - sz / 2 : F.anchor[3 * id + a] + sz + sz / 2;
  nb[t] = -1;
  rel[t] = 0;
  if (!f_contains(F, ctr)) {
    rep[t] = 1;  // boundary face
    return;
  }
  const int q = f_locate(F, ctr, true);
  const int ql = F.level[q];
  if (ql > lev || (ql == lev && q < id)) {
    rep[t] = 0;
    return;
  }
  nb[t] = q;
  rel[t] = ql < lev ? -1 : 0;
  rep[t] = 1;
}

// a field's value / gradient on an active cell at physical x (fem.cpp:269-299)
template <int D>
__device__ void eval_cell(const int* __restrict__ cv, const double* lo, double h, i64 nu,
                          const double* __restrict__ sol, const double* x, double gu[3][3]) {
  double xi[3] = {0, 0, 0};
  for (int a = 0; a < D; ++a) xi[a] = fmin(fmax((x[a] - lo[a]) / h, 0.0), 1.0);
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) gu[a][b] = 0.0;
  for (int k = 0; k < (1 << D); ++k) {
    const i64 v = cv[k];
    double gr[3];
    for (int a = 0; a < D; ++a) {
      double g = (k & (1 << a)) ? 1.0 : -1.0;
      for (int b = 0; b < D; ++b) {
        if (b == a) continue;
        g *= (k & (1 << b)) ? xi[b] : 1.0 - xi[b];
      }
      gr[a] = g;
    }
    for (int a = 0; a < D; ++a) {
      const double uva = sol[v * D + a];
      for (int b = 0; b < D; ++b) gu[a][b] += gr[b] / h * uva;
    }
  }
  (void)nu;
}

// per reported interior face: (h_F / 2) * integral of |[grad u . n]|^2 (adapt.cpp:24-51)
template <int D>
__global__ void k_face_jump(i64 nslots, const i64* __restrict__ rep, const int* __restrict__ nb, DevForest F,
                            const int* __restrict__ pos_of, const int* __restrict__ cid,
                            const int* __restrict__ cvert, double K, double unit, const double* __restrict__ hlev,
                            const double* __restrict__ fmeas, const double* __restrict__ fp,
                            const double* __restrict__ fw, i64 nu, const double* __restrict__ sol,
                            double* __restrict__ contrib) {
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nslots) return;
  contrib[t] = 0.0;
  if (!rep[t] || nb[t] < 0) return;
  const i64 c = t / (2 * D);
  const int a = int((t / 2) % D), s = int(t % 2);
  const int id = cid[c], q = nb[t];
  const int lev = F.level[id], lq = F.level[q];
  const double h = hlev[lev], hq = hlev[lq];
  double lo[3] = {0, 0, 0}, loq[3] = {0, 0, 0};
  for (int b = 0; b < D; ++b) {
    lo[b] = -K + double(F.anchor[3 * id + b]) * unit;
    loq[b] = -K + double(F.anchor[3 * q + b]) * unit;
  }
  double base[3] = {lo[0], lo[1], lo[2]};
  if (s == 1) base[a] += h;
  int span[2] = {-1, -1}, ns = 0;
  for (int b = 0; b < D; ++b)
    if (b != a) span[ns++] = b;
  const int* cva = cvert + c * (1 << D);
  const int* cvb = cvert + i64(pos_of[q]) * (1 << D);
  double jump2 = 0.0;
  for (int qq = 0; qq < (1 << (D - 1)); ++qq) {
    double x[3] = {base[0], base[1], base[2]};
    for (int k = 0; k < ns; ++k) x[span[k]] += fp[qq * (D - 1) + k] * h;
    double ga[3][3], gb[3][3];
    eval_cell<D>(cva, lo, h, nu, sol, x, ga);
    eval_cell<D>(cvb, loq, hq, nu, sol, x, gb);
    const double j0 = ga[0][a] - gb[0][a], j1 = ga[1][a] - gb[1][a], j2 = ga[2][a] - gb[2][a];
    jump2 += fw[qq] * (j0 * j0 + j1 * j1 + j2 * j2);
  }
  contrib[t] = 0.5 * h * jump2 * fmeas[lev];
}

// the two halves of every face, keyed by target cell position, in face-list order
__global__ void k_eta_emit(i64 nslots, int d, const i64* __restrict__ rep, const int* __restrict__ nb,
                           const int* __restrict__ pos_of, const double* __restrict__ contrib, i64* __restrict__ key,
                           double* __restrict__ val) {
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nslots) return;
  const bool on = rep[t] && nb[t] >= 0;
  key[2 * t] = on ? t / (2 * d) : -1;
  key[2 * t + 1] = on ? pos_of[nb[t]] : -1;
  val[2 * t] = 0.5 * contrib[t];
  val[2 * t + 1] = 0.5 * contrib[t];
}

__global__ void k_pos_of(i64 nact, const int* __restrict__ cid, int* __restrict__ pos) {
  const i64 c = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c < nact) pos[cid[c]] = int(c);
}

__global__ void k_eta_sum(i64 nact, const i64* __restrict__ ptr, const double* __restrict__ v, double* __restrict__ eta) {
  const i64 c = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= nact) return;
  double s = 0.0;
  for (i64 e = ptr[c]; e < ptr[c + 1]; ++e) s += v[e];
  eta[c] = sqrt(s);
}

__global__ void k_lb(i64 n, const i64* __restrict__ key, i64 nq, i64* __restrict__ out) {
  const i64 q = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  i64 lo = 0, hi = n;
  while (lo < hi) {
    const i64 mid = (lo + hi) >> 1;
    if (key[mid] < q) lo = mid + 1; else hi = mid;
  }
  out[q] = lo;
}

// band clause of mark_cells (adapt.cpp:63-72)
__global__ void k_mark_band(i64 nact, int d, const int* __restrict__ clevel, const int* __restrict__ cvert,
                            const double* __restrict__ hlev, i64 nu, const double* __restrict__ sol, double thr,
                            double h_target, int max_level, std::uint8_t* __restrict__ mark) {
  const i64 c = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= nact) return;
  const int lev = clevel[c];
  std::uint8_t m = 0;
  if (lev < max_level && !(hlev[lev] <= h_target * (1.0 + 1e-9))) {
    double pm = 1e300;
    for (int k = 0; k < (1 << d); ++k) pm = fmin(pm, sol[nu + cvert[c * (1 << d) + k]]);
    m = pm < thr ? 1 : 0;
  }
  mark[c] = m;
}

__global__ void k_e2(i64 n, const double* __restrict__ eta, unsigned long long* __restrict__ key,
                     double* __restrict__ e2, int* __restrict__ pos) {
  const i64 c = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const double v = eta[c] * eta[c];
  e2[c] = v;
  key[c] = __double_as_longlong(v);  // non-negative: the bit pattern orders like the value
  pos[c] = int(c);
}

// the fixed-fraction cut, sequential as adapt.cpp:75-91 (total summed in active-cell order)
__global__ void k_mark_cut(i64 n, const double* __restrict__ e2, const int* __restrict__ spos,
                           const int* __restrict__ clevel, double theta, int max_level, std::uint8_t* __restrict__ mark) {
  double total = 0.0;
  for (i64 c = 0; c < n; ++c) total += e2[c];
  double acc = 0.0;
  for (i64 i = 0; i < n; ++i) {
    if (total <= 0.0 || acc >= theta * total) break;
    const int c = spos[i];
    acc += e2[c];
    if (clevel[c] < max_level && e2[c] > 0.0) mark[c] = 1;
  }
}

// transfer (fem.cpp:318-333): each new vertex evaluates the old field on the old active cell
// (smallest id) holding it
__global__ void k_transfer(i64 Vn, int d, double K, double unit, const i64* __restrict__ nkey, DevForest Fo,
                           const int* __restrict__ opos, const int* __restrict__ ocvert,
                           const double* __restrict__ ohlev, i64 Vo, const double* __restrict__ ov,
                           double* __restrict__ nv, int* __restrict__ bad) {
  const i64 v = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= Vn) return;
  i64 p[3];
  vcoord(nkey[v], p);
  const int cell = f_locate(Fo, p, false);
  if (cell < 0) {
    *bad = 1;
    return;
  }
  const double h = ohlev[Fo.level[cell]];
  double x[3], xi[3] = {0, 0, 0};
  for (int a = 0; a < d; ++a) {
    x[a] = -K + double(p[a]) * unit;
    const double lo = -K + double(Fo.anchor[3 * cell + a]) * unit;
    xi[a] = fmin(fmax((x[a] - lo) / h, 0.0), 1.0);
  }
  const int* cv = ocvert + i64(opos[cell]) * (1 << d);
  const i64 nuo = i64(d) * Vo;
  double u[3] = {0, 0, 0}, ph = 0.0;
  for (int k = 0; k < (1 << d); ++k) {
    double s = 1.0;
    for (int a = 0; a < d; ++a) s *= (k & (1 << a)) ? xi[a] : 1.0 - xi[a];
    const i64 w = cv[k];
    ph += s * ov[nuo + w];
    for (int a = 0; a < d; ++a) u[a] += s * ov[w * d + a];
  }
  for (int a = 0; a < d; ++a) nv[v * d + a] = u[a];
  nv[i64(d) * Vn + v] = ph;
}

__global__ void k_mask_band_eta(i64 nact, int d, const int* __restrict__ clevel, const int* __restrict__ cvert,
                                const double* __restrict__ hlev, i64 nu, const double* __restrict__ sol, double thr,
                                double h_target, double* __restrict__ eta) {
  const i64 c = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= nact) return;
  if (hlev[clevel[c]] <= h_target * (1.0 + 1e-9)) return;
  double pm = 1e300;
  for (int k = 0; k < (1 << d); ++k) pm = fmin(pm, sol[nu + cvert[c * (1 << d) + k]]);
  if (pm < thr) eta[c] = 0.0;
}

struct HLev {
  DevBuf<double> h, fm;
  explicit HLev(const MeshDisc& m) {
    std::vector<double> hh(size_t(m.max_level + 1)), f(size_t(m.max_level + 1));
    for (int l = 0; l <= m.max_level; ++l) {
      hh[size_t(l)] = m.level_edge(l);
      f[size_t(l)] = std::pow(hh[size_t(l)], m.d - 1);
    }
    h.alloc(i64(hh.size()));
    fm.alloc(i64(f.size()));
    CF_CUDA(cudaMemcpyAsync(h.p, hh.data(), hh.size() * sizeof(double), cudaMemcpyHostToDevice, stream()));
    CF_CUDA(cudaMemcpyAsync(fm.p, f.data(), f.size() * sizeof(double), cudaMemcpyHostToDevice, stream()));
    CF_CUDA(cudaStreamSynchronize(stream()));
  }
};

struct FaceSlots {
  i64 n = 0;
  DevBuf<int> nb, rel;
  DevBuf<i64> rep;
};

FaceSlots face_slots(MeshDisc& m) {
  FaceSlots f;
  f.n = m.nact * m.d * 2;
  f.nb.alloc(f.n);
  f.rel.alloc(f.n);
  f.rep.alloc(f.n + 1);
  k_faces<<<grid_for(f.n, 128), 128, 0, stream()>>>(m.nact, m.forest(), m.cid.p, f.nb.p, f.rel.p, f.rep.p);
  CF_LAUNCHED();
  return f;
}

}  // namespace

std::vector<int> mesh_faces(MeshDisc& m) {
  FaceSlots f = face_slots(m);
  std::vector<i64> rep = dl(f.rep.p, f.n);
  std::vector<int> nb = dl(f.nb.p, f.n), rel = dl(f.rel.p, f.n);
  std::vector<int> out;
  for (i64 t = 0; t < f.n; ++t) {
    if (!rep[size_t(t)]) continue;
    out.push_back(m.active[size_t(t / (2 * m.d))]);
    out.push_back(int((t / 2) % m.d));
    out.push_back(int(t % 2));
    out.push_back(nb[size_t(t)]);
    out.push_back(rel[size_t(t)]);
  }
  return out;
}

void mesh_jump_estimator(MeshDisc& m, const double* sol, double* eta) {  // adapt.cpp:16-55
  const int d = m.d;
  FaceSlots f = face_slots(m);
  HLev hl(m);
  DevBuf<int> pos(i64(m.cells.size()));
  k_pos_of<<<grid_for(m.nact, 256), 256, 0, stream()>>>(m.nact, m.cid.p, pos.p);
  CF_LAUNCHED();
  // face rule = cell_rule(d - 1, 2) (fem.cpp:53-74)
  const double a1 = 1.0 / std::sqrt(3.0), x1[2] = {-a1, a1};
  double fp[4 * 2] = {0}, fw[4];
  const int nq = 1 << (d - 1);
  for (int q = 0; q < nq; ++q) {
    int rem = q;
    double wt = 1.0;
    for (int a = 0; a < d - 1; ++a) {
      const int i = rem % 2;
      rem /= 2;
      fp[q * (d - 1) + a] = 0.5 * (x1[i] + 1.0);
      wt *= 0.5 * 1.0;
    }
    fw[q] = wt;
  }
  DevBuf<double> dfp(8), dfw(4), contrib(std::max<i64>(f.n, 1));
  CF_CUDA(cudaMemcpyAsync(dfp.p, fp, sizeof(fp), cudaMemcpyHostToDevice, stream()));
  CF_CUDA(cudaMemcpyAsync(dfw.p, fw, sizeof(fw), cudaMemcpyHostToDevice, stream()));
  if (d == 2)
    k_face_jump<2><<<grid_for(f.n, 128), 128, 0, stream()>>>(f.n, f.rep.p, f.nb.p, m.forest(), pos.p, m.cid.p,
                                                             m.cvert.p, m.K, m.unit, hl.h.p, hl.fm.p, dfp.p, dfw.p,
                                                             m.n_u(), sol, contrib.p);
  else
    k_face_jump<3><<<grid_for(f.n, 128), 128, 0, stream()>>>(f.n, f.rep.p, f.nb.p, m.forest(), pos.p, m.cid.p,
                                                             m.cvert.p, m.K, m.unit, hl.h.p, hl.fm.p, dfp.p, dfw.p,
                                                             m.n_u(), sol, contrib.p);
  CF_LAUNCHED();
  const i64 ne = 2 * f.n;
  DevBuf<i64> key(std::max<i64>(ne, 1)), key_s(std::max<i64>(ne, 1));
  DevBuf<double> val(std::max<i64>(ne, 1)), val_s(std::max<i64>(ne, 1));
  k_eta_emit<<<grid_for(f.n, 256), 256, 0, stream()>>>(f.n, d, f.rep.p, f.nb.p, pos.p, contrib.p, key.p, val.p);
  CF_LAUNCHED();
  if (ne > 0) {  // stable: every cell's halves stay in face-list order
    size_t bytes = 0;
    CF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key.p, key_s.p, val.p, val_s.p, ne, 0, 64, stream()));
    DevBuf<unsigned char> tmp{i64(bytes)};
    CF_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, key.p, key_s.p, val.p, val_s.p, ne, 0, 64, stream()));
    count_launch();
  }
  // segment pointers per cell position by lower bound (the -1 keys of boundary slots sort first)
  DevBuf<i64> ptr(m.nact + 1);
  k_lb<<<grid_for(m.nact + 1, 256), 256, 0, stream()>>>(ne, key_s.p, m.nact + 1, ptr.p);
  CF_LAUNCHED();
  k_eta_sum<<<grid_for(m.nact, 256), 256, 0, stream()>>>(m.nact, ptr.p, val_s.p, eta);
  CF_LAUNCHED();
  CF_CUDA(cudaStreamSynchronize(stream()));
}

// adapt.cpp:158-170: band cells above the target leave the fixed-fraction ranking
void mesh_mask_band_eta(MeshDisc& m, const double* sol, double* eta, const cf_refinement_policy& pol) {
  HLev hl(m);
  k_mask_band_eta<<<grid_for(m.nact, 256), 256, 0, stream()>>>(m.nact, m.d, m.clevel.p, m.cvert.p, hl.h.p, m.n_u(),
                                                               sol, pol.phi_threshold, pol.h_target, eta);
  CF_LAUNCHED();
}

std::vector<int> mesh_mark_cells(MeshDisc& m, const double* sol, const double* eta, const cf_refinement_policy& pol) {
  if (!(pol.phi_threshold > 0.0 && pol.phi_threshold < 1.0))
    fail(CF_ERR_INVALID_ARGUMENT, "RefinementPolicy: phi_threshold must be in (0,1)");
  if (!(pol.theta >= 0.0 && pol.theta <= 1.0))
    fail(CF_ERR_INVALID_ARGUMENT, "RefinementPolicy: theta must be in [0,1]");
  HLev hl(m);
  DevBuf<std::uint8_t> mark(std::max<i64>(m.nact, 1));
  k_mark_band<<<grid_for(m.nact, 256), 256, 0, stream()>>>(m.nact, m.d, m.clevel.p, m.cvert.p, hl.h.p, m.n_u(), sol,
                                                           pol.phi_threshold, pol.h_target, pol.max_level, mark.p);
  CF_LAUNCHED();
  if (pol.estimator && pol.theta > 0.0 && eta && m.nact > 0) {
    const i64 n = m.nact;
    DevBuf<unsigned long long> key(n), key_s(n);
    DevBuf<double> e2(n);
    DevBuf<int> pos(n), pos_s(n);
    k_e2<<<grid_for(n, 256), 256, 0, stream()>>>(n, eta, key.p, e2.p, pos.p);
    CF_LAUNCHED();
    size_t bytes = 0;
    CF_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, key.p, key_s.p, pos.p, pos_s.p, n, 0, 64,
                                                      stream()));
    DevBuf<unsigned char> tmp{i64(bytes)};
    CF_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp.p, bytes, key.p, key_s.p, pos.p, pos_s.p, n, 0, 64,
                                                      stream()));
    count_launch();
    k_mark_cut<<<1, 1, 0, stream()>>>(n, e2.p, pos_s.p, m.clevel.p, pol.theta, pol.max_level, mark.p);
    CF_LAUNCHED();
  }
  std::vector<std::uint8_t> mk = dl(mark.p, m.nact);
  std::vector<int> out;
  for (i64 c = 0; c < m.nact; ++c)
    if (mk[size_t(c)]) out.push_back(m.active[size_t(c)]);
  return out;
}

void mesh_transfer(MeshDisc& om, const double* ov, MeshDisc& nm, double* nvec) {
  if (om.d != nm.d || om.n0 != nm.n0 || om.K != nm.K) fail(CF_ERR_INVALID_ARGUMENT, "transfer: meshes are unrelated");
  HLev hl(om);
  DevBuf<int> pos(i64(om.cells.size())), bad(1);
  bad.zero();
  k_pos_of<<<grid_for(om.nact, 256), 256, 0, stream()>>>(om.nact, om.cid.p, pos.p);
  CF_LAUNCHED();
  k_transfer<<<grid_for(nm.V, 128), 128, 0, stream()>>>(nm.V, nm.d, nm.K, nm.unit, nm.vkey.p, om.forest(), pos.p,
                                                        om.cvert.p, hl.h.p, om.V, ov, nvec, bad.p);
  CF_LAUNCHED();
  if (dl(bad.p, 1)[0]) fail(CF_ERR_INVALID_ARGUMENT, "transfer: meshes are unrelated");
}

}  // namespace cfb

// General (adaptive) meshes on the device — SURVEY §8f row 2 (element-table assembly with
// hanging-node constraints, device DofMap / build_constraints) and row 3 (estimator, marking,
// transfer; adapt.cu).  See cf_mesh.hpp for the split between host forest and device work.
//
// Assembly on a general mesh reproduces the reference's condensation and its triplet sums bit
// for bit with two precomputed plans per mesh:
//  * residual plan: for every dof, the ordered list of (element-residual entry, weight) that
//    Scatter::vector_add (model.cpp:74-80) adds into it, in the reference's cell / corner /
//    component / line-entry order;
//  * Jacobian plans: for every (row, column) of M_uu, M_phiu, M_phiphi, the ordered list of
//    (element-matrix entry, weight product) that Scatter::matrix_add (model.cpp:82-101) emits
//    for it, i.e. Eigen's setFromTriplets duplicate sum in insertion order, computed once by a
//    stable radix sort of the emitted triplet keys.
// Per Newton iteration only the element kernels run, then one pass sums each plan slot.  The
// active set changes no weight: active phi dofs simply stop being targets (their rows and
// columns are dropped, their rows keep the summed element diagonal, model.cpp:295-311).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>

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
std::vector<T> to_host(const T* p, i64 n) {
  std::vector<T> h(size_t(std::max<i64>(n, 0)));
  if (n > 0) {
    read_small(h.data(), p, size_t(n) * sizeof(T));
  }
  return h;
}

template <class T>
void to_dev(DevBuf<T>& b, const std::vector<T>& h) {
  b.alloc(i64(h.size()));
  if (!h.empty()) CF_CUDA(cudaMemcpyAsync(b.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, stream()));
}

// exclusive scan in place over n+1 entries (the last input entry is ignored; it receives the total)
template <class T>
void scan_ex(T* data, i64 n1) {
  size_t bytes = 0;
  CF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, data, data, n1, stream()));
  DevBuf<unsigned char> tmp{i64(bytes)};
  CF_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, data, data, n1, stream()));
  count_launch();
}

// ------------------------------------------------------------------ forest (host, mesh.cpp)
bool h_contains(const MeshDisc& m, const i64* p) {
  for (int a = 0; a < m.d; ++a)
    if (p[a] < 0 || p[a] > m.extent()) return false;
  return true;
}

// active cells whose closed box holds p, ascending (mesh.cpp:101-141)
std::vector<int> h_cells_at(const MeshDisc& m, const i64* p) {
  std::vector<int> out;
  if (!h_contains(m, p)) return out;
  const int n0 = m.n0, d = m.d;
  int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  for (int a = 0; a < d; ++a) {
    const i64 i = p[a] / kUnit;
    lo[a] = int(std::max<i64>(0, (p[a] % kUnit == 0) ? i - 1 : i));
    hi[a] = int(std::min<i64>(n0 - 1, i));
    lo[a] = std::min(lo[a], n0 - 1);
  }
  std::vector<int> st;
  for (int k = lo[2]; k <= (d == 3 ? hi[2] : 0); ++k)
    for (int j = lo[1]; j <= hi[1]; ++j)
      for (int i = lo[0]; i <= hi[0]; ++i) st.push_back(m.roots[i + n0 * j + (d == 3 ? n0 * n0 * k : 0)]);
  while (!st.empty()) {
    const int id = st.back();
    st.pop_back();
    const HostCell& c = m.cells[id];
    bool in = true;
    for (int a = 0; a < d; ++a) in = in && p[a] >= c.anchor[a] && p[a] <= c.anchor[a] + c.isize();
    if (!in) continue;
    if (c.active) {
      out.push_back(id);
      continue;
    }
    for (int ch : c.child)
      if (ch >= 0) st.push_back(ch);
  }
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
  return out;
}

void h_split(MeshDisc& m, int id);

// mesh.cpp:178-201: before a level-l cell splits, every face neighbour reaches level >= l
void h_ensure_neighbor_level(MeshDisc& m, int id) {
  for (;;) {
    const HostCell c = m.cells[id];
    bool changed = false;
    for (int a = 0; a < m.d && !changed; ++a)
      for (int s = 0; s < 2 && !changed; ++s) {
        i64 ctr[3] = {c.anchor[0], c.anchor[1], c.anchor[2]};
        for (int b = 0; b < m.d; ++b) ctr[b] += c.isize() / 2;
        ctr[a] = (s == 0) ? c.anchor[a] - c.isize() / 2 : c.anchor[a] + c.isize() + c.isize() / 2;
        if (!h_contains(m, ctr)) continue;
        for (int nb : h_cells_at(m, ctr))
          if (m.cells[nb].level < c.level) {
            h_split(m, nb);
            changed = true;
            break;
          }
      }
    if (!changed) return;
  }
}

void h_split(MeshDisc& m, int id) {  // mesh.cpp:152-175
  if (!m.cells[id].active) return;
  if (m.cells[id].level + 1 > kLevelBits)
    fail(CF_ERR_NUMERICAL, "Mesh: refinement depth exceeds integer coordinate resolution");
  h_ensure_neighbor_level(m, id);
  const i64 half = m.cells[id].isize() / 2;
  m.cells[id].active = false;
  for (int k = 0; k < (1 << m.d); ++k) {
    HostCell ch;
    ch.level = m.cells[id].level + 1;
    for (int a = 0; a < 3; ++a) ch.anchor[a] = m.cells[id].anchor[a];
    for (int a = 0; a < m.d; ++a)
      if (k & (1 << a)) ch.anchor[a] += half;
    ch.parent = id;
    m.cells[id].child[k] = int(m.cells.size());
    m.cells.push_back(ch);
  }
  ++m.revision;
}

// ------------------------------------------------------------------ device forest / DofMap
__device__ __forceinline__ i64 pack_key(i64 x, i64 y, i64 z) { return x | (y << 21) | (z << 42); }

__device__ __forceinline__ bool d_contains(const DevForest& F, const i64* p) {
  const i64 ext = i64(F.n0) * kUnit;
  for (int a = 0; a < F.d; ++a)
    if (p[a] < 0 || p[a] > ext) return false;
  return true;
}

// smallest id among the active cells whose closed box holds p (coarsest = false), or among the
// coarsest of them (coarsest = true: the smallest level first, then the smallest id); -1 outside
__device__ int d_locate(const DevForest& F, const i64* p, bool coarsest) {
  if (!d_contains(F, p)) return -1;
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

__device__ __forceinline__ i64 d_vertex_index(const i64* __restrict__ keys, i64 V, i64 k) {
  i64 lo = 0, hi = V;
  while (lo < hi) {
    const i64 mid = (lo + hi) >> 1;
    if (keys[mid] < k) lo = mid + 1; else hi = mid;
  }
  return (lo < V && keys[lo] == k) ? lo : -1;
}

__global__ void k_corner_keys(i64 nact, int d, const int* __restrict__ cid, DevForest F, i64* __restrict__ keys) {
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  const int nv = 1 << d;
  if (t >= nact * nv) return;
  const i64 c = t / nv;
  const int k = int(t % nv);
  const int id = cid[c];
  const i64 sz = kUnit >> F.level[id];
  i64 p[3] = {F.anchor[3 * id], F.anchor[3 * id + 1], F.anchor[3 * id + 2]};
  for (int a = 0; a < d; ++a)
    if (k & (1 << a)) p[a] += sz;
  keys[t] = pack_key(p[0], p[1], p[2]);
}

__global__ void k_cell_vertices(i64 nact, int d, const int* __restrict__ cid, DevForest F,
                                const i64* __restrict__ vkey, i64 V, int* __restrict__ cvert,
                                int* __restrict__ clevel) {
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  const int nv = 1 << d;
  if (t >= nact * nv) return;
  const i64 c = t / nv;
  const int k = int(t % nv);
  const int id = cid[c];
  const i64 sz = kUnit >> F.level[id];
  i64 p[3] = {F.anchor[3 * id], F.anchor[3 * id + 1], F.anchor[3 * id + 2]};
  for (int a = 0; a < d; ++a)
    if (k & (1 << a)) p[a] += sz;
  cvert[t] = int(d_vertex_index(vkey, V, pack_key(p[0], p[1], p[2])));
  if (k == 0) clevel[c] = F.level[id];
}

void upload(MeshDisc& m) {
  m.active.clear();
  for (int i = 0; i < int(m.cells.size()); ++i)
    if (m.cells[i].active) m.active.push_back(i);
  m.max_level = 0;
  for (int id : m.active) m.max_level = std::max(m.max_level, m.cells[id].level);
  const i64 nc = i64(m.cells.size());
  std::vector<int> lev(nc), ch(nc * 8);
  std::vector<i64> anc(nc * 3);
  std::vector<std::uint8_t> act(nc);
  for (i64 i = 0; i < nc; ++i) {
    const HostCell& c = m.cells[i];
    lev[i] = c.level;
    act[i] = c.active;
    for (int a = 0; a < 3; ++a) anc[3 * i + a] = c.anchor[a];
    for (int k = 0; k < 8; ++k) ch[8 * i + k] = c.child[k];
  }
  to_dev(m.t_level, lev);
  to_dev(m.t_child, ch);
  to_dev(m.t_anchor, anc);
  to_dev(m.t_active, act);
  to_dev(m.t_roots, m.roots);
  to_dev(m.cid, m.active);
  m.nact = i64(m.active.size());
  const int nv = 1 << m.d;
  const i64 nk = m.nact * nv;
  // DofMap (fem.cpp:98-116): sorted unique packed corner keys
  DevBuf<i64> keys(nk), sorted(nk);
  k_corner_keys<<<grid_for(nk, 256), 256, 0, stream()>>>(m.nact, m.d, m.cid.p, m.forest(), keys.p);
  CF_LAUNCHED();
  {
    size_t bytes = 0;
    CF_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, keys.p, sorted.p, nk, 0, 63, stream()));
    DevBuf<unsigned char> tmp{i64(bytes)};
    CF_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, bytes, keys.p, sorted.p, nk, 0, 63, stream()));
    count_launch();
  }
  DevBuf<i64> nsel(1);
  {
    size_t bytes = 0;
    CF_CUDA(cub::DeviceSelect::Unique(nullptr, bytes, sorted.p, keys.p, nsel.p, nk, stream()));
    DevBuf<unsigned char> tmp{i64(bytes)};
    CF_CUDA(cub::DeviceSelect::Unique(tmp.p, bytes, sorted.p, keys.p, nsel.p, nk, stream()));
    count_launch();
  }
  m.V = read1(nsel.p);
  m.vkey.alloc(m.V);
  CF_CUDA(cudaMemcpyAsync(m.vkey.p, keys.p, size_t(m.V) * sizeof(i64), cudaMemcpyDeviceToDevice, stream()));
  m.cvert.alloc(nk);
  m.clevel.alloc(m.nact);
  k_cell_vertices<<<grid_for(nk, 256), 256, 0, stream()>>>(m.nact, m.d, m.cid.p, m.forest(), m.vkey.p, m.V,
                                                           m.cvert.p, m.clevel.p);
  CF_LAUNCHED();
  m.plans_ready = false;
  m.tab_mu = m.tab_lam = -1.0;
  m.base_cache.reset();
}

// ------------------------------------------------------------------ constraints (fem.cpp:189-267)
__device__ __forceinline__ void vcoord(i64 key, i64* c) {
  const i64 msk = (i64(1) << 21) - 1;
  c[0] = key & msk;
  c[1] = (key >> 21) & msk;
  c[2] = (key >> 42) & msk;
}

__global__ void k_mesh_dirichlet(i64 V, int d, i64 ext, int clamp, const i64* __restrict__ vkey,
                                 std::uint8_t* __restrict__ flag) {
  const i64 v = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= V) return;
  i64 c[3];
  vcoord(vkey[v], c);
  bool bnd = false;
  for (int a = 0; a < d; ++a) bnd = bnd || c[a] == 0 || c[a] == ext;
  for (int a = 0; a < d; ++a) flag[v * d + a] = (clamp && bnd) ? 1 : 0;
  flag[i64(d) * V + v] = 0;
}

// hanging vertex v: the coarsest active cell (first found among equals) that holds one of the
// 2^d diagonal probes around v without having v as a corner hosts it; its Q1 shape values at v
// with |value| >= 1e-12 weight the host corners (fem.cpp:207-238).  Up to 2^d entries.
__global__ void k_mesh_hanging(i64 V, DevForest F, const i64* __restrict__ vkey, int* __restrict__ hn,
                               int* __restrict__ hm, double* __restrict__ hw) {
  const i64 v = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= V) return;
  const int d = F.d, nv = 1 << d;
  i64 p[3];
  vcoord(vkey[v], p);
  int host = -1;
  for (int k = 0; k < nv; ++k) {
    i64 pr[3] = {p[0], p[1], p[2]};
    for (int a = 0; a < d; ++a) pr[a] += (k & (1 << a)) ? 1 : -1;
    if (!d_contains(F, pr)) continue;
    const int c = d_locate(F, pr, false);
    if (c < 0) continue;
    const i64 sz = kUnit >> F.level[c];
    bool corner = true;
    for (int a = 0; a < d; ++a) corner = corner && (p[a] == F.anchor[3 * c + a] || p[a] == F.anchor[3 * c + a] + sz);
    if (!corner && (host < 0 || F.level[c] < F.level[host])) host = c;
  }
  int n = 0;
  if (host >= 0) {
    const i64 sz = kUnit >> F.level[host];
    double xi[3] = {0, 0, 0};
    for (int a = 0; a < d; ++a) xi[a] = double(p[a] - F.anchor[3 * host + a]) / double(sz);
    for (int k = 0; k < nv; ++k) {
      double s = 1.0;
      for (int a = 0; a < d; ++a) s *= (k & (1 << a)) ? xi[a] : 1.0 - xi[a];
      if (fabs(s) < 1e-12) continue;
      i64 q[3] = {F.anchor[3 * host], F.anchor[3 * host + 1], F.anchor[3 * host + 2]};
      for (int a = 0; a < d; ++a)
        if (k & (1 << a)) q[a] += sz;
      hm[v * 8 + n] = int(d_vertex_index(vkey, V, pack_key(q[0], q[1], q[2])));
      hw[v * 8 + n] = s;
      ++n;
    }
  }
  hn[v] = n;
}

// Closure (fem.cpp:151-184) of the lines with entries, on the host: they are the hanging dofs
// only.  Lines are closed in ascending dof order until no line changes; hanging weights are
// dyadic, so every closed weight is exact in any order (see oracle_mesh.inc).
struct HLine {
  std::vector<std::pair<i64, double>> e;
  double inhom = 0.0;
  bool entries = false;
};

void close_lines(std::map<i64, HLine>& L, const std::vector<std::uint8_t>& flag, const std::vector<double>& inh) {
  bool changed = true;
  int rounds = 0;
  while (changed) {
    if (++rounds > 32) fail(CF_ERR_NUMERICAL, "ConstraintSet: constraint graph has a cycle");
    changed = false;
    for (auto& [dof, line] : L) {
      HLine next;
      next.inhom = line.inhom;
      next.entries = true;
      bool touched = false;
      for (auto& [mm, w] : line.e) {
        if (!flag[size_t(mm)]) {
          next.e.emplace_back(mm, w);
          continue;
        }
        touched = true;
        auto it = L.find(mm);
        if (it == L.end()) {  // entry-free line (Dirichlet, active set)
          next.inhom += w * inh[size_t(mm)];
        } else {
          next.inhom += w * it->second.inhom;
          for (auto& [m2, w2] : it->second.e) next.e.emplace_back(m2, w * w2);
        }
      }
      if (touched) {
        std::sort(next.e.begin(), next.e.end());
        HLine merged;
        merged.inhom = next.inhom;
        merged.entries = true;
        for (auto& [mm, w] : next.e) {
          if (!merged.e.empty() && merged.e.back().first == mm)
            merged.e.back().second += w;
          else
            merged.e.emplace_back(mm, w);
        }
        line = std::move(merged);
        changed = true;
      }
    }
  }
}

__global__ void k_apply_active_dofs(i64 n, const i64* __restrict__ dofs, const double* __restrict__ vals, i64 nt,
                                    std::uint8_t* __restrict__ flag, double* __restrict__ inh, int* __restrict__ bad) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const i64 dof = dofs[i];
  if (dof < 0 || dof >= nt) {
    *bad = 1;
    return;
  }
  if (flag[dof] == 1) return;  // already constrained (Dirichlet / hanging priority)
  flag[dof] = 2;               // active (normalised to 1 after all are applied)
  inh[dof] = vals[i];
}

__global__ void k_flags_one(i64 n, std::uint8_t* f) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n && f[i]) f[i] = 1;
}

// full lines: the base line's entries whose master is constrained in the full set (the active
// phi dofs) are dropped, each adding weight * inhomogeneity in entry order
__global__ void k_full_lines_count(i64 nl, const i64* __restrict__ ptr, const int* __restrict__ m,
                                   const std::uint8_t* __restrict__ flag, i64* __restrict__ cnt) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nl) return;
  i64 c = 0;
  for (i64 k = ptr[i]; k < ptr[i + 1]; ++k) c += flag[m[k]] ? 0 : 1;
  cnt[i] = c;
}

__global__ void k_full_lines_fill(i64 nl, const int* __restrict__ ldof, const i64* __restrict__ ptr,
                                  const int* __restrict__ m, const double* __restrict__ w,
                                  const double* __restrict__ binh, const std::uint8_t* __restrict__ flag,
                                  const i64* __restrict__ optr, int* __restrict__ om, double* __restrict__ ow,
                                  double* __restrict__ inh) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nl) return;
  const int dof = ldof[i];
  double g = binh[dof];
  i64 o = optr[i];
  for (i64 k = ptr[i]; k < ptr[i + 1]; ++k) {
    if (flag[m[k]]) {
      g += w[k] * inh[m[k]];
    } else {
      om[o] = m[k];
      ow[o] = w[k];
      ++o;
    }
  }
  inh[dof] = g;
}

__global__ void k_distribute_lines(i64 nl, const int* __restrict__ ldof, const i64* __restrict__ ptr,
                                   const int* __restrict__ m, const double* __restrict__ w,
                                   const double* __restrict__ inh, double* __restrict__ v, int homogeneous) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nl) return;
  double val = homogeneous ? 0.0 : inh[ldof[i]];
  for (i64 k = ptr[i]; k < ptr[i + 1]; ++k) val += w[k] * v[m[k]];
  v[ldof[i]] = val;
}

}  // namespace

// ------------------------------------------------------------------ public: forest
MeshDisc* mesh_create(int d, double K, int n0) {
  if (d != 2 && d != 3) fail(CF_ERR_INVALID_ARGUMENT, "DomainSpec: dimension must be 2 or 3");
  if (!(K > 0.0)) fail(CF_ERR_INVALID_ARGUMENT, "DomainSpec: half_width must be positive");
  if (n0 < 1 || n0 > 16) fail(CF_ERR_INVALID_ARGUMENT, "DomainSpec: initial_cells_per_side must be in [1,16]");
  auto* m = new MeshDisc;
  m->d = d;
  m->K = K;
  m->n0 = n0;
  m->unit = 2.0 * K / (n0 * double(kUnit));
  const int nz = (d == 3) ? n0 : 1;
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < n0; ++j)
      for (int i = 0; i < n0; ++i) {
        HostCell c;
        c.anchor[0] = i * kUnit;
        c.anchor[1] = j * kUnit;
        c.anchor[2] = i64(k) * kUnit;
        m->roots.push_back(int(m->cells.size()));
        m->cells.push_back(c);
      }
  upload(*m);
  return m;
}

std::unique_ptr<MeshDisc> mesh_copy(const MeshDisc& src) {
  auto m = std::make_unique<MeshDisc>();
  m->d = src.d;
  m->n0 = src.n0;
  m->K = src.K;
  m->unit = src.unit;
  m->cells = src.cells;
  m->roots = src.roots;
  m->revision = src.revision;
  upload(*m);
  return m;
}

void mesh_refine(MeshDisc& m, std::vector<int> ids) {  // mesh.cpp:203-215
  std::sort(ids.begin(), ids.end());
  ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
  for (int id : ids) {
    if (id < 0 || id >= int(m.cells.size())) fail(CF_ERR_INVALID_ARGUMENT, "refine: unknown cell id");
    if (!m.cells[id].active) fail(CF_ERR_INVALID_ARGUMENT, "refine: cell is not active");
  }
  for (int id : ids) h_split(m, id);
  upload(m);
}

void mesh_uniform_refine(MeshDisc& m, int times) {  // mesh.cpp:217-223
  if (times < 0) fail(CF_ERR_INVALID_ARGUMENT, "uniform_refine: times must be >= 0");
  for (int t = 0; t < times; ++t) {
    std::vector<int> all;
    for (int i = 0; i < int(m.cells.size()); ++i)
      if (m.cells[i].active) all.push_back(i);
    for (int id : all) h_split(m, id);
  }
  upload(m);
}

int mesh_find_cell(const MeshDisc& m, const double* x) {
  i64 p[3] = {0, 0, 0};
  for (int a = 0; a < m.d; ++a) p[a] = std::llround((x[a] + m.K) / m.unit);
  const std::vector<int> cs = h_cells_at(m, p);
  return cs.empty() ? -1 : cs.front();
}

// ------------------------------------------------------------------ public: constraints
std::unique_ptr<Constraints> mesh_build_constraints(MeshDisc& m, bool clamp, i64 n_active, const i64* dofs_dev,
                                                    const double* vals_dev) {
  static std::uint64_t next_uid = 0;
  auto c = std::make_unique<Constraints>();
  c->mesh = &m;
  c->uid = ++next_uid;
  const i64 V = m.V, nt = m.n_total(), nu = m.n_u();
  const int d = m.d;
  c->flag.alloc(nt);
  c->inhom.alloc(nt);
  c->inhom.zero();
  // Dirichlet lines first, then the hanging lines of the dofs they leave free, then the active
  // set on the dofs still free (fem.cpp:194-263)
  k_mesh_dirichlet<<<grid_for(V, 256), 256, 0, stream()>>>(V, d, m.extent(), clamp ? 1 : 0, m.vkey.p, c->flag.p);
  CF_LAUNCHED();
  DevBuf<int> hn(V), hm(V * 8);
  DevBuf<double> hw(V * 8);
  k_mesh_hanging<<<grid_for(V, 128), 128, 0, stream()>>>(V, m.forest(), m.vkey.p, hn.p, hm.p, hw.p);
  CF_LAUNCHED();
  const std::vector<std::uint8_t> dir = to_host(c->flag.p, nt);
  const std::vector<int> hnh = to_host(hn.p, V), hmh = to_host(hm.p, V * 8);
  const std::vector<double> hwh = to_host(hw.p, V * 8);
  std::map<i64, HLine> L;
  std::vector<std::uint8_t> fl = dir;
  for (int comp = 0; comp <= d; ++comp)
    for (i64 v = 0; v < V; ++v) {
      if (hnh[size_t(v)] == 0) continue;
      const i64 dof = comp < d ? v * d + comp : nu + v;
      if (dir[size_t(dof)]) continue;  // Dirichlet priority
      HLine l;
      l.entries = true;
      for (int j = 0; j < hnh[size_t(v)]; ++j) {
        const i64 mv = hmh[size_t(v * 8 + j)];
        l.e.emplace_back(comp < d ? mv * d + comp : nu + mv, hwh[size_t(v * 8 + j)]);
      }
      L[dof] = std::move(l);
      fl[size_t(dof)] = 1;
    }
  CF_CUDA(cudaMemcpyAsync(c->flag.p, fl.data(), size_t(nt), cudaMemcpyHostToDevice, stream()));
  if (n_active > 0) {
    DevBuf<int> bad(1);
    bad.zero();
    k_apply_active_dofs<<<grid_for(n_active, 256), 256, 0, stream()>>>(n_active, dofs_dev, vals_dev, nt, c->flag.p,
                                                                        c->inhom.p, bad.p);
    CF_LAUNCHED();
    if (read1(bad.p)) fail(CF_ERR_INVALID_ARGUMENT, "build_constraints: dof out of range");
    k_flags_one<<<grid_for(nt, 256), 256, 0, stream()>>>(nt, c->flag.p);
    CF_LAUNCHED();
  }
  std::vector<std::uint8_t> fall = to_host(c->flag.p, nt);
  std::vector<double> inh = to_host(c->inhom.p, nt);
  close_lines(L, fall, inh);
  std::vector<int> ldof;
  std::vector<i64> lptr{0};
  std::vector<int> lm;
  std::vector<double> lw;
  for (auto& [dof, l] : L) {
    ldof.push_back(int(dof));
    inh[size_t(dof)] = l.inhom;
    for (auto& [mm, w] : l.e) {
      lm.push_back(int(mm));
      lw.push_back(w);
    }
    lptr.push_back(i64(lm.size()));
  }
  CF_CUDA(cudaMemcpyAsync(c->inhom.p, inh.data(), size_t(nt) * sizeof(double), cudaMemcpyHostToDevice, stream()));
  c->n_lines = i64(ldof.size());
  to_dev(c->line_dof, ldof);
  to_dev(c->line_ptr, lptr);
  to_dev(c->line_m, lm);
  to_dev(c->line_w, lw);
  i64 cnt = 0;
  for (auto f : fall) cnt += f;
  c->count = cnt;
  CF_CUDA(cudaStreamSynchronize(stream()));  // the host staging vectors go out of scope
  return c;
}

void mesh_full_lines(const Constraints& base, Constraints& full) {
  full.mesh = base.mesh;
  full.n_lines = base.n_lines;
  full.line_dof.alloc(base.n_lines);
  full.line_ptr.alloc(base.n_lines + 1);
  if (base.n_lines == 0) {
    CF_CUDA(cudaMemsetAsync(full.line_ptr.p, 0, sizeof(i64), stream()));
    full.line_m.alloc(0);
    full.line_w.alloc(0);
    return;
  }
  CF_CUDA(cudaMemcpyAsync(full.line_dof.p, base.line_dof.p, size_t(base.n_lines) * sizeof(int),
                          cudaMemcpyDeviceToDevice, stream()));
  const i64 nl = base.n_lines;
  k_full_lines_count<<<grid_for(nl, 256), 256, 0, stream()>>>(nl, base.line_ptr.p, base.line_m.p, full.flag.p,
                                                             full.line_ptr.p);
  CF_LAUNCHED();
  CF_CUDA(cudaMemsetAsync(full.line_ptr.p + nl, 0, sizeof(i64), stream()));
  scan_ex(full.line_ptr.p, nl + 1);
  const i64 ne = read1(full.line_ptr.p + nl);
  full.line_m.alloc(std::max<i64>(ne, 1));
  full.line_w.alloc(std::max<i64>(ne, 1));
  k_full_lines_fill<<<grid_for(nl, 256), 256, 0, stream()>>>(nl, base.line_dof.p, base.line_ptr.p, base.line_m.p,
                                                            base.line_w.p, base.inhom.p, full.flag.p,
                                                            full.line_ptr.p, full.line_m.p, full.line_w.p,
                                                            full.inhom.p);
  CF_LAUNCHED();
}

void distribute_lines(const Constraints& c, double* v, bool homogeneous) {
  if (c.n_lines == 0) return;
  k_distribute_lines<<<grid_for(c.n_lines, 256), 256, 0, stream()>>>(c.n_lines, c.line_dof.p, c.line_ptr.p,
                                                                      c.line_m.p, c.line_w.p, c.inhom.p, v,
                                                                      homogeneous ? 1 : 0);
  CF_LAUNCHED();
}

// ------------------------------------------------------------------ element tables per level
void mesh_tables(MeshDisc& m, double mu, double lam) {
  if (m.tab_mu == mu && m.tab_lam == lam && int(m.host_tabs.size()) == m.max_level + 1) return;
  const int d = m.d;
  m.host_tabs.assign(size_t(m.max_level + 1), Tables{});
  for (int l = 0; l <= m.max_level; ++l) {
    const double h = m.level_edge(l);
    fill_tables(m.host_tabs[size_t(l)], d, h, std::pow(h, d), mu, lam);
  }
  m.tabs.alloc(m.max_level + 1);
  CF_CUDA(cudaMemcpyAsync(m.tabs.p, m.host_tabs.data(), m.host_tabs.size() * sizeof(Tables), cudaMemcpyHostToDevice,
                          stream()));
  m.tab_mu = mu;
  m.tab_lam = lam;
}


// ------------------------------------------------------------------ model helpers on meshes
namespace {

__device__ __forceinline__ double d_phys(double K, double unit, i64 c) { return -K + double(c) * unit; }

__global__ void k_mesh_rigid(i64 V, int d, double K, double unit, const i64* __restrict__ vkey,
                             const std::uint8_t* __restrict__ flag, double* __restrict__ B) {
  const i64 v = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= V) return;
  i64 c[3];
  vcoord(vkey[v], c);
  const double x0 = d_phys(K, unit, c[0]), x1 = d_phys(K, unit, c[1]), x2 = d == 3 ? d_phys(K, unit, c[2]) : 0.0;
  const i64 n = i64(d) * V;
  const int m = (d == 2) ? 3 : 6;
  double row[3][6];
  for (int a = 0; a < 3; ++a)
    for (int k = 0; k < 6; ++k) row[a][k] = 0.0;
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
    for (int k = 0; k < m; ++k) B[i64(k) * n + v * d + a] = con ? 0.0 : row[a][k];
  }
}

// model.cpp:324-349: phi = 0 on the vertices of the slab around the slit
__global__ void k_mesh_crack(i64 V, int d, double K, double unit, double l0, double band, const i64* __restrict__ vkey,
                             double* __restrict__ phi, unsigned long long* __restrict__ counts) {
  const i64 v = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= V) return;
  i64 c[3];
  vcoord(vkey[v], c);
  const double x0 = d_phys(K, unit, c[0]), x1 = d_phys(K, unit, c[1]), x2 = d == 3 ? d_phys(K, unit, c[2]) : 0.0;
  const double tol = 1e-9 * band;
  bool in;
  if (d == 2)
    in = fabs(x0) <= l0 + tol && fabs(x1) <= band + tol;
  else
    in = hypot(x0, x1) <= l0 + tol && fabs(x2) <= band + tol;
  phi[v] = in ? 0.0 : 1.0;
  if (in) {
    atomicAdd(&counts[0], 1ull);
    if (fabs(d == 2 ? x1 : x2) <= tol) atomicAdd(&counts[1], 1ull);
  }
}

// u . grad(phi) of a field on an active cell at physical x (fem.cpp:269-299)
template <int D>
__device__ double m_u_dot_gradphi(const int* __restrict__ cv, double lo0, double lo1, double lo2, double h, i64 nu,
                                  const double* __restrict__ sol, const double* x) {
  const double lo[3] = {lo0, lo1, lo2};
  double xi[3] = {0, 0, 0};
  for (int a = 0; a < D; ++a) xi[a] = fmin(fmax((x[a] - lo[a]) / h, 0.0), 1.0);
  double u[3] = {0, 0, 0}, gp[3] = {0, 0, 0};
  for (int k = 0; k < (1 << D); ++k) {
    double s = 1.0;
    for (int a = 0; a < D; ++a) s *= (k & (1 << a)) ? xi[a] : 1.0 - xi[a];
    const i64 v = cv[k];
    const double phi = sol[nu + v];
    for (int a = 0; a < D; ++a) {
      double gr = (k & (1 << a)) ? 1.0 : -1.0;
      for (int b = 0; b < D; ++b) {
        if (b == a) continue;
        gr *= (k & (1 << b)) ? xi[b] : 1.0 - xi[b];
      }
      gp[a] += gr / h * phi;
      u[a] += s * sol[v * D + a];
    }
  }
  double dot = 0.0;
  for (int a = 0; a < 3; ++a) dot += u[a] * gp[a];
  return dot;
}

struct CellGeo {
  const int* cid;
  const int* clevel;
  const i64* anchor;
  double K, unit;
  const double* hlev;
  const double* detj;
};

template <int D>
__global__ void __launch_bounds__(256) k_mesh_tcv(i64 nact, CellGeo G, const int* __restrict__ cvert, i64 nu,
                                                  const double* __restrict__ sol, const double* __restrict__ qp,
                                                  const double* __restrict__ qw, double* __restrict__ part) {
  __shared__ double sh[256];
  double s = 0.0;
  for (i64 c = i64(blockIdx.x) * 256 + threadIdx.x; c < nact; c += i64(gridDim.x) * 256) {
    const int id = G.cid[c], lev = G.clevel[c];
    const double h = G.hlev[lev], dj = G.detj[lev];
    double lo[3] = {0, 0, 0};
    for (int a = 0; a < D; ++a) lo[a] = d_phys(G.K, G.unit, G.anchor[3 * id + a]);
    double cs = 0.0;
    for (int q = 0; q < (1 << D); ++q) {
      double x[3] = {lo[0], lo[1], lo[2]};
      for (int a = 0; a < D; ++a) x[a] += qp[q * 3 + a] * h;
      cs += qw[q] * dj * m_u_dot_gradphi<D>(cvert + c * (1 << D), lo[0], lo[1], lo[2], h, nu, sol, x);
    }
    s += cs;
  }
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

// one CTA per station, over every active cell whose column owns it (postproc.cpp:39-66)
template <int D>
__global__ void __launch_bounds__(256) k_mesh_cod(i64 nact, CellGeo G, const int* __restrict__ cvert, i64 nu,
                                                  const double* __restrict__ sol, const double* __restrict__ st,
                                                  const double* __restrict__ lp, const double* __restrict__ lw,
                                                  double* __restrict__ out) {
  __shared__ double sh[256];
  const double s = st[blockIdx.x];
  const double K = G.K;
  auto owns = [K](double lo, double hi, double x) { return (x < K) ? (lo <= x && x < hi) : (lo < x && x <= hi); };
  const int axis = D - 1;
  double acc = 0.0;
  for (i64 c = threadIdx.x; c < nact; c += blockDim.x) {
    const int id = G.cid[c], lev = G.clevel[c];
    const double h = G.hlev[lev];
    const i64 sz = kUnit >> lev;
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int a = 0; a < D; ++a) {
      lo[a] = d_phys(G.K, G.unit, G.anchor[3 * id + a]);
      hi[a] = d_phys(G.K, G.unit, G.anchor[3 * id + a] + sz);
    }
    if (!owns(lo[0], hi[0], s)) continue;
    if (D == 3 && !owns(lo[1], hi[1], 0.0)) continue;
    double cs = 0.0;
    for (int q = 0; q < 4; ++q) {
      double x[3] = {s, 0.0, 0.0};
      x[axis] = lo[axis] + lp[q] * h;
      cs += lw[q] * h * m_u_dot_gradphi<D>(cvert + c * (1 << D), lo[0], lo[1], lo[2], h, nu, sol, x);
    }
    acc += cs;
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = 0.5 * fabs(sh[0]);
}

__global__ void k_msum(int nb, const double* __restrict__ part, double* out) {
  __shared__ double sh[256];
  double s = 0.0;
  for (int b = threadIdx.x; b < nb; b += 256) s += part[b];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

struct LevelGeo {
  DevBuf<double> h, detj;
  LevelGeo(const MeshDisc& m) {
    std::vector<double> hh(size_t(m.max_level + 1)), dj(size_t(m.max_level + 1));
    for (int l = 0; l <= m.max_level; ++l) {
      hh[size_t(l)] = m.level_edge(l);
      dj[size_t(l)] = std::pow(hh[size_t(l)], m.d);
    }
    to_dev(h, hh);
    to_dev(detj, dj);
    CF_CUDA(cudaStreamSynchronize(stream()));
  }
};

}  // namespace

void mesh_rigid_body_modes(const MeshDisc& m, const Constraints& c, double* B) {
  k_mesh_rigid<<<grid_for(m.V, 256), 256, 0, stream()>>>(m.V, m.d, m.K, m.unit, m.vkey.p, c.flag.p, B);
  CF_LAUNCHED();
}

double mesh_slit_band_edge(const MeshDisc& m, const cf_material& mat) {  // model.cpp:28-50
  const int d = m.d;
  double edge = -1.0;
  for (int id : m.active) {
    const HostCell& c = m.cells[id];
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int a = 0; a < d; ++a) {
      lo[a] = m.to_physical(c.anchor[a]);
      hi[a] = m.to_physical(c.anchor[a] + c.isize());
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
      const double h = m.level_edge(c.level);
      if (edge < 0.0 || h < edge) edge = h;
    }
  }
  if (edge < 0.0) fail(CF_ERR_NUMERICAL, "slit_band_edge: no active cell meets the slit");
  return edge;
}

cf_regularization mesh_resolve_regularization(const MeshDisc& m, const cf_material& mat, double band_edge) {
  cf_regularization reg;  // model.cpp:52-58
  const double diam = band_edge * std::sqrt(double(m.d));
  reg.eps = (mat.eps_mode == 0) ? mat.c_eps * diam : mat.eps_fixed;
  reg.kappa = mat.kappa_factor * m.level_edge(m.max_level);
  return reg;
}

std::vector<double> mesh_initial_crack(MeshDisc& m, const cf_material& mat, double band_half, double* band_edge) {
  const double be = band_half > 0.0 ? band_half : mesh_slit_band_edge(m, mat);
  DevBuf<double> phi(m.V);
  DevBuf<unsigned long long> cnt(2);
  cnt.zero();
  k_mesh_crack<<<grid_for(m.V, 256), 256, 0, stream()>>>(m.V, m.d, m.K, m.unit, mat.l0, be, m.vkey.p, phi.p, cnt.p);
  CF_LAUNCHED();
  std::vector<unsigned long long> c = to_host(cnt.p, 2);
  if (c[0] == 0 || c[1] == 0)
    fail(CF_ERR_NUMERICAL, "initial_crack: slit is not resolved by the mesh (no vertex layer inside the band)");
  if (band_edge) *band_edge = be;
  return to_host(phi.p, m.V);
}

double mesh_compute_tcv(MeshDisc& m, const double* sol) {
  const int d = m.d;
  double pts[8 * 3] = {0}, wts[8];
  const double a1 = 1.0 / std::sqrt(3.0), x1[2] = {-a1, a1};
  for (int q = 0; q < (1 << d); ++q) {
    int rem = q;
    double wt = 1.0;
    for (int a = 0; a < d; ++a) {
      const int i = rem % 2;
      rem /= 2;
      pts[q * 3 + a] = 0.5 * (x1[i] + 1.0);
      wt *= 0.5 * 1.0;
    }
    wts[q] = wt;
  }
  LevelGeo lg(m);
  DevBuf<double> dq(24), dw(8), part(1024), out(1);
  CF_CUDA(cudaMemcpyAsync(dq.p, pts, sizeof(pts), cudaMemcpyHostToDevice, stream()));
  CF_CUDA(cudaMemcpyAsync(dw.p, wts, sizeof(wts), cudaMemcpyHostToDevice, stream()));
  const int nb = int(std::min<i64>(1024, std::max<i64>(1, (m.nact + 255) / 256)));
  CellGeo G{m.cid.p, m.clevel.p, m.t_anchor.p, m.K, m.unit, lg.h.p, lg.detj.p};
  if (d == 2)
    k_mesh_tcv<2><<<nb, 256, 0, stream()>>>(m.nact, G, m.cvert.p, m.n_u(), sol, dq.p, dw.p, part.p);
  else
    k_mesh_tcv<3><<<nb, 256, 0, stream()>>>(m.nact, G, m.cvert.p, m.n_u(), sol, dq.p, dw.p, part.p);
  CF_LAUNCHED();
  k_msum<<<1, 256, 0, stream()>>>(nb, part.p, out.p);
  CF_LAUNCHED();
  return read1(out.p);
}

void mesh_compute_cod(MeshDisc& m, const double* sol, const double* stations_host, int ns, double* out_host) {
  for (int i = 1; i < ns; ++i)
    if (!(stations_host[i] > stations_host[i - 1]))
      fail(CF_ERR_INVALID_ARGUMENT, "compute_cod: stations must be strictly increasing");
  for (int i = 0; i < ns; ++i)
    if (std::abs(stations_host[i]) > m.K) fail(CF_ERR_INVALID_ARGUMENT, "compute_cod: station outside domain");
  if (ns == 0) return;
  const double a = std::sqrt(3.0 / 7.0 - 2.0 / 7.0 * std::sqrt(6.0 / 5.0));
  const double b = std::sqrt(3.0 / 7.0 + 2.0 / 7.0 * std::sqrt(6.0 / 5.0));
  const double wa = (18.0 + std::sqrt(30.0)) / 36.0, wb = (18.0 - std::sqrt(30.0)) / 36.0;
  const double xs[4] = {-b, -a, a, b}, ws[4] = {wb, wa, wa, wb};
  double lp[4], lw[4];
  for (int q = 0; q < 4; ++q) {
    lp[q] = 0.5 * (xs[q] + 1.0);
    lw[q] = 1.0 * (0.5 * ws[q]);
  }
  LevelGeo lg(m);
  DevBuf<double> dst(ns), dlp(4), dlw(4), dout(ns);
  CF_CUDA(cudaMemcpyAsync(dst.p, stations_host, size_t(ns) * sizeof(double), cudaMemcpyHostToDevice, stream()));
  CF_CUDA(cudaMemcpyAsync(dlp.p, lp, sizeof(lp), cudaMemcpyHostToDevice, stream()));
  CF_CUDA(cudaMemcpyAsync(dlw.p, lw, sizeof(lw), cudaMemcpyHostToDevice, stream()));
  CellGeo G{m.cid.p, m.clevel.p, m.t_anchor.p, m.K, m.unit, lg.h.p, lg.detj.p};
  if (m.d == 2)
    k_mesh_cod<2><<<ns, 256, 0, stream()>>>(m.nact, G, m.cvert.p, m.n_u(), sol, dst.p, dlp.p, dlw.p, dout.p);
  else
    k_mesh_cod<3><<<ns, 256, 0, stream()>>>(m.nact, G, m.cvert.p, m.n_u(), sol, dst.p, dlp.p, dlw.p, dout.p);
  CF_LAUNCHED();
  CF_CUDA(cudaMemcpyAsync(out_host, dout.p, size_t(ns) * sizeof(double), cudaMemcpyDeviceToHost, stream()));
  CF_CUDA(cudaStreamSynchronize(stream()));
}

}  // namespace cfb

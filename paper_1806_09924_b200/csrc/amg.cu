// K7/K8: smoothed-aggregation AMG setup and V-cycle on the device (linsolve.cpp:117-318).
//
// Setup per level, all on the device and deterministic (compiled with -fmad=false so every
// floating-point expression is the reference's sequence of IEEE operations):
//   strength   node blocks grouped by a stable radix sort of node_of_dof; per node, the
//              Frobenius^2 sums of its coupling blocks accumulated in (row, column) order into a
//              small sorted key list (std::map semantics); strong iff
//              sqrt(s_ij) > theta sqrt(sqrt(s_ii) sqrt(s_jj))          (linsolve.cpp:185-201)
//   aggregate  the reference's sequential greedy (linsolve.cpp:142-166) computed EXACTLY in
//              parallel: pass-1 roots are the lexicographically-first MIS of the directed
//              distance-2 dependency graph N2(i) = S[i] u S^T[i] u S^T[S[i]] (i is a root iff no
//              root r < i lies in N2(i)), resolved by a persistent cooperative kernel that
//              pushes decisions along N2 frontier by frontier; pass 2/3 by ordered fix-point
//              rounds.  Identical output to the sequential loop for any strength graph.
//   tentative  one thread per aggregate runs the column-pivoting Householder QR of its
//              near-nullspace block (Eigen ColPivHouseholderQR semantics, threshold 1e-10)
//   smoothing  D^-1 from the diagonal, lambda_max by 15 power iterations, P = T - w D^-1 A T
//   Galerkin   Ac = P^T (A P) with the deterministic SpGEMM of spgemm.cu, pruned
// V-cycle: damped Jacobi pre/post sweeps, restriction with an explicit R = P^T, dense LU on the
// coarsest level (one CTA).
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <unordered_map>

#include "cf_comm.hpp"
#include "cf_vec.hpp"

namespace cg = cooperative_groups;

namespace cfb {

namespace {

template <class T>
void scan_excl(T* data, i64 n_plus_1) {
  size_t bytes = 0;
  CF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, data, data, n_plus_1, stream()));
  DevBuf<unsigned char> tmp{static_cast<i64>(bytes)};
  CF_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, data, data, n_plus_1, stream()));
  count_launch();
}

template <class T>
T read_dev(const T* p) {
  T h{};
  read_small(&h, p, sizeof(T));
  return h;
}

int bits_for(i64 n) {
  int b = 1;
  while ((i64(1) << b) < n) ++b;
  return b;
}

// CF_TIMING=1: per-phase device times of build_amg on stderr (profiling aid, off by default)
struct PhaseClock {
  bool on;
  cudaEvent_t last;
  int lev = 0;
  long syncs = 0;  // host round trips at the previous mark
  PhaseClock() : on(std::getenv("CF_TIMING") != nullptr) {
    syncs = host_sync_count();
    if (on) {
      cudaEventCreate(&last);
      cudaEventRecord(last, stream());
    }
  }
  void mark(const char* what) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, stream());
    cudaEventSynchronize(e);
    float ms = 0;
    cudaEventElapsedTime(&ms, last, e);
    const long ns = host_sync_count();
    std::fprintf(stderr, "[amg L%d] %-12s %8.3f ms %4ld host syncs\n", lev, what, ms, ns - syncs);
    syncs = ns;
    cudaEventDestroy(last);
    last = e;
  }
  ~PhaseClock() {
    if (on) cudaEventDestroy(last);
  }
};

i64 pow2_at_least(i64 n) {
  i64 c = 16;
  while (c < n) c <<= 1;
  return c;
}

__global__ void k_iota(i64 n, int* out) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = int(i);
}

__global__ void k_flag_list(i64 n, const int* __restrict__ flag, int* __restrict__ list, int* __restrict__ count);

struct OvfList {
  DevBuf<int> list;
  int n = 0;
};

// ascending list of flagged nodes
OvfList make_ovf_list(i64 n, const int* flag) {
  OvfList o;
  DevBuf<int> c(1);
  c.zero();
  o.list.alloc(std::max<i64>(n, 1));
  k_flag_list<<<grid_for(n, 256), 256, 0, stream()>>>(n, flag, o.list.p, c.p);
  CF_LAUNCHED();
  o.n = read_dev(c.p);  // list order is irrelevant: every listed node is processed independently
  return o;
}

__global__ void k_count_keys(i64 n, const int* __restrict__ key, i64* __restrict__ cnt) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(reinterpret_cast<unsigned long long*>(cnt + key[i]), 1ull);
}

// Stable grouping of items 0..n-1 by key in [0, nkeys): ptr (nkeys+1) and ascending items.
void group_by_key(i64 n, const int* key, i64 nkeys, DevBuf<i64>& ptr, DevBuf<int>& items) {
  ptr.alloc(nkeys + 1);
  ptr.zero();
  items.alloc(std::max<i64>(n, 1));
  if (n == 0) return;
  k_count_keys<<<grid_for(n, 256), 256, 0, stream()>>>(n, key, ptr.p);
  CF_LAUNCHED();
  scan_excl(ptr.p, nkeys + 1);
  DevBuf<int> iota(n), keys_out(n);
  k_iota<<<grid_for(n, 256), 256, 0, stream()>>>(n, iota.p);
  CF_LAUNCHED();
  size_t bytes = 0;
  const int eb = bits_for(nkeys + 1);
  CF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key, keys_out.p, iota.p, items.p, n, 0, eb, stream()));
  DevBuf<unsigned char> tmp{static_cast<i64>(bytes)};
  CF_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, key, keys_out.p, iota.p, items.p, n, 0, eb, stream()));
  count_launch();
}

// ------------------------------------------------------------------ strength (linsolve.cpp:185-201)
constexpr int SCAP = 96;        // distinct neighbour nodes per node in the register/local tier
constexpr int SWARP_MIN = 320;  // nodes with more entries than this use the warp tier

// Overflow tier: nodes with more distinct neighbour nodes than SCAP get a private open-addressing
// table in global memory (capacity = next pow2 >= 2 x their entry count); one thread per node
// keeps the (row, column) accumulation order, then compacts and heap-sorts its keys.
__device__ __forceinline__ unsigned hash_u(int k) { return unsigned(k) * 2654435761u; }
// slot in a power-of-two table: the high bits of the Fibonacci product (the low bits collide for
// clustered node ids); the tables are sets or per-key sums, so the slot function never changes a result
__device__ __forceinline__ unsigned hslot_u(int k, unsigned mask) {
#ifdef CF_LOWHASH
  return hash_u(k) & mask;
#else
  return mask ? (hash_u(k) >> (32 - __popc(mask))) : 0u;
#endif
}

__device__ void heap_sort_pairs(int* key, double* val, int n) {
  auto sift = [&](int start, int end) {
    int root = start;
    while (2 * root + 1 <= end) {
      int child = 2 * root + 1, sw = root;
      if (key[sw] < key[child]) sw = child;
      if (child + 1 <= end && key[sw] < key[child + 1]) sw = child + 1;
      if (sw == root) return;
      const int tk = key[root]; key[root] = key[sw]; key[sw] = tk;
      if (val) { const double tv = val[root]; val[root] = val[sw]; val[sw] = tv; }
      root = sw;
    }
  };
  for (int s = (n - 2) / 2; s >= 0; --s) sift(s, n - 1);
  for (int e = n - 1; e > 0; --e) {
    const int tk = key[0]; key[0] = key[e]; key[e] = tk;
    if (val) { const double tv = val[0]; val[0] = val[e]; val[e] = tv; }
    sift(0, e - 1);
  }
}

__global__ void k_node_entries(i64 nov, const int* __restrict__ list, const i64* __restrict__ nptr,
                               const int* __restrict__ ndofs, const i64* __restrict__ Ap, i64 cap_max,
                               i64* __restrict__ cap) {
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nov) return;
  const int i = list[t];
  i64 e = 0;
  for (i64 k = nptr[i]; k < nptr[i + 1]; ++k) e += Ap[ndofs[k] + 1] - Ap[ndofs[k]];
  i64 c = 16;
  while (c < 2 * e && c < cap_max) c <<= 1;
  cap[t] = c;
}

__global__ void k_strength_big(i64 nov, const int* __restrict__ list, const i64* __restrict__ off,
                               const i64* __restrict__ nptr, const int* __restrict__ ndofs, const i64* __restrict__ Ap,
                               const int* __restrict__ Ac, const double* __restrict__ Av, const int* __restrict__ nod,
                               int* __restrict__ keys, double* __restrict__ sums, int* __restrict__ len_out) {
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nov) return;
  const int i = list[t];
  int* K = keys + off[t];
  double* S = sums + off[t];
  const unsigned mask = unsigned(off[t + 1] - off[t]) - 1u;
  int len = 0;
  for (i64 q = nptr[i]; q < nptr[i + 1]; ++q) {
    const int r = ndofs[q];
    for (i64 k = Ap[r]; k < Ap[r + 1]; ++k) {
      const int nj = nod[Ac[k]];
      const double a2 = Av[k] * Av[k];
      unsigned s = hslot_u(nj, mask);
      while (K[s] != -1 && K[s] != nj) s = (s + 1) & mask;
      if (K[s] == nj) {
        S[s] += a2;
      } else {
        K[s] = nj;
        S[s] = a2;
        ++len;
      }
    }
  }
  int p = 0;
  for (unsigned s = 0; s <= mask; ++s)
    if (K[s] != -1) {
      K[p] = K[s];
      S[p] = S[s];
      ++p;
    }
  heap_sort_pairs(K, S, len);
  len_out[t] = len;
}

// Warp-per-node variant of k_strength_big (the same table, sums and ascending output): the 32 lanes
// take consecutive entries of one dof row; lanes that hit the same neighbour node are applied by the
// lowest of them in lane (= column) order, and rows follow one another, so every sum is accumulated
// in exactly the serial (row, column) order.  Tables come in with keys = -1 and sums = 0.
constexpr int SBW_WPB = 4;
__global__ void __launch_bounds__(SBW_WPB * 32)
    k_strength_bigw(i64 nov, const int* __restrict__ list, const i64* __restrict__ off, const i64* __restrict__ nptr,
                    const int* __restrict__ ndofs, const i64* __restrict__ Ap, const int* __restrict__ Ac,
                    const double* __restrict__ Av, const int* __restrict__ nod, int* __restrict__ keys,
                    double* __restrict__ sums, int* __restrict__ len_out) {
  __shared__ double sbuf[SBW_WPB][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const i64 t = i64(blockIdx.x) * SBW_WPB + w;
  if (t >= nov) return;
  const int i = list[t];
  int* K = keys + off[t];
  double* S = sums + off[t];
  const unsigned cap = unsigned(off[t + 1] - off[t]), mask = cap - 1u;
  for (i64 q = nptr[i]; q < nptr[i + 1]; ++q) {
    const int r = ndofs[q];
    const i64 e0 = Ap[r], e1 = Ap[r + 1];
    for (i64 b = e0; b < e1; b += 32) {
      const i64 k = b + lane;
      const bool v = k < e1;
      int slot = -1;
      if (v) {
        const int nj = nod[Ac[k]];
        const double x = Av[k];
        sbuf[w][lane] = x * x;
        unsigned s = hslot_u(nj, mask);
        for (unsigned p = 0; p < cap; ++p) {
          int cur = K[s];
          if (cur == -1) cur = atomicCAS(&K[s], -1, nj);
          if (cur == -1 || cur == nj) break;
          s = (s + 1) & mask;
        }
        slot = int(s);
      }
      __syncwarp();
      const unsigned act = __ballot_sync(0xffffffffu, v);
      const unsigned peers = __match_any_sync(0xffffffffu, slot);
      if (v && (peers & act & ((1u << lane) - 1u)) == 0) {  // lowest lane of its group
        double acc = S[slot];
        for (unsigned m = peers & act; m; m &= m - 1) acc += sbuf[w][__ffs(m) - 1];
        S[slot] = acc;
      }
      __syncwarp();
    }
  }
  // compact the occupied slots (ascending slot order) to the front, pad, bitonic-sort by key
  int len = 0;
  for (unsigned b = 0; b < cap; b += 32) {
    const unsigned s = b + lane;
    const int key = s < cap ? K[s] : -1;
    const double sm = s < cap ? S[s] : 0.0;
    const unsigned occ = __ballot_sync(0xffffffffu, key != -1);
    __syncwarp();
    if (key != -1) {
      const int dst = len + __popc(occ & ((1u << lane) - 1u));
      K[dst] = key;
      S[dst] = sm;
    }
    len += __popc(occ);
    __syncwarp();
  }
  unsigned n2 = 1;
  while (n2 < unsigned(len)) n2 <<= 1;
  for (unsigned s = len + lane; s < n2; s += 32) K[s] = INT_MAX;
  __syncwarp();
  for (unsigned k2 = 2; k2 <= n2; k2 <<= 1)
    for (unsigned j = k2 >> 1; j > 0; j >>= 1) {
      for (unsigned s = lane; s < n2; s += 32) {
        const unsigned o = s ^ j;
        if (o > s) {
          const int a = K[s], c = K[o];
          if ((a > c) == ((s & k2) == 0)) {
            K[s] = c;
            K[o] = a;
            const double ta = S[s];
            S[s] = S[o];
            S[o] = ta;
          }
        }
      }
      __syncwarp();
    }
  if (lane == 0) len_out[t] = len;
}

// strong test on the sorted overflow lists; mode 0 counts, mode 1 writes
__global__ void k_strength_big_emit(i64 nov, const int* __restrict__ list, const i64* __restrict__ off,
                                    const int* __restrict__ keys, const double* __restrict__ sums,
                                    const int* __restrict__ len, const double* __restrict__ dsq, double theta,
                                    i64* __restrict__ cnt, const i64* __restrict__ sptr, int* __restrict__ sidx,
                                    int mode) {
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nov) return;
  const int i = list[t];
  const int* K = keys + off[t];
  const double* S = sums + off[t];
  const double dii = dsq[i];
  i64 n = 0;
  const i64 base = mode ? sptr[i] : 0;
  for (int s = 0; s < len[t]; ++s) {
    const int j = K[s];
    if (j == i) continue;
    if (sqrt(S[s]) > theta * sqrt(dii * dsq[j])) {
      if (mode) sidx[base + n] = j;
      ++n;
    }
  }
  if (!mode) cnt[i] = n;
}

__global__ void k_flag_list(i64 n, const int* __restrict__ flag, int* __restrict__ list, int* __restrict__ count) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n && flag[i]) list[atomicAdd(count, 1)] = int(i);
}

__global__ void k_strength_diag(i64 nn, const i64* __restrict__ nptr, const int* __restrict__ ndofs,
                                const i64* __restrict__ Ap, const int* __restrict__ Ac, const double* __restrict__ Av,
                                const int* __restrict__ nod, double* __restrict__ dsq) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nn) return;
  double s = 0.0;
  bool present = false;
  for (i64 t = nptr[i]; t < nptr[i + 1]; ++t) {
    const int r = ndofs[t];
    for (i64 k = Ap[r]; k < Ap[r + 1]; ++k)
      if (nod[Ac[k]] == int(i)) {
        s += Av[k] * Av[k];
        present = true;
      }
  }
  dsq[i] = sqrt(present ? s : 0.0);  // sqrt(blk[i].count(i) ? blk[i][i] : 0)
}

// mode 0: count strong neighbours; mode 1: write them (ascending node id)
__global__ void k_strength(i64 nn, const i64* __restrict__ nptr, const int* __restrict__ ndofs,
                           const i64* __restrict__ Ap, const int* __restrict__ Ac, const double* __restrict__ Av,
                           const int* __restrict__ nod, const double* __restrict__ dsq, double theta,
                           i64* __restrict__ cnt, const i64* __restrict__ sptr, int* __restrict__ sidx, int mode,
                           int* __restrict__ ovf, int* __restrict__ stmp) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nn) return;
  if (mode && ovf[i]) return;  // handled by the overflow tier
  if (!mode) {  // long nodes go straight to the warp tier (one thread would walk them serially)
    i64 e = 0;
    for (i64 t = nptr[i]; t < nptr[i + 1]; ++t) e += Ap[ndofs[t] + 1] - Ap[ndofs[t]];
    if (e > SWARP_MIN) {
      ovf[i] = 1;
      return;
    }
  }
  int keys[SCAP];
  double sums[SCAP];
  int len = 0;
  for (i64 t = nptr[i]; t < nptr[i + 1]; ++t) {
    const int r = ndofs[t];
    for (i64 k = Ap[r]; k < Ap[r + 1]; ++k) {
      const int nj = nod[Ac[k]];
      const double a2 = Av[k] * Av[k];
      int lo = 0, hi = len;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (keys[mid] < nj) lo = mid + 1; else hi = mid;
      }
      if (lo < len && keys[lo] == nj) {
        sums[lo] += a2;
      } else {
        if (len == SCAP) {
          ovf[i] = 1;
          return;
        }
        for (int s = len; s > lo; --s) {
          keys[s] = keys[s - 1];
          sums[s] = sums[s - 1];
        }
        keys[lo] = nj;
        sums[lo] = a2;
        ++len;
      }
    }
  }
  const double dii = dsq[i];
  i64 n = 0;
  const i64 base = mode ? sptr[i] : 0;
  for (int s = 0; s < len; ++s) {
    const int j = keys[s];
    if (j == int(i)) continue;
    const double djj = dsq[j];
    if (sqrt(sums[s]) > theta * sqrt(dii * djj)) {
      if (mode) sidx[base + n] = j;
      else if (stmp) stmp[i64(i) * SCAP + n] = j;  // kept for k_strength_compact (n < SCAP)
      ++n;
    }
  }
  if (!mode) cnt[i] = n;
}

// the strong lists stored by the counting pass -> CSR (warp per node; overflow-tier nodes skipped)
// G lanes per node: 32 for the fine levels (tens of strong neighbours), 1 where most nodes have
// none (the dof-less coarse nodes of the phi levels), so the launch is not a warp per empty node
template <int G>
__global__ void k_strength_compact(i64 nn, const int* __restrict__ ovf, const int* __restrict__ stmp,
                                   const i64* __restrict__ sptr, int* __restrict__ sidx) {
  const i64 i = (i64(blockIdx.x) * blockDim.x + threadIdx.x) / G;
  const int lane = threadIdx.x % G;
  if (i >= nn || ovf[i]) return;
  const i64 b = sptr[i], n = sptr[i + 1] - b;
  for (i64 t = lane; t < n; t += G) sidx[b + t] = stmp[i * SCAP + t];
}

// ------------------------------------------------------------------ N2 dependency graph
// N2(i) = S[i] u T[i] u T[S[i]] (T = S^T): per node a hash set (k_n2w: warp, shared memory;
// k_n2_big: global memory for high-degree nodes).  mode 0 counts the lower (< i) and upper (> i)
// members; mode 1 writes the upper members (the dependents).

// overflow tier of N2: a private hash set per node in global memory
__global__ void k_n2_cap(i64 nov, const int* __restrict__ list, const i64* __restrict__ sp, const int* __restrict__ si,
                         const i64* __restrict__ tp, i64 cap_max, i64* __restrict__ cap) {
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nov) return;
  const int i = list[t];
  i64 e = (sp[i + 1] - sp[i]) + (tp[i + 1] - tp[i]);
  for (i64 k = sp[i]; k < sp[i + 1]; ++k) e += tp[si[k] + 1] - tp[si[k]];
  i64 c = 16;
  while (c < 2 * e && c < cap_max) c <<= 1;
  cap[t] = c;
}

__device__ __forceinline__ void set_insert(int* K, unsigned mask, int v) {
  unsigned s = hslot_u(v, mask);
  while (K[s] != -1 && K[s] != v) s = (s + 1) & mask;
  K[s] = v;
}

__global__ void k_n2_big(i64 nov, const int* __restrict__ list, const i64* __restrict__ off, const i64* __restrict__ sp,
                         const int* __restrict__ si, const i64* __restrict__ tp, const int* __restrict__ ti,
                         int* __restrict__ keys, int* __restrict__ lower, i64* __restrict__ upcnt,
                         const i64* __restrict__ upptr, int* __restrict__ up, int mode) {
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nov) return;
  const int i = list[t];
  int* K = keys + off[t];
  const unsigned mask = unsigned(off[t + 1] - off[t]) - 1u;
  if (mode == 0) {
    for (i64 k = sp[i]; k < sp[i + 1]; ++k) set_insert(K, mask, si[k]);
    for (i64 k = tp[i]; k < tp[i + 1]; ++k) set_insert(K, mask, ti[k]);
    for (i64 k = sp[i]; k < sp[i + 1]; ++k) {
      const int j = si[k];
      for (i64 q = tp[j]; q < tp[j + 1]; ++q) set_insert(K, mask, ti[q]);
    }
    int nlow = 0;
    i64 nup = 0;
    for (unsigned s = 0; s <= mask; ++s) {
      if (K[s] < 0) continue;
      if (K[s] < i) ++nlow;
      else if (K[s] > i) ++nup;
    }
    lower[i] = nlow;
    upcnt[i] = nup;
  } else {
    i64 n = 0;
    const i64 base = upptr[i];
    for (unsigned s = 0; s <= mask; ++s)
      if (K[s] > i) up[base + n++] = K[s];
  }
}

// warp per node, shared-memory hash set of N2(i) (set semantics: the insertion order is
// irrelevant); more than 3/4 x N2CAP members -> overflow tier
constexpr int N2CAP = 1024, N2WPB = 4;
// mode 0 also stores up to N2UPC upper members per node in ups[i * N2UPC ...] (redo[i] = 0), so
// mode 1 (which rebuilds the set) runs only for the nodes with more (redo[i] = 1); k_n2_compact
// then moves the stored lists into the CSR of the dependents
constexpr int N2UPC = 96;
// the nodes with a strong edge (either direction); isolated nodes (the dof-less coarse nodes of
// the phi levels, active phi dofs) get their empty N2 here, so the warp kernels visit only the list
__global__ void k_n2_nodes(i64 nn, const i64* __restrict__ sp, const i64* __restrict__ tp, int* __restrict__ lower,
                           i64* __restrict__ upcnt, int* __restrict__ redo, int* __restrict__ list,
                           int* __restrict__ count) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nn) return;
  if (sp[i + 1] == sp[i] && tp[i + 1] == tp[i]) {
    lower[i] = 0;
    upcnt[i] = 0;
    redo[i] = 0;
  } else {
    list[atomicAdd(count, 1)] = int(i);
  }
}

__global__ void __launch_bounds__(N2WPB * 32) k_n2w(i64 nn, const int* __restrict__ list, const i64* __restrict__ sp,
                                                    const int* __restrict__ si, const i64* __restrict__ tp,
                                                    const int* __restrict__ ti, int* __restrict__ lower,
                                                    i64* __restrict__ upcnt, const i64* __restrict__ upptr,
                                                    int* __restrict__ up, int mode, int* __restrict__ ovf,
                                                    int* __restrict__ ups, int* __restrict__ redo) {
  __shared__ int tab[N2WPB][N2CAP];
  __shared__ int cnt[N2WPB];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const i64 node = i64(blockIdx.x) * N2WPB + w;
  if (node >= nn) return;
  const int i = list ? list[node] : int(node);
  if (mode == 1 && (ovf[i] || !redo[i])) return;
  if (sp[i + 1] == sp[i] && tp[i + 1] == tp[i]) {  // isolated node: N2(i) is empty
    if (mode == 0 && lane == 0) {
      lower[i] = 0;
      upcnt[i] = 0;
      redo[i] = 0;
    }
    return;
  }
  int* T = tab[w];
  for (int s = lane; s < N2CAP; s += 32) T[s] = -1;
  if (lane == 0) cnt[w] = 0;
  __syncwarp();
  const unsigned mask = N2CAP - 1;
  bool full = false;
  auto ins = [&](int v) {
    unsigned s = hslot_u(v, mask);
    for (int p = 0; p < N2CAP; ++p) {
      const int cur = T[s];
      if (cur == v) return;
      if (cur == -1) {
        const int old = atomicCAS(&T[s], -1, v);
        if (old == -1) {
          atomicAdd(&cnt[w], 1);
          return;
        }
        if (old == v) return;
      }
      s = (s + 1) & mask;
    }
    full = true;
  };
  for (i64 k = sp[i] + lane; k < sp[i + 1]; k += 32) ins(si[k]);
  for (i64 k = tp[i] + lane; k < tp[i + 1]; k += 32) ins(ti[k]);
  for (i64 k = sp[i]; k < sp[i + 1]; ++k) {
    const int j = si[k];
    for (i64 q = tp[j] + lane; q < tp[j + 1]; q += 32) ins(ti[q]);
    if (__any_sync(0xffffffffu, full) || cnt[w] > (N2CAP * 3) / 4) {
      full = true;
      break;
    }
  }
  __syncwarp();
  if (__any_sync(0xffffffffu, full) || cnt[w] > (N2CAP * 3) / 4) {
    if (mode == 0 && lane == 0) ovf[i] = 1;
    return;
  }
  if (mode == 0) {
    __syncwarp();
    if (lane == 0) cnt[w] = 0;
    __syncwarp();
    int nl = 0, nu = 0;
    int* my = ups + i64(i) * N2UPC;
    for (int s = lane; s < N2CAP; s += 32) {
      const int v = T[s];
      if (v < 0) continue;
      nl += v < i;
      if (v > i) {
        ++nu;
        const int pos = atomicAdd(&cnt[w], 1);
        if (pos < N2UPC) my[pos] = v;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      nl += __shfl_xor_sync(0xffffffffu, nl, o);
      nu += __shfl_xor_sync(0xffffffffu, nu, o);
    }
    if (lane == 0) {
      lower[i] = nl;
      upcnt[i] = nu;
      redo[i] = nu > N2UPC ? 1 : 0;
    }
  } else {
    __syncwarp();
    if (lane == 0) cnt[w] = 0;
    __syncwarp();
    const i64 base = upptr[i];
    for (int s = lane; s < N2CAP; s += 32) {
      const int v = T[s];
      if (v > i) up[base + atomicAdd(&cnt[w], 1)] = v;
    }
  }
}


// stored upper lists -> CSR of the dependents (warp per node; nodes handled by mode 1 or by the
// global-memory tier are skipped)
__global__ void k_n2_compact(i64 nn, const int* __restrict__ list, const int* __restrict__ ovf,
                             const int* __restrict__ redo, const int* __restrict__ ups, const i64* __restrict__ upptr,
                             int* __restrict__ up) {
  const i64 t = (i64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= nn) return;
  const i64 i = list ? list[t] : t;
  if (ovf[i] || redo[i]) return;
  const i64 b = upptr[i], n = upptr[i + 1] - b;
  for (i64 t = lane; t < n; t += 32) up[b + t] = ups[i * N2UPC + t];
}

// ------------------------------------------------------------------ pass 1: LFMIS frontier rounds
constexpr int UND = 0, ROOT = 1, NOTROOT = 2;

// roots without dependents (isolated nodes: active phi dofs, dof-less coarse nodes) are decided
// here and never enter a frontier (they would message nobody)
__global__ void k_lfmis_init(i64 nn, const int* __restrict__ lower, const i64* __restrict__ up_ptr,
                             int* __restrict__ status, int* __restrict__ front, int* __restrict__ fsize) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nn) return;
  if (lower[i] == 0) {
    status[i] = ROOT;
    if (up_ptr[i + 1] > up_ptr[i]) front[atomicAdd(fsize, 1)] = int(i);
  } else {
    status[i] = UND;
  }
}

__global__ void k_lfmis(const i64* __restrict__ up_ptr, const int* __restrict__ up, int* cnt, int* status, int* f0,
                        int* f1, int* sizes, int* rounds) {
  cg::grid_group g = cg::this_grid();
  int r = 0;
  while (true) {
    int* F = (r & 1) ? f1 : f0;
    int* G = (r & 1) ? f0 : f1;
    const int nf = *((volatile int*)&sizes[r % 3]);
    if (nf == 0) break;
    if (g.thread_rank() == 0) sizes[(r + 2) % 3] = 0;
    int* nxt = &sizes[(r + 1) % 3];
    // one warp per frontier node, lanes over its dependents: a node's ~100 dependents would
    // otherwise be a serial chain of returning atomics on one thread (the round's critical path)
    const long long nwarps = g.size() / 32;
    const int lane = threadIdx.x & 31;
    for (long long t = g.thread_rank() / 32; t < nf; t += nwarps) {
      const int v = F[t];
      const int st = *((volatile int*)&status[v]);
      for (i64 k = up_ptr[v] + lane; k < up_ptr[v + 1]; k += 32) {
        const int i = up[k];
        // a decided dependent needs no message: its status is final (a pending count is only
        // consulted while the node is undecided), so skip the atomic after a plain read
        if (*((volatile int*)&status[i]) != UND) continue;
        if (st == ROOT) {
          if (atomicCAS(&status[i], UND, NOTROOT) == UND) G[atomicAdd(nxt, 1)] = i;
        } else {
          if (atomicSub(&cnt[i], 1) == 1)
            if (atomicCAS(&status[i], UND, ROOT) == UND) G[atomicAdd(nxt, 1)] = i;
        }
      }
    }
    g.sync();
    ++r;
  }
  if (g.thread_rank() == 0) *rounds = r;
}

__global__ void k_root_flags(i64 nn, const int* __restrict__ status, int* __restrict__ flag) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < nn) flag[i] = status[i] == ROOT ? 1 : 0;
}

// roots claim their strong neighbours (disjoint by construction)
__global__ void k_claim(i64 nn, const int* __restrict__ status, const int* __restrict__ rootid,
                        const i64* __restrict__ sp, const int* __restrict__ si, int* __restrict__ agg) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nn || status[i] != ROOT) return;
  const int a = rootid[i];
  agg[i] = a;
  for (i64 k = sp[i]; k < sp[i + 1]; ++k) agg[si[k]] = a;
}

// pass 2 (linsolve.cpp:157-161): p2 state -1 unresolved, -2 unassignable, >=0 assigned aggregate.
__global__ void k_pass2(i64 nn, const i64* __restrict__ sp, const int* __restrict__ si, const int* __restrict__ agg1,
                        int* __restrict__ p2, int* __restrict__ changed) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nn || agg1[i] >= 0 || p2[i] != -1) return;
  for (i64 k = sp[i]; k < sp[i + 1]; ++k) {
    const int j = si[k];
    if (agg1[j] >= 0) {
      p2[i] = agg1[j];
      *changed = 1;
      return;
    }
    if (j < int(i)) {
      const int s = *((volatile int*)&p2[j]);
      if (s >= 0) {
        p2[i] = s;
        *changed = 1;
        return;
      }
      if (s == -1) return;  // wait for j
    }
  }
  p2[i] = -2;
  *changed = 1;
}

__global__ void k_pass3_flags(i64 nn, const int* __restrict__ agg1, const int* __restrict__ p2, int* __restrict__ f) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < nn) f[i] = (agg1[i] < 0 && p2[i] == -2) ? 1 : 0;
}

__global__ void k_final_agg(i64 nn, const int* __restrict__ agg1, const int* __restrict__ p2,
                            const int* __restrict__ p3id, int n1, int* __restrict__ agg) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nn) return;
  agg[i] = agg1[i] >= 0 ? agg1[i] : (p2[i] >= 0 ? p2[i] : n1 + p3id[i]);
}

// ------------------------------------------------------------------ tentative prolongator (QR)
__global__ void k_agg_of_dof(i64 n, const int* __restrict__ nod, const int* __restrict__ agg, int* __restrict__ out) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = agg[nod[i]];
}

// Column-pivoting Householder QR of one aggregate's near-nullspace block (Eigen 3.3
// ColPivHouseholderQR::computeInPlace / rank / householderQ, sequential sums), m <= 8.
__global__ void k_agg_qr(i64 na, const i64* __restrict__ aptr, const int* __restrict__ adofs,
                         const double* __restrict__ B, i64 n, int m, double* __restrict__ W, double* __restrict__ Q,
                         double* __restrict__ hc_all, int* __restrict__ perm_all, int* __restrict__ rank_out,
                         int st) {
  const i64 a = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a >= na) return;
  const i64 off = aptr[a];
  const int rows = int(aptr[a + 1] - off);
  double* qr = W + off * m;  // column-major, ld = rows, element stride st
  for (int c = 0; c < m; ++c)
    for (int r = 0; r < rows; ++r) qr[(c * rows + r) * st] = B[i64(c) * n + adofs[off + r]];
  const int cols = m, size = rows < cols ? rows : cols;
  double upd[8], dir[8], hc[8];
  int transp[8], perm[8];
  for (int k = 0; k < cols; ++k) {
    double s = 0.0;
    for (int r = 0; r < rows; ++r) s += qr[(k * rows + r) * st] * qr[(k * rows + r) * st];
    dir[k] = sqrt(s);
    upd[k] = dir[k];
  }
  double mx = 0.0;
  for (int k = 0; k < cols; ++k) mx = (k == 0 || upd[k] > mx) ? upd[k] : mx;
  const double eps = 2.220446049250313e-16;
  const double th_helper = (mx * eps) * (mx * eps) / double(rows);
  const double ndt = sqrt(eps);
  int nonzero = size;
  double maxpivot = 0.0;
  for (int k = 0; k < size; ++k) {
    int bi = k;
    double bv = upd[k];
    for (int j = k + 1; j < cols; ++j)
      if (upd[j] > bv) {
        bv = upd[j];
        bi = j;
      }
    const double bsq = bv * bv;
    if (nonzero == size && bsq < th_helper * double(rows - k)) nonzero = k;
    transp[k] = bi;
    if (k != bi) {
      for (int r = 0; r < rows; ++r) {
        const double t = qr[(k * rows + r) * st];
        qr[(k * rows + r) * st] = qr[(bi * rows + r) * st];
        qr[(bi * rows + r) * st] = t;
      }
      double t = upd[k]; upd[k] = upd[bi]; upd[bi] = t;
      t = dir[k]; dir[k] = dir[bi]; dir[bi] = t;
    }
    double beta, tau;
    {
      const double c0 = qr[(k * rows + k) * st];
      double tsq = 0.0;
      for (int r = k + 1; r < rows; ++r) tsq += qr[(k * rows + r) * st] * qr[(k * rows + r) * st];
      if (tsq <= 2.2250738585072014e-308) {
        tau = 0.0;
        beta = c0;
        for (int r = k + 1; r < rows; ++r) qr[(k * rows + r) * st] = 0.0;
      } else {
        beta = sqrt(c0 * c0 + tsq);
        if (c0 >= 0.0) beta = -beta;
        for (int r = k + 1; r < rows; ++r) qr[(k * rows + r) * st] = qr[(k * rows + r) * st] / (c0 - beta);
        tau = (beta - c0) / beta;
      }
    }
    hc[k] = tau;
    qr[(k * rows + k) * st] = beta;
    if (fabs(beta) > maxpivot) maxpivot = fabs(beta);
    for (int j = k + 1; j < cols; ++j) {
      if (rows - k == 1) {
        qr[(j * rows + k) * st] *= (1.0 - tau);
      } else if (tau != 0.0) {
        double t = 0.0;
        for (int r = k + 1; r < rows; ++r) t += qr[(k * rows + r) * st] * qr[(j * rows + r) * st];
        t += qr[(j * rows + k) * st];
        qr[(j * rows + k) * st] -= tau * t;
        for (int r = k + 1; r < rows; ++r) qr[(j * rows + r) * st] -= (tau * qr[(k * rows + r) * st]) * t;
      }
    }
    for (int j = k + 1; j < cols; ++j) {
      if (upd[j] != 0.0) {
        double tmp = fabs(qr[(j * rows + k) * st]) / upd[j];
        tmp = (1.0 + tmp) * (1.0 - tmp);
        tmp = tmp < 0.0 ? 0.0 : tmp;
        const double ratio = upd[j] / dir[j];
        const double tmp2 = tmp * (ratio * ratio);
        if (tmp2 <= ndt) {
          double s = 0.0;
          for (int r = k + 1; r < rows; ++r) s += qr[(j * rows + r) * st] * qr[(j * rows + r) * st];
          dir[j] = sqrt(s);
          upd[j] = dir[j];
        } else {
          upd[j] *= sqrt(tmp);
        }
      }
    }
  }
  for (int k = 0; k < cols; ++k) perm[k] = k;
  for (int k = 0; k < size; ++k) {
    const int t = perm[k];
    perm[k] = perm[transp[k]];
    perm[transp[k]] = t;
  }
  const double pt = fabs(maxpivot) * 1e-10;
  int rank = 0;
  for (int i = 0; i < nonzero; ++i) rank += (fabs(qr[(i * rows + i) * st]) > pt) ? 1 : 0;
  rank = rank < 0 ? 0 : rank;
  if (rank > size) rank = size;
  rank_out[a] = rank;
  for (int k = 0; k < m; ++k) {
    hc_all[a * 8 + k] = k < size ? hc[k] : 0.0;
    perm_all[a * 8 + k] = perm[k];
  }
  // Q columns c < rank: H_0 ... H_{size-1} e_c
  double* q = Q + off * m;
  for (int c = 0; c < rank; ++c) {
    double* out = q + c * rows;
    for (int r = 0; r < rows; ++r) out[(r) * st] = (r == c) ? 1.0 : 0.0;
    for (int k = size - 1; k >= 0; --k) {
      const double tau = hc[k];
      if (rows - k == 1) {
        out[(k) * st] *= (1.0 - tau);
      } else if (tau != 0.0) {
        double t = 0.0;
        for (int r = k + 1; r < rows; ++r) t += qr[(k * rows + r) * st] * out[(r) * st];
        t += out[(k) * st];
        out[(k) * st] -= tau * t;
        for (int r = k + 1; r < rows; ++r) out[(r) * st] -= (tau * qr[(k * rows + r) * st]) * t;
      }
    }
  }
}

__global__ void k_pos_in_agg(i64 na, const i64* __restrict__ aptr, const int* __restrict__ adofs, int* __restrict__ pos,
                             int* __restrict__ agg_of) {
  const i64 a = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a >= na) return;
  for (i64 t = aptr[a]; t < aptr[a + 1]; ++t) {
    pos[adofs[t]] = int(t - aptr[a]);
    agg_of[adofs[t]] = int(a);
  }
}

// T rows: row i -> entries (agg_offset[a] + c, Q(pos, c)) with |Q| > 1e-300 (linsolve.cpp:230-238)
__global__ void k_build_T(i64 n, int m, const int* __restrict__ agg_of, const int* __restrict__ pos,
                          const i64* __restrict__ aptr, const int* __restrict__ rank, const i64* __restrict__ aoff,
                          const double* __restrict__ Q, i64* __restrict__ tp, int* __restrict__ tc,
                          double* __restrict__ tv, int mode) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int a = agg_of[i], r = pos[i];
  const i64 off = aptr[a];
  const int rows = int(aptr[a + 1] - off);
  const double* q = Q + off * m;
  i64 cnt = 0;
  const i64 base = mode ? tp[i] : 0;
  for (int c = 0; c < rank[a]; ++c) {
    const double v = q[c * rows + r];
    if (fabs(v) > 1e-300) {
      if (mode) {
        tc[base + cnt] = int(aoff[a] + c);
        tv[base + cnt] = v;
      }
      ++cnt;
    }
  }
  if (!mode) tp[i] = cnt;
}

// coarse near-nullspace Bc = [R_a Pi_a^T] and coarse node ids (linsolve.cpp:265-270)
__global__ void k_build_Bc(i64 na, int m, const i64* __restrict__ aptr, const int* __restrict__ rank,
                           const i64* __restrict__ aoff, const double* __restrict__ W, const int* __restrict__ perm_all,
                           i64 nc, double* __restrict__ Bc, int* __restrict__ cnode) {
  const i64 a = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a >= na) return;
  const i64 off = aptr[a];
  const int rows = int(aptr[a + 1] - off);
  const double* qr = W + off * m;
  for (int i = 0; i < rank[a]; ++i) {
    const i64 row = aoff[a] + i;
    cnode[row] = int(a);
    for (int c = 0; c < m; ++c) Bc[i64(c) * nc + row] = 0.0;
    for (int k = i; k < m; ++k) Bc[i64(perm_all[a * 8 + k]) * nc + row] = qr[k * rows + i];
  }
}

// ---- empty coarse nodes (DESIGN.md §4 K7) --------------------------------------------------------
// A level's nodes are the previous level's aggregates, and an aggregate whose near-nullspace block
// has rank 0 (every constrained phi dof is one) carries no coarse dof: in the reference it is an
// isolated node and seeds its own, again empty, aggregate in pass 1 (linsolve.cpp:146-154).  The
// build runs on the non-empty nodes only (ascending order kept, so every aggregate keeps its place
// among the others) and restores the reference numbering for what it reports: nodes counted with
// the empty ones, pass-1 aggregates numbered over all roots by ascending node id.
__global__ void k_nonempty_flags(i64 na, const int* __restrict__ rank, int* __restrict__ f) {
  const i64 a = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a < na) f[a] = rank[a] > 0 ? 1 : 0;
}
// compact id -> reference id of the next level's nodes (aorig: this level's compact -> reference
// aggregate ids, null = identity)
__global__ void k_compact_orig(i64 na, const int* __restrict__ rank, const int* __restrict__ cid,
                               const int* __restrict__ aorig, int* __restrict__ orig_next) {
  const i64 a = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a < na && rank[a] > 0) orig_next[cid[a]] = aorig ? aorig[a] : int(a);
}
__global__ void k_renumber(i64 n, const int* __restrict__ cid, int* __restrict__ node) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) node[i] = cid[node[i]];
}
__global__ void k_fill_ones(i64 n, int* __restrict__ f) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) f[i] = 1;
}
// root flags over the reference node numbering (empty nodes are roots) and each pass-1 aggregate's root
__global__ void k_root_scatter(i64 nn, const int* __restrict__ status, const int* __restrict__ rootid,
                               const int* __restrict__ orig, int* __restrict__ rflag, int* __restrict__ root_of_agg) {
  const i64 c = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= nn) return;
  const bool root = status[c] == ROOT;
  rflag[orig[c]] = root ? 1 : 0;
  if (root) root_of_agg[rootid[c]] = int(c);
}
// reference id of compact aggregate a: pass-1 aggregates by their root's rank among all roots,
// pass-3 singletons after all pass-1 aggregates
__global__ void k_agg_orig(i64 na, int n1, const int* __restrict__ root_of_agg, const int* __restrict__ orig,
                           const int* __restrict__ rid, i64 nn_orig, int* __restrict__ aorig) {
  const i64 a = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a >= na) return;
  aorig[a] = a < n1 ? rid[orig[root_of_agg[a]]] : rid[nn_orig] + int(a - n1);
}
__global__ void k_agg_full(i64 nn, const int* __restrict__ agg, const int* __restrict__ orig,
                           const int* __restrict__ aorig, int* __restrict__ agg_full) {
  const i64 c = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c < nn) agg_full[orig[c]] = aorig[agg[c]];
}

__global__ void k_inv_diag(i64 n, double* d) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) d[i] = d[i] != 0.0 ? 1.0 / d[i] : 0.0;
}
// diagonal preconditioner: 1/d, 1 where d == 0 (linsolve.cpp:382-391)
__global__ void k_inv_diag_one(i64 n, double* d) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) d[i] = d[i] != 0.0 ? 1.0 / d[i] : 1.0;
}
__global__ void k_int_to_i64(i64 n, const int* __restrict__ a, i64* __restrict__ b) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}
__global__ void k_graph_rows(i64 nn, const i64* __restrict__ ptr, int* __restrict__ src) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nn) return;
  for (i64 k = ptr[i]; k < ptr[i + 1]; ++k) src[k] = int(i);
}
__global__ void k_gather_int(i64 n, const int* __restrict__ idx, const int* __restrict__ src, int* __restrict__ out) {
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < n) out[t] = src[idx[t]];
}

// ------------------------------------------------------------------ dense LU (one CTA)
__global__ void k_dense_from_csr(i64 n, const i64* __restrict__ p, const int* __restrict__ c,
                                 const double* __restrict__ v, double* __restrict__ a) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (i64 k = p[i]; k < p[i + 1]; ++k) a[i64(c[k]) * n + i] = v[k];
}

// Eigen PartialPivLU semantics (unblocked): first maximal |pivot|, row swap, column divide,
// rank-1 update.  column-major n x n.
__global__ void __launch_bounds__(1024) k_dense_lu(int n, double* a, int* piv, double* minpiv) {
  __shared__ double sv[1024];
  __shared__ int si[1024];
  for (int k = 0; k < n; ++k) {
    double best = -1.0;
    int bi = k;
    for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
      const double v = fabs(a[i64(k) * n + i]);
      if (v > best) {
        best = v;
        bi = i;
      }
    }
    sv[threadIdx.x] = best;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
      if (threadIdx.x < s) {
        const double o = sv[threadIdx.x + s];
        const int oi = si[threadIdx.x + s];
        if (o > sv[threadIdx.x] || (o == sv[threadIdx.x] && oi < si[threadIdx.x])) {
          sv[threadIdx.x] = o;
          si[threadIdx.x] = oi;
        }
      }
      __syncthreads();
    }
    const double big = sv[0];
    const int p = si[0];
    __syncthreads();
    if (threadIdx.x == 0) piv[k] = p;
    if (big != 0.0) {
      if (p != k)
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
          const double t = a[i64(j) * n + k];
          a[i64(j) * n + k] = a[i64(j) * n + p];
          a[i64(j) * n + p] = t;
        }
      __syncthreads();
      const double akk = a[i64(k) * n + k];
      for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) a[i64(k) * n + i] /= akk;
    }
    __syncthreads();
    const int rem = n - k - 1;
    for (long long t = threadIdx.x; t < (long long)rem * rem; t += blockDim.x) {
      const int i = k + 1 + int(t % rem), j = k + 1 + int(t / rem);
      a[i64(j) * n + i] -= a[i64(k) * n + i] * a[i64(j) * n + k];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double m = INFINITY;
    for (int i = 0; i < n; ++i) m = fmin(m, fabs(a[i64(i) * n + i]));
    *minpiv = m;
  }
}

// Multi-CTA form of k_dense_lu for coarsest matrices beyond one CTA (n > 16384; the reference
// LU-factors a coarsest matrix of any size, linsolve.cpp:277-285): per column k a pivot search
// (one CTA, first maximal |a_ik|), the row swap and column division, and the rank-1 update of the
// trailing block over the whole grid.  Every entry receives its updates in ascending k with the
// same operands, so the factors are bitwise those of the one-CTA kernel and the oracle.
__global__ void __launch_bounds__(1024) k_lu_pivot(int n, int k, const double* __restrict__ a, int* __restrict__ piv,
                                                   double* __restrict__ big) {
  __shared__ double sv[1024];
  __shared__ int si[1024];
  double best = -1.0;
  int bi = k;
  for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
    const double v = fabs(a[i64(k) * n + i]);
    if (v > best) {
      best = v;
      bi = i;
    }
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double o = sv[threadIdx.x + s];
      const int oi = si[threadIdx.x + s];
      if (o > sv[threadIdx.x] || (o == sv[threadIdx.x] && oi < si[threadIdx.x])) {
        sv[threadIdx.x] = o;
        si[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    piv[k] = si[0];
    *big = sv[0];
  }
}
__global__ void k_lu_swap(int n, int k, double* __restrict__ a, const int* __restrict__ piv,
                          const double* __restrict__ big) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int p = piv[k];
  if (j >= n || *big == 0.0 || p == k) return;
  const double t = a[i64(j) * n + k];
  a[i64(j) * n + k] = a[i64(j) * n + p];
  a[i64(j) * n + p] = t;
}
__global__ void k_lu_scale(int n, int k, double* __restrict__ a, const double* __restrict__ big) {
  const int i = k + 1 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || *big == 0.0) return;
  a[i64(k) * n + i] /= a[i64(k) * n + k];
}
__global__ void k_lu_update(int n, int k, double* __restrict__ a) {
  const int i = k + 1 + blockIdx.x * blockDim.x + threadIdx.x;
  const int j = k + 1 + blockIdx.y;
  if (i >= n) return;
  a[i64(j) * n + i] -= a[i64(k) * n + i] * a[i64(j) * n + k];
}
__global__ void k_lu_minpiv(int n, const double* __restrict__ a, double* minpiv) {
  __shared__ double sm[256];
  double m = INFINITY;
  for (int i = threadIdx.x; i < n; i += blockDim.x) m = fmin(m, fabs(a[i64(i) * n + i]));
  sm[threadIdx.x] = m;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sm[threadIdx.x] = fmin(sm[threadIdx.x], sm[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *minpiv = sm[0];
}

// is the CSR diagonal (no off-diagonal entries)?  diag[i] = a_ii (0 when absent)
__global__ void k_check_diag(i64 n, const i64* __restrict__ p, const int* __restrict__ c,
                             const double* __restrict__ v, double* __restrict__ diag, int* __restrict__ offdiag) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double d = 0.0;
  for (i64 k = p[i]; k < p[i + 1]; ++k) {
    if (c[k] == int(i)) d = v[k];
    else atomicOr(offdiag, 1);
  }
  diag[i] = d;
}

__global__ void k_diag_solve(i64 n, const double* __restrict__ d, const double* __restrict__ b,
                             double* __restrict__ x) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) x[i] = b[i] / d[i];
}

__global__ void k_min_abs(i64 n, const double* __restrict__ d, unsigned long long* __restrict__ out) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) atomicMin(out, __double_as_longlong(fabs(d[i])));  // non-negative doubles order as integers
}

// solve (single thread: sequential substitutions, as the oracle)
__global__ void k_dense_solve(int n, const double* __restrict__ a, const int* __restrict__ piv,
                              const double* __restrict__ b, double* __restrict__ x) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int i = 0; i < n; ++i) x[i] = b[i];
  for (int k = 0; k < n; ++k)
    if (piv[k] != k) {
      const double t = x[k];
      x[k] = x[piv[k]];
      x[piv[k]] = t;
    }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j) x[i] -= a[i64(j) * n + i] * x[j];
  for (int i = n - 1; i >= 0; --i) {
    for (int j = i + 1; j < n; ++j) x[i] -= a[i64(j) * n + i] * x[j];
    x[i] /= a[i64(i) * n + i];
  }
}

// Shared-memory variant for small coarsest systems (n <= DENSE_SM_MAX): the factors are staged in
// shared memory; the forward substitution runs column by column over all threads (each x_i still
// receives its updates in ascending j with the same operands, so it is bitwise the row form above);
// the backward substitution is the same serial loop, reading shared memory.
constexpr int DENSE_SM_MAX = 128;
__global__ void __launch_bounds__(256) k_dense_solve_sm(int n, const double* __restrict__ a,
                                                        const int* __restrict__ piv, const double* __restrict__ b,
                                                        double* __restrict__ x) {
  extern __shared__ double dsm[];
  double* A = dsm;      // n * n, column-major
  double* X = dsm + n * n;
  for (int t = threadIdx.x; t < n * n; t += blockDim.x) A[t] = a[t];
  for (int t = threadIdx.x; t < n; t += blockDim.x) X[t] = b[t];
  __syncthreads();
  if (threadIdx.x == 0)
    for (int k = 0; k < n; ++k)
      if (piv[k] != k) {
        const double t = X[k];
        X[k] = X[piv[k]];
        X[piv[k]] = t;
      }
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    const double xj = X[j];
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) X[i] -= A[j * n + i] * xj;
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int i = n - 1; i >= 0; --i) {
      double xi = X[i];
      for (int j = i + 1; j < n; ++j) xi -= A[j * n + i] * X[j];
      X[i] = xi / A[i * n + i];
    }
  __syncthreads();
  for (int t = threadIdx.x; t < n; t += blockDim.x) x[t] = X[t];
}

// ------------------------------------------------------------------ V-cycle pieces
// x = w * (d .* b)
__global__ void k_jacobi0(i64 n, double w, const double* __restrict__ d, const double* __restrict__ b,
                          double* __restrict__ x) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) x[i] = w * (d[i] * b[i]);
}
// x += w * (d .* (b - ax))
__global__ void k_jacobi_upd(i64 n, double w, const double* __restrict__ d, const double* __restrict__ b,
                             const double* __restrict__ ax, double* __restrict__ x) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) x[i] += w * (d[i] * (b[i] - ax[i]));
}

// power-iteration start vector v_i = 1 + 0.5 sin(1 + i) (linsolve.cpp:123): computed on the host
// with the C library's sin (correctly rounded).  v_i does not depend on the length, so one buffer
// holds the longest prefix seen so far and every level (of every hierarchy) reads a prefix of it.
// Chebyshev smoothing on D^-1 A (smoother 1): the first step d = D^-1 r / theta, then
// d = c1 d + c2 D^-1 r, x += d (the standard three-term recurrence)
__global__ void k_cheb_init(i64 n, double inv_theta, const double* __restrict__ dinv, const double* __restrict__ r,
                            double* __restrict__ d, double* __restrict__ x, int zero) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double di = inv_theta * (dinv[i] * r[i]);
  d[i] = di;
  x[i] = zero ? di : x[i] + di;
}
__global__ void k_cheb_step(i64 n, double c1, double c2, const double* __restrict__ dinv,
                            const double* __restrict__ r, double* __restrict__ d, double* __restrict__ x) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double di = c1 * d[i] + c2 * (dinv[i] * r[i]);
  d[i] = di;
  x[i] += di;
}

// Gershgorin bound of D^-1 A, row i: |d_i| sum_j |a_ij| (the Chebyshev smoother's upper bound)
__global__ void k_gershgorin_rows(i64 n, const i64* __restrict__ ptr, const double* __restrict__ val,
                                  const double* __restrict__ dinv, double* __restrict__ out) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (i64 k = ptr[i]; k < ptr[i + 1]; ++k) s += fabs(val[k]);
  out[i] = fabs(dinv[i]) * s;
}

double gershgorin_bound(const Csr& A, const double* inv_diag) {
  const i64 n = A.rows;
  if (n == 0) return 1.0;
  DevBuf<double> rows(n), mx(1);
  k_gershgorin_rows<<<grid_for(n, 256), 256, 0, stream()>>>(n, A.ptr.p, A.val.p, inv_diag, rows.p);
  CF_LAUNCHED();
  size_t bytes = 0;
  CF_CUDA(cub::DeviceReduce::Max(nullptr, bytes, rows.p, mx.p, n, stream()));
  DevBuf<unsigned char> tmp{static_cast<i64>(bytes)};
  CF_CUDA(cub::DeviceReduce::Max(tmp.p, bytes, rows.p, mx.p, n, stream()));
  count_launch();
  return read_dev(mx.p);
}

const double* lambda_start(i64 n) {
  static DevBuf<double> buf;
  static std::vector<double> host;
  if (i64(host.size()) >= n) return buf.p;
  const i64 old = i64(host.size());
  const i64 cap = std::max<i64>(n, old + old / 2);
  host.resize(cap);
  for (i64 i = old; i < cap; ++i) host[i] = 1.0 + 0.5 * std::sin(1.0 + double(i));
  DevBuf<double> nb(cap);
  CF_CUDA(cudaMemcpyAsync(nb.p, host.data(), size_t(cap) * sizeof(double), cudaMemcpyHostToDevice, stream()));
  CF_CUDA(cudaStreamSynchronize(stream()));
  ++host_sync_count();
  buf = std::move(nb);
  return buf.p;
}

// power-iteration bookkeeping on the device: st = {lambda, done}; the first zero norm freezes
// lambda at 1.0 (the reference returns 1.0 there), later iterations (NaN) change nothing
__global__ void k_lambda_step(const double* __restrict__ nw, double* __restrict__ st) {
  if (st[1] != 0.0) return;
  if (nw[0] == 0.0) {
    st[0] = 1.0;
    st[1] = 1.0;
  } else {
    st[0] = nw[0];
  }
}

double estimate_lambda_max(const Csr& A, const double* inv_diag) {  // linsolve.cpp:120-134
  const i64 n = A.rows;
  DevBuf<double> v(n), w(n);
  double* s = scalar_buf(4);  // s[0]: norm; s[2], s[3]: lambda, done
  const double* v0 = lambda_start(n);
  vdot_dev(v0, v0, n, s, true);
  vdiv_dev(v0, s, v.p, n);
  const double init[2] = {1.0, 0.0};
  CF_CUDA(cudaMemcpyAsync(s + 2, init, sizeof(init), cudaMemcpyHostToDevice, stream()));
  // 15 iterations without a host round trip each (the reference's early return on a zero norm is
  // the device flag; the values are the same IEEE sequence)
  for (int it = 0; it < 15; ++it) {
    SpmvEpi ep;  // w = 1.0 * (D^-1 (A v)): vdiag_mul's expression in the SpMV epilogue
    ep.d = inv_diag;
    ep.w = 1.0;
    ep.mode = 3;
    csr_spmv_epi(A, v.p, w.p, ep);
    vdot_dev(w.p, w.p, n, s, true);
    k_lambda_step<<<1, 1, 0, stream()>>>(s, s + 2);
    CF_LAUNCHED();
    vdiv_dev(w.p, s, v.p, n);
  }
  double st[2];
  read_small(st, s + 2, sizeof(st));
  if (st[1] != 0.0) return 1.0;
  return std::max(st[0], 1e-12);
}

}  // namespace

// ------------------------------------------------------------------ dense LU host side
void DenseLu::factor_from_csr(const Csr& A) {
  n = A.rows;
  diagonal = false;
  // CF_LU_MULTICTA_MIN (test switch): smallest n factorised by the multi-CTA kernels (default 16385)
  static const i64 multi_min = std::getenv("CF_LU_MULTICTA_MIN") ? std::atoll(std::getenv("CF_LU_MULTICTA_MIN")) : 16385;
  if (n >= multi_min) {
    if (n > 65535) fail(CF_ERR_UNSUPPORTED, "dense LU: coarsest matrix above 65535 rows (n^2 doubles)");
    lu.alloc(n);
    DevBuf<int> off(1);
    off.zero();
    k_check_diag<<<grid_for(n, 256), 256, 0, stream()>>>(n, A.ptr.p, A.col.p, A.val.p, lu.p, off.p);
    CF_LAUNCHED();
    DevBuf<unsigned long long> mn(1);
    const unsigned long long inf_bits = 0x7ff0000000000000ull;
    CF_CUDA(cudaMemcpyAsync(mn.p, &inf_bits, sizeof(inf_bits), cudaMemcpyHostToDevice, stream()));
    k_min_abs<<<grid_for(n, 256), 256, 0, stream()>>>(n, lu.p, mn.p);
    CF_LAUNCHED();
    int h_off = 0;
    unsigned long long h_mn = 0;
    CF_CUDA(cudaMemcpyAsync(&h_off, off.p, sizeof(int), cudaMemcpyDeviceToHost, stream()));
    read_small(&h_mn, mn.p, sizeof(h_mn));
    if (!h_off) {  // a diagonal coarsest matrix: the LU is the diagonal itself
      std::memcpy(&min_abs_pivot, &h_mn, sizeof(double));
      diagonal = true;
      return;
    }
    // a general coarsest matrix beyond one CTA: the multi-CTA factorisation (n^2 doubles)
    lu.alloc(n * n);
    lu.zero();
    piv.alloc(n);
    k_dense_from_csr<<<grid_for(n, 256), 256, 0, stream()>>>(n, A.ptr.p, A.col.p, A.val.p, lu.p);
    CF_LAUNCHED();
    double* big = scalar_buf(2);
    for (int k = 0; k < int(n); ++k) {
      k_lu_pivot<<<1, 1024, 0, stream()>>>(int(n), k, lu.p, piv.p, big);
      k_lu_swap<<<grid_for(n, 256), 256, 0, stream()>>>(int(n), k, lu.p, piv.p, big);
      const int rem = int(n) - k - 1;
      if (rem > 0) {
        k_lu_scale<<<grid_for(rem, 256), 256, 0, stream()>>>(int(n), k, lu.p, big);
        k_lu_update<<<dim3(grid_for(rem, 256), unsigned(rem)), 256, 0, stream()>>>(int(n), k, lu.p);
      }
      count_launch(rem > 0 ? 4 : 2);
    }
    CF_CUDA(cudaGetLastError());
    k_lu_minpiv<<<1, 256, 0, stream()>>>(int(n), lu.p, big + 1);
    CF_LAUNCHED();
    min_abs_pivot = read_dev(big + 1);
    return;
  }
  lu.alloc(std::max<i64>(n * n, 1));
  lu.zero();
  piv.alloc(std::max<i64>(n, 1));
  if (n == 0) {
    min_abs_pivot = INFINITY;
    return;
  }
  k_dense_from_csr<<<grid_for(n, 256), 256, 0, stream()>>>(n, A.ptr.p, A.col.p, A.val.p, lu.p);
  CF_LAUNCHED();
  double* mp = scalar_buf(1);
  k_dense_lu<<<1, 1024, 0, stream()>>>(int(n), lu.p, piv.p, mp);
  CF_LAUNCHED();
  min_abs_pivot = read_dev(mp);
}

void DenseLu::solve(const double* b, double* x) const {
  if (n == 0) return;
  if (diagonal) {
    k_diag_solve<<<grid_for(n, 256), 256, 0, stream()>>>(n, lu.p, b, x);
    CF_LAUNCHED();
    return;
  }
  if (n <= DENSE_SM_MAX) {
    const size_t sm = size_t(n) * (n + 1) * sizeof(double);
    static bool attr = false;
    if (!attr) {
      CF_CUDA(cudaFuncSetAttribute(k_dense_solve_sm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(size_t(DENSE_SM_MAX) * (DENSE_SM_MAX + 1) * sizeof(double))));
      attr = true;
    }
    k_dense_solve_sm<<<1, 256, sm, stream()>>>(int(n), lu.p, piv.p, b, x);
  } else {
    k_dense_solve<<<1, 32, 0, stream()>>>(int(n), lu.p, piv.p, b, x);
  }
  CF_LAUNCHED();
}

// ------------------------------------------------------------------ build_amg (linsolve.cpp:170-287)
std::unique_ptr<Amg> build_amg(std::shared_ptr<Csr> A0, const int* node_of_dof, const double* B0, int m,
                               const cf_amg_options& opts) {
  if (m < 1 || m > 8) fail(CF_ERR_UNSUPPORTED, "build_amg: near-nullspace width must be 1..8");
  auto h = std::make_unique<Amg>();
  h->opts = opts;
  h->n = A0->rows;
  h->A0 = A0;
  h->m0 = m;
  h->nod0.alloc(A0->rows);
  h->B0.alloc(A0->rows * m);
  std::shared_ptr<Csr> A = A0;
  // a level-0 operator most of whose rows are a lone diagonal (the phi block's active rows): its
  // SpMVs (power iteration, residual and smoothing sweeps) run the heavy rows from a list
  if (m == 1 && !A0->split) csr_enable_row_split(*A0);
  DevBuf<int> nod(A->rows);
  DevBuf<double> B(A->rows * m);
  if (A->rows) {
    CF_CUDA(cudaMemcpyAsync(nod.p, node_of_dof, size_t(A->rows) * sizeof(int), cudaMemcpyDeviceToDevice, stream()));
    CF_CUDA(cudaMemcpyAsync(B.p, B0, size_t(A->rows) * m * sizeof(double), cudaMemcpyDeviceToDevice, stream()));
    CF_CUDA(cudaMemcpyAsync(h->nod0.p, node_of_dof, size_t(A->rows) * sizeof(int), cudaMemcpyDeviceToDevice,
                            stream()));
    CF_CUDA(cudaMemcpyAsync(h->B0.p, B0, size_t(A->rows) * m * sizeof(double), cudaMemcpyDeviceToDevice, stream()));
  }
  DevBuf<int> err(1);
  PhaseClock clk;
  // compact -> reference node ids of the current level (empty: identity, no empty nodes)
  DevBuf<int> orig_of_c;
  static const bool no_compact = std::getenv("CF_AMG_NO_COMPACT") != nullptr;  // A/B switch
  for (int lev = 0; lev < opts.max_levels; ++lev) {
    clk.lev = lev;
    const i64 n = A->rows;
    if (n <= opts.coarse_size) break;
    // n_nodes = max(node_of_dof) + 1
    i64 n_nodes;
    {
      DevBuf<int> mx(1);
      size_t bytes = 0;
      CF_CUDA(cub::DeviceReduce::Max(nullptr, bytes, nod.p, mx.p, n, stream()));
      DevBuf<unsigned char> tmp{static_cast<i64>(bytes)};
      CF_CUDA(cub::DeviceReduce::Max(tmp.p, bytes, nod.p, mx.p, n, stream()));
      count_launch();
      n_nodes = i64(read_dev(mx.p)) + 1;
    }
    // the reference's node count includes the empty nodes below the last non-empty one
    i64 n_nodes_ref = n_nodes;
    if (orig_of_c.n > 0) {
      n_nodes_ref = i64(read_dev(orig_of_c.p + n_nodes - 1)) + 1;
      if (n_nodes_ref == n_nodes) orig_of_c.release();  // no empty node: identity
    }
    // strength graph S (ascending neighbour lists)
    DevBuf<i64> nptr;
    DevBuf<int> ndofs;
    group_by_key(n, nod.p, n_nodes, nptr, ndofs);
    DevBuf<double> dsq(n_nodes);
    k_strength_diag<<<grid_for(n_nodes, 128), 128, 0, stream()>>>(n_nodes, nptr.p, ndofs.p, A->ptr.p, A->col.p,
                                                                   A->val.p, nod.p, dsq.p);
    CF_LAUNCHED();
    DevBuf<i64> sptr(n_nodes + 1);
    sptr.zero();
    DevBuf<int> ovf(n_nodes);
    ovf.zero();
    // the counting pass also stores each node's strong list (persistent scratch, SCAP per node), so
    // the fill is a compaction instead of a second pass over the matrix
    static DevBuf<int> stmp;
    if (stmp.n < n_nodes * SCAP) stmp.alloc(n_nodes * SCAP);
    k_strength<<<grid_for(n_nodes, 128), 128, 0, stream()>>>(n_nodes, nptr.p, ndofs.p, A->ptr.p, A->col.p, A->val.p,
                                                              nod.p, dsq.p, opts.strength_threshold, sptr.p, nullptr,
                                                              nullptr, 0, ovf.p, stmp.p);
    CF_LAUNCHED();
    // overflow tier for high-degree nodes
    OvfList big = make_ovf_list(n_nodes, ovf.p);
    DevBuf<i64> boff;
    DevBuf<int> bkeys, blen;
    DevBuf<double> bsums;
    if (big.n) {
      boff.alloc(big.n + 1);
      k_node_entries<<<grid_for(big.n, 128), 128, 0, stream()>>>(big.n, big.list.p, nptr.p, ndofs.p, A->ptr.p,
                                                                 pow2_at_least(2 * n_nodes), boff.p);
      CF_LAUNCHED();
      CF_CUDA(cudaMemsetAsync(boff.p + big.n, 0, sizeof(i64), stream()));
      scan_excl(boff.p, big.n + 1);
      const i64 tot = read_dev(boff.p + big.n);
      bkeys.alloc(tot);
      bsums.alloc(tot);
      blen.alloc(big.n);
      CF_CUDA(cudaMemsetAsync(bkeys.p, 0xff, size_t(tot) * sizeof(int), stream()));
      if (std::getenv("CF_STRENGTH_SERIAL")) {  // A/B switch: the one-thread-per-node tier
        k_strength_big<<<grid_for(big.n, 64), 64, 0, stream()>>>(big.n, big.list.p, boff.p, nptr.p, ndofs.p,
                                                                 A->ptr.p, A->col.p, A->val.p, nod.p, bkeys.p, bsums.p,
                                                                 blen.p);
      } else {
        CF_CUDA(cudaMemsetAsync(bsums.p, 0, size_t(tot) * sizeof(double), stream()));
        k_strength_bigw<<<grid_for(big.n, SBW_WPB), SBW_WPB * 32, 0, stream()>>>(
            big.n, big.list.p, boff.p, nptr.p, ndofs.p, A->ptr.p, A->col.p, A->val.p, nod.p, bkeys.p, bsums.p, blen.p);
      }
      CF_LAUNCHED();
      k_strength_big_emit<<<grid_for(big.n, 128), 128, 0, stream()>>>(big.n, big.list.p, boff.p, bkeys.p, bsums.p,
                                                                      blen.p, dsq.p, opts.strength_threshold, sptr.p,
                                                                      nullptr, nullptr, 0);
      CF_LAUNCHED();
    }
    scan_excl(sptr.p, n_nodes + 1);
    const i64 ns = read_dev(sptr.p + n_nodes);
    DevBuf<int> sidx(std::max<i64>(ns, 1));
    if (ns >= 8 * n_nodes)
      k_strength_compact<32><<<grid_for(n_nodes * 32, 256), 256, 0, stream()>>>(n_nodes, ovf.p, stmp.p, sptr.p, sidx.p);
    else
      k_strength_compact<1><<<grid_for(n_nodes, 256), 256, 0, stream()>>>(n_nodes, ovf.p, stmp.p, sptr.p, sidx.p);
    CF_LAUNCHED();
    if (big.n) {
      k_strength_big_emit<<<grid_for(big.n, 128), 128, 0, stream()>>>(big.n, big.list.p, boff.p, bkeys.p, bsums.p,
                                                                      blen.p, dsq.p, opts.strength_threshold, nullptr,
                                                                      sptr.p, sidx.p, 1);
      CF_LAUNCHED();
    }
    bkeys.release();
    bsums.release();
    clk.mark("strength");
    // transpose T = S^T (ascending lists): stable grouping of edges by destination
    DevBuf<i64> tptr;
    DevBuf<int> tidx(std::max<i64>(ns, 1));
    {
      DevBuf<int> src(std::max<i64>(ns, 1)), order;
      k_graph_rows<<<grid_for(n_nodes, 256), 256, 0, stream()>>>(n_nodes, sptr.p, src.p);
      CF_LAUNCHED();
      group_by_key(ns, sidx.p, n_nodes, tptr, order);
      k_gather_int<<<grid_for(ns, 256), 256, 0, stream()>>>(ns, order.p, src.p, tidx.p);
      CF_LAUNCHED();
    }
    // dependency graph N2: lower counts + upper (dependent) lists
    DevBuf<int> lower(n_nodes);
    DevBuf<i64> uptr(n_nodes + 1);
    uptr.zero();
    ovf.zero();
    // the stored upper lists: a persistent scratch (hundreds of MB at the fine levels; allocating
    // it per build from the caching allocator costs more than the pass it saves)
    static DevBuf<int> ups;
    if (ups.n < n_nodes * N2UPC) ups.alloc(n_nodes * N2UPC);
    DevBuf<int> redo(n_nodes), nlist(n_nodes), ncount(1);
    ncount.zero();
    k_n2_nodes<<<grid_for(n_nodes, 256), 256, 0, stream()>>>(n_nodes, sptr.p, tptr.p, lower.p, uptr.p, redo.p,
                                                             nlist.p, ncount.p);
    CF_LAUNCHED();
    const int nl = read_dev(ncount.p);
    if (nl > 0)
      k_n2w<<<grid_for(nl, N2WPB), N2WPB * 32, 0, stream()>>>(nl, nlist.p, sptr.p, sidx.p, tptr.p, tidx.p, lower.p,
                                                              uptr.p, nullptr, nullptr, 0, ovf.p, ups.p, redo.p);
    CF_LAUNCHED();
    clk.mark("S^T + N2 count");
    OvfList big2 = make_ovf_list(n_nodes, ovf.p);
    DevBuf<i64> noff;
    DevBuf<int> nkeys;
    if (big2.n) {
      noff.alloc(big2.n + 1);
      k_n2_cap<<<grid_for(big2.n, 128), 128, 0, stream()>>>(big2.n, big2.list.p, sptr.p, sidx.p, tptr.p,
                                                            pow2_at_least(2 * n_nodes), noff.p);
      CF_LAUNCHED();
      CF_CUDA(cudaMemsetAsync(noff.p + big2.n, 0, sizeof(i64), stream()));
      scan_excl(noff.p, big2.n + 1);
      const i64 tot = read_dev(noff.p + big2.n);
      nkeys.alloc(tot);
      CF_CUDA(cudaMemsetAsync(nkeys.p, 0xff, size_t(tot) * sizeof(int), stream()));
      k_n2_big<<<grid_for(big2.n, 64), 64, 0, stream()>>>(big2.n, big2.list.p, noff.p, sptr.p, sidx.p, tptr.p, tidx.p,
                                                          nkeys.p, lower.p, uptr.p, nullptr, nullptr, 0);
      CF_LAUNCHED();
    }
    scan_excl(uptr.p, n_nodes + 1);
    const i64 nup = read_dev(uptr.p + n_nodes);
    DevBuf<int> up(std::max<i64>(nup, 1));
    if (nl > 0) {
      k_n2w<<<grid_for(nl, N2WPB), N2WPB * 32, 0, stream()>>>(nl, nlist.p, sptr.p, sidx.p, tptr.p, tidx.p, nullptr,
                                                              nullptr, uptr.p, up.p, 1, ovf.p, nullptr, redo.p);
      CF_LAUNCHED();
      k_n2_compact<<<grid_for(i64(nl) * 32, 256), 256, 0, stream()>>>(nl, nlist.p, ovf.p, redo.p, ups.p, uptr.p, up.p);
      CF_LAUNCHED();
    }
    if (big2.n) {
      k_n2_big<<<grid_for(big2.n, 64), 64, 0, stream()>>>(big2.n, big2.list.p, noff.p, sptr.p, sidx.p, tptr.p, tidx.p,
                                                          nkeys.p, nullptr, nullptr, uptr.p, up.p, 1);
      CF_LAUNCHED();
    }
    nkeys.release();
    if (clk.on) {
      std::vector<int> rd(n_nodes);
      if (n_nodes) CF_CUDA(cudaMemcpy(rd.data(), redo.p, size_t(n_nodes) * sizeof(int), cudaMemcpyDeviceToHost));
      long long nredo = 0;
      for (int v : rd) nredo += v != 0;
      std::fprintf(stderr, "[amg L%d] n2: listed %d, global-tier %lld, strength global-tier %lld, upper %lld, redo %lld\n",
                   lev, nl, (long long)big2.n, (long long)big.n, (long long)nup, nredo);
    }
    clk.mark("S^T + N2");
    // pass 1: lexicographically-first MIS of N2 (persistent cooperative frontier kernel)
    DevBuf<int> status(n_nodes), f0(n_nodes), f1(n_nodes), sizes(3), rounds(1);
    sizes.zero();
    k_lfmis_init<<<grid_for(n_nodes, 256), 256, 0, stream()>>>(n_nodes, lower.p, uptr.p, status.p, f0.p, sizes.p);
    CF_LAUNCHED();
    {
      int bps = 0;
      CF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_lfmis, 256, 0));
      static const int bps_cap = [] {  // CF_LFMIS_BPS: blocks per SM of the cooperative grid (A/B)
        const char* e = std::getenv("CF_LFMIS_BPS");
        return e ? std::max(1, std::atoi(e)) : 4;
      }();
      const int grid = std::max(1, std::min(bps, bps_cap)) * rt().sm_count;
      const i64* a1 = uptr.p;
      const int* a2 = up.p;
      int* a3 = lower.p;  // consumed as the pending-dependency counter
      int* a4 = status.p;
      int* a5 = f0.p;
      int* a6 = f1.p;
      int* a7 = sizes.p;
      int* a8 = rounds.p;
      void* args[] = {&a1, &a2, &a3, &a4, &a5, &a6, &a7, &a8};
      CF_CUDA(cudaLaunchCooperativeKernel((void*)k_lfmis, grid, 256, args, 0, stream()));
      CF_LAUNCHED();
    }
    clk.mark("lfmis");
    if (clk.on) std::fprintf(stderr, "[amg L%d] nodes %lld strong edges %lld lfmis rounds %d\n", lev,
                             (long long)n_nodes, (long long)ns, read_dev(rounds.p));
    // aggregate ids of the roots (ascending), claims
    DevBuf<int> rootid(n_nodes + 1), agg1(n_nodes);
    k_root_flags<<<grid_for(n_nodes, 256), 256, 0, stream()>>>(n_nodes, status.p, rootid.p);
    CF_LAUNCHED();
    CF_CUDA(cudaMemsetAsync(rootid.p + n_nodes, 0, sizeof(int), stream()));
    scan_excl(rootid.p, n_nodes + 1);
    const int n1 = read_dev(rootid.p + n_nodes);
    CF_CUDA(cudaMemsetAsync(agg1.p, 0xff, size_t(n_nodes) * sizeof(int), stream()));
    k_claim<<<grid_for(n_nodes, 256), 256, 0, stream()>>>(n_nodes, status.p, rootid.p, sptr.p, sidx.p, agg1.p);
    CF_LAUNCHED();
    // pass 2 (ordered fix point) and pass 3 (new singletons, ascending)
    // (a sweep that changes nothing leaves every later sweep without effect, so sweeps run in
    // batches of P2B with one flag each and one host round trip per batch)
    constexpr int P2B = 4;
    DevBuf<int> p2(n_nodes), changed(P2B);
    CF_CUDA(cudaMemsetAsync(p2.p, 0xff, size_t(n_nodes) * sizeof(int), stream()));
    for (i64 guard = 0;; guard += P2B) {
      changed.zero();
      for (int b = 0; b < P2B; ++b) {
        k_pass2<<<grid_for(n_nodes, 256), 256, 0, stream()>>>(n_nodes, sptr.p, sidx.p, agg1.p, p2.p, changed.p + b);
        CF_LAUNCHED();
      }
      int hc[P2B];
      read_small(hc, changed.p, sizeof(hc));
      bool done = false;
      for (int b = 0; b < P2B; ++b) done = done || hc[b] == 0;
      if (done) break;
      if (guard > n_nodes + 2) fail(CF_ERR_LOGIC, "build_amg: pass-2 resolution did not converge");
    }
    DevBuf<int> p3(n_nodes + 1), agg(n_nodes);
    k_pass3_flags<<<grid_for(n_nodes, 256), 256, 0, stream()>>>(n_nodes, agg1.p, p2.p, p3.p);
    CF_LAUNCHED();
    CF_CUDA(cudaMemsetAsync(p3.p + n_nodes, 0, sizeof(int), stream()));
    scan_excl(p3.p, n_nodes + 1);
    const int n3 = read_dev(p3.p + n_nodes);
    k_final_agg<<<grid_for(n_nodes, 256), 256, 0, stream()>>>(n_nodes, agg1.p, p2.p, p3.p, n1, agg.p);
    CF_LAUNCHED();
    const i64 n_agg = i64(n1) + n3;
    if (n_agg >= n_nodes && n_nodes_ref > 1) break;  // no coarsening possible (linsolve.cpp:203)
    // reference numbering of the aggregates when empty nodes were left out
    DevBuf<int> aorig, agg_ref;
    if (orig_of_c.n > 0) {
      DevBuf<int> rid(n_nodes_ref + 1), root_of_agg(std::max(n1, 1));
      k_fill_ones<<<grid_for(n_nodes_ref, 256), 256, 0, stream()>>>(n_nodes_ref, rid.p);
      CF_LAUNCHED();
      CF_CUDA(cudaMemsetAsync(rid.p + n_nodes_ref, 0, sizeof(int), stream()));
      k_root_scatter<<<grid_for(n_nodes, 256), 256, 0, stream()>>>(n_nodes, status.p, rootid.p, orig_of_c.p, rid.p,
                                                                   root_of_agg.p);
      CF_LAUNCHED();
      scan_excl(rid.p, n_nodes_ref + 1);  // rid[i]: roots below i; rid[n_nodes_ref]: all pass-1 aggregates
      aorig.alloc(n_agg);
      k_agg_orig<<<grid_for(n_agg, 256), 256, 0, stream()>>>(n_agg, n1, root_of_agg.p, orig_of_c.p, rid.p,
                                                             n_nodes_ref, aorig.p);
      CF_LAUNCHED();
      agg_ref.alloc(n_nodes_ref);
      CF_CUDA(cudaMemcpyAsync(agg_ref.p, rid.p, size_t(n_nodes_ref) * sizeof(int), cudaMemcpyDeviceToDevice,
                              stream()));  // an empty node's aggregate: its rank among the roots
      k_agg_full<<<grid_for(n_nodes, 256), 256, 0, stream()>>>(n_nodes, agg.p, orig_of_c.p, aorig.p, agg_ref.p);
      CF_LAUNCHED();
    }

    clk.mark("pass 2/3");
    // tentative prolongator: per-aggregate QR of the near-nullspace rows
    DevBuf<int> aod(n);
    k_agg_of_dof<<<grid_for(n, 256), 256, 0, stream()>>>(n, nod.p, agg.p, aod.p);
    CF_LAUNCHED();
    DevBuf<i64> aptr;
    DevBuf<int> adofs;
    group_by_key(n, aod.p, n_agg, aptr, adofs);
    DevBuf<double> W(n * m), Q(n * m), hc(n_agg * 8);
    DevBuf<int> perm(n_agg * 8);
    DevBuf<i64> rank64(n_agg + 1);
    DevBuf<int> rank(n_agg);
    {
      // element stride st = 1 passed at run time: measured 13 ms against 40 ms for the config-3
      // u-hierarchy when the unit stride is a compile-time constant (slower generated loop nest)
      k_agg_qr<<<grid_for(n_agg, 64), 64, 0, stream()>>>(n_agg, aptr.p, adofs.p, B.p, n, m, W.p, Q.p, hc.p, perm.p,
                                                         rank.p, 1);
    }
    CF_LAUNCHED();
    k_int_to_i64<<<grid_for(n_agg, 256), 256, 0, stream()>>>(n_agg, rank.p, rank64.p);
    CF_LAUNCHED();
    CF_CUDA(cudaMemsetAsync(rank64.p + n_agg, 0, sizeof(i64), stream()));
    scan_excl(rank64.p, n_agg + 1);  // aggregate column offsets
    const i64 nc = read_dev(rank64.p + n_agg);
    if (nc == 0 || nc >= n) break;  // linsolve.cpp:226
    DevBuf<int> pos(n), agg_of(n);
    k_pos_in_agg<<<grid_for(n_agg, 256), 256, 0, stream()>>>(n_agg, aptr.p, adofs.p, pos.p, agg_of.p);
    CF_LAUNCHED();
    Csr T;
    T.rows = n;
    T.cols = nc;
    T.ptr.alloc(n + 1);
    T.ptr.zero();
    k_build_T<<<grid_for(n, 256), 256, 0, stream()>>>(n, m, agg_of.p, pos.p, aptr.p, rank.p, rank64.p, Q.p, T.ptr.p,
                                                      nullptr, nullptr, 0);
    CF_LAUNCHED();
    scan_excl(T.ptr.p, n + 1);
    T.nnz = read_dev(T.ptr.p + n);
    T.col.alloc(std::max<i64>(T.nnz, 1));
    T.val.alloc(std::max<i64>(T.nnz, 1));
    k_build_T<<<grid_for(n, 256), 256, 0, stream()>>>(n, m, agg_of.p, pos.p, aptr.p, rank.p, rank64.p, Q.p, T.ptr.p,
                                                      T.col.p, T.val.p, 1);
    CF_LAUNCHED();

    // smoothing: P = T - (w_P 2/lambda) D^-1 A T, pruned (linsolve.cpp:240-251)
    auto L = std::make_unique<AmgLevel>();
    L->inv_diag.alloc(n);
    csr_diagonal(*A, L->inv_diag.p);
    k_inv_diag<<<grid_for(n, 256), 256, 0, stream()>>>(n, L->inv_diag.p);
    CF_LAUNCHED();
    clk.mark("qr+T");
    const double lambda = estimate_lambda_max(*A, L->inv_diag.p);
    clk.mark("lambda");
    const double wp = opts.prolongation_omega * 2.0 / lambda;
    auto DAT = spgemm(*A, T, L->inv_diag.p);
    clk.mark("spgemm DAT");
    L->P = csr_axpy_prune(T, wp, *DAT);
    DAT.reset();
    L->R = transpose(*L->P);
    // row groups for the V-cycle SpMVs of the coarse levels (an aggregate's coarse dofs share their
    // pattern in A, P and R); on level 0 the row-wise kernel wins (3x the threads in flight: P
    // 0.53 vs 0.58 ms, R 0.34 vs 0.36 ms on config 3), on level 1 the groups do (A 0.117 vs
    // 0.143, P 0.041 vs 0.047, R 0.043 vs 0.051 ms)
    if (lev == 0 && m == 1) csr_enable_row_split(*L->P);  // (mostly empty rows: the active phi dofs)
    if (lev > 0) {
      L->P->grp = csr_row_groups(*L->P, 6);
      L->R->grp = csr_row_groups(*L->R, 6);
      if (!A->grp) A->grp = csr_row_groups(*A, 6);
    }
    clk.mark("P+R");
    L->A = A;
    L->jacobi_weight = opts.jacobi_omega * 2.0 / lambda;
    L->lambda = lambda;
    if (opts.smoother == 1) L->cheb_hi = gershgorin_bound(*A, L->inv_diag.p);
    L->n_nodes = n_nodes_ref;
    L->n_aggregates = n_agg + (n_nodes_ref - n_nodes);  // every empty node is its own aggregate
    L->strong_edges = ns;
    L->lfmis_rounds = read_dev(rounds.p);
    L->agg_of_node = orig_of_c.n > 0 ? std::move(agg_ref) : std::move(agg);
    // Galerkin coarse operator Ac = P^T (A P), pruned; coarse nullspace and node ids
    auto AP = spgemm(*A, *L->P);
    clk.mark("spgemm AP");
    auto Ac = spgemm(*L->R, *AP);
    clk.mark("spgemm RAP");
    AP.reset();
    csr_prune(*Ac);
    DevBuf<double> Bc(nc * m);
    DevBuf<int> cnode(nc);
    k_build_Bc<<<grid_for(n_agg, 256), 256, 0, stream()>>>(n_agg, m, aptr.p, rank.p, rank64.p, W.p, perm.p, nc, Bc.p,
                                                           cnode.p);
    CF_LAUNCHED();
    // next level's nodes: the aggregates that carry coarse dofs, renumbered in order
    if (!no_compact) {
      DevBuf<int> cid(n_agg + 1), orig_next(n_agg);
      k_nonempty_flags<<<grid_for(n_agg, 256), 256, 0, stream()>>>(n_agg, rank.p, cid.p);
      CF_LAUNCHED();
      CF_CUDA(cudaMemsetAsync(cid.p + n_agg, 0, sizeof(int), stream()));
      scan_excl(cid.p, n_agg + 1);
      k_compact_orig<<<grid_for(n_agg, 256), 256, 0, stream()>>>(n_agg, rank.p, cid.p, aorig.n > 0 ? aorig.p : nullptr,
                                                                 orig_next.p);
      CF_LAUNCHED();
      k_renumber<<<grid_for(nc, 256), 256, 0, stream()>>>(nc, cid.p, cnode.p);
      CF_LAUNCHED();
      orig_of_c = std::move(orig_next);
    }
    L->tmp_r.alloc(n);
    L->tmp_b.alloc(nc);
    L->tmp_x.alloc(nc);
    h->levels.push_back(std::move(L));
    A = std::shared_ptr<Csr>(std::move(Ac));
    B = std::move(Bc);
    nod = std::move(cnode);
  }
  if (clk.on) std::fprintf(stderr, "[amg] coarsest dense LU n=%lld after %zu levels\n", (long long)A->rows,
                           h->levels.size());
  h->coarse.factor_from_csr(*A);
  clk.mark("coarse LU");
  if (A->rows > 0 && h->coarse.min_abs_pivot == 0.0)
    fail(CF_ERR_NUMERICAL, "build_amg: coarsest-level matrix is singular");
  h->cb.alloc(std::max<i64>(A->rows, 1));
  h->cx.alloc(std::max<i64>(A->rows, 1));
  h->coarse_A = A;
  return h;
}

// linsolve.cpp:295-312, zero initial guess.  The residual r = b - A x and the post-smoothing sweep
// x + w D^-1 (b - A x) are fused into the SpMV's row epilogue (SpmvEpi), the prolongation
// x + P x_c lands in the level's scratch vector so the fused sweep can read it while writing x;
// the same IEEE operations as the separate kernels (CF_VCYCLE_UNFUSED=1 runs those).
void Amg::vcycle(const double* r, double* x) const {
  if (!dist.empty()) {
    vcycle_dist(r, x);
    return;
  }
  vcycle_range(0, r, x);
}

// the V-cycle of levels l0.. for the right-hand side b0 of level l0, output x0 (linsolve.cpp:295-312)
void Amg::vcycle_range(size_t l0, const double* b0, double* x0) const {
  static const bool unfused = std::getenv("CF_VCYCLE_UNFUSED") != nullptr;
  // A x (+ epilogue) of level l: matrix-free on the finest level when mf0 is set
  auto apply = [&](size_t l, const double* xin, double* yout, const SpmvEpi& ep) {
    if (l == 0 && mf0)
      mf_apply(*mf0, xin, yout, ep);
    else
      csr_spmv_epi(*levels[l]->A, xin, yout, ep);
  };
  // Chebyshev smoothing of level l (opts.smoother == 1) on D^-1 A over [hi / 10, hi], hi the
  // Gershgorin bound (the 15-step power estimate undershoots lambda_max by enough that the
  // polynomial amplifies the top of the spectrum: GMRES stagnated on config 3 with 1.1 lambda)
  auto chebyshev = [&](size_t l, const double* bl, double* xl, bool zero) {
    const AmgLevel& L = *levels[l];
    const i64 n = L.A->rows;
    if (L.tmp_d.n < n) L.tmp_d.alloc(n);
    const double hi = L.cheb_hi, lo = hi / 10.0;
    const double theta = 0.5 * (hi + lo), delta = 0.5 * (hi - lo), sigma = theta / delta;
    const int deg = std::max(1, opts.chebyshev_degree);
    for (int sweep = 0; sweep < std::max(1, opts.smoothing_sweeps); ++sweep) {
      const bool z = zero && sweep == 0;
      const double* r = bl;
      if (!z) {
        SpmvEpi ep;
        ep.b = bl;
        ep.mode = 1;
        apply(l, xl, L.tmp_r.p, ep);  // r = b - A x
        r = L.tmp_r.p;
      }
      k_cheb_init<<<grid_for(n, 256), 256, 0, stream()>>>(n, 1.0 / theta, L.inv_diag.p, r, L.tmp_d.p, xl, z ? 1 : 0);
      CF_LAUNCHED();
      double rho = 1.0 / sigma;
      for (int k = 1; k < deg; ++k) {
        SpmvEpi ep;
        ep.b = bl;
        ep.mode = 1;
        apply(l, xl, L.tmp_r.p, ep);
        const double rho_new = 1.0 / (2.0 * sigma - rho);
        k_cheb_step<<<grid_for(n, 256), 256, 0, stream()>>>(n, rho_new * rho, 2.0 * rho_new / delta, L.inv_diag.p,
                                                            L.tmp_r.p, L.tmp_d.p, xl);
        CF_LAUNCHED();
        rho = rho_new;
      }
    }
  };
  const bool cheb = opts.smoother == 1;
  const double* b = b0;
  for (size_t l = l0; l < levels.size(); ++l) {
    const AmgLevel& L = *levels[l];
    const i64 n = L.A->rows;
    double* xl = (l == l0) ? x0 : levels[l - 1]->tmp_x.p;
    const double w = L.jacobi_weight;
    if (cheb) {
      chebyshev(l, b, xl, true);
      SpmvEpi ep;
      ep.b = b;
      ep.mode = 1;
      apply(l, xl, L.tmp_r.p, ep);  // r = b - A x
      csr_spmv_add(*L.R, L.tmp_r.p, L.tmp_b.p, nullptr);
      b = L.tmp_b.p;
      continue;
    }
    k_jacobi0<<<grid_for(n, 256), 256, 0, stream()>>>(n, w, L.inv_diag.p, b, xl);
    CF_LAUNCHED();
    for (int s = 1; s < opts.smoothing_sweeps; ++s) {
      apply(l, xl, L.tmp_r.p, SpmvEpi{});
      k_jacobi_upd<<<grid_for(n, 256), 256, 0, stream()>>>(n, w, L.inv_diag.p, b, L.tmp_r.p, xl);
      CF_LAUNCHED();
    }
    if (unfused) {
      apply(l, xl, L.tmp_r.p, SpmvEpi{});
      vsub(b, L.tmp_r.p, L.tmp_r.p, n);  // r = b - A x
    } else {
      SpmvEpi ep;
      ep.b = b;
      ep.mode = 1;
      apply(l, xl, L.tmp_r.p, ep);  // r = b - A x
    }
    csr_spmv_add(*L.R, L.tmp_r.p, L.tmp_b.p, nullptr);  // b_c = P^T r
    b = L.tmp_b.p;
  }
  // coarsest
  const double* bc = b;
  double* xc = (levels.size() == l0) ? x0 : levels.back()->tmp_x.p;
  coarse.solve(bc, xc);
  for (size_t l = levels.size(); l-- > l0;) {
    const AmgLevel& L = *levels[l];
    const i64 n = L.A->rows;
    double* xl = (l == l0) ? x0 : levels[l - 1]->tmp_x.p;
    const double* bl = (l == l0) ? b0 : levels[l - 1]->tmp_b.p;
    if (cheb) {
      csr_spmv_add(*L.P, L.tmp_x.p, xl, xl);  // x += P x_c
      chebyshev(l, bl, xl, false);
      continue;
    }
    int s = 0;
    if (unfused || opts.smoothing_sweeps < 1) {
      csr_spmv_add(*L.P, L.tmp_x.p, xl, xl);  // x += P x_c
    } else {
      csr_spmv_add(*L.P, L.tmp_x.p, L.tmp_r.p, xl);  // t = x + P x_c
      SpmvEpi ep;
      ep.b = bl;
      ep.d = L.inv_diag.p;
      ep.w = L.jacobi_weight;
      ep.mode = 2;
      apply(l, L.tmp_r.p, xl, ep);  // x = t + w D^-1 (b - A t)
      s = 1;
    }
    for (; s < opts.smoothing_sweeps; ++s) {
      apply(l, xl, L.tmp_r.p, SpmvEpi{});
      k_jacobi_upd<<<grid_for(n, 256), 256, 0, stream()>>>(n, L.jacobi_weight, L.inv_diag.p, bl, L.tmp_r.p, xl);
      CF_LAUNCHED();
    }
  }
}

// ------------------------------------------------------------------ distributed V-cycle (§8e)
// The hierarchy is built identically on every rank; the leading levels with at least min_rows rows
// are then split by rows: each rank keeps row slices of A, P and R (carrying the undivided lane
// split) and applies only its rows, the level vectors travel by in-place all-gathers, and the
// remaining small levels run redundantly on every rank.  Every row is computed exactly as on one
// GPU, so the V-cycle output is bitwise independent of the rank count.
void Amg::distribute(const Comm* cm, i64 min_rows) {
  dist.clear();
  comm = cm;
  if (!cm || !cm->distributed() || opts.smoothing_sweeps != 1 || opts.smoother != 0) return;
  static const bool unfused = std::getenv("CF_VCYCLE_UNFUSED") != nullptr;
  if (unfused) return;
  const int P = cm->size, r = cm->rank;
  for (size_t l = 0; l < levels.size(); ++l) {
    const AmgLevel& L = *levels[l];
    const i64 n = L.A->rows, nc = L.P->cols;
    if (n < min_rows) break;
    DistLevel D;
    // row chunks aligned to the stencil format's vertex rows (d rows per vertex)
    const i64 align = L.A->st.kind == 1 ? L.A->st.d : 1;
    D.chunk = ((n + P - 1) / P + align - 1) / align * align;
    D.cchunk = (nc + P - 1) / P;
    D.lo = std::min(n, r * D.chunk);
    D.hi = std::min(n, (r + 1) * D.chunk);
    D.clo = std::min(nc, r * D.cchunk);
    D.chi = std::min(nc, (r + 1) * D.cchunk);
    D.A = csr_extract_rows(*L.A, D.lo, D.hi);
    if (L.A->st.kind == 1)
      csr_enable_stencil(*D.A, StencilCols{1, L.A->st.d, L.A->st.nn, D.lo / L.A->st.d, 0, L.A->st.inv_nn});
    D.P = csr_extract_rows(*L.P, D.lo, D.hi);
    D.R = csr_extract_rows(*L.R, D.clo, D.chi);
    D.x.alloc(P * D.chunk);
    D.r.alloc(P * D.chunk);
    D.bc.alloc(P * D.cchunk);
    dist.push_back(std::move(D));
  }
}

void Amg::vcycle_dist(const double* r, double* x) const {
  // own rows of level l's A (x global): matrix-free on the finest level when mf0 is set (the rows
  // of the vertices [lo/d, hi/d), bitwise the rows of the undivided matrix-free apply)
  auto dist_apply = [&](size_t l, const DistLevel& D, const double* xin, double* yout, const SpmvEpi& ep) {
    if (l == 0 && mf0) {
      MfOp op = *mf0;
      const i64 dd = mf0->P->g.d;
      op.x_off = 0;
      op.y_lo = D.lo / dd;
      op.y_hi = D.hi / dd;
      mf_apply(op, xin, yout, ep);
    } else {
      csr_spmv_epi(*D.A, xin, yout, ep);
    }
  };
  const size_t nd = dist.size();
  const double* b = r;
  for (size_t l = 0; l < nd; ++l) {  // down: pre-smooth (redundant), own residual rows, own R rows
    const AmgLevel& L = *levels[l];
    const DistLevel& D = dist[l];
    const i64 n = L.A->rows;
    k_jacobi0<<<grid_for(n, 256), 256, 0, stream()>>>(n, L.jacobi_weight, L.inv_diag.p, b, D.x.p);
    CF_LAUNCHED();
    SpmvEpi ep;
    ep.b = b + D.lo;
    ep.mode = 1;
    if (D.hi > D.lo) dist_apply(l, D, D.x.p, D.r.p + D.lo, ep);  // r = b - A x (own rows)
    comm->allgather_inplace(D.r.p, D.chunk);
    if (D.chi > D.clo) csr_spmv_add(*D.R, D.r.p, D.bc.p + D.clo, nullptr);  // b_c = P^T r (own rows)
    comm->allgather_inplace(D.bc.p, D.cchunk);
    b = D.bc.p;
  }
  // the small levels and the coarsest solve: redundant on every rank
  double* xc = levels[nd - 1]->tmp_x.p;
  vcycle_range(nd, b, xc);
  for (size_t l = nd; l-- > 0;) {  // up: own rows of t = x + P x_c and of the post-smoothing sweep
    const AmgLevel& L = *levels[l];
    const DistLevel& D = dist[l];
    const double* bl = (l == 0) ? r : dist[l - 1].bc.p;
    const double* xcl = (l + 1 == nd) ? levels[l]->tmp_x.p : dist[l + 1].x.p;
    if (D.hi > D.lo) csr_spmv_add(*D.P, xcl, D.r.p + D.lo, D.x.p + D.lo);
    comm->allgather_inplace(D.r.p, D.chunk);
    SpmvEpi ep;
    ep.b = bl + D.lo;
    ep.d = L.inv_diag.p + D.lo;
    ep.w = L.jacobi_weight;
    ep.mode = 2;
    ep.xoff = D.lo;
    if (D.hi > D.lo) dist_apply(l, D, D.r.p, D.x.p + D.lo, ep);
    comm->allgather_inplace(D.x.p, D.chunk);
  }
  vcopy(x, dist[0].x.p, levels[0]->A->rows);
}

// ------------------------------------------------------------------ input identity (reuse)
namespace {
__global__ void k_neq(i64 nwords, const unsigned* __restrict__ a, const unsigned* __restrict__ b, int* flag) {
  for (i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x; i < nwords; i += i64(gridDim.x) * blockDim.x)
    if (a[i] != b[i]) {
      *flag = 1;
      return;
    }
}
}  // namespace

bool bitwise_equal(const void* a, const void* b, size_t bytes) {
  if (bytes == 0 || a == b) return true;
  if (bytes % 4) fail(CF_ERR_LOGIC, "bitwise_equal: size must be a multiple of 4");
  DevBuf<int> flag(1);
  flag.zero();
  const i64 nw = i64(bytes / 4);
  k_neq<<<int(std::min<i64>(4096, (nw + 255) / 256)), 256, 0, stream()>>>(nw, static_cast<const unsigned*>(a),
                                                                         static_cast<const unsigned*>(b), flag.p);
  CF_LAUNCHED();
  return read_dev(flag.p) == 0;
}

bool Amg::same_inputs(const Csr& A, const int* node_of_dof, const double* B, int m, const cf_amg_options& o) const {
  if (!A0 || m != m0 || A.rows != A0->rows || A.cols != A0->cols || A.nnz != A0->nnz) return false;
  if (o.strength_threshold != opts.strength_threshold || o.prolongation_omega != opts.prolongation_omega ||
      o.jacobi_omega != opts.jacobi_omega || o.smoothing_sweeps != opts.smoothing_sweeps ||
      o.coarse_size != opts.coarse_size || o.max_levels != opts.max_levels || o.smoother != opts.smoother ||
      o.chebyshev_degree != opts.chebyshev_degree)
    return false;
  const bool same_matrix = &A == A0.get() ||  // the very matrix the hierarchy was built from
                           (bitwise_equal(A.ptr.p, A0->ptr.p, size_t(A.rows + 1) * sizeof(i64)) &&
                            bitwise_equal(A.col.p, A0->col.p, size_t(A.nnz) * sizeof(int)) &&
                            bitwise_equal(A.val.p, A0->val.p, size_t(A.nnz) * sizeof(double)));
  return same_matrix && bitwise_equal(node_of_dof, nod0.p, size_t(A.rows) * sizeof(int)) &&
         bitwise_equal(B, B0.p, size_t(A.rows) * m * sizeof(double));
}

// ------------------------------------------------------------------ block preconditioner
std::unique_ptr<BlockPrec> build_block_prec(const BlockSystem& J, int kind, const cf_amg_options& o,
                                            const NullspaceDev* ns, const BlockPrec* prev) {
  auto p = std::make_unique<BlockPrec>();
  p->kind = kind;
  p->nu = J.nu;
  p->np = J.np;
  static const bool no_reuse = std::getenv("CF_NO_AMG_REUSE") != nullptr;  // rebuild every hierarchy
  if (kind == 1 && ns && prev && prev->kind == 1 && !no_reuse) {
    if (prev->amg_u && prev->amg_u->same_inputs(*J.uu, ns->u_node, ns->u_modes, ns->m_u, o)) p->amg_u = prev->amg_u;
    if (prev->amg_p && prev->amg_p->same_inputs(*J.pp, ns->p_node, ns->p_modes, 1, o)) p->amg_p = prev->amg_p;
    if (!p->amg_u) p->amg_u = build_amg(J.uu, ns->u_node, ns->u_modes, ns->m_u, o);
    if (!p->amg_p) p->amg_p = build_amg(J.pp, ns->p_node, ns->p_modes, 1, o);
    return p;
  }
  if (kind == 0) {  // exact: dense LU of each diagonal block (small systems only)
    p->lu_u = std::make_shared<DenseLu>();
    p->lu_p = std::make_shared<DenseLu>();
    p->lu_u->factor_from_csr(*J.uu);
    p->lu_p->factor_from_csr(*J.pp);
    if ((J.nu > 0 && p->lu_u->min_abs_pivot == 0.0) || (J.np > 0 && p->lu_p->min_abs_pivot == 0.0))
      fail(CF_ERR_NUMERICAL, "BlockPreconditioner: block factorization failed");
  } else if (kind == 1) {
    if (ns) {
      p->amg_u = build_amg(J.uu, ns->u_node, ns->u_modes, ns->m_u, o);
      p->amg_p = build_amg(J.pp, ns->p_node, ns->p_modes, 1, o);
    } else {
      DevBuf<int> idu(J.nu), idp(J.np);
      DevBuf<double> onu(J.nu), onp(J.np);
      k_iota<<<grid_for(J.nu, 256), 256, 0, stream()>>>(J.nu, idu.p);
      CF_LAUNCHED();
      k_iota<<<grid_for(J.np, 256), 256, 0, stream()>>>(J.np, idp.p);
      CF_LAUNCHED();
      vfill(onu.p, 1.0, J.nu);
      vfill(onp.p, 1.0, J.np);
      p->amg_u = build_amg(J.uu, idu.p, onu.p, 1, o);
      p->amg_p = build_amg(J.pp, idp.p, onp.p, 1, o);
    }
  } else if (kind == 2) {
    p->inv_u.alloc(J.nu);
    p->inv_p.alloc(J.np);
    csr_diagonal(*J.uu, p->inv_u.p);
    csr_diagonal(*J.pp, p->inv_p.p);
    k_inv_diag_one<<<grid_for(J.nu, 256), 256, 0, stream()>>>(J.nu, p->inv_u.p);
    CF_LAUNCHED();
    k_inv_diag_one<<<grid_for(J.np, 256), 256, 0, stream()>>>(J.np, p->inv_p.p);
    CF_LAUNCHED();
  } else {
    fail(CF_ERR_INVALID_ARGUMENT, "unknown preconditioner kind");
  }
  return p;
}

void BlockPrec::apply(const double* r, double* z) const {  // linsolve.cpp:398-415
  if (kind == 0) {
    lu_u->solve(r, z);
    lu_p->solve(r + nu, z + nu);
  } else if (kind == 1) {
    // the two V-cycles are independent (separate hierarchies, work vectors and output ranges): the
    // phi cycle runs on the auxiliary stream while the u cycle runs on the library stream, so
    // the small coarse-level kernels of one overlap the other
    static const bool serial_env = std::getenv("CF_SERIAL_VCYCLES") != nullptr;
    Runtime& R = rt();
    if (serial_env || serial || np == 0) {
      amg_u->vcycle(r, z);
      amg_p->vcycle(r + nu, z + nu);
      return;
    }
    if (!R.aux) {
      CF_CUDA(cudaStreamCreateWithFlags(&R.aux, cudaStreamNonBlocking));
      CF_CUDA(cudaEventCreateWithFlags(&R.ev_fork, cudaEventDisableTiming));
      CF_CUDA(cudaEventCreateWithFlags(&R.ev_join, cudaEventDisableTiming));
    }
    const cudaStream_t main = R.stream;
    CF_CUDA(cudaEventRecord(R.ev_fork, main));
    CF_CUDA(cudaStreamWaitEvent(R.aux, R.ev_fork, 0));
    R.stream = R.aux;
    try {
      amg_p->vcycle(r + nu, z + nu);
    } catch (...) {
      R.stream = main;
      throw;
    }
    R.stream = main;
    CF_CUDA(cudaEventRecord(R.ev_join, R.aux));
    amg_u->vcycle(r, z);
    CF_CUDA(cudaStreamWaitEvent(main, R.ev_join, 0));
  } else {
    vdiag_mul(inv_u.p, r, z, 1.0, nu);
    vdiag_mul(inv_p.p, r + nu, z + nu, 1.0, np);
  }
}

}  // namespace cfb

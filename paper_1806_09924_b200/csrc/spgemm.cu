// Deterministic sparse kernels for the AMG setup: Gustavson SpGEMM,
// transpose, union-axpy with pruning, prune, diagonal extraction.
//
// SpGEMM C = diag(s) A B (linsolve.cpp:248-263: D^-1 A T, A P, P^T (A P)) in three passes:
//   1. symbolic count — per row a shared-memory hash set of the output columns (warp per row,
//      512 slots; rows that overflow retry with 2048 slots, then a CTA with 16384 slots);
//   2. symbolic fill  — the same hash sized to the known row length, then a bitonic sort of the
//      unique columns (sorted CSR);
//   3. numeric        — the row's columns are loaded into a shared-memory hash whose slots carry
//      the accumulators.  A warp processes G = 32/L consecutive A entries at once (L lanes per
//      B row); lanes compute (slot, value) pairs in parallel, then the G groups add in ascending
//      k order, so every C(i,j) is the k-ascending sequential sum sum_k (s_i A_ik) B_kj — the same
//      IEEE sequence as Eigen's conservative sparse product and the oracle, with no
//      floating-point atomics and independent of the launch configuration.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <climits>
#include <cstdlib>

#include "cf_vec.hpp"

namespace cfb {

namespace {

constexpr int EMPTY = -1;

// Fibonacci hashing: the HIGH bits of the product (the low bits of key * odd only permute the
// residues of key mod cap, so clustered keys - the coarse dofs of neighbouring aggregates -
// collide in runs).  mask = cap - 1 with cap a power of two (-DCF_LOWHASH: the low-bit form, A/B).
__device__ __forceinline__ unsigned hslot(int key, unsigned mask) {
  const unsigned h = unsigned(key) * 2654435761u;
#ifdef CF_LOWHASH
  return h & mask;
#else
  return mask ? (h >> (32 - __popc(mask))) : 0u;
#endif
}

// insert key; returns 1 if newly inserted, 0 if present, -1 if the table is full (bounded
// probing: a full table can never hang the kernel)
__device__ __forceinline__ int hinsert(int* tab, unsigned mask, int key) {
  unsigned s = hslot(key, mask);
  for (unsigned p = 0; p <= mask; ++p) {
    const int cur = tab[s];
    if (cur == key) return 0;
    if (cur == EMPTY) {
      const int old = atomicCAS(&tab[s], EMPTY, key);
      if (old == EMPTY) return 1;
      if (old == key) return 0;
    }
    s = (s + 1) & mask;
  }
  return -1;
}

// slot of a present key (read-only probe)
__device__ __forceinline__ int hfind(const int* tab, unsigned mask, int key) {
  unsigned s = hslot(key, mask);
  for (unsigned p = 0; p <= mask; ++p) {
    const int cur = tab[s];
    if (cur == key) return int(s);
    if (cur == EMPTY) return -1;
    s = (s + 1) & mask;
  }
  return -1;
}

__global__ void k_row_bound(i64 rows, const i64* __restrict__ ap, const int* __restrict__ ac,
                            const i64* __restrict__ bp, i64* __restrict__ ub) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  i64 s = 0;
  for (i64 k = ap[i]; k < ap[i + 1]; ++k) {
    const int c = ac[k];
    s += bp[c + 1] - bp[c];
  }
  ub[i] = s;
}

__global__ void k_max_row(i64 rows, const i64* __restrict__ p, unsigned long long* __restrict__ mx) {
  __shared__ unsigned long long sm[256];
  unsigned long long m = 0;
  for (i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x; i < rows; i += i64(gridDim.x) * blockDim.x)
    m = max(m, (unsigned long long)(p[i + 1] - p[i]));
  sm[threadIdx.x] = m;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sm[threadIdx.x] = max(sm[threadIdx.x], sm[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) atomicMax(mx, sm[0]);  // one atomic per block
}

template <int WPB>
__device__ __forceinline__ void bitonic_warp(int* Bf, int n2, int lane) {
  for (int k2 = 2; k2 <= n2; k2 <<= 1)
    for (int j = k2 >> 1; j > 0; j >>= 1) {
      for (int t = lane; t < n2; t += 32) {
        const int ixj = t ^ j;
        if (ixj > t) {
          const int a = Bf[t], b = Bf[ixj];
          const bool up = (t & k2) == 0;
          if ((a > b) == up) {
            Bf[t] = b;
            Bf[ixj] = a;
          }
        }
      }
      __syncwarp();
    }
}

// --- symbolic, warp per row: G = 32/L consecutive A entries per step (set semantics, any order)
// mode 0: cnt[row] = unique count or -1 (overflow); mode 1: sorted columns -> ccol
template <int CAP, int L, int WPB, int MODE>
__global__ void __launch_bounds__(WPB * 32) k_sym(const int* __restrict__ rowlist, i64 nrows,
                                                  const i64* __restrict__ ap, const int* __restrict__ ac,
                                                  const i64* __restrict__ bp, const int* __restrict__ bc,
                                                  i64* __restrict__ cnt, const i64* __restrict__ cptr,
                                                  int* __restrict__ ccol) {
  constexpr int G = 32 / L;
  __shared__ int tab[WPB][CAP];
  __shared__ int buf[MODE == 1 ? WPB : 1][MODE == 1 ? CAP : 1];
  __shared__ int nuniq[WPB];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const i64 r = i64(blockIdx.x) * WPB + w;
  if (r >= nrows) return;
  const i64 i = rowlist ? rowlist[r] : r;
  int* T = tab[w];
  for (int s = lane; s < CAP; s += 32) T[s] = EMPTY;
  __syncwarp();
  const unsigned mask = CAP - 1;
  const int g = lane / L, lig = lane % L;
  int mine = 0;
  bool full = false;
  const i64 a0 = ap[i], a1 = ap[i + 1];
  for (i64 kb0 = a0; kb0 < a1 && !full; kb0 += G) {
    const i64 ka = kb0 + g;
    if (ka < a1) {
      const int k = ac[ka];
      for (i64 q = bp[k] + lig; q < bp[k + 1]; q += L) {
        const int r2 = hinsert(T, mask, bc[q]);
        if (r2 < 0) full = true; else mine += r2;
      }
    }
    int tot = mine;
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    full = __any_sync(0xffffffffu, full) || tot > (CAP * 3) / 4;
  }
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  __syncwarp();
  if (full || mine > (CAP * 3) / 4) {
    if (MODE != 1 && lane == 0) cnt[i] = -1;  // overflow: retried by the next tier
    return;
  }
  if (MODE == 0) {
    if (lane == 0) cnt[i] = mine;
    return;
  }
  if (MODE == 2) {  // count + spill the unsorted unique columns to scratch (ccol at cptr[i])
    if (lane == 0) nuniq[w] = 0;
    __syncwarp();
    const i64 base = cptr[i];
    for (int s = lane; s < CAP; s += 32) {
      const int key = T[s];
      if (key != EMPTY) ccol[base + atomicAdd(&nuniq[w], 1)] = key;
    }
    if (lane == 0) cnt[i] = mine;
    return;
  }
  int* Bf = buf[w];
  if (lane == 0) nuniq[w] = 0;
  __syncwarp();
  for (int s = lane; s < CAP; s += 32) {
    const int key = T[s];
    if (key != EMPTY) Bf[atomicAdd(&nuniq[w], 1)] = key;
  }
  __syncwarp();
  int n2 = 1;
  while (n2 < mine) n2 <<= 1;
  for (int s = mine + lane; s < n2; s += 32) Bf[s] = INT_MAX;
  __syncwarp();
  bitonic_warp<WPB>(Bf, n2, lane);
  const i64 base = cptr[i];
  for (int t = lane; t < mine; t += 32) ccol[base + t] = Bf[t];
}

// sort each row's spilled columns (scratch at soff[i], length cnt) into the CSR (warp per row)
template <int CAP, int WPB>
__global__ void __launch_bounds__(WPB * 32) k_sort_rows(const int* __restrict__ rowlist, i64 nrows,
                                                        const i64* __restrict__ soff, const int* __restrict__ scratch,
                                                        const i64* __restrict__ cptr, int* __restrict__ ccol) {
  __shared__ int Bf[WPB][CAP];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const i64 r = i64(blockIdx.x) * WPB + w;
  if (r >= nrows) return;
  const i64 i = rowlist ? rowlist[r] : r;
  const i64 c0 = cptr[i];
  const int n = int(cptr[i + 1] - c0);
  const int* src = scratch + soff[i];
  int n2 = 1;
  while (n2 < n) n2 <<= 1;
  for (int t = lane; t < n2; t += 32) Bf[w][t] = t < n ? src[t] : INT_MAX;
  __syncwarp();
  bitonic_warp<WPB>(Bf[w], n2, lane);
  for (int t = lane; t < n; t += 32) ccol[c0 + t] = Bf[w][t];
}

__global__ void k_scatter_len(const int* __restrict__ list, int n, const i64* __restrict__ len, i64* __restrict__ out) {
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < n) out[list[t]] = len[list[t]];
}

__global__ void k_spill_cap(i64 m, const i64* __restrict__ ub, i64 cap, i64* __restrict__ out) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < m) out[i] = ub[i] < cap ? ub[i] : cap;
}

// --- symbolic, CTA per row (rows beyond the warp tiers) -----------------------------------
template <int CAP>
__global__ void __launch_bounds__(256) k_sym_cta(const int* __restrict__ rowlist, i64 nrows,
                                                 const i64* __restrict__ ap, const int* __restrict__ ac,
                                                 const i64* __restrict__ bp, const int* __restrict__ bc,
                                                 i64* __restrict__ cnt, const i64* __restrict__ cptr,
                                                 int* __restrict__ ccol, int mode, int* __restrict__ overflow) {
  extern __shared__ int sm[];
  int* T = sm;         // CAP
  int* Bf = sm + CAP;  // CAP (mode 1)
  __shared__ int nuniq;
  __shared__ int sfull;
  const i64 r = blockIdx.x;
  if (r >= nrows) return;
  const i64 i = rowlist ? rowlist[r] : r;
  for (int s = threadIdx.x; s < CAP; s += blockDim.x) T[s] = EMPTY;
  if (threadIdx.x == 0) {
    nuniq = 0;
    sfull = 0;
  }
  __syncthreads();
  const unsigned mask = CAP - 1;
  for (i64 ka = ap[i]; ka < ap[i + 1]; ++ka) {
    const int k = ac[ka];
    for (i64 kb = bp[k] + threadIdx.x; kb < bp[k + 1]; kb += blockDim.x) {
      const int r2 = hinsert(T, mask, bc[kb]);
      if (r2 > 0) atomicAdd(&nuniq, 1);
      if (r2 < 0) sfull = 1;
    }
    if (nuniq > (CAP * 3) / 4 || sfull) break;  // benign race: only an early exit
  }
  __syncthreads();
  const int mine = nuniq;
  if (mine > (CAP * 3) / 4 || sfull) {
    if (threadIdx.x == 0) *overflow = 1;
    return;
  }
  if (mode == 0) {
    if (threadIdx.x == 0) cnt[i] = mine;
    return;
  }
  int n2 = 1;
  while (n2 < mine) n2 <<= 1;
  __syncthreads();
  if (threadIdx.x == 0) nuniq = 0;
  __syncthreads();
  for (int s = threadIdx.x; s < CAP; s += blockDim.x) {
    const int key = T[s];
    if (key != EMPTY) Bf[atomicAdd(&nuniq, 1)] = key;
  }
  __syncthreads();
  for (int s = mine + threadIdx.x; s < n2; s += blockDim.x) Bf[s] = INT_MAX;
  __syncthreads();
  for (int k2 = 2; k2 <= n2; k2 <<= 1)
    for (int j = k2 >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < n2; t += blockDim.x) {
        const int ixj = t ^ j;
        if (ixj > t) {
          const int a = Bf[t], b = Bf[ixj];
          const bool up = (t & k2) == 0;
          if ((a > b) == up) {
            Bf[t] = b;
            Bf[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  const i64 base = cptr[i];
  for (int t = threadIdx.x; t < mine; t += blockDim.x) ccol[base + t] = Bf[t];
}

// --- numeric, warp per row: hash slots carry the accumulators; ordered group adds ------------
template <int CAP, int L, int WPB, int CMAX>
__global__ void __launch_bounds__(WPB * 32) k_num(const int* __restrict__ rowlist, i64 nrows,
                                                  const i64* __restrict__ ap, const int* __restrict__ ac,
                                                  const double* __restrict__ av, const double* __restrict__ rs,
                                                  const i64* __restrict__ bp, const int* __restrict__ bc,
                                                  const double* __restrict__ bv, const i64* __restrict__ cp,
                                                  const int* __restrict__ cc, double* __restrict__ cv) {
  constexpr int G = 32 / L;
  __shared__ int tab[WPB][CAP];
  __shared__ double acc[WPB][CAP];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const i64 r = i64(blockIdx.x) * WPB + w;
  if (r >= nrows) return;
  const i64 i = rowlist ? rowlist[r] : r;
  int* T = tab[w];
  double* Acc = acc[w];
  for (int s = lane; s < CAP; s += 32) {
    T[s] = EMPTY;
    Acc[s] = 0.0;
  }
  __syncwarp();
  const unsigned mask = CAP - 1;
  const i64 c0 = cp[i];
  const int nc = int(cp[i + 1] - c0);
  for (int t = lane; t < nc; t += 32) hinsert(T, mask, cc[c0 + t]);
  __syncwarp();
  const double si = rs ? rs[i] : 1.0;
  const int g = lane / L, lig = lane % L;
  const i64 a0 = ap[i], a1 = ap[i + 1];
  static_assert(CMAX <= 16, "k_num: product buffer");
  for (i64 kb0 = a0; kb0 < a1; kb0 += G) {
    const i64 ka = kb0 + g;
    int slot[CMAX];
    double val[CMAX];
    int np = 0;
    if (ka < a1) {
      const int k = ac[ka];
      const double a = rs ? si * av[ka] : av[ka];
      if constexpr (L >= 16) {  // measured: a loss for the 4- and 8-lane groups
        // issue all of the lane's B loads first (in flight together), then the hash lookups
        const i64 q0 = bp[k] + lig, q1 = bp[k + 1];
        const i64 nq = q1 > q0 ? (q1 - q0 + L - 1) / L : 0;
        np = int(nq < CMAX ? nq : CMAX);
        int cb[CMAX];
        double vb[CMAX];
#pragma unroll
        for (int t = 0; t < CMAX; ++t)
          if (t < np) {
            cb[t] = bc[q0 + i64(t) * L];
            vb[t] = bv[q0 + i64(t) * L];
          }
#pragma unroll
        for (int t = 0; t < CMAX; ++t)
          if (t < np) {
            slot[t] = hfind(T, mask, cb[t]);
            val[t] = a * vb[t];
          }
      } else {
        for (i64 q = bp[k] + lig; q < bp[k + 1] && np < CMAX; q += L) {
          slot[np] = hfind(T, mask, bc[q]);
          val[np] = a * bv[q];
          ++np;
        }
      }
    }
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {  // ascending k: group gg holds A entry kb0 + gg
      if (g == gg)
        for (int t = 0; t < np; ++t) Acc[slot[t]] += val[t];
      __syncwarp();
    }
  }
  for (int t = lane; t < nc; t += 32) cv[c0 + t] = Acc[hfind(T, mask, cc[c0 + t])];
}

__device__ __forceinline__ int lower_bound_sm(const int* a, int n, int key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// numeric, CTA per row (long rows): sorted columns in smem, binary-search slots, k sequential
__global__ void __launch_bounds__(256) k_num_cta(const int* __restrict__ rowlist, i64 nrows,
                                                 const i64* __restrict__ ap, const int* __restrict__ ac,
                                                 const double* __restrict__ av, const double* __restrict__ rs,
                                                 const i64* __restrict__ bp, const int* __restrict__ bc,
                                                 const double* __restrict__ bv, const i64* __restrict__ cp,
                                                 const int* __restrict__ cc, double* __restrict__ cv) {
  extern __shared__ unsigned char smraw[];
  const i64 r = blockIdx.x;
  if (r >= nrows) return;
  const i64 i = rowlist ? rowlist[r] : r;
  const i64 c0 = cp[i];
  const int nc = int(cp[i + 1] - c0);
  double* acc = reinterpret_cast<double*>(smraw);
  int* cols = reinterpret_cast<int*>(acc + nc);
  for (int t = threadIdx.x; t < nc; t += blockDim.x) {
    cols[t] = cc[c0 + t];
    acc[t] = 0.0;
  }
  __syncthreads();
  const double si = rs ? rs[i] : 1.0;
  for (i64 ka = ap[i]; ka < ap[i + 1]; ++ka) {
    const int k = ac[ka];
    const double a = rs ? si * av[ka] : av[ka];
    for (i64 kb = bp[k] + threadIdx.x; kb < bp[k + 1]; kb += blockDim.x) {
      const int pos = lower_bound_sm(cols, nc, bc[kb]);
      acc[pos] += a * bv[kb];
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < nc; t += blockDim.x) cv[c0 + t] = acc[t];
}

// numeric, CTA per row for products with few, long rows (the coarse levels' P^T (A P): a few
// hundred output rows of B rows with hundreds of entries, too few rows to occupy the GPU one warp
// each).  As k_num_cta, with the entries of B row k+1 (E per thread) loaded while row k is applied
// and shared memory sized to the longest output row, so several CTAs share an SM.
template <int E>
__global__ void __launch_bounds__(256) k_num_cta_pf(const int* __restrict__ rowlist, i64 nrows,
                                                    const i64* __restrict__ ap, const int* __restrict__ ac,
                                                    const double* __restrict__ av, const double* __restrict__ rs,
                                                    const i64* __restrict__ bp, const int* __restrict__ bc,
                                                    const double* __restrict__ bv, const i64* __restrict__ cp,
                                                    const int* __restrict__ cc, double* __restrict__ cv) {
  extern __shared__ unsigned char smraw[];
  const i64 r = blockIdx.x;
  if (r >= nrows) return;
  const i64 i = rowlist ? rowlist[r] : r;
  const i64 c0 = cp[i];
  const int nc = int(cp[i + 1] - c0);
  double* acc = reinterpret_cast<double*>(smraw);
  int* cols = reinterpret_cast<int*>(acc + nc);
  for (int t = threadIdx.x; t < nc; t += blockDim.x) {
    cols[t] = cc[c0 + t];
    acc[t] = 0.0;
  }
  __syncthreads();
  const double si = rs ? rs[i] : 1.0;
  const i64 a0 = ap[i], a1 = ap[i + 1];
  int cb[E], nb[E];
  double vb[E], wb[E], ca = 0.0, na = 0.0;
  auto load = [&](i64 ka, int* kc, double* kv, double& a) {
    const int k = ac[ka];
    a = rs ? si * av[ka] : av[ka];
    const i64 q0 = bp[k], q1 = bp[k + 1];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const i64 q = q0 + threadIdx.x + i64(e) * blockDim.x;
      kc[e] = q < q1 ? bc[q] : -1;
      kv[e] = q < q1 ? bv[q] : 0.0;
    }
  };
  if (a0 < a1) load(a0, cb, vb, ca);
  for (i64 ka = a0; ka < a1; ++ka) {
    if (ka + 1 < a1) load(ka + 1, nb, wb, na);
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (cb[e] >= 0) {
        const int pos = lower_bound_sm(cols, nc, cb[e]);
        acc[pos] += ca * vb[e];
      }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; ++e) {
      cb[e] = nb[e];
      vb[e] = wb[e];
    }
    ca = na;
  }
  for (int t = threadIdx.x; t < nc; t += blockDim.x) cv[c0 + t] = acc[t];
}

// symbolic, CTA per row with one byte flag per output column (columns < FLAG_MAX): the row's B
// rows set their flags (benign identical writes, no atomics), then MODE 0 counts them and MODE 1
// writes the set columns in ascending order (a block scan over contiguous column ranges).
constexpr int FLAG_MAX = 96 * 1024;
template <int MODE>
__global__ void __launch_bounds__(256) k_sym_flags(i64 rows, const i64* __restrict__ ap, const int* __restrict__ ac,
                                                   const i64* __restrict__ bp, const int* __restrict__ bc, int ncols,
                                                   i64* __restrict__ cnt_or_ptr, int* __restrict__ ccol) {
  extern __shared__ unsigned char flg[];
  __shared__ int part[256];
  const i64 i = blockIdx.x;
  if (i >= rows) return;
  for (int t = threadIdx.x; t < ncols; t += blockDim.x) flg[t] = 0;
  __syncthreads();
  for (i64 ka = ap[i]; ka < ap[i + 1]; ++ka) {
    const int k = ac[ka];
    for (i64 q = bp[k] + threadIdx.x; q < bp[k + 1]; q += blockDim.x) flg[bc[q]] = 1;
  }
  __syncthreads();
  const int chunk = (ncols + blockDim.x - 1) / blockDim.x;
  const int lo = min(ncols, int(threadIdx.x) * chunk), hi = min(ncols, lo + chunk);
  int c = 0;
  for (int t = lo; t < hi; ++t) c += flg[t];
  part[threadIdx.x] = c;
  __syncthreads();
  if (MODE == 0) {
    if (threadIdx.x == 0) {
      int s = 0;
      for (int t = 0; t < int(blockDim.x); ++t) s += part[t];
      cnt_or_ptr[i] = s;
    }
    return;
  }
  // exclusive scan of the per-thread counts (256 values, one warp of partial sums)
  if (threadIdx.x < 32) {
    int run = 0;
    for (int w = 0; w < 8; ++w) {
      const int t = w * 32 + int(threadIdx.x);
      const int v = part[t];
      int incl = v;
      for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(0xffffffffu, incl, o);
        if (threadIdx.x >= o) incl += n;
      }
      part[t] = run + incl - v;
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
  __syncthreads();
  i64 o = cnt_or_ptr[i] + part[threadIdx.x];
  for (int t = lo; t < hi; ++t)
    if (flg[t]) ccol[o++] = t;
}

// ---- staged CTA-per-row kernels of the small-product path --------------------------------------
// k_sym_flags / k_num_cta_pf walk a row's A entries one after the other, each a dependent global
// round trip (column -> B row pointers -> B row), so a row of R with 800 entries takes ~1 ms
// whatever the GPU (56 such launches were 31 ms of the config-3 step).  Here the row's (A entry,
// B entry) products are flattened: a chunk of up to 256 A entries loads its B row ranges at once,
// a block scan numbers the products, and every thread fetches products f, f + 256, ... (all loads
// independent).  The symbolic pass sets their flags; the numeric pass stages product and output
// slot in shared memory and then adds them A entry by A entry (one barrier each, shared memory
// only), which is the order of every other numeric kernel.
constexpr int ST_CH = 2048;  // staged products per sub-chunk (>= the longest B row of the path, 1024)

// exclusive block scan of one int per thread (256 threads); returns the total; off[256] in smem
__device__ __forceinline__ int block_scan_256(int v, int* off, int* wsum) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += n;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  int base = 0, tot = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int x = wsum[i];
    if (i < w) base += x;
    tot += x;
  }
  off[threadIdx.x] = base + incl - v;
  if (threadIdx.x == 255) off[256] = tot;
  __syncthreads();
  return tot;
}
// last e in [0, n) with off[e] <= f (off ascending, off[0] = 0)
__device__ __forceinline__ int seg_of(const int* off, int n, int f) {
  int lo = 0, hi = n;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (off[mid] <= f) lo = mid; else hi = mid;
  }
  return lo;
}

template <int MODE>
__global__ void __launch_bounds__(256) k_sym_flags_st(i64 rows, const i64* __restrict__ ap, const int* __restrict__ ac,
                                                      const i64* __restrict__ bp, const int* __restrict__ bc,
                                                      int ncols, i64* __restrict__ cnt_or_ptr,
                                                      int* __restrict__ ccol) {
  extern __shared__ unsigned char flg[];
  __shared__ int off[257], wsum[8];
  __shared__ i64 q0s[256];
  const i64 i = blockIdx.x;
  if (i >= rows) return;
  for (int t = threadIdx.x; t < ncols; t += blockDim.x) flg[t] = 0;
  const i64 a0 = ap[i], a1 = ap[i + 1];
  for (i64 base = a0; base < a1; base += 256) {
    const i64 ka = base + threadIdx.x;
    int len = 0;
    if (ka < a1) {
      const int k = ac[ka];
      const i64 q0 = bp[k];
      len = int(bp[k + 1] - q0);
      q0s[threadIdx.x] = q0;
    }
    const int tot = block_scan_256(len, off, wsum);  // (its barriers also order the flag zeroing)
    const int ne = int(min(i64(256), a1 - base));
    for (int f = threadIdx.x; f < tot; f += 256) {
      const int e = seg_of(off, ne, f);
      flg[bc[q0s[e] + (f - off[e])]] = 1;
    }
    __syncthreads();
  }
  __syncthreads();
  const int chunk = (ncols + blockDim.x - 1) / blockDim.x;
  const int lo = min(ncols, int(threadIdx.x) * chunk), hi = min(ncols, lo + chunk);
  int c = 0;
  for (int t = lo; t < hi; ++t) c += flg[t];
  const int tot = block_scan_256(c, off, wsum);
  if (MODE == 0) {
    if (threadIdx.x == 0) cnt_or_ptr[i] = tot;
    return;
  }
  i64 o = cnt_or_ptr[i] + off[threadIdx.x];
  for (int t = lo; t < hi; ++t)
    if (flg[t]) ccol[o++] = t;
}

__global__ void __launch_bounds__(256) k_num_cta_st(const int* __restrict__ rowlist, i64 nrows,
                                                    const i64* __restrict__ ap, const int* __restrict__ ac,
                                                    const double* __restrict__ av, const double* __restrict__ rs,
                                                    const i64* __restrict__ bp, const int* __restrict__ bc,
                                                    const double* __restrict__ bv, const i64* __restrict__ cp,
                                                    const int* __restrict__ cc, double* __restrict__ cv) {
  extern __shared__ unsigned char smraw[];
  __shared__ int off[257], wsum[8];
  __shared__ i64 q0s[256];
  __shared__ double as[256];
  if (i64(blockIdx.x) >= nrows) return;
  const i64 i = rowlist ? rowlist[blockIdx.x] : i64(blockIdx.x);
  const i64 c0 = cp[i];
  const int nc = int(cp[i + 1] - c0);
  double* prod = reinterpret_cast<double*>(smraw);
  double* acc = prod + ST_CH;
  int* cols = reinterpret_cast<int*>(acc + nc);
  int* pos = cols + nc;
  for (int t = threadIdx.x; t < nc; t += blockDim.x) {
    cols[t] = cc[c0 + t];
    acc[t] = 0.0;
  }
  const double si = rs ? rs[i] : 1.0;
  const i64 a0 = ap[i], a1 = ap[i + 1];
  for (i64 base = a0; base < a1; base += 256) {
    const i64 ka = base + threadIdx.x;
    int len = 0;
    if (ka < a1) {
      const int k = ac[ka];
      const i64 q0 = bp[k];
      len = int(bp[k + 1] - q0);
      q0s[threadIdx.x] = q0;
      as[threadIdx.x] = rs ? si * av[ka] : av[ka];
    }
    block_scan_256(len, off, wsum);  // (its barriers also order the cols / acc initialisation)
    const int ne = int(min(i64(256), a1 - base));
    // sub-chunks of whole A entries with at most ST_CH products
    for (int e_lo = 0; e_lo < ne;) {
      const int f0 = off[e_lo];
      int e_hi = seg_of(off, ne + 1, f0 + ST_CH);  // last e with off[e] <= f0 + ST_CH
      if (e_hi <= e_lo) e_hi = e_lo + 1;            // (a single B row never exceeds ST_CH)
      const int f1 = off[e_hi];
      for (int f = f0 + int(threadIdx.x); f < f1; f += 256) {
        const int e = e_lo + seg_of(off + e_lo, e_hi - e_lo, f);
        const i64 kb = q0s[e] + (f - off[e]);
        prod[f - f0] = as[e] * bv[kb];
        pos[f - f0] = lower_bound_sm(cols, nc, bc[kb]);
      }
      __syncthreads();
      for (int e = e_lo; e < e_hi; ++e) {
        const int b = off[e] - f0, n = off[e + 1] - off[e];
        if (n == 0) continue;
        for (int t = threadIdx.x; t < n; t += 256) acc[pos[b + t]] += prod[b + t];
        __syncthreads();
      }
      e_lo = e_hi;
    }
    __syncthreads();
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nc; t += blockDim.x) cv[c0 + t] = acc[t];
}

// partition rows by a predicate on a per-row value (order within a bin is irrelevant: every
// listed row is processed independently)
__global__ void k_bin_rows(i64 rows, const i64* __restrict__ v, i64 lo, i64 hi, int* __restrict__ list,
                           int* __restrict__ count) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const i64 x = v[i];
  if (x > lo && x <= hi) list[atomicAdd(count, 1)] = int(i);
}
__global__ void k_row_len(i64 m, const i64* __restrict__ p, i64* __restrict__ out) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < m) out[i] = p[i + 1] - p[i];
}
__global__ void k_bin_overflow(i64 rows, const int* __restrict__ list, int n, const i64* __restrict__ cnt,
                               int* __restrict__ out, int* __restrict__ count) {
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < n && cnt[list[t]] < 0) out[atomicAdd(count, 1)] = list[t];
}

template <class T>
void scan_excl(T* data, i64 n_plus_1) {
  size_t bytes = 0;
  CF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, data, data, n_plus_1, stream()));
  DevBuf<unsigned char> tmp{static_cast<i64>(bytes)};
  CF_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, data, data, n_plus_1, stream()));
  count_launch();
}

i64 read_i64(const i64* p) {
  i64 h = 0;
  read_small(&h, p, sizeof(i64));
  return h;
}
int read_int(const int* p) {
  int h = 0;
  read_small(&h, p, sizeof(int));
  return h;
}

struct RowBin {
  DevBuf<int> list;
  int n = 0;
};

RowBin make_bin(i64 rows, const i64* v, i64 lo, i64 hi) {
  RowBin b;
  b.list.alloc(std::max<i64>(rows, 1));
  DevBuf<int> c(1);
  c.zero();
  k_bin_rows<<<grid_for(rows, 256), 256, 0, stream()>>>(rows, v, lo, hi, b.list.p, c.p);
  CF_LAUNCHED();
  b.n = read_int(c.p);
  return b;
}

RowBin overflow_of(const RowBin& in, const i64* cnt) {
  RowBin o;
  o.list.alloc(std::max(in.n, 1));
  if (!in.n) return o;
  DevBuf<int> c(1);
  c.zero();
  k_bin_overflow<<<grid_for(in.n, 256), 256, 0, stream()>>>(0, in.list.p, in.n, cnt, o.list.p, c.p);
  CF_LAUNCHED();
  o.n = read_int(c.p);
  return o;
}

constexpr int SYM_BIG = 16384;
constexpr i64 SMALL_ROWS = 16384, SMALL_COLS = 8192;  // the one-round-trip path of spgemm()

// lanes per A entry in the warp kernels, from the longest B row
// 8 lanes (4 A entries in flight per step, <= 16 independent B loads per lane) unless B rows are
// long; this is what hides the per-A-entry dependency chain (ac -> bp -> bc -> hash)
// lanes per B row in the symbolic and numeric kernels (measured on config 3: 4 lanes for the <= 6
// entry rows of the tentative prolongator, 16 lanes beat 8 lanes with 16 buffered products per
// lane for B rows of 65-128 entries, 32 lanes beat 16 beyond 128)
int lanes_for(i64 maxb) { return maxb <= 8 ? 4 : (maxb <= 64 ? 8 : (maxb <= 128 ? 16 : 32)); }

template <int L>
void sym_launch(int mode, const RowBin& b, int cap, const Csr& A, const Csr& B, i64* cnt, const Csr* C) {
  if (!b.n) return;
  if (cap == 512) {
    if (mode == 0)
      k_sym<512, L, 8, 0><<<grid_for(b.n, 8), 256, 0, stream()>>>(b.list.p, b.n, A.ptr.p, A.col.p, B.ptr.p, B.col.p,
                                                                  cnt, nullptr, nullptr);
    else
      k_sym<512, L, 8, 1><<<grid_for(b.n, 8), 256, 0, stream()>>>(b.list.p, b.n, A.ptr.p, A.col.p, B.ptr.p, B.col.p,
                                                                  nullptr, C->ptr.p, C->col.p);
  } else {
    if (mode == 0)
      k_sym<2048, L, 4, 0><<<grid_for(b.n, 4), 128, 0, stream()>>>(b.list.p, b.n, A.ptr.p, A.col.p, B.ptr.p, B.col.p,
                                                                   cnt, nullptr, nullptr);
    else
      k_sym<2048, L, 2, 1><<<grid_for(b.n, 2), 64, 0, stream()>>>(b.list.p, b.n, A.ptr.p, A.col.p, B.ptr.p, B.col.p,
                                                                  nullptr, C->ptr.p, C->col.p);
  }
  CF_LAUNCHED();
}

void sym_dispatch(int L, int mode, const RowBin& b, int cap, const Csr& A, const Csr& B, i64* cnt, const Csr* C) {
  if (L == 4) sym_launch<4>(mode, b, cap, A, B, cnt, C);
  else if (L == 8) sym_launch<8>(mode, b, cap, A, B, cnt, C);
  else if (L == 16) sym_launch<16>(mode, b, cap, A, B, cnt, C);
  else sym_launch<32>(mode, b, cap, A, B, cnt, C);
}

template <int L, int CMAX>
void num_launch(const RowBin& b, int cap, const Csr& A, const Csr& B, const double* rs, Csr& C) {
  if (!b.n) return;
  if (cap == 512)
    k_num<512, L, 8, CMAX><<<grid_for(b.n, 8), 256, 0, stream()>>>(b.list.p, b.n, A.ptr.p, A.col.p, A.val.p, rs,
                                                                   B.ptr.p, B.col.p, B.val.p, C.ptr.p, C.col.p,
                                                                   C.val.p);
  else
    k_num<2048, L, 2, CMAX><<<grid_for(b.n, 2), 64, 0, stream()>>>(b.list.p, b.n, A.ptr.p, A.col.p, A.val.p, rs,
                                                                   B.ptr.p, B.col.p, B.val.p, C.ptr.p, C.col.p,
                                                                   C.val.p);
  CF_LAUNCHED();
}

// --- row groups: runs of consecutive A rows with one column pattern ------------------------
// Rows of one mesh node (or of one aggregate on the coarse levels) share their pattern, and so do
// their product rows: the symbolic phase runs once per group and the numeric kernel below applies
// each B row once for all rows of the group.  Per row, every C(i,j) is still the k-ascending
// sequential sum, so C is bitwise that of the row-wise kernels.
__global__ void k_same_prev(i64 rows, const i64* __restrict__ p, const int* __restrict__ c, int* __restrict__ head) {
  const i64 i = (i64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= rows) return;
  bool same = i > 0;
  i64 n = 0, b0 = 0, b1 = 0;
  if (same) {
    b0 = p[i - 1];
    b1 = p[i];
    n = p[i + 1] - b1;
    same = n > 0 && n == b1 - b0;
  }
  for (i64 t = lane; same && t < n; t += 32)
    if (c[b0 + t] != c[b1 + t]) same = false;
  same = __all_sync(0xffffffffu, same);
  if (lane == 0) head[i] = same ? 0 : 1;
}

__global__ void k_not_head(i64 rows, const int* __restrict__ head, unsigned char* __restrict__ same) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < rows) same[i] = head[i] ? 0 : 1;
}

// run start of each row: max over j <= i of (head[j] ? j : 0) via a max-scan of these keys
__global__ void k_head_key(i64 rows, const int* __restrict__ head, int* __restrict__ key) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < rows) key[i] = head[i] ? int(i) : 0;
}
__global__ void k_chunk_heads(i64 rows, const int* __restrict__ runstart, int gm, int* __restrict__ head) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < rows) head[i] = ((int(i) - runstart[i]) % gm) == 0 ? 1 : 0;
}
__global__ void k_group_len(int ng, const int* __restrict__ heads, i64 rows, int* __restrict__ glen) {
  const i64 g = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g < ng) glen[g] = (g + 1 < ng ? heads[g + 1] : int(rows)) - heads[g];
}

// gathered head rows (pattern only)
__global__ void k_head_len_rows(int ng, const int* __restrict__ rows, const i64* __restrict__ p, i64* __restrict__ out) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g < ng) out[g] = p[rows[g] + 1] - p[rows[g]];
}
__global__ void k_head_len(int ng, const int* __restrict__ heads, const i64* __restrict__ p, i64* __restrict__ out) {
  const i64 g = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g < ng) out[g] = p[heads[g] + 1] - p[heads[g]];
}
__global__ void k_gather_rows(int ng, const int* __restrict__ heads, const i64* __restrict__ p,
                              const int* __restrict__ c, const i64* __restrict__ gp, int* __restrict__ gc) {
  const i64 g = (i64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (g >= ng) return;
  const i64 b = p[heads[g]], n = gp[g + 1] - gp[g];
  for (i64 t = lane; t < n; t += 32) gc[gp[g] + t] = c[b + t];
}
// expand the group pattern to the rows: lengths, then columns
__global__ void k_expand_len(int ng, const int* __restrict__ heads, const int* __restrict__ glen,
                             const i64* __restrict__ gp, i64* __restrict__ cnt) {
  const i64 g = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= ng) return;
  const i64 n = gp[g + 1] - gp[g];
  for (int r = 0; r < glen[g]; ++r) cnt[heads[g] + r] = n;
}
__global__ void k_expand_cols(int ng, const int* __restrict__ heads, const int* __restrict__ glen,
                              const i64* __restrict__ gp, const int* __restrict__ gc, const i64* __restrict__ cp,
                              int* __restrict__ cc) {
  const i64 g = (i64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (g >= ng) return;
  const i64 b = gp[g], n = gp[g + 1] - b;
  for (int r = 0; r < glen[g]; ++r) {
    const i64 o = cp[heads[g] + r];
    for (i64 t = lane; t < n; t += 32) cc[o + t] = gc[b + t];
  }
}
// per-row selection of the rows of the listed groups (their C row length), for the row-wise tiers
__global__ void k_select_group_rows(int n, const int* __restrict__ list, const int* __restrict__ heads,
                                    const int* __restrict__ glen, const i64* __restrict__ cp, i64* __restrict__ sel) {
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int g = list[t];
  for (int r = 0; r < glen[g]; ++r) {
    const i64 i = heads[g] + r;
    sel[i] = cp[i + 1] - cp[i];
  }
}

constexpr int GRP_MAX = 6;  // rows per group (longer runs are chunked)

// numeric, warp per group: the group's (shared) columns in a hash of cap slots, one accumulator row
// per group row.  The A positions k are taken in ascending order, one at a time; the lanes cover
// the entries of B row k (CB per lane), find each slot once and apply it to every row of the group.
// Within one k the slots are distinct, so no two lanes touch one accumulator; __syncwarp orders
// successive k.  The next k's B row and A values are loaded while the current one is applied.
// The position loop is instantiated per group size NR (a warp-uniform switch), and the per-lane
// entry loop stops at the row's length, so no predicated-off row or entry slots are issued.
template <int CB, int NR>
__device__ __forceinline__ void num_grp_rows(double* __restrict__ Acc, const int* __restrict__ T, unsigned mask,
                                             int cap, int row0, int lane, const i64* __restrict__ ap,
                                             const int* __restrict__ ac, const double* __restrict__ av,
                                             const double* __restrict__ rs, const i64* __restrict__ bp,
                                             const int* __restrict__ bc, const double* __restrict__ bv) {
  double si[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) si[r] = rs ? rs[row0 + r] : 1.0;
  const i64 a0 = ap[row0];
  const int alen = int(ap[row0 + 1] - a0);
  int ck[CB], nk[CB];
  double cb[CB], nb[CB], ca[NR], na[NR];
  int cn = 0, nn = 0;
  auto load = [&](int pos, int* kc, double* kv, double* ka, int& n) {
    const int k = ac[a0 + pos];
    const i64 q0 = bp[k];
    n = int(bp[k + 1] - q0);
#pragma unroll
    for (int t = 0; t < CB; ++t) {
      const int e = t * 32 + lane;
      if (e < n) {
        kc[t] = bc[q0 + e];
        kv[t] = bv[q0 + e];
      }
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) ka[r] = rs ? si[r] * av[a0 + i64(r) * alen + pos] : av[a0 + i64(r) * alen + pos];
  };
  if (alen > 0) load(0, ck, cb, ca, cn);
  // slot of the previous position's entry t: the d rows of a mesh node (or an aggregate's coarse
  // dofs) repeat one column pattern, so the lookup is reused when the column is the same
  int pk[CB], ps[CB];
#pragma unroll
  for (int t = 0; t < CB; ++t) pk[t] = -1;
  for (int pos = 0; pos < alen; ++pos) {
    if (pos + 1 < alen) load(pos + 1, nk, nb, na, nn);
#pragma unroll
    for (int t = 0; t < CB; ++t) {
      if (t * 32 >= cn) break;  // warp-uniform
      const int e = t * 32 + lane;
      if (e < cn) {
        const int sl = ck[t] == pk[t] ? ps[t] : hfind(T, mask, ck[t]);
        pk[t] = ck[t];
        ps[t] = sl;
#pragma unroll
        for (int r = 0; r < NR; ++r) Acc[size_t(r) * cap + sl] += ca[r] * cb[t];
      }
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < CB; ++t) {
      ck[t] = nk[t];
      cb[t] = nb[t];
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) ca[r] = na[r];
    cn = nn;
  }
}

// Runs of B rows: consecutive A positions k, k+1, .. (the d dofs of one mesh node, or the coarse
// dofs of one aggregate) whose B rows repeat one column pattern (bsame[k + j]: row k + j has row
// k + j - 1's columns) are applied together, up to MR rows per step: the lane of entry e loads its
// column once and the m values (the rows are contiguous, row k + j at bp[k] + j n), finds the slot
// once and adds the m products to each accumulator in ascending k — per C(i,j) the same
// k-ascending sequence of IEEE additions as one position at a time (any split of the positions
// into runs gives it), with a third of the steps, slot lookups and shared-memory updates.
// The positions are taken in windows of 32: lane p loads position base + p's column k, B-row
// offset and length and the group's A values there in one round, so a run's step waits only on its
// own B entries; the runs of a window are the ballot of run starts (chain starts, and every MR-th
// link of a chain).  B rows longer than 32 entries are taken 32 CH entries per load round.
template <int NR, int MR, int CH>
__device__ __forceinline__ void num_grp_runs(double* __restrict__ Acc, const int* __restrict__ T, unsigned mask,
                                             int cap, int row0, int lane, const i64* __restrict__ ap,
                                             const int* __restrict__ ac, const double* __restrict__ av,
                                             const double* __restrict__ rs, const i64* __restrict__ bp,
                                             const int* __restrict__ bc, const double* __restrict__ bv,
                                             const unsigned char* __restrict__ bsame, double* __restrict__ wa,
                                             i64* __restrict__ wq, int* __restrict__ wn) {
  constexpr unsigned FULL = 0xffffffffu;
  const i64 a0 = ap[row0];
  const int alen = int(ap[row0 + 1] - a0);
  for (int base = 0; base < alen; base += 32) {
    // the window's positions: B-row offsets and lengths and the group's A values, in shared memory
    const int p = base + lane;
    const bool in = p < alen;
    int k = -1;
    if (in) {
      k = ac[a0 + p];
      const i64 q0 = bp[k];
      wq[lane] = q0;
      wn[lane] = int(bp[k + 1] - q0);
#pragma unroll
      for (int r = 0; r < NR; ++r)
        wa[r * 32 + lane] = rs ? rs[row0 + r] * av[a0 + i64(r) * alen + p] : av[a0 + i64(r) * alen + p];
    }
    const int kprev = __shfl_up_sync(FULL, k, 1);
    const bool link = in && lane > 0 && k == kprev + 1 && bsame[k];
    const unsigned lm = __ballot_sync(FULL, link);
    const unsigned nl = ~lm & __ballot_sync(FULL, in);
    const int cs = 31 - __clz(nl & (FULL >> (31 - lane)));  // chain start (lane 0 is never a link)
    unsigned starts = __ballot_sync(FULL, in && (lane - cs) % MR == 0);
    __syncwarp();
    // software pipeline over the window's runs: the first 32 entries of the next run are loaded
    // while the current run is applied (longer rows: the rest is taken CH chunks per round)
    auto run_len = [&](int st) {
      return st < 31 ? 1 + min(MR - 1, __ffs(~(lm >> (st + 1))) - 1) : 1;
    };
    auto load0 = [&](int st, int m, int& col, double* b) {
      const i64 rq = wq[st];
      const int rn = wn[st];
      if (lane < rn) {
        col = bc[rq + lane];
#pragma unroll
        for (int j = 0; j < MR; ++j)
          if (j < m) b[j] = bv[rq + i64(j) * rn + lane];
      }
    };
    int pcol = 0;
    double pb[MR];
    int st = -1, m = 1;
    if (starts) {
      st = __ffs(starts) - 1;
      starts &= starts - 1;
      m = run_len(st);
      load0(st, m, pcol, pb);
    }
    while (st >= 0) {
      const i64 rq = wq[st];
      const int rn = wn[st];
      double ca[MR][NR];
#pragma unroll
      for (int j = 0; j < MR; ++j)
        if (j < m) {
#pragma unroll
          for (int r = 0; r < NR; ++r) ca[j][r] = wa[r * 32 + st + j];
        }
      const int ccol = pcol;
      double cb[MR];
#pragma unroll
      for (int j = 0; j < MR; ++j) cb[j] = pb[j];
      const int cm = m;
      // next run of the window: start its loads now
      st = -1;
      if (starts) {
        st = __ffs(starts) - 1;
        starts &= starts - 1;
        m = run_len(st);
        load0(st, m, pcol, pb);
      }
      if (lane < rn) {
        const int sl = hfind(T, mask, ccol);
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          double acc = Acc[size_t(r) * cap + sl];
#pragma unroll
          for (int j = 0; j < MR; ++j)
            if (j < cm) acc += ca[j][r] * cb[j];
          Acc[size_t(r) * cap + sl] = acc;
        }
      }
      for (int c0 = 32; c0 < rn; c0 += 32 * CH) {
        int col[CH];
        double b[CH][MR];
#pragma unroll
        for (int h = 0; h < CH; ++h) {
          const int e = c0 + h * 32 + lane;
          if (e < rn) {
            col[h] = bc[rq + e];
#pragma unroll
            for (int j = 0; j < MR; ++j)
              if (j < cm) b[h][j] = bv[rq + i64(j) * rn + e];
          }
        }
#pragma unroll
        for (int h = 0; h < CH; ++h) {
          const int e = c0 + h * 32 + lane;
          if (e < rn) {
            const int sl = hfind(T, mask, col[h]);
#pragma unroll
            for (int r = 0; r < NR; ++r) {
              double acc = Acc[size_t(r) * cap + sl];
#pragma unroll
              for (int j = 0; j < MR; ++j)
                if (j < cm) acc += ca[j][r] * b[h][j];
              Acc[size_t(r) * cap + sl] = acc;
            }
          }
        }
      }
      __syncwarp();
    }
    __syncwarp();
  }
}

// per-warp window scratch of the run kernel (after the hash tables): A values, B-row offsets, lengths
#ifndef CF_RUN_MINB
#define CF_RUN_MINB 4
#endif
#ifndef CF_RUN_MINB6
#define CF_RUN_MINB6 2
#endif
constexpr size_t RUN_WIN_BYTES = size_t(GRP_MAX) * 32 * sizeof(double) + 32 * sizeof(i64) + 32 * sizeof(int);

template <int NRMAX, int CH>
__global__ void __launch_bounds__(256, NRMAX <= 3 ? CF_RUN_MINB : CF_RUN_MINB6) k_num_grp_run(const int* __restrict__ glist, int ng, const int* __restrict__ heads,
                                                 const int* __restrict__ glen, int cap, int wpb, int gm,
                                                 const i64* __restrict__ ap, const int* __restrict__ ac,
                                                 const double* __restrict__ av, const double* __restrict__ rs,
                                                 const i64* __restrict__ bp, const int* __restrict__ bc,
                                                 const double* __restrict__ bv, const unsigned char* __restrict__ bsame,
                                                 const i64* __restrict__ cp, const int* __restrict__ cc,
                                                 double* __restrict__ cv) {
  extern __shared__ double grp_sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const i64 gi = i64(blockIdx.x) * wpb + w;
  if (gi >= ng) return;
  const int grp = glist[gi];
  const int row0 = heads[grp], nr = glen[grp];
  double* Acc = grp_sm + size_t(w) * cap * gm;
  int* T = reinterpret_cast<int*>(grp_sm + size_t(wpb) * cap * gm) + size_t(w) * cap;
  for (int s = lane; s < cap; s += 32) T[s] = EMPTY;
  for (int s = lane; s < cap * nr; s += 32) Acc[s] = 0.0;
  __syncwarp();
  const unsigned mask = unsigned(cap) - 1u;
  const i64 c0 = cp[row0];
  const int nc = int(cp[row0 + 1] - c0);
  for (int t = lane; t < nc; t += 32) hinsert(T, mask, cc[c0 + t]);
  unsigned char* win = reinterpret_cast<unsigned char*>(reinterpret_cast<int*>(grp_sm + size_t(wpb) * cap * gm) +
                                                        size_t(wpb) * cap) + size_t(w) * RUN_WIN_BYTES;
  double* wa = reinterpret_cast<double*>(win);
  i64* wq = reinterpret_cast<i64*>(win + size_t(GRP_MAX) * 32 * sizeof(double));
  int* wn = reinterpret_cast<int*>(win + size_t(GRP_MAX) * 32 * sizeof(double) + 32 * sizeof(i64));
  __syncwarp();
  switch (nr) {
#define CFB_NR(R) \
  case R: if (R <= NRMAX) num_grp_runs<R <= NRMAX ? R : 1, 3, CH>(Acc, T, mask, cap, row0, lane, ap, ac, av, rs, bp, bc, bv, bsame, wa, wq, wn); break;
    CFB_NR(1) CFB_NR(2) CFB_NR(3) CFB_NR(4) CFB_NR(5) CFB_NR(6)
#undef CFB_NR
  }
  for (int t = lane; t < nc; t += 32) {
    const int sl = hfind(T, mask, cc[c0 + t]);
    for (int r = 0; r < nr; ++r) cv[c0 + i64(r) * nc + t] = Acc[size_t(r) * cap + sl];
  }
}

template <int CB>
__global__ void __launch_bounds__(256, CB >= 8 ? 2 : 3) k_num_grp(const int* __restrict__ glist, int ng, const int* __restrict__ heads,
                                                 const int* __restrict__ glen, int cap, int wpb, int gm,
                                                 const i64* __restrict__ ap, const int* __restrict__ ac,
                                                 const double* __restrict__ av, const double* __restrict__ rs,
                                                 const i64* __restrict__ bp, const int* __restrict__ bc,
                                                 const double* __restrict__ bv, const i64* __restrict__ cp,
                                                 const int* __restrict__ cc, double* __restrict__ cv) {
  extern __shared__ double grp_sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const i64 gi = i64(blockIdx.x) * wpb + w;
  if (gi >= ng) return;
  const int grp = glist[gi];
  const int row0 = heads[grp], nr = glen[grp];
  double* Acc = grp_sm + size_t(w) * cap * gm;  // [gm][cap], gm = the longest group
  int* T = reinterpret_cast<int*>(grp_sm + size_t(wpb) * cap * gm) + size_t(w) * cap;
  for (int s = lane; s < cap; s += 32) T[s] = EMPTY;
  for (int s = lane; s < cap * nr; s += 32) Acc[s] = 0.0;
  __syncwarp();
  const unsigned mask = unsigned(cap) - 1u;
  const i64 c0 = cp[row0];
  const int nc = int(cp[row0 + 1] - c0);
  for (int t = lane; t < nc; t += 32) hinsert(T, mask, cc[c0 + t]);
  __syncwarp();
  switch (nr) {
#define CFB_NR(R) \
  case R: num_grp_rows<CB, R>(Acc, T, mask, cap, row0, lane, ap, ac, av, rs, bp, bc, bv); break;
    CFB_NR(1) CFB_NR(2) CFB_NR(3) CFB_NR(4) CFB_NR(5) CFB_NR(6)
#undef CFB_NR
  }
  for (int t = lane; t < nc; t += 32) {
    const int sl = hfind(T, mask, cc[c0 + t]);
    for (int r = 0; r < nr; ++r) cv[c0 + i64(r) * nc + t] = Acc[size_t(r) * cap + sl];
  }
}

// Group numeric for short B rows (<= 8 entries: the tentative prolongator of D^-1 A T): 8 lanes per
// B row, so one step covers G = 4 consecutive A positions; slots and products are formed in
// parallel, then the 4 position groups add in ascending k (one at a time, __syncwarp between), so
// every accumulator sees k_num_grp's sequence.  Each slot lookup serves the NR rows of the group.
template <int NR>
__device__ __forceinline__ void num_grp_short_rows(double* __restrict__ Acc, const int* __restrict__ T,
                                                   unsigned mask, int cap, int row0, int lane,
                                                   const i64* __restrict__ ap, const int* __restrict__ ac,
                                                   const double* __restrict__ av, const double* __restrict__ rs,
                                                   const i64* __restrict__ bp, const int* __restrict__ bc,
                                                   const double* __restrict__ bv) {
  constexpr int L = 8, G = 32 / L;
  const int g = lane / L, lig = lane % L;
  double si[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) si[r] = rs ? rs[row0 + r] : 1.0;
  const i64 a0 = ap[row0];
  const int alen = int(ap[row0 + 1] - a0);
  for (int p0 = 0; p0 < alen; p0 += G) {
    const int pos = p0 + g;
    int sl = -1;
    double b = 0.0, a[NR];
    if (pos < alen) {
      const int k = ac[a0 + pos];
      const i64 q = bp[k] + lig;
      if (q < bp[k + 1]) {
        const int c = bc[q];
        b = bv[q];
#pragma unroll
        for (int r = 0; r < NR; ++r) a[r] = rs ? si[r] * av[a0 + i64(r) * alen + pos] : av[a0 + i64(r) * alen + pos];
        sl = hfind(T, mask, c);
      }
    }
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
      if (g == gg && sl >= 0) {
#pragma unroll
        for (int r = 0; r < NR; ++r) Acc[size_t(r) * cap + sl] += a[r] * b;
      }
      __syncwarp();
    }
  }
}

__global__ void __launch_bounds__(256) k_num_grp_short(const int* __restrict__ glist, int ng,
                                                       const int* __restrict__ heads, const int* __restrict__ glen,
                                                       int cap, int wpb, int gm, const i64* __restrict__ ap,
                                                       const int* __restrict__ ac, const double* __restrict__ av,
                                                       const double* __restrict__ rs, const i64* __restrict__ bp,
                                                       const int* __restrict__ bc, const double* __restrict__ bv,
                                                       const i64* __restrict__ cp, const int* __restrict__ cc,
                                                       double* __restrict__ cv) {
  extern __shared__ double grp_sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const i64 gi = i64(blockIdx.x) * wpb + w;
  if (gi >= ng) return;
  const int grp = glist[gi];
  const int row0 = heads[grp], nr = glen[grp];
  double* Acc = grp_sm + size_t(w) * cap * gm;
  int* T = reinterpret_cast<int*>(grp_sm + size_t(wpb) * cap * gm) + size_t(w) * cap;
  for (int s = lane; s < cap; s += 32) T[s] = EMPTY;
  for (int s = lane; s < cap * nr; s += 32) Acc[s] = 0.0;
  __syncwarp();
  const unsigned mask = unsigned(cap) - 1u;
  const i64 c0 = cp[row0];
  const int nc = int(cp[row0 + 1] - c0);
  for (int t = lane; t < nc; t += 32) hinsert(T, mask, cc[c0 + t]);
  __syncwarp();
  switch (nr) {
#define CFB_NR(R) \
  case R: num_grp_short_rows<R>(Acc, T, mask, cap, row0, lane, ap, ac, av, rs, bp, bc, bv); break;
    CFB_NR(1) CFB_NR(2) CFB_NR(3) CFB_NR(4) CFB_NR(5) CFB_NR(6)
#undef CFB_NR
  }
  for (int t = lane; t < nc; t += 32) {
    const int sl = hfind(T, mask, cc[c0 + t]);
    for (int r = 0; r < nr; ++r) cv[c0 + i64(r) * nc + t] = Acc[size_t(r) * cap + sl];
  }
}

// CB = 0: the short-row kernel (B rows of <= 8 entries); bsame: the run kernel
template <int CB>
void num_grp_launch(const RowBin& b, int cap, const int* heads, const int* glen, const Csr& A, const Csr& B,
                    const double* rs, Csr& C, int gm, const unsigned char* bsame = nullptr) {
  if (!b.n) return;
  const size_t per_warp = size_t(cap) * (sizeof(int) + sizeof(double) * gm);
  const int wpb = int(std::min<size_t>(8, std::max<size_t>(1, (100u << 10) / per_warp)));
  const size_t sm = per_warp * wpb;
  if (bsame) {
    const size_t per_warp_r = per_warp + RUN_WIN_BYTES;
    const int wpb = int(std::min<size_t>(8, std::max<size_t>(1, (100u << 10) / per_warp_r)));
    const size_t sm = per_warp_r * wpb;
    auto rk = gm <= 3 ? k_num_grp_run<3, 1> : k_num_grp_run<6, 1>;
    CF_CUDA(cudaFuncSetAttribute(rk, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
    rk<<<grid_for(b.n, wpb), wpb * 32, sm, stream()>>>(b.list.p, b.n, heads, glen, cap, wpb, gm, A.ptr.p, A.col.p,
                                                      A.val.p, rs, B.ptr.p, B.col.p, B.val.p, bsame, C.ptr.p,
                                                      C.col.p, C.val.p);
    CF_LAUNCHED();
    return;
  }
  auto kern = CB == 0 ? k_num_grp_short : k_num_grp<CB == 0 ? 1 : CB>;
  CF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
  kern<<<grid_for(b.n, wpb), wpb * 32, sm, stream()>>>(b.list.p, b.n, heads, glen, cap, wpb, gm, A.ptr.p, A.col.p,
                                                      A.val.p, rs, B.ptr.p, B.col.p, B.val.p, C.ptr.p, C.col.p,
                                                      C.val.p);
  CF_LAUNCHED();
}

__global__ void k_max_int(i64 n, const int* __restrict__ v, int* __restrict__ mx) {
  int m = 0;
  for (i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += i64(gridDim.x) * blockDim.x) m = max(m, v[i]);
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(mx, m);
}

__global__ void k_group_clen(int ng, const int* __restrict__ heads, const i64* __restrict__ cp, i64* __restrict__ out) {
  const i64 g = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g < ng) out[g] = cp[heads[g] + 1] - cp[heads[g]];
}

// ---- giant rows (more than GIANT output columns, beyond the 16384-slot CTA hash): sort tier.
// The row's products are expanded in A-position order (k ascending, then B-row order), keyed by
// (giant row, column) and stably radix-sorted; equal keys then sit in k order, and each output
// entry is the first product followed by the others added one by one — the k-ascending
// sequential sum of every other tier (and of Eigen's conservative product).  Any row length.
constexpr i64 GIANT = 12288;

__global__ void k_giant_len(int ng, const int* __restrict__ rows, const i64* __restrict__ ap,
                            const int* __restrict__ ac, const i64* __restrict__ bp, i64* __restrict__ len) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ng) return;
  const int i = rows[g];
  i64 s = 0;
  for (i64 k = ap[i]; k < ap[i + 1]; ++k) s += bp[ac[k] + 1] - bp[ac[k]];
  len[g] = s;
}
__global__ void k_giant_expand(int ng, const int* __restrict__ rows, const i64* __restrict__ ap,
                               const int* __restrict__ ac, const double* __restrict__ av,
                               const double* __restrict__ rs, const i64* __restrict__ bp,
                               const int* __restrict__ bc, const double* __restrict__ bv,
                               const i64* __restrict__ off, unsigned long long* __restrict__ key,
                               double* __restrict__ val) {
  const int g = blockIdx.x;
  const int i = rows[g];
  i64 o = off[g];
  for (i64 ka = ap[i]; ka < ap[i + 1]; ++ka) {
    const int k = ac[ka];
    const double a = rs ? rs[i] * av[ka] : (av ? av[ka] : 0.0);
    const i64 q0 = bp[k];
    const int n = int(bp[k + 1] - q0);
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      key[o + t] = (static_cast<unsigned long long>(g) << 32) | static_cast<unsigned>(bc[q0 + t]);
      if (val) val[o + t] = a * bv[q0 + t];
    }
    o += n;
  }
}
__global__ void k_zero_rows(int ng, const int* __restrict__ rows, i64* __restrict__ cnt) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g < ng) cnt[rows[g]] = 0;
}
__global__ void k_giant_heads(i64 n, const unsigned long long* __restrict__ key, int* __restrict__ head) {
  const i64 p = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p < n) head[p] = (p == 0 || key[p] != key[p - 1]) ? 1 : 0;
}
__global__ void k_giant_count(i64 nu, const i64* __restrict__ hpos, const unsigned long long* __restrict__ key,
                              const int* __restrict__ rows, i64* __restrict__ cnt) {
  const i64 u = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u < nu) atomicAdd(reinterpret_cast<unsigned long long*>(&cnt[rows[int(key[hpos[u]] >> 32)]]), 1ull);
}
// unique u (in (giant row, column) order) -> its place in C: ptr[row] + (u - first[g])
__global__ void k_giant_emit(i64 nu, i64 n, const i64* __restrict__ hpos, const unsigned long long* __restrict__ key,
                             const double* __restrict__ val, const int* __restrict__ rows,
                             const i64* __restrict__ first, const i64* __restrict__ cptr, int* __restrict__ ccol,
                             double* __restrict__ cval) {
  const i64 u = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= nu) return;
  const i64 p0 = hpos[u], p1 = (u + 1 < nu) ? hpos[u + 1] : n;
  const unsigned long long kk = key[p0];
  const int g = int(kk >> 32);
  const i64 pos = cptr[rows[g]] + (u - first[g]);
  if (ccol) ccol[pos] = int(kk & 0xffffffffull);
  if (cval) {
    double s = val[p0];
    for (i64 p = p0 + 1; p < p1; ++p) s += val[p];
    cval[pos] = s;
  }
}

// mode 0: cnt[row] := the row's number of distinct columns; mode 1: C.col of the rows;
// mode 2: C.val of the rows.  rows: device list of ng giant rows.
void giant_rows(int mode, const int* rows, int ng, const Csr& A, const Csr& B, const double* rs, i64* cnt, Csr* C) {
  if (ng <= 0) return;
  DevBuf<i64> off(ng + 1);
  CF_CUDA(cudaMemsetAsync(off.p + ng, 0, sizeof(i64), stream()));
  k_giant_len<<<grid_for(ng, 128), 128, 0, stream()>>>(ng, rows, A.ptr.p, A.col.p, B.ptr.p, off.p);
  CF_LAUNCHED();
  scan_excl(off.p, ng + 1);
  const i64 n = read_i64(off.p + ng);
  DevBuf<unsigned long long> key(n), key2(n);
  DevBuf<double> val(mode == 2 ? n : 0), val2(mode == 2 ? n : 0);
  k_giant_expand<<<ng, 256, 0, stream()>>>(ng, rows, A.ptr.p, A.col.p, mode == 2 ? A.val.p : nullptr, rs, B.ptr.p,
                                           B.col.p, B.val.p, off.p, key.p, mode == 2 ? val.p : nullptr);
  CF_LAUNCHED();
  int hi_bit = 32;
  while ((1ll << (hi_bit - 32)) < ng) ++hi_bit;
  {
    size_t bytes = 0;
    if (mode == 2) {
      CF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key.p, key2.p, val.p, val2.p, n, 0, hi_bit, stream()));
      DevBuf<unsigned char> tmp{static_cast<i64>(bytes)};
      CF_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, key.p, key2.p, val.p, val2.p, n, 0, hi_bit, stream()));
    } else {
      CF_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, key.p, key2.p, n, 0, hi_bit, stream()));
      DevBuf<unsigned char> tmp{static_cast<i64>(bytes)};
      CF_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, bytes, key.p, key2.p, n, 0, hi_bit, stream()));
    }
    count_launch();
  }
  key.release();
  DevBuf<int> head(n);
  k_giant_heads<<<grid_for(n, 256), 256, 0, stream()>>>(n, key2.p, head.p);
  CF_LAUNCHED();
  DevBuf<i64> hpos(n);
  DevBuf<i64> nsel(1);
  {
    size_t bytes = 0;
    thrust::counting_iterator<i64> it(0);
    CF_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, head.p, hpos.p, nsel.p, n, stream()));
    DevBuf<unsigned char> tmp{static_cast<i64>(bytes)};
    CF_CUDA(cub::DeviceSelect::Flagged(tmp.p, bytes, it, head.p, hpos.p, nsel.p, n, stream()));
    count_launch();
  }
  const i64 nu = read_i64(nsel.p);
  if (mode == 0) {
    k_zero_rows<<<grid_for(ng, 256), 256, 0, stream()>>>(ng, rows, cnt);  // drop the overflow marks
    CF_LAUNCHED();
    k_giant_count<<<grid_for(nu, 256), 256, 0, stream()>>>(nu, hpos.p, key2.p, rows, cnt);
    CF_LAUNCHED();
    return;
  }
  // first unique of every giant row: exclusive prefix of the rows' lengths, in giant order
  DevBuf<i64> first(ng + 1);
  CF_CUDA(cudaMemsetAsync(first.p + ng, 0, sizeof(i64), stream()));
  k_head_len_rows<<<grid_for(ng, 256), 256, 0, stream()>>>(ng, rows, C->ptr.p, first.p);
  CF_LAUNCHED();
  scan_excl(first.p, ng + 1);
  k_giant_emit<<<grid_for(nu, 256), 256, 0, stream()>>>(nu, n, hpos.p, key2.p, mode == 2 ? val2.p : nullptr, rows,
                                                        first.p, C->ptr.p, mode == 1 ? C->col.p : nullptr,
                                                        mode == 2 ? C->val.p : nullptr);
  CF_LAUNCHED();
}

}  // namespace

// pattern of C = A B (sorted columns; values allocated, not computed); L lanes per B row
static std::unique_ptr<Csr> spgemm_symbolic(const Csr& A, const Csr& B, int L, i64 maxb) {
  auto C = std::make_unique<Csr>();
  C->rows = A.rows;
  C->cols = B.cols;
  C->ptr.alloc(A.rows + 1);
  C->ptr.zero();
  const i64 m = A.rows;
  if (m == 0) return C;
  i64* cnt = C->ptr.p;  // row counts in place, scanned into offsets afterwards
  // few rows into a narrow column space (coarse-level products): CTA per row, byte flags
  // test switches: CF_SPGEMM_NO_FLAGS=1 never, CF_SPGEMM_FORCE_PATHS=1 whenever the columns fit
  static const bool no_flags = std::getenv("CF_SPGEMM_NO_FLAGS") != nullptr;
  static const bool force = std::getenv("CF_SPGEMM_FORCE_PATHS") != nullptr;
  if (!no_flags && B.cols <= FLAG_MAX && m < INT_MAX && (force || (m <= 32768 && maxb >= 64))) {
    const size_t sm = size_t(B.cols) + 16;
    static const bool no_staged = std::getenv("CF_SPGEMM_NO_STAGED") != nullptr;
    if (!no_staged) {
      CF_CUDA(cudaFuncSetAttribute(k_sym_flags_st<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
      k_sym_flags_st<0><<<int(m), 256, sm, stream()>>>(m, A.ptr.p, A.col.p, B.ptr.p, B.col.p, int(B.cols), cnt,
                                                       nullptr);
      CF_LAUNCHED();
      scan_excl(C->ptr.p, m + 1);
      C->nnz = read_i64(C->ptr.p + m);
      C->col.alloc(std::max<i64>(C->nnz, 1));
      C->val.alloc(std::max<i64>(C->nnz, 1));
      CF_CUDA(cudaFuncSetAttribute(k_sym_flags_st<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
      k_sym_flags_st<1><<<int(m), 256, sm, stream()>>>(m, A.ptr.p, A.col.p, B.ptr.p, B.col.p, int(B.cols), C->ptr.p,
                                                       C->col.p);
      CF_LAUNCHED();
      return C;
    }
    CF_CUDA(cudaFuncSetAttribute(k_sym_flags<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
    k_sym_flags<0><<<int(m), 256, sm, stream()>>>(m, A.ptr.p, A.col.p, B.ptr.p, B.col.p, int(B.cols), cnt, nullptr);
    CF_LAUNCHED();
    scan_excl(C->ptr.p, m + 1);
    C->nnz = read_i64(C->ptr.p + m);
    C->col.alloc(std::max<i64>(C->nnz, 1));
    C->val.alloc(std::max<i64>(C->nnz, 1));
    CF_CUDA(cudaFuncSetAttribute(k_sym_flags<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
    k_sym_flags<1><<<int(m), 256, sm, stream()>>>(m, A.ptr.p, A.col.p, B.ptr.p, B.col.p, int(B.cols), C->ptr.p,
                                                  C->col.p);
    CF_LAUNCHED();
    return C;
  }
  // 1. symbolic count: all rows with products try the 512-slot tier, which also spills its
  //    unsorted unique columns (<= 384 per row) to scratch; overflow -> 2048 -> CTA tiers
  DevBuf<i64> soff(m + 1);
  DevBuf<int> spill;
  RowBin spilled;
  RowBin o1;
  {
    DevBuf<i64> ub(m);
    k_row_bound<<<grid_for(m, 256), 256, 0, stream()>>>(m, A.ptr.p, A.col.p, B.ptr.p, ub.p);
    CF_LAUNCHED();
    k_spill_cap<<<grid_for(m, 256), 256, 0, stream()>>>(m, ub.p, 384, soff.p);
    CF_LAUNCHED();
    CF_CUDA(cudaMemsetAsync(soff.p + m, 0, sizeof(i64), stream()));
    scan_excl(soff.p, m + 1);
    spill.alloc(std::max<i64>(1, read_i64(soff.p + m)));
    RowBin all = make_bin(m, ub.p, 0, LLONG_MAX);
    if (all.n) {
      if (L == 4)
        k_sym<512, 4, 8, 2><<<grid_for(all.n, 8), 256, 0, stream()>>>(all.list.p, all.n, A.ptr.p, A.col.p, B.ptr.p,
                                                                      B.col.p, cnt, soff.p, spill.p);
      else if (L == 8)
        k_sym<512, 8, 8, 2><<<grid_for(all.n, 8), 256, 0, stream()>>>(all.list.p, all.n, A.ptr.p, A.col.p, B.ptr.p,
                                                                      B.col.p, cnt, soff.p, spill.p);
      else if (L == 16)
        k_sym<512, 16, 8, 2><<<grid_for(all.n, 8), 256, 0, stream()>>>(all.list.p, all.n, A.ptr.p, A.col.p,
                                                                       B.ptr.p, B.col.p, cnt, soff.p, spill.p);
      else
        k_sym<512, 32, 8, 2><<<grid_for(all.n, 8), 256, 0, stream()>>>(all.list.p, all.n, A.ptr.p, A.col.p,
                                                                       B.ptr.p, B.col.p, cnt, soff.p, spill.p);
      CF_LAUNCHED();
    }
    o1 = overflow_of(all, cnt);
    spilled = make_bin(m, cnt, 0, LLONG_MAX);  // rows fully handled by the spill tier (cnt >= 1)
    sym_dispatch(L, 0, o1, 2048, A, B, cnt, nullptr);
    RowBin o2 = overflow_of(o1, cnt);
    if (o2.n) {
      DevBuf<int> flag(1);
      flag.zero();
      const size_t sm = size_t(2) * SYM_BIG * sizeof(int);
      CF_CUDA(cudaFuncSetAttribute(k_sym_cta<SYM_BIG>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
      k_sym_cta<SYM_BIG><<<o2.n, 256, sm, stream()>>>(o2.list.p, o2.n, A.ptr.p, A.col.p, B.ptr.p, B.col.p, cnt,
                                                      nullptr, nullptr, 0, flag.p);
      CF_LAUNCHED();
      if (read_int(flag.p)) {  // rows beyond the CTA hash: the sort tier counts them exactly
        RowBin o3 = overflow_of(o2, cnt);
        giant_rows(0, o3.list.p, o3.n, A, B, nullptr, cnt, nullptr);
      }
    }
  }
  scan_excl(C->ptr.p, m + 1);
  C->nnz = read_i64(C->ptr.p + m);
  C->col.alloc(C->nnz);
  C->val.alloc(C->nnz);
  // 2. symbolic fill
  DevBuf<i64> len(m);
  k_row_len<<<grid_for(m, 256), 256, 0, stream()>>>(m, C->ptr.p, len.p);
  CF_LAUNCHED();
  // spilled rows: sort their scratch columns; overflow rows: hash again in the 2048/CTA tiers
  if (spilled.n) {
    k_sort_rows<512, 8><<<grid_for(spilled.n, 8), 256, 0, stream()>>>(spilled.list.p, spilled.n, soff.p, spill.p,
                                                                       C->ptr.p, C->col.p);
    CF_LAUNCHED();
  }
  spill.release();
  RowBin g2, g3;
  {
    // overflow rows split by exact length (they are > 384 columns)
    DevBuf<i64> olen(m);
    CF_CUDA(cudaMemsetAsync(olen.p, 0, size_t(m) * sizeof(i64), stream()));
    k_scatter_len<<<grid_for(o1.n, 256), 256, 0, stream()>>>(o1.list.p, o1.n, len.p, olen.p);
    CF_LAUNCHED();
    g2 = make_bin(m, olen.p, 0, 1024);
    g3 = make_bin(m, olen.p, 1024, GIANT);
    RowBin g4 = make_bin(m, olen.p, GIANT, LLONG_MAX);
    giant_rows(1, g4.list.p, g4.n, A, B, nullptr, nullptr, C.get());
  }
  sym_dispatch(L, 1, g2, 2048, A, B, nullptr, C.get());
  if (g3.n) {
    RowBin& f3 = g3;
    DevBuf<int> flag(1);
    flag.zero();
    const size_t sm = size_t(2) * SYM_BIG * sizeof(int);
    CF_CUDA(cudaFuncSetAttribute(k_sym_cta<SYM_BIG>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
    k_sym_cta<SYM_BIG><<<f3.n, 256, sm, stream()>>>(f3.list.p, f3.n, A.ptr.p, A.col.p, B.ptr.p, B.col.p, nullptr,
                                                    C->ptr.p, C->col.p, 1, flag.p);
    CF_LAUNCHED();
  }
  return C;
}

// values of C = diag(rs) A B on the rows whose entry of lensel (the C row length, 0 = skip) is
// positive, binned by that length: k-grouped warp kernels (G = 32/L A entries per step), CTA beyond
static void spgemm_numeric(const Csr& A, const Csr& B, const double* row_scale, Csr& C, i64 maxb, int L,
                           const i64* lensel) {
  const i64 m = A.rows;
  // few rows of long B rows (coarse-level RAP): one CTA per row, B rows prefetched
  static const bool no_cta_pf = std::getenv("CF_SPGEMM_NO_CTA_PF") != nullptr;
  static const bool force = std::getenv("CF_SPGEMM_FORCE_PATHS") != nullptr;  // test switch
  if (!no_cta_pf && m > 0 && m < INT_MAX && maxb <= 1024 && (force || (m <= 32768 && maxb >= 128))) {
    RowBin all = make_bin(m, lensel, 0, LLONG_MAX);  // rows with >= 1 output column
    if (all.n) {
      DevBuf<unsigned long long> mx(1);
      mx.zero();
      k_max_row<<<int(std::min<i64>(1024, grid_for(m, 256))), 256, 0, stream()>>>(m, C.ptr.p, mx.p);
      CF_LAUNCHED();
      const i64 ncmax = read_i64(reinterpret_cast<const i64*>(mx.p));
      if (ncmax <= SYM_BIG) {
        const size_t sm = size_t(ncmax) * (sizeof(double) + sizeof(int)) + 16;
        auto launch = [&](auto kern) {
          CF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
          kern<<<all.n, 256, sm, stream()>>>(all.list.p, all.n, A.ptr.p, A.col.p, A.val.p, row_scale, B.ptr.p,
                                             B.col.p, B.val.p, C.ptr.p, C.col.p, C.val.p);
          CF_LAUNCHED();
        };
        // staged form (all B-row loads of 256 A entries in flight at once) when its sub-chunk
        // buffers fit beside the row's accumulators; CF_SPGEMM_NO_STAGED=1: the prefetching kernel
        static const bool no_staged = std::getenv("CF_SPGEMM_NO_STAGED") != nullptr;
        const size_t sms = sm + size_t(ST_CH) * (sizeof(double) + sizeof(int));
        if (!no_staged && sms <= size_t(200) * 1024) {
          CF_CUDA(cudaFuncSetAttribute(k_num_cta_st, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sms)));
          k_num_cta_st<<<all.n, 256, sms, stream()>>>(all.list.p, all.n, A.ptr.p, A.col.p, A.val.p, row_scale, B.ptr.p,
                                                      B.col.p, B.val.p, C.ptr.p, C.col.p, C.val.p);
          CF_LAUNCHED();
          return;
        }
        if (maxb <= 256) launch(k_num_cta_pf<1>);
        else if (maxb <= 512) launch(k_num_cta_pf<2>);
        else launch(k_num_cta_pf<4>);
        return;
      }
    } else {
      return;
    }
  }
  RowBin f1 = make_bin(m, lensel, 0, 256);
  RowBin f2 = make_bin(m, lensel, 256, 1024);
  RowBin f3 = make_bin(m, lensel, 1024, GIANT);
  {
    RowBin f4 = make_bin(m, lensel, GIANT, LLONG_MAX);  // beyond the CTA hash: the sort tier
    giant_rows(2, f4.list.p, f4.n, A, B, row_scale, nullptr, &C);
  }
  const i64 cmax_need = (maxb + L - 1) / L;
  bool warp_ok = true;
  if (cmax_need <= 8) {
    if (L == 4) { num_launch<4, 2>(f1, 512, A, B, row_scale, C); num_launch<4, 2>(f2, 2048, A, B, row_scale, C); }
    else if (L == 8) { num_launch<8, 8>(f1, 512, A, B, row_scale, C); num_launch<8, 8>(f2, 2048, A, B, row_scale, C); }
    else if (L == 16) { num_launch<16, 8>(f1, 512, A, B, row_scale, C); num_launch<16, 8>(f2, 2048, A, B, row_scale, C); }
    else { num_launch<32, 8>(f1, 512, A, B, row_scale, C); num_launch<32, 8>(f2, 2048, A, B, row_scale, C); }
  } else if (cmax_need <= 16) {
    if (L == 8) { num_launch<8, 16>(f1, 512, A, B, row_scale, C); num_launch<8, 16>(f2, 2048, A, B, row_scale, C); }
    else if (L == 16) { num_launch<16, 16>(f1, 512, A, B, row_scale, C); num_launch<16, 16>(f2, 2048, A, B, row_scale, C); }
    else { num_launch<32, 16>(f1, 512, A, B, row_scale, C); num_launch<32, 16>(f2, 2048, A, B, row_scale, C); }
  } else {
    warp_ok = false;
  }
  RowBin n3 = warp_ok ? std::move(f3) : make_bin(m, lensel, 0, GIANT);
  if (n3.n) {
    const size_t sm = size_t(SYM_BIG) * (sizeof(double) + sizeof(int));
    CF_CUDA(cudaFuncSetAttribute(k_num_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
    k_num_cta<<<n3.n, 256, sm, stream()>>>(n3.list.p, n3.n, A.ptr.p, A.col.p, A.val.p, row_scale, B.ptr.p, B.col.p,
                                           B.val.p, C.ptr.p, C.col.p, C.val.p);
    CF_LAUNCHED();
  }
}


std::unique_ptr<Csr> spgemm(const Csr& A, const Csr& B, const double* row_scale) {
  if (A.cols != B.rows) fail(CF_ERR_LOGIC, "spgemm: inner dimensions differ");
  const i64 m = A.rows;
  i64 maxb = 0;
  if (m > 0) {
    DevBuf<unsigned long long> mx(1);
    mx.zero();
    k_max_row<<<int(std::min<i64>(1024, grid_for(B.rows, 256))), 256, 0, stream()>>>(B.rows, B.ptr.p, mx.p);
    CF_LAUNCHED();
    unsigned long long h = 0;
    read_small(&h, mx.p, sizeof(h));
    maxb = i64(h);
  }
  const int L = lanes_for(maxb);
  // Small products (the coarse levels of every hierarchy, eight phi-hierarchies per Newton step):
  // the tiered paths below cost 13-15 host round trips per product to size their row bins, which
  // is all the time such a product takes.  One CTA per row instead, byte-flag symbolic and
  // prefetching numeric over all rows with shared memory for B.cols columns: one round trip (nnz).
  // Same per-entry summation order as every other path (CF_SPGEMM_NO_SMALL=1: tiered paths).
  static const bool no_small = std::getenv("CF_SPGEMM_NO_SMALL") != nullptr;
  static const i64 small_rows = [] {  // CF_SPGEMM_SMALL_ROWS: A/B override of the row limit
    const char* e = std::getenv("CF_SPGEMM_SMALL_ROWS");
    return e ? i64(std::atoll(e)) : SMALL_ROWS;
  }();
  if (!no_small && m > 0 && m <= small_rows && B.cols <= SMALL_COLS && maxb >= 1 && maxb <= 1024) {
    auto C = std::make_unique<Csr>();
    C->rows = m;
    C->cols = B.cols;
    C->ptr.alloc(m + 1);
    CF_CUDA(cudaMemsetAsync(C->ptr.p + m, 0, sizeof(i64), stream()));
    const size_t smf = size_t(B.cols) + 16;
    CF_CUDA(cudaFuncSetAttribute(k_sym_flags_st<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smf)));
    k_sym_flags_st<0><<<int(m), 256, smf, stream()>>>(m, A.ptr.p, A.col.p, B.ptr.p, B.col.p, int(B.cols), C->ptr.p,
                                                      nullptr);
    CF_LAUNCHED();
    scan_excl(C->ptr.p, m + 1);
    C->nnz = read_i64(C->ptr.p + m);
    C->col.alloc(std::max<i64>(C->nnz, 1));
    C->val.alloc(std::max<i64>(C->nnz, 1));
    CF_CUDA(cudaFuncSetAttribute(k_sym_flags_st<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smf)));
    k_sym_flags_st<1><<<int(m), 256, smf, stream()>>>(m, A.ptr.p, A.col.p, B.ptr.p, B.col.p, int(B.cols), C->ptr.p,
                                                      C->col.p);
    CF_LAUNCHED();
    if (C->nnz > 0) {
      // products + slots of a sub-chunk, accumulators and sorted columns of the longest possible row
      const size_t sm = size_t(ST_CH) * (sizeof(double) + sizeof(int)) +
                        size_t(B.cols) * (sizeof(double) + sizeof(int)) + 16;
      CF_CUDA(cudaFuncSetAttribute(k_num_cta_st, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
      k_num_cta_st<<<int(m), 256, sm, stream()>>>(nullptr, m, A.ptr.p, A.col.p, A.val.p, row_scale, B.ptr.p, B.col.p,
                                                  B.val.p,
                                                  C->ptr.p, C->col.p, C->val.p);
      CF_LAUNCHED();
    }
    return C;
  }
  // A/B and test switches: CF_SPGEMM_NOGROUP=1 row-wise only; CF_SPGEMM_GROUP_ALL=1 groups every
  // product the grouped kernel can take (small matrices, short B rows, few shared patterns)
  static const bool no_group = std::getenv("CF_SPGEMM_NOGROUP") != nullptr;
  static const bool group_all = std::getenv("CF_SPGEMM_GROUP_ALL") != nullptr;
  static const bool no_short = std::getenv("CF_SPGEMM_NO_SHORT_GROUP") != nullptr;  // A/B switch
  const bool try_group = group_all ? (m >= 1 && maxb >= 1) : (m >= 1024 && (maxb > 16 || (!no_short && maxb >= 2 && maxb <= 8)));
  if (!no_group && try_group && maxb <= 256 && m < INT_MAX) {
    // row groups, chunked to GRP_MAX rows
    DevBuf<int> head(m), key(m), runstart(m);
    k_same_prev<<<grid_for(m * 32, 256), 256, 0, stream()>>>(m, A.ptr.p, A.col.p, head.p);
    CF_LAUNCHED();
    k_head_key<<<grid_for(m, 256), 256, 0, stream()>>>(m, head.p, key.p);
    CF_LAUNCHED();
    {
      size_t bytes = 0;
      CF_CUDA(cub::DeviceScan::InclusiveScan(nullptr, bytes, key.p, runstart.p, cub::Max(), m, stream()));
      DevBuf<unsigned char> tmp{static_cast<i64>(bytes)};
      CF_CUDA(cub::DeviceScan::InclusiveScan(tmp.p, bytes, key.p, runstart.p, cub::Max(), m, stream()));
      count_launch();
    }
    k_chunk_heads<<<grid_for(m, 256), 256, 0, stream()>>>(m, runstart.p, GRP_MAX, head.p);
    CF_LAUNCHED();
    DevBuf<int> heads(m), nsel(1);
    {
      size_t bytes = 0;
      thrust::counting_iterator<int> it(0);
      CF_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, head.p, heads.p, nsel.p, m, stream()));
      DevBuf<unsigned char> tmp{static_cast<i64>(bytes)};
      CF_CUDA(cub::DeviceSelect::Flagged(tmp.p, bytes, it, head.p, heads.p, nsel.p, m, stream()));
      count_launch();
    }
    const int ng = read_int(nsel.p);
    if (group_all || double(ng) <= 0.6 * double(m)) {
      key.release();
      runstart.release();
      head.release();
      DevBuf<int> glen(ng);
      k_group_len<<<grid_for(ng, 256), 256, 0, stream()>>>(ng, heads.p, m, glen.p);
      CF_LAUNCHED();
      // accumulator rows per warp = the longest group (3 on the node-structured fine level, 6 on
      // coarse levels): the shared-memory footprint, hence the resident warps, follows it
      int gmax = GRP_MAX;
      {
        DevBuf<int> mx(1);
        mx.zero();
        k_max_int<<<int(std::min<i64>(1024, grid_for(ng, 256))), 256, 0, stream()>>>(ng, glen.p, mx.p);
        CF_LAUNCHED();
        gmax = std::max(1, std::min(GRP_MAX, read_int(mx.p)));
      }
      // symbolic on the head rows
      Csr Ag;
      Ag.rows = ng;
      Ag.cols = A.cols;
      Ag.ptr.alloc(ng + 1);
      CF_CUDA(cudaMemsetAsync(Ag.ptr.p + ng, 0, sizeof(i64), stream()));
      k_head_len<<<grid_for(ng, 256), 256, 0, stream()>>>(ng, heads.p, A.ptr.p, Ag.ptr.p);
      CF_LAUNCHED();
      scan_excl(Ag.ptr.p, ng + 1);
      Ag.nnz = read_i64(Ag.ptr.p + ng);
      Ag.col.alloc(std::max<i64>(Ag.nnz, 1));
      k_gather_rows<<<grid_for(i64(ng) * 32, 256), 256, 0, stream()>>>(ng, heads.p, A.ptr.p, A.col.p, Ag.ptr.p,
                                                                      Ag.col.p);
      CF_LAUNCHED();
      auto Cg = spgemm_symbolic(Ag, B, L, maxb);
      Ag.col.release();
      // expand to the rows
      auto C = std::make_unique<Csr>();
      C->rows = m;
      C->cols = B.cols;
      C->ptr.alloc(m + 1);
      CF_CUDA(cudaMemsetAsync(C->ptr.p + m, 0, sizeof(i64), stream()));
      k_expand_len<<<grid_for(ng, 256), 256, 0, stream()>>>(ng, heads.p, glen.p, Cg->ptr.p, C->ptr.p);
      CF_LAUNCHED();
      scan_excl(C->ptr.p, m + 1);
      C->nnz = read_i64(C->ptr.p + m);
      C->col.alloc(std::max<i64>(C->nnz, 1));
      C->val.alloc(std::max<i64>(C->nnz, 1));
      k_expand_cols<<<grid_for(i64(ng) * 32, 256), 256, 0, stream()>>>(ng, heads.p, glen.p, Cg->ptr.p, Cg->col.p,
                                                                      C->ptr.p, C->col.p);
      CF_LAUNCHED();
      Cg.reset();
      // numeric: groups binned by their row length (hash tiers); beyond 384 columns row-wise
      DevBuf<i64> gl(ng);
      k_group_clen<<<grid_for(ng, 256), 256, 0, stream()>>>(ng, heads.p, C->ptr.p, gl.p);
      CF_LAUNCHED();
      const int caps[3] = {128, 256, 512};
      const i64 lims[4] = {0, 96, 192, 384};
      // runs of B rows with one pattern (CF_SPGEMM_NO_RUNS=1: one position at a time; A/B switch)
      static const bool no_runs = std::getenv("CF_SPGEMM_NO_RUNS") != nullptr;
      DevBuf<unsigned char> bsame;
      static const bool short_runs = std::getenv("CF_SPGEMM_SHORT_RUNS") != nullptr;  // A/B switch
      if (!no_runs && (short_runs || !(maxb <= 8 && !no_short)) && B.rows > 1) {
        DevBuf<int> bh(B.rows);
        k_same_prev<<<grid_for(B.rows * 32, 256), 256, 0, stream()>>>(B.rows, B.ptr.p, B.col.p, bh.p);
        CF_LAUNCHED();
        bsame.alloc(B.rows);
        k_not_head<<<grid_for(B.rows, 256), 256, 0, stream()>>>(B.rows, bh.p, bsame.p);
        CF_LAUNCHED();
      }
      const unsigned char* bs = bsame.n ? bsame.p : nullptr;
      for (int t = 0; t < 3; ++t) {
        RowBin b = make_bin(ng, gl.p, lims[t], lims[t + 1]);
        if (maxb <= 8 && !no_short) num_grp_launch<0>(b, caps[t], heads.p, glen.p, A, B, row_scale, *C, gmax, bs);
        else if (maxb <= 32) num_grp_launch<1>(b, caps[t], heads.p, glen.p, A, B, row_scale, *C, gmax, bs);
        else if (maxb <= 64) num_grp_launch<2>(b, caps[t], heads.p, glen.p, A, B, row_scale, *C, gmax, bs);
        else if (maxb <= 128) num_grp_launch<4>(b, caps[t], heads.p, glen.p, A, B, row_scale, *C, gmax, bs);
        else num_grp_launch<8>(b, caps[t], heads.p, glen.p, A, B, row_scale, *C, gmax, bs);
      }
      RowBin big = make_bin(ng, gl.p, 384, LLONG_MAX);
      if (big.n) {
        DevBuf<i64> sel(m);
        CF_CUDA(cudaMemsetAsync(sel.p, 0, size_t(m) * sizeof(i64), stream()));
        k_select_group_rows<<<grid_for(big.n, 256), 256, 0, stream()>>>(big.n, big.list.p, heads.p, glen.p, C->ptr.p,
                                                                        sel.p);
        CF_LAUNCHED();
        spgemm_numeric(A, B, row_scale, *C, maxb, L, sel.p);
      }
      return C;
    }
  }
  auto C = spgemm_symbolic(A, B, L, maxb);
  if (m > 0) {
    DevBuf<i64> len(m);
    k_row_len<<<grid_for(m, 256), 256, 0, stream()>>>(m, C->ptr.p, len.p);
    CF_LAUNCHED();
    spgemm_numeric(A, B, row_scale, *C, maxb, L, len.p);
  }
  return C;
}

std::shared_ptr<RowGroups> csr_row_groups(const Csr& A, int gmax) {
  const i64 m = A.rows;
  if (m < 1024 || m >= INT_MAX || A.nnz < 8 * m || gmax < 2) return nullptr;
  DevBuf<int> head(m), key(m), runstart(m);
  k_same_prev<<<grid_for(m * 32, 256), 256, 0, stream()>>>(m, A.ptr.p, A.col.p, head.p);
  CF_LAUNCHED();
  k_head_key<<<grid_for(m, 256), 256, 0, stream()>>>(m, head.p, key.p);
  CF_LAUNCHED();
  {
    size_t bytes = 0;
    CF_CUDA(cub::DeviceScan::InclusiveScan(nullptr, bytes, key.p, runstart.p, cub::Max(), m, stream()));
    DevBuf<unsigned char> tmp{static_cast<i64>(bytes)};
    CF_CUDA(cub::DeviceScan::InclusiveScan(tmp.p, bytes, key.p, runstart.p, cub::Max(), m, stream()));
    count_launch();
  }
  k_chunk_heads<<<grid_for(m, 256), 256, 0, stream()>>>(m, runstart.p, gmax, head.p);
  CF_LAUNCHED();
  auto g = std::make_shared<RowGroups>();
  g->heads.alloc(m);
  DevBuf<int> nsel(1);
  {
    size_t bytes = 0;
    thrust::counting_iterator<int> it(0);
    CF_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, head.p, g->heads.p, nsel.p, m, stream()));
    DevBuf<unsigned char> tmp{static_cast<i64>(bytes)};
    CF_CUDA(cub::DeviceSelect::Flagged(tmp.p, bytes, it, head.p, g->heads.p, nsel.p, m, stream()));
    count_launch();
  }
  const int ng = read_int(nsel.p);
  if (double(ng) * 4.0 > double(m) * 3.0) return nullptr;
  g->n = ng;
  g->len.alloc(ng);
  k_group_len<<<grid_for(ng, 256), 256, 0, stream()>>>(ng, g->heads.p, m, g->len.p);
  CF_LAUNCHED();
  DevBuf<int> mx(1);
  mx.zero();
  k_max_int<<<int(std::min<i64>(1024, grid_for(ng, 256))), 256, 0, stream()>>>(ng, g->len.p, mx.p);
  CF_LAUNCHED();
  g->gmax = read_int(mx.p);
  return g;
}

// ------------------------------------------------------------------ transpose (stable)
namespace {
__global__ void k_iota64(i64 n, i64* out) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = i;
}
__global__ void k_row_of_entry(i64 rows, const i64* __restrict__ ptr, int* __restrict__ row_of) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  for (i64 k = ptr[i]; k < ptr[i + 1]; ++k) row_of[k] = int(i);
}
__global__ void k_gather_t(i64 nnz, const i64* __restrict__ perm, const int* __restrict__ row_of,
                           const double* __restrict__ val, int* __restrict__ tcol, double* __restrict__ tval) {
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nnz) return;
  const i64 e = perm[t];
  tcol[t] = row_of[e];
  tval[t] = val[e];
}
__global__ void k_count_cols(i64 nnz, const int* __restrict__ col, i64* __restrict__ cnt) {
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < nnz) atomicAdd(reinterpret_cast<unsigned long long*>(cnt + col[t]), 1ull);
}
int bits_for(i64 n) {
  int b = 1;
  while ((i64(1) << b) < n) ++b;
  return b;
}
}  // namespace

std::unique_ptr<Csr> transpose(const Csr& A) {
  auto T = std::make_unique<Csr>();
  T->rows = A.cols;
  T->cols = A.rows;
  T->nnz = A.nnz;
  T->ptr.alloc(A.cols + 1);
  T->ptr.zero();
  T->col.alloc(A.nnz);
  T->val.alloc(A.nnz);
  if (A.nnz == 0) return T;
  k_count_cols<<<grid_for(A.nnz, 256), 256, 0, stream()>>>(A.nnz, A.col.p, T->ptr.p);
  CF_LAUNCHED();
  scan_excl(T->ptr.p, A.cols + 1);
  // stable sort of entry indices by column: within a column, rows stay ascending
  DevBuf<i64> idx(A.nnz), perm(A.nnz);
  DevBuf<int> keys_out(A.nnz);
  k_iota64<<<grid_for(A.nnz, 256), 256, 0, stream()>>>(A.nnz, idx.p);
  CF_LAUNCHED();
  size_t bytes = 0;
  const int eb = bits_for(A.cols + 1);
  CF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, A.col.p, keys_out.p, idx.p, perm.p, A.nnz, 0, eb, stream()));
  {
    DevBuf<unsigned char> tmp{static_cast<i64>(bytes)};
    CF_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, A.col.p, keys_out.p, idx.p, perm.p, A.nnz, 0, eb,
                                            stream()));
    count_launch();
  }
  DevBuf<int> row_of(A.nnz);
  k_row_of_entry<<<grid_for(A.rows, 256), 256, 0, stream()>>>(A.rows, A.ptr.p, row_of.p);
  CF_LAUNCHED();
  k_gather_t<<<grid_for(A.nnz, 256), 256, 0, stream()>>>(A.nnz, perm.p, row_of.p, A.val.p, T->col.p, T->val.p);
  CF_LAUNCHED();
  return T;
}

// ------------------------------------------------------------------ union axpy + prune
namespace {
// mode 0: count; mode 1: write.  P(i,:) = T(i,:) - w DAT(i,:) over the union, |v| > 1e-300 kept.
__global__ void k_axpy_merge(i64 rows, const i64* __restrict__ tp, const int* __restrict__ tc,
                             const double* __restrict__ tv, double w, const i64* __restrict__ dp,
                             const int* __restrict__ dc, const double* __restrict__ dv, i64* __restrict__ pp,
                             int* __restrict__ pc, double* __restrict__ pv, int mode) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  i64 a = tp[i], ae = tp[i + 1], b = dp[i], be = dp[i + 1];
  i64 out = mode ? pp[i] : 0;
  i64 n = 0;
  while (a < ae || b < be) {
    int c;
    double v;
    if (b >= be || (a < ae && tc[a] < dc[b])) {
      c = tc[a];
      v = tv[a];
      ++a;
    } else if (a >= ae || dc[b] < tc[a]) {
      c = dc[b];
      v = 0.0 - w * dv[b];
      ++b;
    } else {
      c = tc[a];
      v = tv[a] - w * dv[b];
      ++a;
      ++b;
    }
    if (fabs(v) > 1e-300) {
      if (mode) {
        pc[out + n] = c;
        pv[out + n] = v;
      }
      ++n;
    }
  }
  if (!mode) pp[i] = n;
}

// P = T - w D^-1 A T, warp per row: when T's pattern is contained in DAT's (A carries its
// diagonal, so it always is for the AMG products) the merged row is DAT's pattern; lanes take DAT's
// entries coalesced, look their column up among T's <= 32 entries (registers + shuffles) and
// compact the kept values with a ballot.  Rows where T has a column DAT lacks are left to the
// serial merge (flag).  The values are k_axpy_merge's expressions.
__global__ void k_axpy_merge_w(i64 rows, const i64* __restrict__ tp, const int* __restrict__ tc,
                               const double* __restrict__ tv, double w, const i64* __restrict__ dp,
                               const int* __restrict__ dc, const double* __restrict__ dv, i64* __restrict__ pp,
                               int* __restrict__ pc, double* __restrict__ pv, int mode, int* __restrict__ serial) {
  const i64 i = (i64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= rows) return;
  const i64 a = tp[i], na = tp[i + 1] - a, b = dp[i], nb = dp[i + 1] - b;
  if (na > 32) {  // not handled here
    if (mode == 0 && lane == 0) serial[i] = 1;
    return;
  }
  if (mode == 1 && serial[i]) return;
  const int myc = lane < na ? tc[a + lane] : -1;
  const double mytv = lane < na ? tv[a + lane] : 0.0;
  int matched = 0;
  i64 n = 0;
  const i64 out = mode ? pp[i] : 0;
  for (i64 base = 0; base < nb; base += 32) {
    const i64 e = base + lane;
    const bool in = e < nb;
    const int c = in ? dc[b + e] : -2;
    const double d = in ? dv[b + e] : 0.0;
    int hit = -1;
    for (int t = 0; t < na; ++t)
      if (__shfl_sync(0xffffffffu, myc, t) == c) hit = t;
    double v = 0.0;
    const double tvh = __shfl_sync(0xffffffffu, mytv, hit < 0 ? 0 : hit);
    if (hit >= 0) v = tvh - w * d;
    else v = 0.0 - w * d;
    const bool keep = in && fabs(v) > 1e-300;
    matched += __popc(__ballot_sync(0xffffffffu, in && hit >= 0));
    const unsigned km = __ballot_sync(0xffffffffu, keep);
    if (mode == 1 && keep) {
      const i64 o = out + n + __popc(km & ((1u << lane) - 1u));
      pc[o] = c;
      pv[o] = v;
    }
    n += __popc(km);
  }
  if (mode == 0 && lane == 0) {
    const bool ok = matched == na;  // every T column found in DAT: the merge is DAT's pattern
    serial[i] = ok ? 0 : 1;
    if (ok) pp[i] = n;
  }
}

// the serial merge restricted to the flagged rows
__global__ void k_axpy_merge_rows(i64 rows, const int* __restrict__ serial, const i64* __restrict__ tp,
                                  const int* __restrict__ tc, const double* __restrict__ tv, double w,
                                  const i64* __restrict__ dp, const int* __restrict__ dc,
                                  const double* __restrict__ dv, i64* __restrict__ pp, int* __restrict__ pc,
                                  double* __restrict__ pv, int mode) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows || !serial[i]) return;
  i64 a = tp[i], ae = tp[i + 1], b = dp[i], be = dp[i + 1];
  i64 out = mode ? pp[i] : 0;
  i64 n = 0;
  while (a < ae || b < be) {
    int c;
    double v;
    if (b >= be || (a < ae && tc[a] < dc[b])) {
      c = tc[a];
      v = tv[a];
      ++a;
    } else if (a >= ae || dc[b] < tc[a]) {
      c = dc[b];
      v = 0.0 - w * dv[b];
      ++b;
    } else {
      c = tc[a];
      v = tv[a] - w * dv[b];
      ++a;
      ++b;
    }
    if (fabs(v) > 1e-300) {
      if (mode) {
        pc[out + n] = c;
        pv[out + n] = v;
      }
      ++n;
    }
  }
  if (!mode) pp[i] = n;
}

__global__ void k_prune(i64 rows, const i64* __restrict__ ip, const int* __restrict__ ic, const double* __restrict__ iv,
                        i64* __restrict__ op, int* __restrict__ oc, double* __restrict__ ov, int mode) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  i64 n = 0;
  const i64 base = mode ? op[i] : 0;
  for (i64 k = ip[i]; k < ip[i + 1]; ++k)
    if (fabs(iv[k]) > 1e-300) {
      if (mode) {
        oc[base + n] = ic[k];
        ov[base + n] = iv[k];
      }
      ++n;
    }
  if (!mode) op[i] = n;
}

// k_prune with a warp per row (coalesced; rows of tens to hundreds of entries): kept entries are
// compacted in order by a ballot prefix
__global__ void k_prune_w(i64 rows, const i64* __restrict__ ip, const int* __restrict__ ic,
                          const double* __restrict__ iv, i64* __restrict__ op, int* __restrict__ oc,
                          double* __restrict__ ov, int mode) {
  const i64 i = (i64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= rows) return;
  const i64 b = ip[i], e = ip[i + 1];
  const i64 base = mode ? op[i] : 0;
  i64 n = 0;
  for (i64 k0 = b; k0 < e; k0 += 32) {
    const i64 k = k0 + lane;
    const bool keep = k < e && fabs(iv[k]) > 1e-300;
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (mode && keep) {
      const i64 o = base + n + __popc(m & ((1u << lane) - 1u));
      oc[o] = ic[k];
      ov[o] = iv[k];
    }
    n += __popc(m);
  }
  if (!mode && lane == 0) op[i] = n;
}

__global__ void k_diag(i64 rows, const i64* __restrict__ p, const int* __restrict__ c, const double* __restrict__ v,
                       double* __restrict__ d) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  i64 lo = p[i], hi = p[i + 1];
  while (lo < hi) {
    const i64 mid = (lo + hi) >> 1;
    if (c[mid] < i) lo = mid + 1; else hi = mid;
  }
  d[i] = (lo < p[i + 1] && c[lo] == i) ? v[lo] : 0.0;
}
}  // namespace

std::unique_ptr<Csr> csr_axpy_prune(const Csr& T, double w, const Csr& DAT) {
  auto P = std::make_unique<Csr>();
  P->rows = T.rows;
  P->cols = T.cols;
  P->ptr.alloc(T.rows + 1);
  P->ptr.zero();
  static const bool serial_only = std::getenv("CF_AXPY_SERIAL") != nullptr;  // A/B switch
  // warp per row pays off for rows of tens of entries (the u-block); short rows stay serial
  if (serial_only || DAT.nnz < 16 * T.rows) {
    k_axpy_merge<<<grid_for(T.rows, 256), 256, 0, stream()>>>(T.rows, T.ptr.p, T.col.p, T.val.p, w, DAT.ptr.p,
                                                              DAT.col.p, DAT.val.p, P->ptr.p, nullptr, nullptr, 0);
    CF_LAUNCHED();
  } else {
    // warp-per-row merge where T's pattern lies in DAT's; the serial merge for the other rows
    DevBuf<int> serial(T.rows);
    k_axpy_merge_w<<<grid_for(T.rows * 32, 256), 256, 0, stream()>>>(T.rows, T.ptr.p, T.col.p, T.val.p, w, DAT.ptr.p,
                                                                     DAT.col.p, DAT.val.p, P->ptr.p, nullptr,
                                                                     nullptr, 0, serial.p);
    CF_LAUNCHED();
    k_axpy_merge_rows<<<grid_for(T.rows, 256), 256, 0, stream()>>>(T.rows, serial.p, T.ptr.p, T.col.p, T.val.p, w,
                                                                   DAT.ptr.p, DAT.col.p, DAT.val.p, P->ptr.p,
                                                                   nullptr, nullptr, 0);
    CF_LAUNCHED();
    scan_excl(P->ptr.p, T.rows + 1);
    P->nnz = read_i64(P->ptr.p + T.rows);
    P->col.alloc(P->nnz);
    P->val.alloc(P->nnz);
    k_axpy_merge_w<<<grid_for(T.rows * 32, 256), 256, 0, stream()>>>(T.rows, T.ptr.p, T.col.p, T.val.p, w, DAT.ptr.p,
                                                                     DAT.col.p, DAT.val.p, P->ptr.p, P->col.p,
                                                                     P->val.p, 1, serial.p);
    CF_LAUNCHED();
    k_axpy_merge_rows<<<grid_for(T.rows, 256), 256, 0, stream()>>>(T.rows, serial.p, T.ptr.p, T.col.p, T.val.p, w,
                                                                   DAT.ptr.p, DAT.col.p, DAT.val.p, P->ptr.p,
                                                                   P->col.p, P->val.p, 1);
    CF_LAUNCHED();
    return P;
  }
  scan_excl(P->ptr.p, T.rows + 1);
  P->nnz = read_i64(P->ptr.p + T.rows);
  P->col.alloc(P->nnz);
  P->val.alloc(P->nnz);
  k_axpy_merge<<<grid_for(T.rows, 256), 256, 0, stream()>>>(T.rows, T.ptr.p, T.col.p, T.val.p, w, DAT.ptr.p,
                                                            DAT.col.p, DAT.val.p, P->ptr.p, P->col.p, P->val.p, 1);
  CF_LAUNCHED();
  return P;
}

void csr_prune(Csr& A) {
  DevBuf<i64> np(A.rows + 1);
  np.zero();
  const bool warp = A.nnz >= 16 * A.rows;  // long rows: warp per row, coalesced
  if (warp)
    k_prune_w<<<grid_for(A.rows * 32, 256), 256, 0, stream()>>>(A.rows, A.ptr.p, A.col.p, A.val.p, np.p, nullptr,
                                                                nullptr, 0);
  else
    k_prune<<<grid_for(A.rows, 256), 256, 0, stream()>>>(A.rows, A.ptr.p, A.col.p, A.val.p, np.p, nullptr, nullptr, 0);
  CF_LAUNCHED();
  scan_excl(np.p, A.rows + 1);
  const i64 nnz = read_i64(np.p + A.rows);
  if (nnz == A.nnz) return;
  DevBuf<int> nc(nnz);
  DevBuf<double> nv(nnz);
  if (warp)
    k_prune_w<<<grid_for(A.rows * 32, 256), 256, 0, stream()>>>(A.rows, A.ptr.p, A.col.p, A.val.p, np.p, nc.p, nv.p,
                                                                1);
  else
    k_prune<<<grid_for(A.rows, 256), 256, 0, stream()>>>(A.rows, A.ptr.p, A.col.p, A.val.p, np.p, nc.p, nv.p, 1);
  CF_LAUNCHED();
  A.ptr = std::move(np);
  A.col = std::move(nc);
  A.val = std::move(nv);
  A.nnz = nnz;
}

void csr_diagonal(const Csr& A, double* d) {
  if (A.rows == 0) return;
  k_diag<<<grid_for(A.rows, 256), 256, 0, stream()>>>(A.rows, A.ptr.p, A.col.p, A.val.p, d);
  CF_LAUNCHED();
}

namespace {
// columns are sorted, so a row's entries in [lo, hi) are one contiguous run
__device__ inline void col_run(const i64* p, const int* c, i64 i, int lo, int hi, i64& b, i64& e) {
  i64 a = p[i], z = p[i + 1];
  while (a < z) {  // first entry >= lo
    const i64 m = (a + z) >> 1;
    if (c[m] < lo) a = m + 1; else z = m;
  }
  b = a;
  z = p[i + 1];
  while (a < z) {  // first entry >= hi
    const i64 m = (a + z) >> 1;
    if (c[m] < hi) a = m + 1; else z = m;
  }
  e = a;
}

__global__ void k_extract_count(i64 rows, const i64* __restrict__ p, const int* __restrict__ c, int lo, int hi,
                                i64* __restrict__ cnt) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  i64 b, e;
  col_run(p, c, i, lo, hi, b, e);
  cnt[i] = e - b;
}

// warp per row: coalesced copy of the row's run, columns shifted by -lo
__global__ void k_extract_fill(i64 rows, const i64* __restrict__ p, const int* __restrict__ c,
                               const double* __restrict__ v, int lo, int hi, const i64* __restrict__ np,
                               int* __restrict__ nc, double* __restrict__ nv) {
  const i64 i = (i64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= rows) return;
  i64 b, e;
  col_run(p, c, i, lo, hi, b, e);
  const i64 o = np[i];
  for (i64 k = b + lane; k < e; k += 32) {
    nc[o + (k - b)] = c[k] - lo;
    nv[o + (k - b)] = v[k];
  }
}
}  // namespace

std::unique_ptr<Csr> csr_extract_cols(const Csr& A, i64 lo, i64 hi) {
  auto C = std::make_unique<Csr>();
  C->rows = A.rows;
  C->cols = hi - lo;
  C->ptr.alloc(A.rows + 1);
  C->ptr.zero();
  k_extract_count<<<grid_for(A.rows, 256), 256, 0, stream()>>>(A.rows, A.ptr.p, A.col.p, int(lo), int(hi), C->ptr.p);
  CF_LAUNCHED();
  scan_excl(C->ptr.p, A.rows + 1);
  C->nnz = read_i64(C->ptr.p + A.rows);
  C->col.alloc(C->nnz);
  C->val.alloc(C->nnz);
  k_extract_fill<<<grid_for(A.rows * 32, 256), 256, 0, stream()>>>(A.rows, A.ptr.p, A.col.p, A.val.p, int(lo),
                                                                   int(hi), C->ptr.p, C->col.p, C->val.p);
  CF_LAUNCHED();
  return C;
}

namespace {
__global__ void k_ptr_sub(const i64* __restrict__ p, i64 n, i64* __restrict__ out) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = p[i] - p[0];
}
}  // namespace

std::unique_ptr<Csr> csr_extract_rows(const Csr& A, i64 lo, i64 hi) {
  auto C = std::make_unique<Csr>();
  lo = std::max<i64>(0, std::min(lo, A.rows));
  hi = std::max(lo, std::min(hi, A.rows));
  C->rows = hi - lo;
  C->cols = A.cols;
  C->ptr.alloc(C->rows + 1);
  k_ptr_sub<<<grid_for(C->rows + 1, 256), 256, 0, stream()>>>(A.ptr.p + lo, C->rows + 1, C->ptr.p);
  CF_LAUNCHED();
  i64 b[2] = {0, 0};
  CF_CUDA(cudaMemcpyAsync(&b[0], A.ptr.p + lo, sizeof(i64), cudaMemcpyDeviceToHost, stream()));
  CF_CUDA(cudaMemcpyAsync(&b[1], A.ptr.p + hi, sizeof(i64), cudaMemcpyDeviceToHost, stream()));
  CF_CUDA(cudaStreamSynchronize(stream()));
  C->nnz = b[1] - b[0];
  C->col.alloc(std::max<i64>(C->nnz, 1));
  C->val.alloc(std::max<i64>(C->nnz, 1));
  if (C->nnz) {
    CF_CUDA(cudaMemcpyAsync(C->col.p, A.col.p + b[0], size_t(C->nnz) * sizeof(int), cudaMemcpyDeviceToDevice,
                            stream()));
    CF_CUDA(cudaMemcpyAsync(C->val.p, A.val.p + b[0], size_t(C->nnz) * sizeof(double), cudaMemcpyDeviceToDevice,
                            stream()));
  }
  // the lane split of the undivided matrix, so every row reduces exactly as there
  C->mean_hint = A.mean_hint >= 0.0 ? A.mean_hint : (A.rows ? double(A.nnz) / double(A.rows) : 0.0);
  return C;
}

std::unique_ptr<Csr> csr_copy(const Csr& A) {
  auto C = std::make_unique<Csr>();
  C->rows = A.rows;
  C->cols = A.cols;
  C->nnz = A.nnz;
  C->ptr.alloc(A.rows + 1);
  C->col.alloc(A.nnz);
  C->val.alloc(A.nnz);
  CF_CUDA(cudaMemcpyAsync(C->ptr.p, A.ptr.p, size_t(A.rows + 1) * sizeof(i64), cudaMemcpyDeviceToDevice, stream()));
  if (A.nnz) {
    CF_CUDA(cudaMemcpyAsync(C->col.p, A.col.p, size_t(A.nnz) * sizeof(int), cudaMemcpyDeviceToDevice, stream()));
    CF_CUDA(cudaMemcpyAsync(C->val.p, A.val.p, size_t(A.nnz) * sizeof(double), cudaMemcpyDeviceToDevice, stream()));
  }
  return C;
}

}  // namespace cfb

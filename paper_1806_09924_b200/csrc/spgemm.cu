// Deterministic sparse kernels for the AMG setup: Gustavson SpGEMM,
// transpose, union-axpy with pruning, prune, diagonal extraction.
//
// SpGEMM C = diag(s) A B (linsolve.cpp:248-263: D^-1 A T, A P, P^T (A P)) in three passes:
//   1. symbolic count — per row, a shared-memory hash set of the output columns (warp per row
//      with 512 / 2048 slots; rows that overflow are redone by a CTA with 16384 slots);
//   2. symbolic fill  — the same hash, then a bitonic sort of the unique columns (sorted CSR);
//   3. numeric        — per row, A's entries are visited in ascending column order and each
//      B row is spread over the lanes; the accumulator slot comes from a binary search in the
//      row's sorted column list.  Every C(i,j) is therefore the k-ascending sequential sum
//      sum_k (s_i A_ik) B_kj — the same IEEE sequence as Eigen's conservative sparse product
//      and the oracle, independent of the launch configuration (no floating-point atomics).
#include <cub/cub.cuh>

#include <climits>

#include "cf_vec.hpp"

namespace cfb {

namespace {

constexpr int EMPTY = -1;

__device__ __forceinline__ unsigned hslot(int key, unsigned mask) { return (unsigned(key) * 2654435761u) & mask; }

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

// --- symbolic, warp per row ---------------------------------------------------------------
// mode 0: count (cnt[row] = unique, or -1 on overflow); mode 1: fill sorted columns into ccol
template <int CAP, int WPB>
__global__ void __launch_bounds__(WPB * 32) k_sym_warp(const int* __restrict__ rowlist, i64 nrows,
                                                       const i64* __restrict__ ap, const int* __restrict__ ac,
                                                       const i64* __restrict__ bp, const int* __restrict__ bc,
                                                       i64* __restrict__ cnt, const i64* __restrict__ cptr,
                                                       int* __restrict__ ccol, int mode) {
  __shared__ int tab[WPB][CAP];
  __shared__ int nuniq[WPB];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const i64 r = i64(blockIdx.x) * WPB + w;
  if (r >= nrows) return;
  const i64 i = rowlist ? rowlist[r] : r;
  int* T = tab[w];
  for (int s = lane; s < CAP; s += 32) T[s] = EMPTY;
  if (lane == 0) nuniq[w] = 0;
  __syncwarp();
  const unsigned mask = CAP - 1;
  int mine = 0;
  bool full = false;
  for (i64 ka = ap[i]; ka < ap[i + 1] && !full; ++ka) {
    const int k = ac[ka];
    for (i64 kb = bp[k] + lane; kb < bp[k + 1]; kb += 32) {
      const int r2 = hinsert(T, mask, bc[kb]);
      if (r2 < 0) full = true; else mine += r2;
    }
    // warp-uniform early exit once the table is 3/4 full (overflow -> CTA tier)
    int tot = mine;
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    full = __any_sync(0xffffffffu, full) || tot > (CAP * 3) / 4;
  }
  // warp total
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  __syncwarp();
  if (full || mine > (CAP * 3) / 4) {
    if (lane == 0 && mode == 0) cnt[i] = -1;
    return;  // mode 1 is only launched for rows known to fit
  }
  if (mode == 0) {
    if (lane == 0) cnt[i] = mine;
    return;
  }
  // compact + bitonic sort (size = next pow2 of the unique count)
  int n2 = 1;
  while (n2 < mine) n2 <<= 1;
  // compact keys to the front of a second region: reuse T by first collecting in registers is
  // impractical, so compact in place through a prefix over slots.
  __shared__ int buf[WPB][CAP];
  int* Bf = buf[w];
  if (lane == 0) nuniq[w] = 0;
  __syncwarp();
  for (int s = lane; s < CAP; s += 32) {
    const int key = T[s];
    if (key != EMPTY) {
      const int p = atomicAdd(&nuniq[w], 1);
      Bf[p] = key;
    }
  }
  __syncwarp();
  for (int s = mine + lane; s < n2; s += 32) Bf[s] = INT_MAX;
  __syncwarp();
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
  const i64 base = cptr[i];
  for (int t = lane; t < mine; t += 32) ccol[base + t] = Bf[t];
}

// --- symbolic, CTA per row (overflow rows) ---------------------------------------------------
template <int CAP>
__global__ void __launch_bounds__(256) k_sym_cta(const int* __restrict__ rowlist, i64 nrows,
                                                 const i64* __restrict__ ap, const int* __restrict__ ac,
                                                 const i64* __restrict__ bp, const int* __restrict__ bc,
                                                 i64* __restrict__ cnt, const i64* __restrict__ cptr,
                                                 int* __restrict__ ccol, int mode, int* __restrict__ overflow) {
  extern __shared__ int sm[];
  int* T = sm;            // CAP
  int* Bf = sm + CAP;     // CAP (mode 1)
  __shared__ int nuniq;
  const i64 r = blockIdx.x;
  if (r >= nrows) return;
  const i64 i = rowlist ? rowlist[r] : r;
  for (int s = threadIdx.x; s < CAP; s += blockDim.x) T[s] = EMPTY;
  if (threadIdx.x == 0) nuniq = 0;
  __syncthreads();
  const unsigned mask = CAP - 1;
  __shared__ int sfull;
  if (threadIdx.x == 0) sfull = 0;
  __syncthreads();
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

__device__ __forceinline__ int lower_bound_sm(const int* a, int n, int key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// --- numeric, warp per row with smem columns/accumulators -----------------------------------
template <int CAP, int WPB>
__global__ void __launch_bounds__(WPB * 32) k_num_warp(const int* __restrict__ rowlist, i64 nrows,
                                                       const i64* __restrict__ ap, const int* __restrict__ ac,
                                                       const double* __restrict__ av,
                                                       const double* __restrict__ rs, const i64* __restrict__ bp,
                                                       const int* __restrict__ bc, const double* __restrict__ bv,
                                                       const i64* __restrict__ cp, const int* __restrict__ cc,
                                                       double* __restrict__ cv) {
  __shared__ int cols[WPB][CAP];
  __shared__ double acc[WPB][CAP];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const i64 r = i64(blockIdx.x) * WPB + w;
  if (r >= nrows) return;
  const i64 i = rowlist ? rowlist[r] : r;
  const i64 c0 = cp[i];
  const int nc = int(cp[i + 1] - c0);
  for (int t = lane; t < nc; t += 32) {
    cols[w][t] = cc[c0 + t];
    acc[w][t] = 0.0;
  }
  __syncwarp();
  const double si = rs ? rs[i] : 1.0;
  for (i64 ka = ap[i]; ka < ap[i + 1]; ++ka) {
    const int k = ac[ka];
    const double a = rs ? si * av[ka] : av[ka];
    for (i64 kb = bp[k] + lane; kb < bp[k + 1]; kb += 32) {
      const int pos = lower_bound_sm(cols[w], nc, bc[kb]);
      acc[w][pos] += a * bv[kb];
    }
    __syncwarp();
  }
  for (int t = lane; t < nc; t += 32) cv[c0 + t] = acc[w][t];
}

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

// partition rows by a predicate on a per-row value: out lists in ascending row order
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
__global__ void k_bin_overflow(i64 rows, const i64* __restrict__ cnt, int* __restrict__ list, int* __restrict__ count) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < rows && cnt[i] < 0) list[atomicAdd(count, 1)] = int(i);
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
  CF_CUDA(cudaMemcpyAsync(&h, p, sizeof(i64), cudaMemcpyDeviceToHost, stream()));
  CF_CUDA(cudaStreamSynchronize(stream()));
  return h;
}
int read_int(const int* p) {
  int h = 0;
  CF_CUDA(cudaMemcpyAsync(&h, p, sizeof(int), cudaMemcpyDeviceToHost, stream()));
  CF_CUDA(cudaStreamSynchronize(stream()));
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

constexpr int SYM_BIG = 16384;

}  // namespace

std::unique_ptr<Csr> spgemm(const Csr& A, const Csr& B, const double* row_scale) {
  if (A.cols != B.rows) fail(CF_ERR_LOGIC, "spgemm: inner dimensions differ");
  auto C = std::make_unique<Csr>();
  C->rows = A.rows;
  C->cols = B.cols;
  C->ptr.alloc(A.rows + 1);
  C->ptr.zero();
  const i64 m = A.rows;
  if (m == 0) return C;
  i64* cnt = C->ptr.p;  // row counts in place, scanned into offsets afterwards
  // 1. symbolic count, binned by the product-count bound U_i (unique columns <= U_i)
  {
    DevBuf<i64> ub(m);
    k_row_bound<<<grid_for(m, 256), 256, 0, stream()>>>(m, A.ptr.p, A.col.p, B.ptr.p, ub.p);
    CF_LAUNCHED();
    RowBin small = make_bin(m, ub.p, 0, 256);
    RowBin large = make_bin(m, ub.p, 256, LLONG_MAX);
    if (small.n) {
      k_sym_warp<512, 8><<<grid_for(small.n, 8), 256, 0, stream()>>>(small.list.p, small.n, A.ptr.p, A.col.p,
                                                                      B.ptr.p, B.col.p, cnt, nullptr, nullptr, 0);
      CF_LAUNCHED();
    }
    if (large.n) {
      k_sym_warp<2048, 2><<<grid_for(large.n, 2), 64, 0, stream()>>>(large.list.p, large.n, A.ptr.p, A.col.p,
                                                                       B.ptr.p, B.col.p, cnt, nullptr, nullptr, 0);
      CF_LAUNCHED();
      RowBin ovf;
      ovf.list.alloc(large.n);
      DevBuf<int> c(1);
      c.zero();
      k_bin_overflow<<<grid_for(m, 256), 256, 0, stream()>>>(m, cnt, ovf.list.p, c.p);
      CF_LAUNCHED();
      ovf.n = read_int(c.p);
      if (ovf.n) {
        DevBuf<int> flag(1);
        flag.zero();
        const size_t sm = size_t(2) * SYM_BIG * sizeof(int);
        CF_CUDA(cudaFuncSetAttribute(k_sym_cta<SYM_BIG>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
        k_sym_cta<SYM_BIG><<<ovf.n, 256, sm, stream()>>>(ovf.list.p, ovf.n, A.ptr.p, A.col.p, B.ptr.p, B.col.p, cnt,
                                                         nullptr, nullptr, 0, flag.p);
        CF_LAUNCHED();
        if (read_int(flag.p)) fail(CF_ERR_UNSUPPORTED, "spgemm: an output row exceeds 12288 columns");
      }
    }
  }
  scan_excl(C->ptr.p, m + 1);
  C->nnz = read_i64(C->ptr.p + m);
  C->col.alloc(C->nnz);
  C->val.alloc(C->nnz);
  // 2. symbolic fill (sorted columns) and 3. numeric, binned by the exact row length
  DevBuf<i64> len(m);
  k_row_len<<<grid_for(m, 256), 256, 0, stream()>>>(m, C->ptr.p, len.p);
  CF_LAUNCHED();
  {
    RowBin f1 = make_bin(m, len.p, 0, 384);
    RowBin f2 = make_bin(m, len.p, 384, 1536);
    RowBin f3 = make_bin(m, len.p, 1536, LLONG_MAX);
    if (f1.n) {
      k_sym_warp<512, 8><<<grid_for(f1.n, 8), 256, 0, stream()>>>(f1.list.p, f1.n, A.ptr.p, A.col.p, B.ptr.p,
                                                                   B.col.p, nullptr, C->ptr.p, C->col.p, 1);
      CF_LAUNCHED();
    }
    if (f2.n) {
      k_sym_warp<2048, 2><<<grid_for(f2.n, 2), 64, 0, stream()>>>(f2.list.p, f2.n, A.ptr.p, A.col.p, B.ptr.p,
                                                                    B.col.p, nullptr, C->ptr.p, C->col.p, 1);
      CF_LAUNCHED();
    }
    if (f3.n) {
      DevBuf<int> flag(1);
      flag.zero();
      const size_t sm = size_t(2) * SYM_BIG * sizeof(int);
      CF_CUDA(cudaFuncSetAttribute(k_sym_cta<SYM_BIG>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
      k_sym_cta<SYM_BIG><<<f3.n, 256, sm, stream()>>>(f3.list.p, f3.n, A.ptr.p, A.col.p, B.ptr.p, B.col.p, nullptr,
                                                      C->ptr.p, C->col.p, 1, flag.p);
      CF_LAUNCHED();
    }
  }
  {
    RowBin n1 = make_bin(m, len.p, 0, 256);
    RowBin n2 = make_bin(m, len.p, 256, 1536);
    RowBin n3 = make_bin(m, len.p, 1536, LLONG_MAX);
    if (n1.n) {
      k_num_warp<256, 8><<<grid_for(n1.n, 8), 256, 0, stream()>>>(n1.list.p, n1.n, A.ptr.p, A.col.p, A.val.p,
                                                                   row_scale, B.ptr.p, B.col.p, B.val.p, C->ptr.p,
                                                                   C->col.p, C->val.p);
      CF_LAUNCHED();
    }
    if (n2.n) {
      k_num_warp<1536, 2><<<grid_for(n2.n, 2), 64, 0, stream()>>>(n2.list.p, n2.n, A.ptr.p, A.col.p, A.val.p,
                                                                    row_scale, B.ptr.p, B.col.p, B.val.p, C->ptr.p,
                                                                    C->col.p, C->val.p);
      CF_LAUNCHED();
    }
    if (n3.n) {
      const size_t sm = size_t(SYM_BIG) * (sizeof(double) + sizeof(int));
      CF_CUDA(cudaFuncSetAttribute(k_num_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
      k_num_cta<<<n3.n, 256, sm, stream()>>>(n3.list.p, n3.n, A.ptr.p, A.col.p, A.val.p, row_scale, B.ptr.p,
                                             B.col.p, B.val.p, C->ptr.p, C->col.p, C->val.p);
      CF_LAUNCHED();
    }
  }
  return C;
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
  k_axpy_merge<<<grid_for(T.rows, 256), 256, 0, stream()>>>(T.rows, T.ptr.p, T.col.p, T.val.p, w, DAT.ptr.p,
                                                            DAT.col.p, DAT.val.p, P->ptr.p, nullptr, nullptr, 0);
  CF_LAUNCHED();
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
  k_prune<<<grid_for(A.rows, 256), 256, 0, stream()>>>(A.rows, A.ptr.p, A.col.p, A.val.p, np.p, nullptr, nullptr, 0);
  CF_LAUNCHED();
  scan_excl(np.p, A.rows + 1);
  const i64 nnz = read_i64(np.p + A.rows);
  if (nnz == A.nnz) return;
  DevBuf<int> nc(nnz);
  DevBuf<double> nv(nnz);
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

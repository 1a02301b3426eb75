// K4: CSR SpMV and the 2x2 lower block-triangular apply (BlockSystem::apply,
// proj/src/linsolve.cpp:13-19).  HBM-bound: the matrix is streamed once with L1-bypassing
// non-coherent loads, x is read through the read-only cache, a group of TPR lanes owns one
// row (TPR picked from the mean row length) and reduces with warp shuffles.
#include "cf_types.hpp"

namespace cfb {

namespace {

__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ld_stream(const int* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

template <int TPR>
__device__ __forceinline__ double group_sum(double s) {
#pragma unroll
  for (int o = TPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, TPR);
  return s;
}

template <int TPR>
__device__ __forceinline__ double row_dot(const i64* __restrict__ ptr, const int* __restrict__ col,
                                          const double* __restrict__ val, const double* __restrict__ x, i64 row,
                                          int lane) {
  double s = 0.0;
  const i64 e = ptr[row + 1];
  for (i64 k = ptr[row] + lane; k < e; k += TPR) s += ld_stream(val + k) * __ldg(x + ld_stream(col + k));
  return s;
}

// y = A x (+ add)  (add may alias y)
template <int TPR>
__global__ void __launch_bounds__(256) k_spmv(i64 rows, const i64* __restrict__ ptr, const int* __restrict__ col,
                                              const double* __restrict__ val, const double* __restrict__ x,
                                              double* y, const double* add) {
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  const i64 row = t / TPR;
  const int lane = int(t % TPR);
  double s = 0.0;
  if (row < rows) s = row_dot<TPR>(ptr, col, val, x, row, lane);
  s = group_sum<TPR>(s);
  if (row < rows && lane == 0) y[row] = add ? add[row] + s : s;
}

// Batched variant: every lane issues U independent (value, column) loads and then U x
// gathers before accumulating, so a warp keeps U x more bytes in flight (the col -> x
// dependency otherwise serialises two HBM round trips per entry).
template <int TPR, int U>
__global__ void __launch_bounds__(256) k_spmv_b(i64 rows, const i64* __restrict__ ptr, const int* __restrict__ col,
                                                const double* __restrict__ val, const double* __restrict__ x,
                                                double* y, const double* add) {
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  const i64 row = t / TPR;
  const int lane = int(t % TPR);
  double s = 0.0;
  if (row < rows) {
    const i64 e = ptr[row + 1];
    for (i64 k0 = ptr[row] + lane; k0 < e; k0 += i64(TPR) * U) {
      double v[U], xv[U];
      int c[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const i64 k = k0 + i64(j) * TPR;
        const bool in = k < e;
        v[j] = in ? ld_stream(val + k) : 0.0;
        c[j] = in ? ld_stream(col + k) : -1;
      }
#pragma unroll
      for (int j = 0; j < U; ++j) xv[j] = c[j] >= 0 ? __ldg(x + c[j]) : 0.0;
#pragma unroll
      for (int j = 0; j < U; ++j) s += v[j] * xv[j];
    }
  }
  s = group_sum<TPR>(s);
  if (row < rows && lane == 0) y[row] = add ? add[row] + s : s;
}

template <int TPR, int U>
__device__ __forceinline__ double row_dot_b(const i64* __restrict__ ptr, const int* __restrict__ col,
                                            const double* __restrict__ val, const double* __restrict__ x, i64 row,
                                            int lane) {
  double s = 0.0;
  const i64 e = ptr[row + 1];
  for (i64 k0 = ptr[row] + lane; k0 < e; k0 += i64(TPR) * U) {
    double v[U], xv[U];
    int c[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const i64 k = k0 + i64(j) * TPR;
      const bool in = k < e;
      v[j] = in ? ld_stream(val + k) : 0.0;
      c[j] = in ? ld_stream(col + k) : -1;
    }
#pragma unroll
    for (int j = 0; j < U; ++j) xv[j] = c[j] >= 0 ? __ldg(x + c[j]) : 0.0;
#pragma unroll
    for (int j = 0; j < U; ++j) s += v[j] * xv[j];
  }
  return s;
}

// y_phi = M_phiu x_u + M_phiphi x_phi, one pass over both blocks per row
template <int TPR, int U>
__global__ void __launch_bounds__(256) k_spmv_phi(i64 rows, const i64* __restrict__ p1, const int* __restrict__ c1,
                                                  const double* __restrict__ v1, const double* __restrict__ x1,
                                                  const i64* __restrict__ p2, const int* __restrict__ c2,
                                                  const double* __restrict__ v2, const double* __restrict__ x2,
                                                  double* __restrict__ y) {
  const i64 t = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  const i64 row = t / TPR;
  const int lane = int(t % TPR);
  double s1 = 0.0, s2 = 0.0;
  if (row < rows) {
    s1 = row_dot_b<TPR, U>(p1, c1, v1, x1, row, lane);
    s2 = row_dot_b<TPR, U>(p2, c2, v2, x2, row, lane);
  }
  s1 = group_sum<TPR>(s1);
  s2 = group_sum<TPR>(s2);
  if (row < rows && lane == 0) y[row] = s1 + s2;
}

template <int TPR>
void launch_spmv(const Csr& A, const double* x, double* y, const double* add) {
  const int block = 256;
  const i64 threads = A.rows * TPR;
  k_spmv<TPR><<<grid_for(threads, block), block, 0, stream()>>>(A.rows, A.ptr.p, A.col.p, A.val.p, x, y, add);
  CF_LAUNCHED();
}

template <int TPR, int U>
void launch_phi(const BlockSystem& J, const double* x, double* y) {
  const int block = 256;
  const i64 threads = J.np * TPR;
  k_spmv_phi<TPR, U><<<grid_for(threads, block), block, 0, stream()>>>(J.np, J.pu->ptr.p, J.pu->col.p, J.pu->val.p, x,
                                                                    J.pp->ptr.p, J.pp->col.p, J.pp->val.p,
                                                                    x + J.in_u(), y + J.nu);
  CF_LAUNCHED();
}

template <int TPR, int U>
void launch_b(const Csr& A, const double* x, double* y, const double* add) {
  const int block = 256;
  const i64 threads = A.rows * TPR;
  k_spmv_b<TPR, U><<<grid_for(threads, block), block, 0, stream()>>>(A.rows, A.ptr.p, A.col.p, A.val.p, x, y, add);
  CF_LAUNCHED();
}

}  // namespace

// Tuning hook: explicit (threads-per-row, unroll) variant.  Returns false for an unknown pair.
bool csr_spmv_variant(const Csr& A, int tpr, int unroll, const double* x, double* y) {
#define CFB_V(T, U) if (tpr == T && unroll == U) { launch_b<T, U>(A, x, y, nullptr); return true; }
  CFB_V(32, 1) CFB_V(32, 2) CFB_V(32, 3) CFB_V(32, 4)
  CFB_V(16, 2) CFB_V(16, 4) CFB_V(16, 6)
  CFB_V(8, 4) CFB_V(8, 6) CFB_V(8, 11)
  CFB_V(4, 3) CFB_V(4, 4) CFB_V(4, 5)
#undef CFB_V
  if (unroll == 0) {
    switch (tpr) {
      case 32: launch_spmv<32>(A, x, y, nullptr); return true;
      case 16: launch_spmv<16>(A, x, y, nullptr); return true;
      case 8: launch_spmv<8>(A, x, y, nullptr); return true;
      case 4: launch_spmv<4>(A, x, y, nullptr); return true;
    }
  }
  return false;
}

// Variant table from the B200 sweep (scripts/spmv_sweep.py, profiles/r01_spmv_sweep.json):
// one batch of TPR*U slots should cover a typical row.
void csr_spmv_add(const Csr& A, const double* x, double* y, const double* add) {
  if (A.rows == 0) return;
  const double mean = A.mean_hint >= 0.0 ? A.mean_hint : double(A.nnz) / double(A.rows);
  if (mean > 64) launch_b<16, 4>(A, x, y, add);
  else if (mean > 24) launch_b<8, 4>(A, x, y, add);
  else if (mean > 12) launch_b<4, 5>(A, x, y, add);
  else launch_b<4, 3>(A, x, y, add);
}

void csr_spmv(const Csr& A, const double* x, double* y, double) { csr_spmv_add(A, x, y, nullptr); }

void block_apply(const BlockSystem& J, const double* x, double* y) {
  csr_spmv_add(*J.uu, x, y, nullptr);
  if (J.np == 0) return;
  const double mean = J.pu->mean_hint >= 0.0 ? J.pu->mean_hint : double(J.pu->nnz) / double(J.np);
  if (mean > 64) launch_phi<16, 4>(J, x, y);
  else if (mean > 24) launch_phi<8, 4>(J, x, y);
  else launch_phi<4, 5>(J, x, y);
}

}  // namespace cfb

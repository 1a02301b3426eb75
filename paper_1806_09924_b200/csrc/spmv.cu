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

// y_phi = M_phiu x_u + M_phiphi x_phi, one pass over both blocks per row
template <int TPR>
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
    s1 = row_dot<TPR>(p1, c1, v1, x1, row, lane);
    s2 = row_dot<TPR>(p2, c2, v2, x2, row, lane);
  }
  s1 = group_sum<TPR>(s1);
  s2 = group_sum<TPR>(s2);
  if (row < rows && lane == 0) y[row] = s1 + s2;
}

int pick_tpr(double mean_row) {
  if (mean_row >= 48) return 32;
  if (mean_row >= 20) return 16;
  if (mean_row >= 8) return 8;
  return 4;
}

template <int TPR>
void launch_spmv(const Csr& A, const double* x, double* y, const double* add) {
  const int block = 256;
  const i64 threads = A.rows * TPR;
  k_spmv<TPR><<<grid_for(threads, block), block, 0, stream()>>>(A.rows, A.ptr.p, A.col.p, A.val.p, x, y, add);
  CF_LAUNCHED();
}

template <int TPR>
void launch_phi(const BlockSystem& J, const double* x, double* y) {
  const int block = 256;
  const i64 threads = J.np * TPR;
  k_spmv_phi<TPR><<<grid_for(threads, block), block, 0, stream()>>>(J.np, J.pu.ptr.p, J.pu.col.p, J.pu.val.p, x,
                                                                    J.pp.ptr.p, J.pp.col.p, J.pp.val.p, x + J.nu,
                                                                    y + J.nu);
  CF_LAUNCHED();
}

}  // namespace

void csr_spmv_add(const Csr& A, const double* x, double* y, const double* add) {
  if (A.rows == 0) return;
  switch (pick_tpr(A.rows ? double(A.nnz) / double(A.rows) : 0.0)) {
    case 32: launch_spmv<32>(A, x, y, add); break;
    case 16: launch_spmv<16>(A, x, y, add); break;
    case 8: launch_spmv<8>(A, x, y, add); break;
    default: launch_spmv<4>(A, x, y, add); break;
  }
}

void csr_spmv(const Csr& A, const double* x, double* y, double) { csr_spmv_add(A, x, y, nullptr); }

void block_apply(const BlockSystem& J, const double* x, double* y) {
  csr_spmv_add(J.uu, x, y, nullptr);
  if (J.np == 0) return;
  const double mean = double(J.pu.nnz + J.pp.nnz) / double(J.np) / 2.0;
  switch (pick_tpr(mean)) {
    case 32: launch_phi<32>(J, x, y); break;
    case 16: launch_phi<16>(J, x, y); break;
    case 8: launch_phi<8>(J, x, y); break;
    default: launch_phi<4>(J, x, y); break;
  }
}

}  // namespace cfb

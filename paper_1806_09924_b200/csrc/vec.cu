// K6: Krylov vector kernels with deterministic (fixed-order, atomic-free) reductions.
// dot/norm: a fixed grid of block partials + one ordered final block; multidot: several basis
// vectors per pass over w (CGS2 orthogonalisation); multi_axpy: w += alpha * V coef.
#include "cf_comm.hpp"
#include "cf_types.hpp"
#include "cf_vec.hpp"

namespace cfb {

namespace {

constexpr int RB = 256;  // reduction block size

__device__ __forceinline__ double block_sum(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(RB) k_dot_partial(const double* __restrict__ x, const double* __restrict__ y, i64 n,
                                                    double* __restrict__ part) {
  __shared__ double sh[RB];
  double s = 0.0;
  for (i64 i = i64(blockIdx.x) * RB + threadIdx.x; i < n; i += i64(gridDim.x) * RB) s += x[i] * y[i];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// MGS step fused with the next dot: w -= (*h) v, then the partials of w . y (y = nullptr: w . w) in
// exactly k_dot_partial's order (same grid, same grid-stride, same block tree)
__global__ void __launch_bounds__(RB) k_axpy_dot_partial(const double* __restrict__ h, const double* __restrict__ v,
                                                         double* __restrict__ w, const double* __restrict__ y, i64 n,
                                                         double* __restrict__ part) {
  __shared__ double sh[RB];
  const double hv = *h;
  double s = 0.0;
  for (i64 i = i64(blockIdx.x) * RB + threadIdx.x; i < n; i += i64(gridDim.x) * RB) {
    double wi = w[i];
    wi -= hv * v[i];
    w[i] = wi;
    s += wi * (y ? y[i] : wi);
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// out[r] = sum_b part[r*nb + b] (fixed tree), optional sqrt
__global__ void __launch_bounds__(RB) k_final(const double* __restrict__ part, int nb, double* out, int do_sqrt) {
  __shared__ double sh[RB];
  const double* p = part + i64(blockIdx.x) * nb;
  double s = 0.0;
  for (int b = threadIdx.x; b < nb; b += RB) s += p[b];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) out[blockIdx.x] = do_sqrt ? sqrt(s) : s;
}

template <int KC>
__global__ void __launch_bounds__(RB) k_multidot_partial(const double* __restrict__ V, i64 ld, int k,
                                                         const double* __restrict__ w, i64 n, double* __restrict__ part,
                                                         int nb) {
  __shared__ double sh[RB];
  const int c0 = blockIdx.y * KC;
  const int kc = min(KC, k - c0);
  double s[KC];
#pragma unroll
  for (int c = 0; c < KC; ++c) s[c] = 0.0;
  for (i64 i = i64(blockIdx.x) * RB + threadIdx.x; i < n; i += i64(gridDim.x) * RB) {
    const double wi = w[i];
#pragma unroll
    for (int c = 0; c < KC; ++c)
      if (c < kc) s[c] += V[(c0 + c) * ld + i] * wi;
  }
  for (int c = 0; c < kc; ++c) {
    const double r = block_sum(s[c], sh);
    if (threadIdx.x == 0) part[i64(c0 + c) * nb + blockIdx.x] = r;
  }
}

// w += alpha * sum_c coef_c V_c: one sequential sum per entry over c ascending; the coefficients
// are staged in shared memory 256 at a time (any number of basis vectors)
__global__ void k_multi_axpy(double* __restrict__ w, const double* __restrict__ V, i64 ld, int k,
                             const double* __restrict__ coef, i64 n, double alpha) {
  __shared__ double cs[256];
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  double s = 0.0;
  for (int c0 = 0; c0 < k; c0 += 256) {
    const int kc = min(256, k - c0);
    __syncthreads();
    for (int c = threadIdx.x; c < kc; c += blockDim.x) cs[c] = coef[c0 + c];
    __syncthreads();
    if (i < n)
      for (int c = 0; c < kc; ++c) s += cs[c] * V[i64(c0 + c) * ld + i];
  }
  if (i < n) w[i] += alpha * s;
}

__global__ void k_fill(double* x, double a, i64 n) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) x[i] = a;
}
__global__ void k_axpby(double a, const double* __restrict__ x, double b, double* __restrict__ y, i64 n) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] = a * x[i] + b * y[i];
}
__global__ void k_axpy(double a, const double* __restrict__ x, double* __restrict__ y, i64 n) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] += a * x[i];
}
__global__ void k_sub(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ o, i64 n) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) o[i] = a[i] - b[i];
}
__global__ void k_div_scalar(const double* __restrict__ x, const double* __restrict__ s, double* __restrict__ y, i64 n) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] = x[i] / *s;
}
__global__ void k_scale(double* x, double a, i64 n) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) x[i] *= a;
}
__global__ void k_diag_mul(const double* __restrict__ d, const double* __restrict__ x, double* __restrict__ y,
                           double a, i64 n) {
  const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] = a * (d[i] * x[i]);
}

// one block per chunk of a plane part (SegLayout); G: the global partial array
template <bool AXPY>
__global__ void __launch_bounds__(RB) k_seg_partial(const double* __restrict__ h, const double* __restrict__ v,
                                                    double* __restrict__ w, const double* __restrict__ y, SegLayout L,
                                                    double* __restrict__ G) {
  __shared__ double sh[RB];
  const int cu = L.cu(), cp = L.cp(), npl = L.p_hi - L.p_lo;
  const int b = blockIdx.x;
  i64 start, len;
  int gi;
  if (b < npl * cu) {
    const int lp = b / cu, c = b % cu;
    start = i64(lp) * L.plane_u + i64(c) * L.chunk;
    len = min(L.chunk, L.plane_u - i64(c) * L.chunk);
    gi = (L.p_lo + lp) * cu + c;
  } else {
    const int bb = b - npl * cu, lp = bb / cp, c = bb % cp;
    start = L.nu_local() + i64(lp) * L.plane_p + i64(c) * L.chunk;
    len = min(L.chunk, L.plane_p - i64(c) * L.chunk);
    gi = L.nplanes * cu + (L.p_lo + lp) * cp + c;
  }
  const double hv = AXPY ? *h : 0.0;
  double s = 0.0;
  for (i64 i = threadIdx.x; i < len; i += RB) {
    double wi = w[start + i];
    if (AXPY) {
      wi -= hv * v[start + i];
      w[start + i] = wi;
    }
    s += wi * (y ? y[start + i] : wi);
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) G[gi] = s;
}

// G := the owning rank's partial of every slot (gathered: size x nparts); owner of plane p is the
// rank r with floor(nplanes r / size) <= p < floor(nplanes (r+1) / size) (rank_slab)
__global__ void k_seg_pick(const double* __restrict__ gathered, int size, SegLayout L, double* __restrict__ G) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = L.nparts(), cu = L.cu(), cp = L.cp();
  if (s >= n) return;
  const int p = s < L.nplanes * cu ? s / cu : (s - L.nplanes * cu) / cp;
  int r = 0;
  while (r + 1 < size && i64(L.nplanes) * (r + 1) / size <= p) ++r;
  G[s] = gathered[i64(r) * n + s];
}

int nblocks_for(i64 n) { return int(std::min<i64>(1024, std::max<i64>(1, (n + 4 * RB - 1) / (4 * RB)))); }

Scratch& scr() {
  static Scratch s;
  return s;
}

double* partial_buf(i64 count) {
  Scratch& s = scr();
  if (s.part.n < count) s.part.alloc(std::max<i64>(count, 1 << 17));
  return s.part.p;
}

}  // namespace

double* scalar_buf(int count) {
  Scratch& s = scr();
  if (s.scal.n < count) s.scal.alloc(std::max(count, 1024));
  return s.scal.p;
}

void vfill(double* x, double a, i64 n) {
  if (n <= 0) return;
  k_fill<<<grid_for(n, 256), 256, 0, stream()>>>(x, a, n);
  CF_LAUNCHED();
}
void vcopy(double* dst, const double* src, i64 n) {
  if (n > 0) CF_CUDA(cudaMemcpyAsync(dst, src, size_t(n) * sizeof(double), cudaMemcpyDeviceToDevice, stream()));
}
void vaxpy(double a, const double* x, double* y, i64 n) {
  if (n <= 0) return;
  k_axpy<<<grid_for(n, 256), 256, 0, stream()>>>(a, x, y, n);
  CF_LAUNCHED();
}
void vaxpby(double a, const double* x, double b, double* y, i64 n) {
  if (n <= 0) return;
  k_axpby<<<grid_for(n, 256), 256, 0, stream()>>>(a, x, b, y, n);
  CF_LAUNCHED();
}
void vsub(const double* a, const double* b, double* out, i64 n) {
  if (n <= 0) return;
  k_sub<<<grid_for(n, 256), 256, 0, stream()>>>(a, b, out, n);
  CF_LAUNCHED();
}
void vscale(double* x, double a, i64 n) {
  if (n <= 0) return;
  k_scale<<<grid_for(n, 256), 256, 0, stream()>>>(x, a, n);
  CF_LAUNCHED();
}
void vdiv_dev(const double* x, const double* s_dev, double* y, i64 n) {
  if (n <= 0) return;
  k_div_scalar<<<grid_for(n, 256), 256, 0, stream()>>>(x, s_dev, y, n);
  CF_LAUNCHED();
}
void vdiag_mul(const double* d, const double* x, double* y, double a, i64 n) {
  if (n <= 0) return;
  k_diag_mul<<<grid_for(n, 256), 256, 0, stream()>>>(d, x, y, a, n);
  CF_LAUNCHED();
}

void vdot_dev(const double* x, const double* y, i64 n, double* out, bool do_sqrt) {
  const int nb = nblocks_for(n);
  double* part = partial_buf(nb);
  k_dot_partial<<<nb, RB, 0, stream()>>>(x, y, n, part);
  CF_LAUNCHED();
  k_final<<<1, RB, 0, stream()>>>(part, nb, out, do_sqrt ? 1 : 0);
  CF_LAUNCHED();
}

void vaxpy_dot_dev(const double* h_dev, const double* v, double* w, const double* y, i64 n, double* out,
                   bool do_sqrt) {
  const int nb = nblocks_for(n);
  double* part = partial_buf(nb);
  k_axpy_dot_partial<<<nb, RB, 0, stream()>>>(h_dev, v, w, y, n, part);
  CF_LAUNCHED();
  k_final<<<1, RB, 0, stream()>>>(part, nb, out, do_sqrt ? 1 : 0);
  CF_LAUNCHED();
}

namespace {
void seg_reduce(const double* h, const double* v, double* w, const double* y, const SegLayout& L, double* out,
                bool do_sqrt, const Comm* comm) {
  const int np = L.nparts();
  const bool dist = comm && comm->distributed();
  double* G = partial_buf(i64(np) * (dist ? comm->size + 1 : 1));
  if (L.nblocks_local() > 0) {
    if (h)
      k_seg_partial<true><<<L.nblocks_local(), RB, 0, stream()>>>(h, v, w, y, L, G);
    else
      k_seg_partial<false><<<L.nblocks_local(), RB, 0, stream()>>>(nullptr, nullptr, w, y, L, G);
    CF_LAUNCHED();
  }
  if (dist) {
    double* gathered = G + np;
    comm->allgather(G, np, gathered);
    k_seg_pick<<<(np + 255) / 256, 256, 0, stream()>>>(gathered, comm->size, L, G);
    CF_LAUNCHED();
  }
  k_final<<<1, RB, 0, stream()>>>(G, np, out, do_sqrt ? 1 : 0);
  CF_LAUNCHED();
}
}  // namespace

void seg_dot_dev(const double* x, const double* y, const SegLayout& L, double* out, bool do_sqrt, const Comm* comm) {
  seg_reduce(nullptr, nullptr, const_cast<double*>(x), y, L, out, do_sqrt, comm);
}

void seg_axpy_dot_dev(const double* h, const double* v, double* w, const double* y, const SegLayout& L, double* out,
                      bool do_sqrt, const Comm* comm) {
  seg_reduce(h, v, w, y, L, out, do_sqrt, comm);
}

double vdot(const double* x, const double* y, i64 n) {
  double* s = scalar_buf(1);
  vdot_dev(x, y, n, s, false);
  double h = 0.0;
  read_small(&h, s, sizeof(double));
  return h;
}

double vnorm(const double* x, i64 n) {
  double* s = scalar_buf(1);
  vdot_dev(x, x, n, s, true);
  double h = 0.0;
  read_small(&h, s, sizeof(double));
  return h;
}

void multidot(const double* V, i64 ld, int k, const double* w, i64 n, double* out_dev) {
  if (k <= 0) return;
  constexpr int KC = 16;
  const int nb = nblocks_for(n);
  double* part = partial_buf(i64(nb) * k);
  dim3 grid(nb, (k + KC - 1) / KC);
  k_multidot_partial<KC><<<grid, RB, 0, stream()>>>(V, ld, k, w, n, part, nb);
  CF_LAUNCHED();
  k_final<<<k, RB, 0, stream()>>>(part, nb, out_dev, 0);
  CF_LAUNCHED();
}

void multi_axpy(double* w, const double* V, i64 ld, int k, const double* coef_dev, i64 n, double alpha) {
  if (k <= 0 || n <= 0) return;
  k_multi_axpy<<<grid_for(n, 256), 256, 0, stream()>>>(w, V, ld, k, coef_dev, n, alpha);
  CF_LAUNCHED();
}

}  // namespace cfb

// K11: total crack volume and crack-opening profile on the device (postproc.cpp:12-99).
//
// TCV = sum_cells sum_qp W u . grad(phi) (2-point Gauss, evaluate_on_cell semantics: the
// reference point is recomputed as clamp((x - lo)/h, 0, 1) from the physical point), reduced with
// a fixed block tree.  COD(x_s) = 0.5 |sum over the cell column owning x_s of the 4-point Gauss
// line integral of u . grad(phi)| along y (2d) / z through (x_s, 0) (3d), one CTA per station.
#include <cmath>

#include "cf_vec.hpp"

namespace cfb {

namespace {

__device__ __forceinline__ double coord(const GridDesc& g, i64 i) {
  return -g.K + double(i * (i64(1) << (16 - g.r))) * g.unit;
}

// u . grad(phi) at physical point x in cell (cx, cy, cz) (fem.cpp:281-309)
template <int D>
__device__ double u_dot_gradphi(const GridDesc& g, const double* __restrict__ sol, i64 cx, i64 cy, i64 cz,
                                const double x[3]) {
  const i64 c[3] = {cx, cy, cz};
  double xi[3] = {0, 0, 0};
  for (int a = 0; a < D; ++a) xi[a] = fmin(fmax((x[a] - coord(g, c[a])) / g.h, 0.0), 1.0);
  double u[3] = {0, 0, 0}, gp[3] = {0, 0, 0};
  const i64 nu = g.n_u();
  for (int k = 0; k < (1 << D); ++k) {
    double s = 1.0;
    for (int a = 0; a < D; ++a) s *= (k & (1 << a)) ? xi[a] : 1.0 - xi[a];
    const i64 v = (cx + (k & 1)) + g.nn * ((cy + ((k >> 1) & 1)) + g.nn * (cz + ((k >> 2) & 1)));
    const double phi = sol[nu + v];
    for (int a = 0; a < D; ++a) {
      double gr = (k & (1 << a)) ? 1.0 : -1.0;
      for (int b = 0; b < D; ++b) {
        if (b == a) continue;
        gr *= (k & (1 << b)) ? xi[b] : 1.0 - xi[b];
      }
      gp[a] += gr / g.h * phi;
      u[a] += s * sol[v * D + a];
    }
  }
  double dot = 0.0;
  for (int a = 0; a < 3; ++a) dot += u[a] * gp[a];
  return dot;
}

template <int D>
__global__ void __launch_bounds__(256) k_tcv(GridDesc g, const double* __restrict__ sol, const double* __restrict__ qp,
                                             const double* __restrict__ qw, double* __restrict__ part) {
  __shared__ double sh[256];
  double s = 0.0;
  for (i64 c = i64(blockIdx.x) * 256 + threadIdx.x; c < g.ncells; c += i64(gridDim.x) * 256) {
    const i64 cx = c % g.nc, cy = (c / g.nc) % g.nc, cz = (D == 3) ? c / (g.nc * g.nc) : 0;
    const double lo[3] = {coord(g, cx), coord(g, cy), D == 3 ? coord(g, cz) : 0.0};
    double cs = 0.0;
    for (int q = 0; q < (1 << D); ++q) {
      double x[3] = {lo[0], lo[1], lo[2]};
      for (int a = 0; a < D; ++a) x[a] += qp[q * 3 + a] * g.h;
      cs += qw[q] * g.detJ * u_dot_gradphi<D>(g, sol, cx, cy, cz, x);
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

// one CTA per station: the owning cell column (postproc.cpp:45-66)
template <int D>
__global__ void __launch_bounds__(256) k_cod(GridDesc g, const double* __restrict__ sol, const double* __restrict__ st,
                                             const double* __restrict__ lp, const double* __restrict__ lw,
                                             double* __restrict__ out) {
  __shared__ double sh[256];
  const double s = st[blockIdx.x];
  const double K = g.K;
  auto owns = [K](double lo, double hi, double x) { return (x < K) ? (lo <= x && x < hi) : (lo < x && x <= hi); };
  i64 cx = -1, cy = -1;
  for (i64 i = 0; i < g.nc; ++i)
    if (owns(coord(g, i), coord(g, i + 1), s)) {
      cx = i;
      break;
    }
  if (D == 3)
    for (i64 i = 0; i < g.nc; ++i)
      if (owns(coord(g, i), coord(g, i + 1), 0.0)) {
        cy = i;
        break;
      }
  double acc = 0.0;
  if (cx >= 0 && (D == 2 || cy >= 0)) {
    const int axis = D - 1;
    for (i64 t = threadIdx.x; t < g.nc; t += blockDim.x) {  // cells along the integration axis
      const i64 ccx = cx, ccy = (D == 2) ? t : cy, ccz = (D == 3) ? t : 0;
      const double lo_ax = coord(g, t);
      double cs = 0.0;
      for (int q = 0; q < 4; ++q) {
        double x[3] = {s, 0.0, 0.0};
        x[axis] = lo_ax + lp[q] * g.h;
        cs += lw[q] * g.h * u_dot_gradphi<D>(g, sol, ccx, ccy, ccz, x);
      }
      acc += cs;
    }
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = 0.5 * fabs(sh[0]);
}

__global__ void k_sum_partials(int nb, const double* __restrict__ part, double* out) {
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

}  // namespace

double compute_tcv(const Problem& P, const double* sol) {
  const GridDesc& g = P.g;
  // cell_rule(d, 2) points/weights (fem.cpp:53-74)
  double pts[8 * 3] = {0}, wts[8];
  const double a1 = 1.0 / std::sqrt(3.0), x1[2] = {-a1, a1};
  for (int q = 0; q < (1 << g.d); ++q) {
    int rem = q;
    double wt = 1.0;
    for (int a = 0; a < g.d; ++a) {
      const int i = rem % 2;
      rem /= 2;
      pts[q * 3 + a] = 0.5 * (x1[i] + 1.0);
      wt *= 0.5 * 1.0;
    }
    wts[q] = wt;
  }
  DevBuf<double> dq(24), dw(8), part(1024), out(1);
  CF_CUDA(cudaMemcpyAsync(dq.p, pts, sizeof(pts), cudaMemcpyHostToDevice, stream()));
  CF_CUDA(cudaMemcpyAsync(dw.p, wts, sizeof(wts), cudaMemcpyHostToDevice, stream()));
  const int nb = int(std::min<i64>(1024, std::max<i64>(1, (g.ncells + 255) / 256)));
  if (g.d == 2)
    k_tcv<2><<<nb, 256, 0, stream()>>>(g, sol, dq.p, dw.p, part.p);
  else
    k_tcv<3><<<nb, 256, 0, stream()>>>(g, sol, dq.p, dw.p, part.p);
  CF_LAUNCHED();
  k_sum_partials<<<1, 256, 0, stream()>>>(nb, part.p, out.p);
  CF_LAUNCHED();
  double h = 0.0;
  CF_CUDA(cudaMemcpyAsync(&h, out.p, sizeof(double), cudaMemcpyDeviceToHost, stream()));
  CF_CUDA(cudaStreamSynchronize(stream()));
  return h;
}

void compute_cod(const Problem& P, const double* sol, const double* stations_host, int ns, double* out_host) {
  const GridDesc& g = P.g;
  for (int i = 1; i < ns; ++i)
    if (!(stations_host[i] > stations_host[i - 1]))
      fail(CF_ERR_INVALID_ARGUMENT, "compute_cod: stations must be strictly increasing");
  for (int i = 0; i < ns; ++i)
    if (std::abs(stations_host[i]) > g.K) fail(CF_ERR_INVALID_ARGUMENT, "compute_cod: station outside domain");
  if (ns == 0) return;
  // line_rule(4) (fem.cpp:76, 30-36): points 0.5(x+1), weights 0.5 w
  const double a = std::sqrt(3.0 / 7.0 - 2.0 / 7.0 * std::sqrt(6.0 / 5.0));
  const double b = std::sqrt(3.0 / 7.0 + 2.0 / 7.0 * std::sqrt(6.0 / 5.0));
  const double wa = (18.0 + std::sqrt(30.0)) / 36.0, wb = (18.0 - std::sqrt(30.0)) / 36.0;
  const double xs[4] = {-b, -a, a, b}, ws[4] = {wb, wa, wa, wb};
  double lp[4], lw[4];
  for (int q = 0; q < 4; ++q) {
    lp[q] = 0.5 * (xs[q] + 1.0);
    lw[q] = 1.0 * (0.5 * ws[q]);
  }
  DevBuf<double> dst(ns), dlp(4), dlw(4), dout(ns);
  CF_CUDA(cudaMemcpyAsync(dst.p, stations_host, size_t(ns) * sizeof(double), cudaMemcpyHostToDevice, stream()));
  CF_CUDA(cudaMemcpyAsync(dlp.p, lp, sizeof(lp), cudaMemcpyHostToDevice, stream()));
  CF_CUDA(cudaMemcpyAsync(dlw.p, lw, sizeof(lw), cudaMemcpyHostToDevice, stream()));
  if (g.d == 2)
    k_cod<2><<<ns, 256, 0, stream()>>>(g, sol, dst.p, dlp.p, dlw.p, dout.p);
  else
    k_cod<3><<<ns, 256, 0, stream()>>>(g, sol, dst.p, dlp.p, dlw.p, dout.p);
  CF_LAUNCHED();
  CF_CUDA(cudaMemcpyAsync(out_host, dout.p, size_t(ns) * sizeof(double), cudaMemcpyDeviceToHost, stream()));
  CF_CUDA(cudaStreamSynchronize(stream()));
}

}  // namespace cfb

// K6: restarted right-preconditioned GMRES (linsolve.cpp:21-115) with a device-resident Krylov
// basis.  The orthogonalisation is the reference's modified Gram-Schmidt: for each basis
// vector a deterministic device dot (fixed-order block tree) and an axpy whose coefficient stays
// in device memory, so the only host round trip per iteration is the (j+2)-entry Hessenberg
// column needed by the Givens logic, which runs on the host exactly as in the reference.
#include <cmath>

#include "cf_comm.hpp"
#include "cf_vec.hpp"

namespace cfb {

namespace {

__global__ void k_sqrt1(double* s) { s[0] = sqrt(s[0]); }

// dot over all ranks' rows: the segmented NP-invariant order when a layout is given, else the
// local fixed-order dot followed by the rank-ordered sum
void gdot(const double* x, const double* y, i64 n, double* out, bool do_sqrt, const Comm* comm,
          const SegLayout* seg) {
  if (seg) {
    seg_dot_dev(x, y, *seg, out, do_sqrt, comm);
    return;
  }
  if (!comm || !comm->distributed()) {
    vdot_dev(x, y, n, out, do_sqrt);
    return;
  }
  vdot_dev(x, y, n, out, false);
  comm->sum_ordered(out, 1);
  if (do_sqrt) {
    k_sqrt1<<<1, 1, 0, stream()>>>(out);
    CF_LAUNCHED();
  }
}

}  // namespace

GmresResult gmres(const DevOp& op, const DevOp* prec, const double* rhs, i64 n, const cf_gmres_options& o,
                  double* x, const Comm* comm, const SegLayout* seg) {
  if (!(o.rtol > 0.0 && o.rtol < 1.0)) fail(CF_ERR_INVALID_ARGUMENT, "gmres: rtol must be in (0,1)");
  if (o.restart < 1) fail(CF_ERR_INVALID_ARGUMENT, "gmres: restart must be >= 1");
  GmresResult res;
  vfill(x, 0.0, n);
  DevBuf<double> sc(2);
  gdot(rhs, rhs, n, sc.p, true, comm, seg);
  double bnorm = 0.0;
  read_small(&bnorm, sc.p, sizeof(double));
  if (bnorm == 0.0) {
    res.converged = true;
    return res;
  }
  const int mmax = std::max(1, std::min(o.restart, o.max_iter));
  // persistent workspace: the basis is GBs at the large configs, and re-allocating it every Newton
  // iteration from a pool fragmented by the AMG setup costs far more than the solve itself
  static struct Work {
    i64 n = -1;
    int m = -1;
    DevBuf<double> r, z, z2, V, hd, yd;
  } ws;
  if (ws.n != n || ws.m < mmax) {
    ws.V.release();
    ws.r.alloc(n);
    ws.z.alloc(n);
    ws.z2.alloc(n);
    ws.V.alloc(n * (mmax + 1));
    ws.hd.alloc(mmax + 2);
    ws.yd.alloc(mmax + 1);
    ws.n = n;
    ws.m = mmax;
  }
  DevBuf<double>&r = ws.r, &z = ws.z, &z2 = ws.z2, &V = ws.V, &hd = ws.hd, &yd = ws.yd;
  vcopy(r.p, rhs, n);
  std::vector<double> H, cs, sn, g, hcol(mmax + 2), y;
  auto apply_op = [&](const double* in, double* out) {
    if (prec) {
      (*prec)(in, z2.p);
      op(z2.p, out);
    } else {
      op(in, out);
    }
  };
  while (res.iterations < o.max_iter) {
    gdot(r.p, r.p, n, sc.p, true, comm, seg);
    double beta = 0.0;
    read_small(&beta, sc.p, sizeof(double));
    if (beta <= o.rtol * bnorm) {
      res.converged = true;
      res.residual = beta / bnorm;
      return res;
    }
    const int m = std::min(o.restart, o.max_iter - res.iterations);
    H.assign(size_t(m + 1) * m, 0.0);
    auto Hij = [&](int i, int j) -> double& { return H[size_t(i) * m + j]; };
    cs.assign(m, 0.0);
    sn.assign(m, 0.0);
    g.assign(m + 1, 0.0);
    g[0] = beta;
    vdiv_dev(r.p, sc.p, V.p, n);  // V(:,0) = r / beta
    int j = 0;
    bool inner_done = false;
    for (; j < m && !inner_done; ++j) {
      double* w = V.p + i64(j + 1) * n;
      apply_op(V.p + i64(j) * n, w);
      // modified Gram-Schmidt: h_i = w . v_i, w -= h_i v_i (i = 0..j), then |w|; each axpy is fused
      // with the following dot (same operations, same reduction order)
      gdot(w, V.p, n, hd.p, false, comm, seg);
      for (int i = 0; i <= j; ++i) {
        const double* next = i < j ? V.p + i64(i + 1) * n : nullptr;
        const bool last = i == j;
        if (seg) {
          seg_axpy_dot_dev(hd.p + i, V.p + i64(i) * n, w, next, *seg, hd.p + i + 1, last, comm);
        } else if (!comm || !comm->distributed()) {
          vaxpy_dot_dev(hd.p + i, V.p + i64(i) * n, w, next, n, hd.p + i + 1, last);
        } else {
          vaxpy_dot_dev(hd.p + i, V.p + i64(i) * n, w, next, n, hd.p + i + 1, false);
          comm->sum_ordered(hd.p + i + 1, 1);
          if (last) {
            k_sqrt1<<<1, 1, 0, stream()>>>(hd.p + i + 1);
            CF_LAUNCHED();
          }
        }
      }
      read_small(hcol.data(), hd.p, size_t(j + 2) * sizeof(double));
      for (int i = 0; i <= j + 1; ++i) Hij(i, j) = hcol[i];
      const bool happy = Hij(j + 1, j) <= 1e-14 * bnorm;
      if (!happy) vdiv_dev(w, hd.p + j + 1, w, n);
      for (int i = 0; i < j; ++i) {  // previous Givens rotations
        const double t = cs[i] * Hij(i, j) + sn[i] * Hij(i + 1, j);
        Hij(i + 1, j) = -sn[i] * Hij(i, j) + cs[i] * Hij(i + 1, j);
        Hij(i, j) = t;
      }
      const double denom = std::hypot(Hij(j, j), Hij(j + 1, j));
      if (denom == 0.0) {
        res.breakdown = true;
        inner_done = true;
        --j;
        break;
      }
      cs[j] = Hij(j, j) / denom;
      sn[j] = Hij(j + 1, j) / denom;
      Hij(j, j) = denom;
      Hij(j + 1, j) = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      ++res.iterations;
      const double rel = std::abs(g[j + 1]) / bnorm;
      res.history.push_back(rel);
      if (rel <= o.rtol || happy || res.iterations >= o.max_iter) inner_done = true;
    }
    const int k = j;
    if (k > 0) {
      y.assign(k, 0.0);
      for (int i = k - 1; i >= 0; --i) {
        double s = g[i];
        for (int l = i + 1; l < k; ++l) s -= Hij(i, l) * y[l];
        if (Hij(i, i) == 0.0) {
          res.breakdown = true;
          y[i] = 0.0;
        } else {
          y[i] = s / Hij(i, i);
        }
      }
      CF_CUDA(cudaMemcpyAsync(yd.p, y.data(), size_t(k) * sizeof(double), cudaMemcpyHostToDevice, stream()));
      vfill(z.p, 0.0, n);
      multi_axpy(z.p, V.p, n, k, yd.p, n, 1.0);  // z = V(:, :k) y
      if (prec) {
        (*prec)(z.p, z2.p);
        vaxpy(1.0, z2.p, x, n);
      } else {
        vaxpy(1.0, z.p, x, n);
      }
    }
    op(x, z.p);
    vsub(rhs, z.p, r.p, n);  // r = b - op(x)
    gdot(r.p, r.p, n, sc.p, true, comm, seg);
    double rn = 0.0;
    read_small(&rn, sc.p, sizeof(double));
    res.residual = rn / bnorm;
    if (res.residual <= o.rtol) {
      res.converged = true;
      return res;
    }
    if (res.breakdown) return res;
  }
  return res;
}

}  // namespace cfb

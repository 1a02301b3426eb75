// C ABI (include/crackfield_b200.h): status codes, last-error text, handle ownership and
// host/device argument staging around the cfb:: implementation.
#include <cstring>
#include <string>

#include "cf_types.hpp"

struct cf_problem_s {
  cfb::Problem* p;
};
struct cf_constraints_s {
  std::unique_ptr<cfb::Constraints> c;
  cf_problem owner;
};
struct cf_block_s {
  std::unique_ptr<cfb::BlockSystem> J;
};

namespace cfb {

Runtime& rt() {
  static Runtime r;
  return r;
}

void ensure_device() {
  Runtime& r = rt();
  if (r.ready) return;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    fail(CF_ERR_CUDA, std::string("crackfield_b200: no CUDA device available (") + cudaGetErrorString(e) +
                          "); there is no CPU fallback");
  CF_CUDA(cudaGetDevice(&r.device));
  CF_CUDA(cudaDeviceGetAttribute(&r.sm_count, cudaDevAttrMultiProcessorCount, r.device));
  // keep freed stream-ordered allocations cached in the pool (per-Newton-iteration reallocation)
  cudaMemPool_t pool;
  CF_CUDA(cudaDeviceGetDefaultMemPool(&pool, r.device));
  uint64_t thr = UINT64_MAX;
  CF_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  r.ready = true;
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace cfb

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return CF_OK;
  } catch (const cfb::Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_err = "out of host memory";
    return CF_ERR_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    g_err = e.what();
    return CF_ERR_LOGIC;
  }
}

#define CHECK_ARG(cond, msg) \
  if (!(cond)) ::cfb::fail(CF_ERR_INVALID_ARGUMENT, msg)

}  // namespace

using namespace cfb;

extern "C" {

const char* cf_last_error(void) { return g_err.c_str(); }
int cf_version(void) { return 1; }

int cf_device_info(int* device, int* sm_count, int64_t* total_mem) {
  return guard([&] {
    ensure_device();
    size_t fr = 0, tot = 0;
    CF_CUDA(cudaMemGetInfo(&fr, &tot));
    if (device) *device = rt().device;
    if (sm_count) *sm_count = rt().sm_count;
    if (total_mem) *total_mem = int64_t(tot);
  });
}

int cf_set_stream(void* s) {
  return guard([&] { rt().stream = static_cast<cudaStream_t>(s); });
}

int cf_synchronize(void) {
  return guard([&] { CF_CUDA(cudaStreamSynchronize(stream())); });
}

int64_t cf_kernel_launches(void) { return rt().launches; }

int cf_problem_create_uniform(int dim, double half_width, int n0, int refinements, cf_problem* out) {
  return guard([&] {
    CHECK_ARG(out, "cf_problem_create_uniform: out is null");
    *out = new cf_problem_s{make_problem(dim, half_width, n0, refinements)};
  });
}

int cf_problem_destroy(cf_problem p) {
  return guard([&] {
    if (p) {
      delete p->p;
      delete p;
    }
  });
}

int cf_problem_info(cf_problem p, int64_t* n_vertices, int64_t* n_cells, double* h) {
  return guard([&] {
    CHECK_ARG(p, "cf_problem_info: null problem");
    if (n_vertices) *n_vertices = p->p->g.V;
    if (n_cells) *n_cells = p->p->g.ncells;
    if (h) *h = p->p->g.h;
  });
}

int cf_constraints_build(cf_problem p, int clamp_boundary, int64_t n_active, const int64_t* active_dofs,
                         const double* active_values, cf_constraints* out) {
  return guard([&] {
    CHECK_ARG(p && out, "cf_constraints_build: null argument");
    CHECK_ARG(n_active >= 0, "cf_constraints_build: negative active count");
    CHECK_ARG(n_active == 0 || (active_dofs && active_values), "cf_constraints_build: null active arrays");
    InArg<i64> dofs(reinterpret_cast<const i64*>(active_dofs), n_active);
    InArg<double> vals(active_values, n_active);
    auto c = build_constraints(*p->p, clamp_boundary != 0, n_active, dofs.dev, vals.dev);
    CF_CUDA(cudaStreamSynchronize(stream()));
    *out = new cf_constraints_s{std::move(c), p};
  });
}

int cf_constraints_destroy(cf_constraints c) {
  return guard([&] { delete c; });
}

int cf_constraints_distribute(cf_constraints c, double* v, int homogeneous) {
  return guard([&] {
    CHECK_ARG(c && v, "cf_constraints_distribute: null argument");
    OutArg<double> out(v, c->owner->p->g.n_total(), true);
    distribute(*c->c, out.dev, homogeneous != 0);
    out.finish();
  });
}

int cf_assemble_residual(cf_problem p, cf_constraints c, const cf_material* mat, const cf_regularization* reg,
                         const double* solution, const double* phi_tilde, double* R) {
  return guard([&] {
    CHECK_ARG(p && c && mat && reg && solution && phi_tilde && R, "cf_assemble_residual: null argument");
    const GridDesc& g = p->p->g;
    InArg<double> x(solution, g.n_total());
    InArg<double> pt(phi_tilde, g.V);
    OutArg<double> out(R, g.n_total());
    assemble_residual(*p->p, *c->c, *mat, *reg, x.dev, pt.dev, out.dev);
    out.finish();
  });
}

int cf_assemble_jacobian(cf_problem p, cf_constraints c, const cf_material* mat, const cf_regularization* reg,
                         const double* solution, const double* phi_tilde, cf_block* outb) {
  return guard([&] {
    CHECK_ARG(p && c && mat && reg && solution && phi_tilde && outb, "cf_assemble_jacobian: null argument");
    const GridDesc& g = p->p->g;
    InArg<double> x(solution, g.n_total());
    InArg<double> pt(phi_tilde, g.V);
    auto J = assemble_jacobian(*p->p, *c->c, *mat, *reg, x.dev, pt.dev);
    CF_CUDA(cudaStreamSynchronize(stream()));
    *outb = new cf_block_s{std::move(J)};
  });
}

int cf_block_info(cf_block b, int64_t* n_u, int64_t* n_phi, int64_t* nnz3) {
  return guard([&] {
    CHECK_ARG(b, "cf_block_info: null block");
    if (n_u) *n_u = b->J->nu;
    if (n_phi) *n_phi = b->J->np;
    if (nnz3) {
      nnz3[0] = b->J->uu.nnz;
      nnz3[1] = b->J->pu.nnz;
      nnz3[2] = b->J->pp.nnz;
    }
  });
}

int cf_block_export(cf_block b, int which, int64_t* rowptr, int32_t* col, double* val) {
  return guard([&] {
    CHECK_ARG(b && which >= 0 && which <= 2, "cf_block_export: bad argument");
    const Csr& A = which == 0 ? b->J->uu : (which == 1 ? b->J->pu : b->J->pp);
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      if (dst && bytes) CF_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, stream()));
    };
    cp(rowptr, A.ptr.p, size_t(A.rows + 1) * sizeof(i64));
    cp(col, A.col.p, size_t(A.nnz) * sizeof(int));
    cp(val, A.val.p, size_t(A.nnz) * sizeof(double));
    CF_CUDA(cudaStreamSynchronize(stream()));
  });
}

int cf_block_apply(cf_block b, const double* x, double* y) {
  return guard([&] {
    CHECK_ARG(b && x && y, "cf_block_apply: null argument");
    const i64 n = b->J->nu + b->J->np;
    InArg<double> xi(x, n);
    OutArg<double> yo(y, n);
    block_apply(*b->J, xi.dev, yo.dev);
    yo.finish();
  });
}

int cf_block_spmv(cf_block b, int which, const double* x, double* y) {
  return guard([&] {
    CHECK_ARG(b && x && y && which >= 0 && which <= 2, "cf_block_spmv: bad argument");
    const Csr& A = which == 0 ? b->J->uu : (which == 1 ? b->J->pu : b->J->pp);
    InArg<double> xi(x, A.cols);
    OutArg<double> yo(y, A.rows);
    csr_spmv_add(A, xi.dev, yo.dev, nullptr);
    yo.finish();
  });
}

int cf_block_destroy(cf_block b) {
  return guard([&] { delete b; });
}

}  // extern "C"

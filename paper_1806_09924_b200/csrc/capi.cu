// C ABI (include/crackfield_b200.h): status codes, last-error text, handle ownership and
// host/device argument staging around the cfb:: implementation.
#include <algorithm>
#include <cstring>
#include <map>
#include <cstdlib>
#include <mutex>
#include <string>
#include <unordered_map>

#include "cf_comm.hpp"
#include "cf_mesh.hpp"
#include "cf_types.hpp"
#include "cf_vec.hpp"

struct cf_problem_s {
  cfb::Problem* p;
};
struct cf_csr_s {
  std::shared_ptr<cfb::Csr> A;
};
struct cf_amg_s {
  std::unique_ptr<cfb::Amg> h;
  cfb::DevBuf<double> mf_pt;         // cf_amg_set_matrix_free: copies of phi_tilde and the flags
  cfb::DevBuf<std::uint8_t> mf_flag;
};
struct cf_prec_s {
  std::unique_ptr<cfb::BlockPrec> p;
};
struct cf_state_s {
  cfb::State st;
  cf_problem prob;
  cf_mesh mesh = nullptr;  // a general-mesh state (prob == nullptr)
};
struct cf_mesh_s {
  std::unique_ptr<cfb::MeshDisc> m;
};
struct cf_constraints_s {
  std::unique_ptr<cfb::Constraints> c;
  cf_problem owner;
};
struct cf_block_s {
  std::unique_ptr<cfb::BlockSystem> J;
};
struct cf_comm_s {
  std::unique_ptr<cfb::Comm> c;
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
  r.ready = true;
}

namespace {
struct BlockCache {
  std::multimap<size_t, void*> free_;
  std::unordered_map<void*, size_t> size_of;
  size_t cached = 0;
  std::mutex mu;
};
BlockCache& block_cache() {
  static BlockCache* c = new BlockCache;  // intentionally leaked: no teardown-order issues at exit
  return *c;
}
size_t round_size(size_t b) {
  if (b < (size_t(1) << 20)) return (b + 511) & ~size_t(511);
  const size_t g = size_t(2) << 20;
  return (b + g - 1) & ~(g - 1);
}
}  // namespace

// CF_GUARD=1 (debug aid; compute-sanitizer is not available on the B200 pool): every block gets a
// 4 KB guard zone after the requested bytes, filled with 0xA5 and verified when the block is freed
// (an out-of-bounds write past the end is reported on stderr and counted), and the requested bytes
// are poisoned with 0xFF (NaN for doubles, -1 for integers) on every allocation, so a read of
// uninitialised device memory shows up as a parity failure against the oracle.
namespace {
bool guard_on() {
  static const bool on = std::getenv("CF_GUARD") != nullptr;
  return on;
}
constexpr size_t kGuard = 4096;
__global__ void k_guard_check(const unsigned char* __restrict__ z, size_t n, int* bad) {
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    if (z[i] != 0xA5) {
      atomicExch(bad, 1);
      return;
    }
}
}  // namespace

long guard_violations = 0;

void* dev_alloc(size_t bytes) {
  ensure_device();
  BlockCache& c = block_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  const size_t need = round_size(guard_on() ? bytes + kGuard : bytes);
  if (guard_on()) {
    void* q = nullptr;
    auto hit = c.free_.lower_bound(need);
    if (hit != c.free_.end() && hit->first <= need + need / 4 + (size_t(1) << 20)) {
      q = hit->second;
      c.cached -= hit->first;
      c.free_.erase(hit);
    } else {
      CF_CUDA(cudaMalloc(&q, need));
      c.size_of[q] = need;
    }
    auto* b = static_cast<unsigned char*>(q);
    CF_CUDA(cudaMemsetAsync(b, 0xFF, bytes, stream()));
    CF_CUDA(cudaMemsetAsync(b + bytes, 0xA5, c.size_of[q] - bytes, stream()));
    return q;
  }
  auto it = c.free_.lower_bound(need);
  if (it != c.free_.end() && it->first <= need + need / 4 + (size_t(1) << 20)) {
    void* p = it->second;
    c.cached -= it->first;
    c.free_.erase(it);
    return p;
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, need);
  if (e == cudaErrorMemoryAllocation) {  // give the cached blocks back and retry once
    cudaGetLastError();
    CF_CUDA(cudaStreamSynchronize(stream()));
    for (auto& kv : c.free_) {
      cudaFree(kv.second);
      c.size_of.erase(kv.second);
    }
    c.free_.clear();
    c.cached = 0;
    e = cudaMalloc(&p, need);
  }
  CF_CUDA(e);
  c.size_of[p] = need;
  return p;
}

void dev_free(void* p, size_t bytes) {
  if (!p) return;
  BlockCache& c = block_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  auto it = c.size_of.find(p);
  if (it == c.size_of.end()) return;
  if (guard_on()) {
    static int* bad = nullptr;
    if (!bad) cudaMalloc(&bad, sizeof(int));
    int h = 0;
    cudaMemsetAsync(bad, 0, sizeof(int), stream());
    k_guard_check<<<64, 256, 0, stream()>>>(static_cast<unsigned char*>(p) + bytes, it->second - bytes, bad);
    cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, stream());
    cudaStreamSynchronize(stream());
    if (h) {
      ++guard_violations;
      std::fprintf(stderr, "CF_GUARD violation: write past the end of a %zu-byte block\n", bytes);
    }
  }
  c.free_.insert({it->second, p});
  c.cached += it->second;
}

size_t dev_cached_bytes() { return block_cache().cached; }

void read_small(void* dst, const void* src, size_t bytes) {
  constexpr size_t kSlot = 4096;
  static void* slot = nullptr;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  ++host_sync_count();
  if (bytes > kSlot) {
    CF_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, stream()));
    CF_CUDA(cudaStreamSynchronize(stream()));
    return;
  }
  if (!slot) CF_CUDA(cudaHostAlloc(&slot, kSlot, cudaHostAllocDefault));
  CF_CUDA(cudaMemcpyAsync(slot, src, bytes, cudaMemcpyDeviceToHost, stream()));
  CF_CUDA(cudaStreamSynchronize(stream()));
  std::memcpy(dst, slot, bytes);
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
  return guard([&] {
    // cached blocks are reused in stream order: drain the old stream before switching
    if (rt().ready && rt().stream != static_cast<cudaStream_t>(s)) CF_CUDA(cudaStreamSynchronize(rt().stream));
    rt().stream = static_cast<cudaStream_t>(s);
  });
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
    OutArg<double> out(v, c->c->flag.n, true);
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

static Slab planes_slab(const GridDesc& g, int64_t p_lo, int64_t p_hi) {
  CHECK_ARG(p_lo >= 0 && p_hi <= g.nn && p_lo < p_hi, "slab planes out of range");
  return make_slab(g, p_lo, p_hi);
}

int cf_slab_info(cf_problem p, int rank, int size, int64_t info[7]) {
  return guard([&] {
    CHECK_ARG(p && info, "cf_slab_info: null argument");
    const Slab s = rank_slab(p->p->g, rank, size);
    const int64_t v[7] = {s.v_lo, s.v_hi, s.ve_lo, s.ve_hi, s.c_lo, s.c_hi, s.plane};
    std::memcpy(info, v, sizeof(v));
  });
}

int cf_assemble_residual_planes(cf_problem p, cf_constraints c, const cf_material* mat, const cf_regularization* reg,
                                const double* solution, const double* phi_tilde, int64_t p_lo, int64_t p_hi,
                                double* R) {
  return guard([&] {
    CHECK_ARG(p && c && mat && reg && solution && phi_tilde && R, "cf_assemble_residual_planes: null argument");
    const GridDesc& g = p->p->g;
    const Slab sl = planes_slab(g, p_lo, p_hi);
    InArg<double> x(solution, g.n_total());
    InArg<double> pt(phi_tilde, g.V);
    OutArg<double> out(R, (g.d + 1) * sl.nv());
    assemble_residual(*p->p, *c->c, *mat, *reg, x.dev, pt.dev, out.dev, &sl);
    out.finish();
  });
}

int cf_assemble_jacobian_planes(cf_problem p, cf_constraints c, const cf_material* mat, const cf_regularization* reg,
                                const double* solution, const double* phi_tilde, int64_t p_lo, int64_t p_hi,
                                cf_block* outb) {
  return guard([&] {
    CHECK_ARG(p && c && mat && reg && solution && phi_tilde && outb, "cf_assemble_jacobian_planes: null argument");
    const GridDesc& g = p->p->g;
    const Slab sl = planes_slab(g, p_lo, p_hi);
    InArg<double> x(solution, g.n_total());
    InArg<double> pt(phi_tilde, g.V);
    auto J = assemble_jacobian(*p->p, *c->c, *mat, *reg, x.dev, pt.dev, &sl);
    CF_CUDA(cudaStreamSynchronize(stream()));
    *outb = new cf_block_s{std::move(J)};
  });
}

int cf_mf_apply_uu(cf_problem p, cf_constraints c, const cf_material* mat, const cf_regularization* reg,
                   const double* phi_tilde, const double* x, double* y) {
  return guard([&] {
    CHECK_ARG(p && c && mat && reg && phi_tilde && x && y, "cf_mf_apply_uu: null argument");
    const GridDesc& g = p->p->g;
    InArg<double> pt(phi_tilde, g.V);
    InArg<double> xi(x, g.n_u());
    OutArg<double> yo(y, g.n_u());
    mf_apply_uu(*p->p, *c->c, *mat, *reg, pt.dev, xi.dev, yo.dev);
    yo.finish();
  });
}

int cf_fp64_peak(double* tflops) {
  return guard([&] {
    CHECK_ARG(tflops, "cf_fp64_peak: null argument");
    ensure_device();
    *tflops = fp64_peak_tflops();
  });
}

int cf_sigma(const double grad_u[9], const cf_material* mat, int d, double out[9]) {
  return guard([&] {
    CHECK_ARG(grad_u && mat && out && (d == 2 || d == 3), "cf_sigma: bad argument");
    double e[3][3];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) e[a][b] = 0.5 * (grad_u[3 * a + b] + grad_u[3 * b + a]);
    double tr = 0.0;
    for (int a = 0; a < d; ++a) tr += e[a][a];
    const double two_mu = 2.0 * mat_mu(*mat);
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) out[3 * a + b] = two_mu * e[a][b];
    for (int a = 0; a < d; ++a) out[3 * a + a] += mat_lambda(*mat) * tr;
  });
}

int cf_q1_shape(int d, const double xi[3], double* values, double* grads) {
  return guard([&] {
    CHECK_ARG(xi && values && grads && (d == 2 || d == 3), "cf_q1_shape: bad argument");
    const int n = 1 << d;
    for (int k = 0; k < n; ++k) {
      double v = 1.0;
      for (int a = 0; a < d; ++a) v *= (k & (1 << a)) ? xi[a] : 1.0 - xi[a];
      values[k] = v;
      for (int a = 0; a < d; ++a) {
        double g = (k & (1 << a)) ? 1.0 : -1.0;
        for (int b = 0; b < d; ++b) {
          if (b == a) continue;
          g *= (k & (1 << b)) ? xi[b] : 1.0 - xi[b];
        }
        grads[k * d + a] = g;
      }
    }
  });
}

int cf_detect_cycles(int n, const int32_t* dofs, const int64_t* offsets, const uint8_t* bits, int window,
                     int toggles, int32_t* out, int* n_out) {
  return guard([&] {
    CHECK_ARG(n >= 0 && n_out && (n == 0 || (dofs && offsets && bits && out)), "cf_detect_cycles: bad argument");
    std::vector<int32_t> found;
    for (int t = 0; t < n; ++t) {
      const i64 lo = offsets[t], len = offsets[t + 1] - offsets[t];
      const i64 start = std::max<i64>(0, len - window);
      int changes = 0;
      for (i64 i = start + 1; i < len; ++i)
        if (bits[lo + i] != bits[lo + i - 1]) ++changes;
      if (changes >= toggles) found.push_back(dofs[t]);
    }
    std::sort(found.begin(), found.end());
    found.erase(std::unique(found.begin(), found.end()), found.end());
    std::copy(found.begin(), found.end(), out);
    *n_out = int(found.size());
  });
}

int cf_assemble_pattern(cf_problem p, cf_constraints c, cf_block* outb) {
  return guard([&] {
    CHECK_ARG(p && c && outb, "cf_assemble_pattern: null argument");
    auto J = assemble_pattern(*p->p, *c->c);
    CF_CUDA(cudaStreamSynchronize(stream()));
    *outb = new cf_block_s{std::move(J)};
  });
}

int cf_block_format(cf_block b, int which, int* format) {
  return guard([&] {
    CHECK_ARG(b && format && which >= 0 && which <= 2, "cf_block_format: bad argument");
    const Csr& A = which == 0 ? *b->J->uu : (which == 1 ? *b->J->pu : *b->J->pp);
    *format = A.st.kind != 0 ? 1 : 0;
  });
}

int cf_block_shape(cf_block b, int64_t shape[4]) {
  return guard([&] {
    CHECK_ARG(b && shape, "cf_block_shape: null argument");
    const BlockSystem& J = *b->J;
    shape[0] = J.nu;
    shape[1] = J.np;
    shape[2] = J.in_u();
    shape[3] = J.np_in >= 0 ? J.np_in : J.np;
  });
}

int cf_block_info(cf_block b, int64_t* n_u, int64_t* n_phi, int64_t* nnz3) {
  return guard([&] {
    CHECK_ARG(b, "cf_block_info: null block");
    if (n_u) *n_u = b->J->nu;
    if (n_phi) *n_phi = b->J->np;
    if (nnz3) {
      nnz3[0] = b->J->uu->nnz;
      nnz3[1] = b->J->pu->nnz;
      nnz3[2] = b->J->pp->nnz;
    }
  });
}

int cf_block_export(cf_block b, int which, int64_t* rowptr, int32_t* col, double* val) {
  return guard([&] {
    CHECK_ARG(b && which >= 0 && which <= 2, "cf_block_export: bad argument");
    const Csr& A = which == 0 ? *b->J->uu : (which == 1 ? *b->J->pu : *b->J->pp);
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
    const BlockSystem& J = *b->J;
    const i64 n = J.nu + J.np, n_in = J.in_u() + (J.np_in >= 0 ? J.np_in : J.np);
    InArg<double> xi(x, n_in);
    OutArg<double> yo(y, n);
    block_apply(*b->J, xi.dev, yo.dev);
    yo.finish();
  });
}

int cf_block_spmv(cf_block b, int which, const double* x, double* y) {
  return guard([&] {
    CHECK_ARG(b && x && y && which >= 0 && which <= 2, "cf_block_spmv: bad argument");
    const Csr& A = which == 0 ? *b->J->uu : (which == 1 ? *b->J->pu : *b->J->pp);
    InArg<double> xi(x, A.cols);
    OutArg<double> yo(y, A.rows);
    csr_spmv_add(A, xi.dev, yo.dev, nullptr);
    yo.finish();
  });
}

int cf_test_div_by(double h, const double* a, int64_t n, double* q) {
  return guard([&] {
    CHECK_ARG(a && q && n >= 0 && h > 0.0, "cf_test_div_by: bad argument");
    InArg<double> ai(a, n);
    OutArg<double> qo(q, n);
    div_by_h(h, ai.dev, n, qo.dev);
    qo.finish();
  });
}

int cf_tune_spmv(cf_block b, int which, int threads_per_row, int unroll, const double* x, double* y) {
  return guard([&] {
    CHECK_ARG(b && x && y && which >= 0 && which <= 2, "cf_tune_spmv: bad argument");
    const Csr& A = which == 0 ? *b->J->uu : (which == 1 ? *b->J->pu : *b->J->pp);
    InArg<double> xi(x, A.cols);
    OutArg<double> yo(y, A.rows);
    if (!csr_spmv_variant(A, threads_per_row, unroll, xi.dev, yo.dev))
      fail(CF_ERR_INVALID_ARGUMENT, "cf_tune_spmv: unknown variant");
    yo.finish();
  });
}

int cf_block_destroy(cf_block b) {
  return guard([&] { delete b; });
}

// ------------------------------------------------------------------ CSR handles
int cf_csr_create(int64_t rows, int64_t cols, const int64_t* rowptr, const int32_t* col, const double* val,
                  cf_csr* out) {
  return guard([&] {
    CHECK_ARG(out && rowptr && rows >= 0 && cols >= 0, "cf_csr_create: bad argument");
    ensure_device();
    auto A = std::make_shared<Csr>();
    A->rows = rows;
    A->cols = cols;
    A->ptr.alloc(rows + 1);
    CF_CUDA(cudaMemcpyAsync(A->ptr.p, rowptr, size_t(rows + 1) * sizeof(i64), cudaMemcpyDefault, stream()));
    CF_CUDA(cudaStreamSynchronize(stream()));
    i64 nnz = 0;
    CF_CUDA(cudaMemcpy(&nnz, A->ptr.p + rows, sizeof(i64), cudaMemcpyDeviceToHost));
    A->nnz = nnz;
    A->col.alloc(nnz);
    A->val.alloc(nnz);
    if (nnz) {
      CHECK_ARG(col && val, "cf_csr_create: null column/value arrays");
      CF_CUDA(cudaMemcpyAsync(A->col.p, col, size_t(nnz) * sizeof(int), cudaMemcpyDefault, stream()));
      CF_CUDA(cudaMemcpyAsync(A->val.p, val, size_t(nnz) * sizeof(double), cudaMemcpyDefault, stream()));
    }
    CF_CUDA(cudaStreamSynchronize(stream()));
    *out = new cf_csr_s{A};
  });
}

int cf_block_csr(cf_block b, int which, cf_csr* out) {
  return guard([&] {
    CHECK_ARG(b && out && which >= 0 && which <= 2, "cf_block_csr: bad argument");
    *out = new cf_csr_s{which == 0 ? b->J->uu : (which == 1 ? b->J->pu : b->J->pp)};
  });
}

int cf_csr_export(cf_csr A, int64_t* rowptr, int32_t* col, double* val) {
  return guard([&] {
    CHECK_ARG(A, "cf_csr_export: null handle");
    const Csr& M = *A->A;
    if (rowptr)
      CF_CUDA(cudaMemcpyAsync(rowptr, M.ptr.p, size_t(M.rows + 1) * sizeof(i64), cudaMemcpyDefault, stream()));
    if (col && M.nnz)
      CF_CUDA(cudaMemcpyAsync(col, M.col.p, size_t(M.nnz) * sizeof(int), cudaMemcpyDefault, stream()));
    if (val && M.nnz)
      CF_CUDA(cudaMemcpyAsync(val, M.val.p, size_t(M.nnz) * sizeof(double), cudaMemcpyDefault, stream()));
    CF_CUDA(cudaStreamSynchronize(stream()));
  });
}

int cf_csr_spgemm(cf_csr A, cf_csr B, const double* row_scale, cf_csr* out) {
  return guard([&] {
    CHECK_ARG(A && B && out, "cf_csr_spgemm: bad argument");
    CHECK_ARG(A->A->cols == B->A->rows, "cf_csr_spgemm: inner dimensions differ");
    InArg<double> rs(row_scale, A->A->rows);
    std::shared_ptr<Csr> C(spgemm(*A->A, *B->A, rs.dev).release());
    CF_CUDA(cudaStreamSynchronize(stream()));
    *out = new cf_csr_s{C};
  });
}

int cf_csr_info(cf_csr A, int64_t* rows, int64_t* cols, int64_t* nnz) {
  return guard([&] {
    CHECK_ARG(A, "cf_csr_info: null handle");
    if (rows) *rows = A->A->rows;
    if (cols) *cols = A->A->cols;
    if (nnz) *nnz = A->A->nnz;
  });
}

int cf_csr_spmv(cf_csr A, const double* x, double* y) {
  return guard([&] {
    CHECK_ARG(A && x && y, "cf_csr_spmv: null argument");
    InArg<double> xi(x, A->A->cols);
    OutArg<double> yo(y, A->A->rows);
    csr_spmv_add(*A->A, xi.dev, yo.dev, nullptr);
    yo.finish();
  });
}

int cf_csr_destroy(cf_csr A) {
  return guard([&] { delete A; });
}

// ------------------------------------------------------------------ AMG
int cf_amg_build(cf_csr A, const int32_t* node_of_dof, const double* B, int m, const cf_amg_options* opts,
                 cf_amg* out) {
  return guard([&] {
    CHECK_ARG(A && opts && out, "cf_amg_build: null argument");
    CHECK_ARG(A->A->rows == A->A->cols, "build_amg: matrix must be square");
    const i64 n = A->A->rows;
    DevBuf<int> nod;
    DevBuf<double> Bd;
    const int* nodp;
    const double* Bp;
    InArg<int> ni(node_of_dof, node_of_dof ? n : 0);
    InArg<double> bi(B, B ? n * m : 0);
    if (node_of_dof && B) {
      nodp = ni.dev;
      Bp = bi.dev;
    } else {
      CHECK_ARG(!node_of_dof && !B, "cf_amg_build: node_of_dof and B must be given together");
      m = 1;
      std::vector<int> h(n);
      for (i64 i = 0; i < n; ++i) h[i] = int(i);
      std::vector<double> one(n, 1.0);
      nod.alloc(n);
      Bd.alloc(n);
      if (n) {
        CF_CUDA(cudaMemcpyAsync(nod.p, h.data(), size_t(n) * sizeof(int), cudaMemcpyHostToDevice, stream()));
        CF_CUDA(cudaMemcpyAsync(Bd.p, one.data(), size_t(n) * sizeof(double), cudaMemcpyHostToDevice, stream()));
        CF_CUDA(cudaStreamSynchronize(stream()));
      }
      nodp = nod.p;
      Bp = Bd.p;
    }
    auto h = build_amg(A->A, nodp, Bp, m, *opts);
    CF_CUDA(cudaStreamSynchronize(stream()));
    *out = new cf_amg_s{std::move(h)};
  });
}

int cf_amg_vcycle(cf_amg h, const double* r, double* x) {
  return guard([&] {
    CHECK_ARG(h && r && x, "cf_amg_vcycle: null argument");
    InArg<double> ri(r, h->h->n);
    OutArg<double> xo(x, h->h->n);
    h->h->vcycle(ri.dev, xo.dev);
    xo.finish();
  });
}

int cf_amg_set_matrix_free(cf_amg h, cf_problem p, cf_constraints c, const cf_material* mat,
                           const cf_regularization* reg, const double* phi_tilde) {
  return guard([&] {
    CHECK_ARG(h && p && c && mat && reg && phi_tilde, "cf_amg_set_matrix_free: null argument");
    const GridDesc& g = p->p->g;
    CHECK_ARG(g.d == 3, "cf_amg_set_matrix_free: the matrix-free M_uu is 3d");
    CHECK_ARG(h->h->n == g.n_u(), "cf_amg_set_matrix_free: the hierarchy is not a u-block hierarchy of this problem");
    h->mf_pt.alloc(g.V);
    h->mf_flag.alloc(g.n_total());
    CF_CUDA(cudaMemcpyAsync(h->mf_pt.p, phi_tilde, size_t(g.V) * sizeof(double), cudaMemcpyDefault, stream()));
    CF_CUDA(cudaMemcpyAsync(h->mf_flag.p, c->c->flag.p, size_t(g.n_total()), cudaMemcpyDeviceToDevice, stream()));
    auto op = std::make_shared<MfOp>();
    op->P = p->p;
    op->flag = h->mf_flag.p;
    op->mu = mat_mu(*mat);
    op->lam = mat_lambda(*mat);
    op->kap = reg->kappa;
    op->pt = h->mf_pt.p;
    h->h->mf0 = op;
    CF_CUDA(cudaStreamSynchronize(stream()));
  });
}

int cf_amg_info(cf_amg h, int* n_levels, int64_t* coarse_dim) {
  return guard([&] {
    CHECK_ARG(h, "cf_amg_info: null handle");
    if (n_levels) *n_levels = int(h->h->levels.size()) + 1;
    if (coarse_dim) *coarse_dim = h->h->coarse.n;
  });
}

int cf_amg_level_info(cf_amg h, int level, int64_t* info8, double* lambda, double* jacobi_weight) {
  return guard([&] {
    CHECK_ARG(h && level >= 0 && level < int(h->h->levels.size()), "cf_amg_level_info: bad level");
    const AmgLevel& L = *h->h->levels[level];
    if (info8) {
      info8[0] = L.A->rows;
      info8[1] = L.A->nnz;
      info8[2] = L.P->nnz;
      info8[3] = L.P->cols;
      info8[4] = L.n_nodes;
      info8[5] = L.n_aggregates;
      info8[6] = L.strong_edges;
      info8[7] = L.lfmis_rounds;
    }
    if (lambda) *lambda = L.lambda;
    if (jacobi_weight) *jacobi_weight = L.jacobi_weight;
  });
}

int cf_amg_level_aggregates(cf_amg h, int level, int32_t* agg) {
  return guard([&] {
    CHECK_ARG(h && agg && level >= 0 && level < int(h->h->levels.size()), "cf_amg_level_aggregates: bad level");
    const AmgLevel& L = *h->h->levels[level];
    CF_CUDA(cudaMemcpyAsync(agg, L.agg_of_node.p, size_t(L.n_nodes) * sizeof(int), cudaMemcpyDefault, stream()));
    CF_CUDA(cudaStreamSynchronize(stream()));
  });
}

int cf_amg_level_export(cf_amg h, int level, int which, int64_t* rowptr, int32_t* col, double* val) {
  return guard([&] {
    CHECK_ARG(h && level >= 0 && level < int(h->h->levels.size()) && (which == 0 || which == 1),
              "cf_amg_level_export: bad argument");
    const AmgLevel& L = *h->h->levels[level];
    const Csr& M = which == 0 ? *L.A : *L.P;
    if (rowptr) CF_CUDA(cudaMemcpyAsync(rowptr, M.ptr.p, size_t(M.rows + 1) * sizeof(i64), cudaMemcpyDefault, stream()));
    if (col && M.nnz) CF_CUDA(cudaMemcpyAsync(col, M.col.p, size_t(M.nnz) * sizeof(int), cudaMemcpyDefault, stream()));
    if (val && M.nnz) CF_CUDA(cudaMemcpyAsync(val, M.val.p, size_t(M.nnz) * sizeof(double), cudaMemcpyDefault, stream()));
    CF_CUDA(cudaStreamSynchronize(stream()));
  });
}

int cf_tune_level_spmv(cf_amg h, int level, int which, int threads_per_row, int unroll, const double* x, double* y) {
  return guard([&] {
    CHECK_ARG(h && x && y && level >= 0 && level < int(h->h->levels.size()) && which >= 0 && which <= 2,
              "cf_tune_level_spmv: bad argument");
    const AmgLevel& L = *h->h->levels[level];
    const Csr& M = which == 0 ? *L.A : (which == 1 ? *L.P : *L.R);
    InArg<double> xi(x, M.cols);
    OutArg<double> yo(y, M.rows);
    if (threads_per_row == 0) csr_spmv_add(M, xi.dev, yo.dev, nullptr);
    else if (!csr_spmv_variant(M, threads_per_row, unroll, xi.dev, yo.dev))
      fail(CF_ERR_INVALID_ARGUMENT, "cf_tune_level_spmv: unknown variant");
    yo.finish();
  });
}

int cf_amg_destroy(cf_amg h) {
  return guard([&] { delete h; });
}

// ------------------------------------------------------------------ block preconditioner
int cf_prec_build(cf_block J, int kind, const cf_amg_options* opts, cf_problem p, cf_constraints c, cf_prec* out) {
  return guard([&] {
    CHECK_ARG(J && opts && out, "cf_prec_build: null argument");
    CHECK_ARG(kind >= 0 && kind <= 2, "unknown preconditioner kind");
    std::unique_ptr<BlockPrec> pr;
    if (p && c && kind == 1) {
      const GridDesc& g = p->p->g;
      const i64 nu = g.n_u(), V = g.V;
      const int m = g.d == 2 ? 3 : 6;
      DevBuf<double> Bu(nu * m), Bp(V);
      DevBuf<int> un(nu), pn(V);
      rigid_body_modes(*p->p, *c->c, Bu.p);
      std::vector<int> hu(nu), hp(V);
      std::vector<double> hb(V);
      std::vector<std::uint8_t> fl(g.n_total());
      CF_CUDA(cudaMemcpyAsync(fl.data(), c->c->flag.p, size_t(g.n_total()), cudaMemcpyDeviceToHost, stream()));
      CF_CUDA(cudaStreamSynchronize(stream()));
      for (i64 i = 0; i < nu; ++i) hu[i] = int(i / g.d);
      for (i64 v = 0; v < V; ++v) {
        hp[v] = int(v);
        hb[v] = fl[nu + v] ? 0.0 : 1.0;
      }
      CF_CUDA(cudaMemcpyAsync(un.p, hu.data(), size_t(nu) * sizeof(int), cudaMemcpyHostToDevice, stream()));
      CF_CUDA(cudaMemcpyAsync(pn.p, hp.data(), size_t(V) * sizeof(int), cudaMemcpyHostToDevice, stream()));
      CF_CUDA(cudaMemcpyAsync(Bp.p, hb.data(), size_t(V) * sizeof(double), cudaMemcpyHostToDevice, stream()));
      NullspaceDev ns{un.p, Bu.p, m, pn.p, Bp.p};
      pr = build_block_prec(*J->J, kind, *opts, &ns);
    } else {
      pr = build_block_prec(*J->J, kind, *opts, nullptr);
    }
    CF_CUDA(cudaStreamSynchronize(stream()));
    *out = new cf_prec_s{std::move(pr)};
  });
}

int cf_prec_apply(cf_prec P, const double* r, double* z) {
  return guard([&] {
    CHECK_ARG(P && r && z, "cf_prec_apply: null argument");
    const i64 n = P->p->nu + P->p->np;
    InArg<double> ri(r, n);
    OutArg<double> zo(z, n);
    P->p->apply(ri.dev, zo.dev);
    zo.finish();
  });
}

int cf_prec_destroy(cf_prec P) {
  return guard([&] { delete P; });
}

int cf_rigid_body_modes(cf_problem p, cf_constraints c, double* B) {
  return guard([&] {
    CHECK_ARG(p && c && B, "cf_rigid_body_modes: null argument");
    const GridDesc& g = p->p->g;
    OutArg<double> bo(B, g.n_u() * (g.d == 2 ? 3 : 6));
    rigid_body_modes(*p->p, *c->c, bo.dev);
    bo.finish();
  });
}

// ------------------------------------------------------------------ GMRES
int cf_gmres(cf_block J, cf_csr A, cf_prec P, cf_amg M, const double* rhs, const cf_gmres_options* opts, double* x,
             cf_gmres_result* result, double* history, int history_cap) {
  return guard([&] {
    CHECK_ARG((J != nullptr) != (A != nullptr), "cf_gmres: give exactly one operator (block or csr)");
    CHECK_ARG(!(P && M), "cf_gmres: give at most one preconditioner");
    CHECK_ARG(rhs && opts && x && result, "cf_gmres: null argument");
    const i64 n = J ? J->J->nu + J->J->np : A->A->rows;
    InArg<double> bi(rhs, n);
    OutArg<double> xo(x, n);
    DevOp op;
    if (J) {
      const BlockSystem* Jp = J->J.get();
      op = [Jp](const double* in, double* out) { block_apply(*Jp, in, out); };
    } else {
      const Csr* Ap = A->A.get();
      op = [Ap](const double* in, double* out) { csr_spmv_add(*Ap, in, out, nullptr); };
    }
    DevOp pop;
    const DevOp* pp = nullptr;
    if (P) {
      const BlockPrec* Pp = P->p.get();
      pop = [Pp](const double* in, double* out) { Pp->apply(in, out); };
      pp = &pop;
    } else if (M) {
      const Amg* Mp = M->h.get();
      pop = [Mp](const double* in, double* out) { Mp->vcycle(in, out); };
      pp = &pop;
    }
    GmresResult r = gmres(op, pp, bi.dev, n, *opts, xo.dev);
    xo.finish();
    CF_CUDA(cudaStreamSynchronize(stream()));
    result->iterations = r.iterations;
    result->converged = r.converged;
    result->breakdown = r.breakdown;
    result->residual = r.residual;
    if (history)
      for (int i = 0; i < int(r.history.size()) && i < history_cap; ++i) history[i] = r.history[i];
  });
}

// ------------------------------------------------------------------ functionals
int cf_compute_tcv(cf_problem p, const double* solution, double* tcv) {
  return guard([&] {
    CHECK_ARG(p && solution && tcv, "cf_compute_tcv: null argument");
    InArg<double> x(solution, p->p->g.n_total());
    *tcv = compute_tcv(*p->p, x.dev);
  });
}

int cf_compute_cod(cf_problem p, const double* solution, const double* stations, int n_stations, double* openings) {
  return guard([&] {
    CHECK_ARG(p && solution && (n_stations == 0 || (stations && openings)) && n_stations >= 0,
              "cf_compute_cod: bad argument");
    InArg<double> x(solution, p->p->g.n_total());
    compute_cod(*p->p, x.dev, stations, n_stations, openings);
  });
}

// ------------------------------------------------------------------ Newton
int cf_slit_band_edge(cf_problem p, const cf_material* mat, double* edge) {
  return guard([&] {
    CHECK_ARG(p && mat && edge, "cf_slit_band_edge: null argument");
    *edge = slit_band_edge(*p->p, *mat);
  });
}

int cf_resolve_regularization(cf_problem p, const cf_material* mat, double band_edge, cf_regularization* out) {
  return guard([&] {
    CHECK_ARG(p && mat && out, "cf_resolve_regularization: null argument");
    *out = resolve_regularization(*p->p, *mat, band_edge);
  });
}

int cf_initial_crack(cf_problem p, const cf_material* mat, double band_half, double* phi, double* band_edge) {
  return guard([&] {
    CHECK_ARG(p && mat && phi, "cf_initial_crack: null argument");
    auto h = initial_crack(*p->p, *mat, band_half, band_edge);
    CF_CUDA(cudaMemcpyAsync(phi, h.data(), h.size() * sizeof(double), cudaMemcpyDefault, stream()));
    CF_CUDA(cudaStreamSynchronize(stream()));
  });
}

int cf_state_create(cf_problem p, const double* solution, const double* phi_old, const double* phi_prev2, int step,
                    cf_state* out) {
  return guard([&] {
    CHECK_ARG(p && out, "cf_state_create: null argument");
    const GridDesc& g = p->p->g;
    auto* s = new cf_state_s;
    s->prob = p;
    s->st.solution.alloc(g.n_total());
    s->st.phi_old.alloc(g.V);
    s->st.phi_prev2.alloc(g.V);
    auto put = [&](DevBuf<double>& d, const double* src) {
      if (src)
        CF_CUDA(cudaMemcpyAsync(d.p, src, size_t(d.n) * sizeof(double), cudaMemcpyDefault, stream()));
      else
        d.zero();
    };
    put(s->st.solution, solution);
    put(s->st.phi_old, phi_old);
    put(s->st.phi_prev2, phi_prev2);
    s->st.step = step;
    CF_CUDA(cudaStreamSynchronize(stream()));
    *out = s;
  });
}

int cf_make_initial_state(cf_problem p, const cf_material* mat, double seed_band, cf_state* out) {
  return guard([&] {
    CHECK_ARG(p && mat && out, "cf_make_initial_state: null argument");
    const GridDesc& g = p->p->g;
    auto phi = initial_crack(*p->p, *mat, seed_band, nullptr);
    std::vector<double> sol(g.n_total(), 0.0);
    std::copy(phi.begin(), phi.end(), sol.begin() + g.n_u());
    cf_state s = nullptr;
    int rc = cf_state_create(p, sol.data(), phi.data(), phi.data(), 0, &s);
    if (rc != CF_OK) fail(rc, g_err);
    *out = s;
  });
}

int cf_state_get(cf_state s, double* solution, double* phi_old, double* phi_prev2, int* step) {
  return guard([&] {
    CHECK_ARG(s, "cf_state_get: null state");
    auto get = [&](double* dst, const DevBuf<double>& d) {
      if (dst) CF_CUDA(cudaMemcpyAsync(dst, d.p, size_t(d.n) * sizeof(double), cudaMemcpyDefault, stream()));
    };
    get(solution, s->st.solution);
    get(phi_old, s->st.phi_old);
    get(phi_prev2, s->st.phi_prev2);
    if (step) *step = s->st.step;
    CF_CUDA(cudaStreamSynchronize(stream()));
  });
}

int cf_extrapolate_phi(cf_state s, double* phi_tilde) {
  return guard([&] {
    CHECK_ARG(s && phi_tilde, "cf_extrapolate_phi: null argument");
    const i64 V = s->st.phi_old.n;
    OutArg<double> out(phi_tilde, V);
    extrapolate_phi(s->st, out.dev, V);
    out.finish();
  });
}

int cf_state_destroy(cf_state s) {
  return guard([&] { delete s; });
}

static void fill_report(const NewtonReport& r, cf_newton_iteration* its, int max_its, int* n_its, int* converged,
                        double* feasibility) {
  if (n_its) *n_its = int(r.its.size());
  if (its)
    for (int i = 0; i < int(r.its.size()) && i < max_its; ++i)
      its[i] = cf_newton_iteration{r.its[i].residual_norm, r.its[i].active_size, r.its[i].set_changes,
                                   r.its[i].gmres_iterations};
  if (converged) *converged = r.converged;
  if (feasibility) *feasibility = r.feasibility;
}

// ------------------------------------------------------------------ I/O
int cf_block_write_matrix_market(cf_block b, int which, const char* path) {
  return guard([&] {
    CHECK_ARG(b && path && which >= 0 && which <= 2, "cf_block_write_matrix_market: bad argument");
    write_matrix_market(which == 0 ? *b->J->uu : (which == 1 ? *b->J->pu : *b->J->pp), path);
  });
}

int cf_csr_write_matrix_market(cf_csr A, const char* path) {
  return guard([&] {
    CHECK_ARG(A && path, "cf_csr_write_matrix_market: null argument");
    write_matrix_market(*A->A, path);
  });
}

int cf_write_vtk(cf_problem p, const double* solution, const double* phi_old, const char* path, int binary) {
  return guard([&] {
    CHECK_ARG(p && solution && path, "cf_write_vtk: null argument");
    InArg<double> x(solution, p->p->g.n_total());
    InArg<double> po(phi_old, phi_old ? p->p->g.V : 0);
    write_vtk(*p->p, x.dev, phi_old ? po.dev : nullptr, path, binary != 0);
  });
}

// ------------------------------------------------------------------ communicator
int cf_comm_unique_id(uint8_t id[128]) {
  return guard([&] {
    CHECK_ARG(id, "cf_comm_unique_id: null argument");
    comm_unique_id(id);
  });
}

int cf_comm_selftest(int* failed_checks) {
  return guard([&] {
    CHECK_ARG(failed_checks, "cf_comm_selftest: null argument");
    ensure_device();
    *failed_checks = comm_selftest();
  });
}

int cf_comm_create_host(int rank, int size, const cf_host_transport* transport, cf_comm* out) {
  return guard([&] {
    CHECK_ARG(out && transport, "cf_comm_create_host: null argument");
    *out = new cf_comm_s{comm_create_host(rank, size, *transport)};
  });
}

int cf_comm_create(const uint8_t id[128], int rank, int size, cf_comm* out) {
  return guard([&] {
    CHECK_ARG(out && (size == 1 || id), "cf_comm_create: null argument");
    unsigned char zero[128] = {0};
    *out = new cf_comm_s{comm_create(id ? id : zero, rank, size)};
  });
}

int cf_comm_info(cf_comm c, int* rank, int* size) {
  return guard([&] {
    CHECK_ARG(c, "cf_comm_info: null communicator");
    if (rank) *rank = c->c->rank;
    if (size) *size = c->c->size;
  });
}

int cf_comm_destroy(cf_comm c) {
  return guard([&] { delete c; });
}

static void newton_timed(cf_problem p, cf_state s, const cf_material* mat, const cf_regularization* reg,
                         const cf_solver_options* opts, const Comm* comm, cf_newton_iteration* its, int max_its,
                         int* n_its, int* converged, double* feasibility, cf_phase_times* times) {
  cudaEvent_t a, b;
  CF_CUDA(cudaEventCreate(&a));
  CF_CUDA(cudaEventCreate(&b));
  CF_CUDA(cudaEventRecord(a, stream()));
  NewtonReport r = newton_active_set_step(*p->p, s->st, *mat, *reg, *opts, comm);
  CF_CUDA(cudaEventRecord(b, stream()));
  CF_CUDA(cudaEventSynchronize(b));
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  fill_report(r, its, max_its, n_its, converged, feasibility);
  if (times)
    *times = cf_phase_times{r.times.residual, r.times.active_set, r.times.jacobian, r.times.amg_setup, r.times.gmres,
                            double(ms)};
}

int cf_newton_active_set_step(cf_problem p, cf_state s, const cf_material* mat, const cf_regularization* reg,
                              const cf_solver_options* opts, cf_newton_iteration* its, int max_its, int* n_its,
                              int* converged, double* feasibility, cf_phase_times* times) {
  return guard([&] {
    CHECK_ARG(p && s && mat && reg && opts, "cf_newton_active_set_step: null argument");
    newton_timed(p, s, mat, reg, opts, nullptr, its, max_its, n_its, converged, feasibility, times);
  });
}

int cf_newton_active_set_step_comm(cf_problem p, cf_state s, const cf_material* mat, const cf_regularization* reg,
                                   const cf_solver_options* opts, cf_comm comm, cf_newton_iteration* its,
                                   int max_its, int* n_its, int* converged, double* feasibility,
                                   cf_phase_times* times) {
  return guard([&] {
    CHECK_ARG(p && s && mat && reg && opts && comm, "cf_newton_active_set_step_comm: null argument");
    newton_timed(p, s, mat, reg, opts, comm->c.get(), its, max_its, n_its, converged, feasibility, times);
  });
}

static void loading_sequence(cf_problem p, cf_state s, const cf_material* mat, const cf_regularization* reg,
                             const cf_solver_options* opts, const Comm* comm, int n_steps, cf_newton_iteration* its,
                             int max_its, int* n_its, int* converged, double* feasibility, int* steps_done) {
  if (n_steps < 1) fail(CF_ERR_INVALID_ARGUMENT, "solve_loading_sequence: n_steps must be >= 1");
  const GridDesc& g = p->p->g;
  int done = 0, off = 0;
  for (int n = 1; n <= n_steps; ++n) {
    State& st = s->st;
    CF_CUDA(cudaMemcpyAsync(st.phi_prev2.p, st.phi_old.p, size_t(g.V) * sizeof(double), cudaMemcpyDeviceToDevice,
                            stream()));
    CF_CUDA(cudaMemcpyAsync(st.phi_old.p, st.solution.p + g.n_u(), size_t(g.V) * sizeof(double),
                            cudaMemcpyDeviceToDevice, stream()));
    st.step = n;
    NewtonReport r = newton_active_set_step(*p->p, st, *mat, *reg, *opts, comm);
    int k = 0;
    fill_report(r, its ? its + off : nullptr, std::max(0, max_its - off), &k, converged ? converged + (n - 1) : nullptr,
                feasibility ? feasibility + (n - 1) : nullptr);
    if (n_its) n_its[n - 1] = k;
    off += std::min(k, std::max(0, max_its - off));
    ++done;
    if (!r.converged) break;
  }
  if (steps_done) *steps_done = done;
}

int cf_solve_loading_sequence(cf_problem p, cf_state s, const cf_material* mat, const cf_regularization* reg,
                              const cf_solver_options* opts, int n_steps, cf_newton_iteration* its, int max_its,
                              int* n_its, int* converged, double* feasibility, int* steps_done) {
  return guard([&] {
    CHECK_ARG(p && s && mat && reg && opts, "cf_solve_loading_sequence: null argument");
    loading_sequence(p, s, mat, reg, opts, nullptr, n_steps, its, max_its, n_its, converged, feasibility, steps_done);
  });
}

int cf_solve_loading_sequence_comm(cf_problem p, cf_state s, const cf_material* mat, const cf_regularization* reg,
                                   const cf_solver_options* opts, cf_comm comm, int n_steps,
                                   cf_newton_iteration* its, int max_its, int* n_its, int* converged,
                                   double* feasibility, int* steps_done) {
  return guard([&] {
    CHECK_ARG(p && s && mat && reg && opts && comm, "cf_solve_loading_sequence_comm: null argument");
    loading_sequence(p, s, mat, reg, opts, comm->c.get(), n_steps, its, max_its, n_its, converged, feasibility,
                     steps_done);
  });
}

}  // extern "C"

// ------------------------------------------------------------------ general meshes
static MeshDisc& M(cf_mesh m) { return *m->m; }

static void mesh_loading_sequence(MeshDisc& m, State& st, const cf_material& mat, const cf_regularization& reg,
                                  const cf_solver_options& opts, int n_steps, std::vector<NewtonReport>& reps) {
  if (n_steps < 1) fail(CF_ERR_INVALID_ARGUMENT, "solve_loading_sequence: n_steps must be >= 1");
  for (int n = 1; n <= n_steps; ++n) {  // solver.cpp:190-204
    CF_CUDA(cudaMemcpyAsync(st.phi_prev2.p, st.phi_old.p, size_t(m.V) * sizeof(double), cudaMemcpyDeviceToDevice,
                            stream()));
    CF_CUDA(cudaMemcpyAsync(st.phi_old.p, st.solution.p + m.n_u(), size_t(m.V) * sizeof(double),
                            cudaMemcpyDeviceToDevice, stream()));
    st.step = n;
    reps.push_back(mesh_newton_step(m, st, mat, reg, opts));
    if (!reps.back().converged) break;
  }
}

// make_initial_state on a mesh (solver.cpp:24-35): u = 0, phi = phi_old = phi_prev2 = seed
static void mesh_initial_state(MeshDisc& m, const cf_material& mat, double seed_band, State& st) {
  const std::vector<double> phi = mesh_initial_crack(m, mat, seed_band, nullptr);
  st.solution.alloc(m.n_total());
  st.phi_old.alloc(m.V);
  st.phi_prev2.alloc(m.V);
  st.solution.zero();
  CF_CUDA(cudaMemcpyAsync(st.solution.p + m.n_u(), phi.data(), size_t(m.V) * sizeof(double), cudaMemcpyHostToDevice,
                          stream()));
  CF_CUDA(cudaMemcpyAsync(st.phi_old.p, phi.data(), size_t(m.V) * sizeof(double), cudaMemcpyHostToDevice, stream()));
  CF_CUDA(cudaMemcpyAsync(st.phi_prev2.p, phi.data(), size_t(m.V) * sizeof(double), cudaMemcpyHostToDevice,
                          stream()));
  st.step = 0;
  CF_CUDA(cudaStreamSynchronize(stream()));
}

// adaptive_cycle (adapt.cpp:122-190)
static std::vector<cf_level_record> mesh_adaptive_cycle(MeshDisc& m, State& st, const cf_material& mat,
                                                        const cf_adaptive_options& o) {
  if (o.cycles < 0) fail(CF_ERR_INVALID_ARGUMENT, "adaptive_cycle: cycles must be >= 0");
  cf_refinement_policy pol = o.policy;
  double seed_band = o.seed_band;
  if (seed_band <= 0.0 && !o.halve_band_target) seed_band = mesh_slit_band_edge(m, mat);
  std::vector<cf_level_record> out;
  for (int cycle = 0; cycle <= o.cycles; ++cycle) {
    const cf_regularization reg = mesh_resolve_regularization(m, mat, mesh_slit_band_edge(m, mat));
    std::vector<NewtonReport> reps;
    mesh_loading_sequence(m, st, mat, reg, o.solver, o.n_steps, reps);
    const NewtonReport& last = reps.back();
    cf_level_record r{};
    r.level = cycle;
    r.dofs = m.n_total();
    r.eps = reg.eps;
    r.h_min = m.level_edge(m.max_level);
    r.tcv = std::abs(mesh_compute_tcv(m, st.solution.p));
    r.newton_iters = int(last.its.size());
    int tot = 0;
    for (const auto& it : last.its) tot += it.gmres_iterations;
    r.gmres_mean = last.its.empty() ? 0.0 : double(tot) / double(last.its.size());
    r.converged = last.converged;
    out.push_back(r);
    if (!last.converged || cycle == o.cycles) break;
    if (o.halve_band_target) pol.h_target = 0.5 * mesh_slit_band_edge(m, mat);
    for (int pass = 0; pass < std::max(1, o.estimator_rounds); ++pass) {
      if (pass > 0) {
        const cf_regularization r2 = mesh_resolve_regularization(m, mat, mesh_slit_band_edge(m, mat));
        std::vector<NewtonReport> rp;
        mesh_loading_sequence(m, st, mat, r2, o.solver, o.n_steps, rp);
        if (!rp.back().converged) break;
      }
      DevBuf<double> eta;
      if (pol.estimator) {
        eta.alloc(m.nact);
        mesh_jump_estimator(m, st.solution.p, eta.p);
        mesh_mask_band_eta(m, st.solution.p, eta.p, pol);
      }
      std::vector<int> marked = mesh_mark_cells(m, st.solution.p, pol.estimator ? eta.p : nullptr, pol);
      if (marked.empty()) break;
      for (int round = 0; round < 10 && !marked.empty(); ++round) {
        std::unique_ptr<MeshDisc> old = mesh_copy(m);
        mesh_refine(m, marked);
        // move_state (adapt.cpp:101-118): u transferred, phi / phi_old / history re-seeded
        DevBuf<double> moved(m.n_total());
        mesh_transfer(*old, st.solution.p, m, moved.p);
        State next;
        mesh_initial_state(m, mat, seed_band, next);
        CF_CUDA(cudaMemcpyAsync(next.solution.p, moved.p, size_t(m.n_u()) * sizeof(double), cudaMemcpyDeviceToDevice,
                                stream()));
        st.solution = std::move(next.solution);
        st.phi_old = std::move(next.phi_old);
        st.phi_prev2 = std::move(next.phi_prev2);
        st.step = 0;
        cf_refinement_policy band_only = pol;
        band_only.estimator = 0;
        marked = mesh_mark_cells(m, st.solution.p, nullptr, band_only);
      }
    }
  }
  return out;
}

extern "C" {

int cf_mesh_create(int dim, double half_width, int n0, cf_mesh* out) {
  return guard([&] {
    CHECK_ARG(out, "cf_mesh_create: null argument");
    *out = new cf_mesh_s{std::unique_ptr<MeshDisc>(mesh_create(dim, half_width, n0))};
  });
}
int cf_mesh_copy(cf_mesh m, cf_mesh* out) {
  return guard([&] {
    CHECK_ARG(m && out, "cf_mesh_copy: null argument");
    *out = new cf_mesh_s{mesh_copy(M(m))};
  });
}
int cf_mesh_destroy(cf_mesh m) {
  return guard([&] { delete m; });
}
int cf_mesh_refine(cf_mesh m, const int32_t* cells, int64_t n) {
  return guard([&] {
    CHECK_ARG(m && (n == 0 || cells) && n >= 0, "cf_mesh_refine: bad argument");
    mesh_refine(M(m), std::vector<int>(cells, cells + n));
  });
}
int cf_mesh_uniform_refine(cf_mesh m, int times) {
  return guard([&] {
    CHECK_ARG(m, "cf_mesh_uniform_refine: null mesh");
    mesh_uniform_refine(M(m), times);
  });
}
int cf_mesh_info(cf_mesh m, int64_t info4[4], double* h_min) {
  return guard([&] {
    CHECK_ARG(m && info4, "cf_mesh_info: null argument");
    const MeshDisc& d = M(m);
    info4[0] = int64_t(d.cells.size());
    info4[1] = d.nact;
    info4[2] = d.max_level;
    info4[3] = d.V;
    if (h_min) *h_min = d.level_edge(d.max_level);
  });
}
int cf_mesh_active_cells(cf_mesh m, int32_t* ids) {
  return guard([&] {
    CHECK_ARG(m && ids, "cf_mesh_active_cells: null argument");
    std::copy(M(m).active.begin(), M(m).active.end(), ids);
  });
}
int cf_mesh_cells(cf_mesh m, int32_t* level, int32_t* parent, int8_t* active, int64_t* anchor) {
  return guard([&] {
    CHECK_ARG(m, "cf_mesh_cells: null mesh");
    const MeshDisc& d = M(m);
    for (size_t i = 0; i < d.cells.size(); ++i) {
      if (level) level[i] = d.cells[i].level;
      if (parent) parent[i] = d.cells[i].parent;
      if (active) active[i] = d.cells[i].active;
      if (anchor)
        for (int a = 0; a < 3; ++a) anchor[3 * i + a] = d.cells[i].anchor[a];
    }
  });
}
int cf_mesh_vertex_keys(cf_mesh m, int64_t* keys) {
  return guard([&] {
    CHECK_ARG(m && keys, "cf_mesh_vertex_keys: null argument");
    CF_CUDA(cudaMemcpyAsync(keys, M(m).vkey.p, size_t(M(m).V) * sizeof(int64_t), cudaMemcpyDefault, stream()));
    CF_CUDA(cudaStreamSynchronize(stream()));
  });
}
int cf_mesh_cell_vertices(cf_mesh m, int64_t* out) {
  return guard([&] {
    CHECK_ARG(m && out, "cf_mesh_cell_vertices: null argument");
    const MeshDisc& d = M(m);
    const i64 n = d.nact * (i64(1) << d.d);
    std::vector<int> cv(size_t(std::max<i64>(n, 0)));
    CF_CUDA(cudaMemcpyAsync(cv.data(), d.cvert.p, size_t(n) * sizeof(int), cudaMemcpyDeviceToHost, stream()));
    CF_CUDA(cudaStreamSynchronize(stream()));
    for (i64 i = 0; i < n; ++i) out[i] = cv[size_t(i)];
  });
}
int cf_mesh_faces(cf_mesh m, int64_t* n, int32_t* out5) {
  return guard([&] {
    CHECK_ARG(m && n, "cf_mesh_faces: null argument");
    const std::vector<int> f = mesh_faces(M(m));
    *n = int64_t(f.size() / 5);
    if (out5) std::copy(f.begin(), f.end(), out5);
  });
}
int cf_mesh_find_cell(cf_mesh m, const double x[3], int32_t* cell) {
  return guard([&] {
    CHECK_ARG(m && x && cell, "cf_mesh_find_cell: null argument");
    *cell = mesh_find_cell(M(m), x);
  });
}
int cf_mesh_constraints_build(cf_mesh m, int clamp_boundary, int64_t n_active, const int64_t* active_dofs,
                              const double* active_values, cf_constraints* out) {
  return guard([&] {
    CHECK_ARG(m && out, "cf_mesh_constraints_build: null argument");
    CHECK_ARG(n_active >= 0, "cf_mesh_constraints_build: negative active count");
    CHECK_ARG(n_active == 0 || (active_dofs && active_values), "cf_mesh_constraints_build: null active arrays");
    InArg<i64> dofs(reinterpret_cast<const i64*>(active_dofs), n_active);
    InArg<double> vals(active_values, n_active);
    auto c = mesh_build_constraints(M(m), clamp_boundary != 0, n_active, dofs.dev, vals.dev);
    *out = new cf_constraints_s{std::move(c), nullptr};
  });
}
int cf_constraint_lines(cf_constraints c, int64_t* n_lines, int64_t* n_entries, int64_t* dofs, int64_t* ptr,
                        int64_t* masters, double* weights, double* inhomogeneities) {
  return guard([&] {
    CHECK_ARG(c && n_lines && n_entries, "cf_constraint_lines: null argument");
    const Constraints& cs = *c->c;
    *n_lines = cs.n_lines;
    std::vector<i64> lp(size_t(cs.n_lines + 1), 0);
    if (cs.n_lines)
      CF_CUDA(cudaMemcpyAsync(lp.data(), cs.line_ptr.p, lp.size() * sizeof(i64), cudaMemcpyDeviceToHost, stream()));
    CF_CUDA(cudaStreamSynchronize(stream()));
    *n_entries = lp.back();
    if (!dofs) return;
    std::vector<int> ld(size_t(cs.n_lines)), lm(size_t(lp.back()));
    std::vector<double> lw(size_t(lp.back())), inh(size_t(cs.flag.n));
    if (cs.n_lines) {
      CF_CUDA(cudaMemcpyAsync(ld.data(), cs.line_dof.p, ld.size() * sizeof(int), cudaMemcpyDeviceToHost, stream()));
      if (!lm.empty()) {
        CF_CUDA(cudaMemcpyAsync(lm.data(), cs.line_m.p, lm.size() * sizeof(int), cudaMemcpyDeviceToHost, stream()));
        CF_CUDA(cudaMemcpyAsync(lw.data(), cs.line_w.p, lw.size() * sizeof(double), cudaMemcpyDeviceToHost,
                                stream()));
      }
    }
    CF_CUDA(cudaMemcpyAsync(inh.data(), cs.inhom.p, inh.size() * sizeof(double), cudaMemcpyDeviceToHost, stream()));
    CF_CUDA(cudaStreamSynchronize(stream()));
    for (i64 i = 0; i < cs.n_lines; ++i) {
      dofs[i] = ld[size_t(i)];
      if (ptr) ptr[i] = lp[size_t(i)];
      if (inhomogeneities) inhomogeneities[i] = inh[size_t(ld[size_t(i)])];
    }
    if (ptr) ptr[cs.n_lines] = lp.back();
    for (i64 k = 0; k < lp.back(); ++k) {
      if (masters) masters[k] = lm[size_t(k)];
      if (weights) weights[k] = lw[size_t(k)];
    }
  });
}
int cf_mesh_assemble_residual(cf_mesh m, cf_constraints c, const cf_material* mat, const cf_regularization* reg,
                              const double* solution, const double* phi_tilde, double* residual) {
  return guard([&] {
    CHECK_ARG(m && c && mat && reg && solution && phi_tilde && residual, "cf_mesh_assemble_residual: null argument");
    MeshDisc& d = M(m);
    InArg<double> x(solution, d.n_total());
    InArg<double> pt(phi_tilde, d.V);
    OutArg<double> out(residual, d.n_total());
    mesh_assemble_residual(d, *c->c, *c->c, *mat, *reg, x.dev, pt.dev, out.dev);
    out.finish();
  });
}
int cf_mesh_assemble_jacobian(cf_mesh m, cf_constraints c, const cf_material* mat, const cf_regularization* reg,
                              const double* solution, const double* phi_tilde, cf_block* out) {
  return guard([&] {
    CHECK_ARG(m && c && mat && reg && solution && phi_tilde && out, "cf_mesh_assemble_jacobian: null argument");
    MeshDisc& d = M(m);
    InArg<double> x(solution, d.n_total());
    InArg<double> pt(phi_tilde, d.V);
    auto J = mesh_assemble_jacobian(d, *c->c, *c->c, *mat, *reg, x.dev, pt.dev);
    CF_CUDA(cudaStreamSynchronize(stream()));
    *out = new cf_block_s{std::move(J)};
  });
}
int cf_mesh_rigid_body_modes(cf_mesh m, cf_constraints c, double* B) {
  return guard([&] {
    CHECK_ARG(m && c && B, "cf_mesh_rigid_body_modes: null argument");
    MeshDisc& d = M(m);
    OutArg<double> out(B, d.n_u() * (d.d == 2 ? 3 : 6));
    mesh_rigid_body_modes(d, *c->c, out.dev);
    out.finish();
  });
}
int cf_mesh_slit_band_edge(cf_mesh m, const cf_material* mat, double* edge) {
  return guard([&] {
    CHECK_ARG(m && mat && edge, "cf_mesh_slit_band_edge: null argument");
    *edge = mesh_slit_band_edge(M(m), *mat);
  });
}
int cf_mesh_resolve_regularization(cf_mesh m, const cf_material* mat, double band_edge, cf_regularization* out) {
  return guard([&] {
    CHECK_ARG(m && mat && out, "cf_mesh_resolve_regularization: null argument");
    *out = mesh_resolve_regularization(M(m), *mat, band_edge);
  });
}
int cf_mesh_initial_crack(cf_mesh m, const cf_material* mat, double band_half, double* phi, double* band_edge) {
  return guard([&] {
    CHECK_ARG(m && mat && phi, "cf_mesh_initial_crack: null argument");
    const std::vector<double> v = mesh_initial_crack(M(m), *mat, band_half, band_edge);
    OutArg<double> out(phi, M(m).V);
    CF_CUDA(cudaMemcpyAsync(out.dev, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice, stream()));
    out.finish();
    CF_CUDA(cudaStreamSynchronize(stream()));
  });
}
int cf_mesh_state_create(cf_mesh m, const double* solution, const double* phi_old, const double* phi_prev2, int step,
                         cf_state* out) {
  return guard([&] {
    CHECK_ARG(m && out, "cf_mesh_state_create: null argument");
    MeshDisc& d = M(m);
    auto* s = new cf_state_s;
    s->prob = nullptr;
    s->mesh = m;
    s->st.solution.alloc(d.n_total());
    s->st.phi_old.alloc(d.V);
    s->st.phi_prev2.alloc(d.V);
    auto put = [&](DevBuf<double>& b, const double* src) {
      if (src)
        CF_CUDA(cudaMemcpyAsync(b.p, src, size_t(b.n) * sizeof(double), cudaMemcpyDefault, stream()));
      else
        b.zero();
    };
    put(s->st.solution, solution);
    put(s->st.phi_old, phi_old);
    put(s->st.phi_prev2, phi_prev2);
    s->st.step = step;
    CF_CUDA(cudaStreamSynchronize(stream()));
    *out = s;
  });
}
int cf_mesh_make_initial_state(cf_mesh m, const cf_material* mat, double seed_band, cf_state* out) {
  return guard([&] {
    CHECK_ARG(m && mat && out, "cf_mesh_make_initial_state: null argument");
    auto* s = new cf_state_s;
    s->prob = nullptr;
    s->mesh = m;
    try {
      mesh_initial_state(M(m), *mat, seed_band, s->st);
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}
int cf_mesh_newton_active_set_step(cf_mesh m, cf_state s, const cf_material* mat, const cf_regularization* reg,
                                   const cf_solver_options* opts, cf_newton_iteration* its, int max_its, int* n_its,
                                   int* converged, double* feasibility, cf_phase_times* times) {
  return guard([&] {
    CHECK_ARG(m && s && mat && reg && opts, "cf_mesh_newton_active_set_step: null argument");
    CHECK_ARG(s->st.solution.n == M(m).n_total(), "cf_mesh_newton_active_set_step: state of another mesh");
    validate_material(*mat);
    cudaEvent_t a, b;
    CF_CUDA(cudaEventCreate(&a));
    CF_CUDA(cudaEventCreate(&b));
    CF_CUDA(cudaEventRecord(a, stream()));
    NewtonReport r = mesh_newton_step(M(m), s->st, *mat, *reg, *opts);
    CF_CUDA(cudaEventRecord(b, stream()));
    CF_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    fill_report(r, its, max_its, n_its, converged, feasibility);
    if (times)
      *times = cf_phase_times{r.times.residual, r.times.active_set, r.times.jacobian, r.times.amg_setup,
                              r.times.gmres, double(ms)};
  });
}
int cf_mesh_solve_loading_sequence(cf_mesh m, cf_state s, const cf_material* mat, const cf_regularization* reg,
                                   const cf_solver_options* opts, int n_steps, cf_newton_iteration* its, int max_its,
                                   int* n_its, int* converged, double* feasibility, int* steps_done) {
  return guard([&] {
    CHECK_ARG(m && s && mat && reg && opts, "cf_mesh_solve_loading_sequence: null argument");
    validate_material(*mat);
    std::vector<NewtonReport> reps;
    mesh_loading_sequence(M(m), s->st, *mat, *reg, *opts, n_steps, reps);
    int off = 0;
    for (size_t n = 0; n < reps.size(); ++n) {
      int k = 0;
      fill_report(reps[n], its ? its + off : nullptr, std::max(0, max_its - off), &k,
                  converged ? converged + n : nullptr, feasibility ? feasibility + n : nullptr);
      if (n_its) n_its[n] = k;
      off += std::min(k, std::max(0, max_its - off));
    }
    if (steps_done) *steps_done = int(reps.size());
  });
}
int cf_mesh_compute_tcv(cf_mesh m, const double* solution, double* tcv) {
  return guard([&] {
    CHECK_ARG(m && solution && tcv, "cf_mesh_compute_tcv: null argument");
    InArg<double> x(solution, M(m).n_total());
    *tcv = mesh_compute_tcv(M(m), x.dev);
  });
}
int cf_mesh_compute_cod(cf_mesh m, const double* solution, const double* stations, int n_stations, double* openings) {
  return guard([&] {
    CHECK_ARG(m && solution && (n_stations == 0 || (stations && openings)), "cf_mesh_compute_cod: null argument");
    InArg<double> x(solution, M(m).n_total());
    mesh_compute_cod(M(m), x.dev, stations, n_stations, openings);
  });
}
int cf_mesh_jump_estimator(cf_mesh m, const double* solution, double* eta) {
  return guard([&] {
    CHECK_ARG(m && solution && eta, "cf_mesh_jump_estimator: null argument");
    InArg<double> x(solution, M(m).n_total());
    OutArg<double> out(eta, M(m).nact);
    mesh_jump_estimator(M(m), x.dev, out.dev);
    out.finish();
  });
}
int cf_mesh_mark_cells(cf_mesh m, const double* solution, const double* eta, const cf_refinement_policy* policy,
                       int32_t* marked, int64_t* n_marked) {
  return guard([&] {
    CHECK_ARG(m && solution && policy && marked && n_marked, "cf_mesh_mark_cells: null argument");
    InArg<double> x(solution, M(m).n_total());
    InArg<double> e(eta, eta ? M(m).nact : 0);
    const std::vector<int> ids = mesh_mark_cells(M(m), x.dev, eta ? e.dev : nullptr, *policy);
    std::copy(ids.begin(), ids.end(), marked);
    *n_marked = int64_t(ids.size());
  });
}
int cf_mesh_transfer(cf_mesh old_mesh, const double* old_vec, cf_mesh new_mesh, double* new_vec) {
  return guard([&] {
    CHECK_ARG(old_mesh && old_vec && new_mesh && new_vec, "cf_mesh_transfer: null argument");
    InArg<double> x(old_vec, M(old_mesh).n_total());
    OutArg<double> out(new_vec, M(new_mesh).n_total());
    mesh_transfer(M(old_mesh), x.dev, M(new_mesh), out.dev);
    out.finish();
  });
}
int cf_mesh_adaptive_cycle(cf_mesh m, cf_state s, cf_material* mat, const cf_adaptive_options* opts,
                           cf_level_record* records, int max_records, int* n_records) {
  return guard([&] {
    CHECK_ARG(m && s && mat && opts, "cf_mesh_adaptive_cycle: null argument");
    validate_material(*mat);
    CHECK_ARG(s->st.solution.n == M(m).n_total(), "cf_mesh_adaptive_cycle: state of another mesh");
    const std::vector<cf_level_record> r = mesh_adaptive_cycle(M(m), s->st, *mat, *opts);
    if (n_records) *n_records = int(r.size());
    for (int i = 0; i < int(r.size()) && i < max_records && records; ++i) records[i] = r[size_t(i)];
  });
}

}  // extern "C"

// NCCL communicator of the slab-decomposed Newton step (cf_comm.hpp).  NCCL is resolved at run
// time from the process (torch.distributed has normally loaded libnccl.so.2 already, so both use
// the same library instance); a single-GPU run never touches it.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "cf_comm.hpp"

namespace cfb {

namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("NCCL not loadable: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p && err.empty()) err = std::string("NCCL symbol missing: ") + name;
      return p;
    };
#define CFB_SYM(f) api.f = reinterpret_cast<decltype(api.f)>(sym("nccl" #f))
    CFB_SYM(GetUniqueId);
    CFB_SYM(CommInitRank);
    CFB_SYM(CommDestroy);
    CFB_SYM(AllGather);
    CFB_SYM(AllReduce);
    CFB_SYM(Broadcast);
    CFB_SYM(Send);
    CFB_SYM(Recv);
    CFB_SYM(GroupStart);
    CFB_SYM(GroupEnd);
    CFB_SYM(GetErrorString);
#undef CFB_SYM
  });
  if (!err.empty()) fail(CF_ERR_COMM, err);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(CF_ERR_COMM, std::string(what) + ": " + nccl().GetErrorString(r));
}
#define CF_NCCL(x) nccl_check((x), #x)

ncclComm_t H(void* p) { return static_cast<ncclComm_t>(p); }

// out[i] = ((g[0][i] + g[1][i]) + ...) + g[P-1][i]: the same left-to-right sum on every rank
__global__ void k_rank_sum(const double* __restrict__ g, int P, int k, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k) return;
  double s = g[i];
  for (int r = 1; r < P; ++r) s += g[size_t(r) * k + i];
  out[i] = s;
}

}  // namespace

void comm_unique_id(unsigned char out[128]) {
  ncclUniqueId id;
  CF_NCCL(nccl().GetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  std::memcpy(out, &id, 128);
}

std::unique_ptr<Comm> comm_create(const unsigned char id_bytes[128], int rank, int size) {
  if (size < 1 || rank < 0 || rank >= size) fail(CF_ERR_INVALID_ARGUMENT, "comm_create: bad rank / size");
  auto c = std::make_unique<Comm>();
  c->rank = rank;
  c->size = size;
  if (size > 1) {
    ncclUniqueId id;
    std::memcpy(&id, id_bytes, 128);
    ncclComm_t h = nullptr;
    CF_NCCL(nccl().CommInitRank(&h, size, id, rank));
    c->nccl = h;
  }
  return c;
}

// Every NCCL entry point the decomposed step uses, executed on a one-rank communicator on the
// library stream and checked on the host (a single-GPU box cannot run two NCCL ranks, so this is
// what can be exercised there: loading libnccl, the symbol table, the id / init / destroy
// sequence, all-gather in and out of place, int64 sum / max all-reduce, broadcast, grouped
// broadcasts and a grouped send / receive to self).  Returns the number of failed checks.
int comm_selftest() {
  const NcclApi& api = nccl();
  ncclUniqueId id;
  CF_NCCL(api.GetUniqueId(&id));
  ncclComm_t h = nullptr;
  CF_NCCL(api.CommInitRank(&h, 1, id, 0));
  int bad = 0;
  constexpr int K = 1000;
  std::vector<double> a(K), b(K, -1.0);
  for (int i = 0; i < K; ++i) a[i] = 0.5 * i + 0.25;
  DevBuf<double> da(K), db(K), dc(K);
  CF_CUDA(cudaMemcpyAsync(da.p, a.data(), K * sizeof(double), cudaMemcpyHostToDevice, stream()));
  CF_NCCL(api.AllGather(da.p, db.p, size_t(K), ncclFloat64, h, stream()));  // out of place
  CF_NCCL(api.AllGather(db.p, db.p, size_t(K), ncclFloat64, h, stream()));  // in place (rank 0's chunk)
  CF_CUDA(cudaMemcpyAsync(b.data(), db.p, K * sizeof(double), cudaMemcpyDeviceToHost, stream()));
  CF_CUDA(cudaStreamSynchronize(stream()));
  bad += std::memcmp(a.data(), b.data(), K * sizeof(double)) != 0;
  long long iv[3] = {7, -3, 1LL << 40}, io[3] = {0, 0, 0};
  DevBuf<long long> di(3);
  CF_CUDA(cudaMemcpyAsync(di.p, iv, sizeof(iv), cudaMemcpyHostToDevice, stream()));
  CF_NCCL(api.AllReduce(di.p, di.p, 3, ncclInt64, ncclSum, h, stream()));
  CF_NCCL(api.AllReduce(di.p, di.p, 3, ncclInt64, ncclMax, h, stream()));
  CF_CUDA(cudaMemcpyAsync(io, di.p, sizeof(io), cudaMemcpyDeviceToHost, stream()));
  CF_CUDA(cudaStreamSynchronize(stream()));
  bad += std::memcmp(iv, io, sizeof(iv)) != 0;
  CF_NCCL(api.Broadcast(da.p, da.p, K * sizeof(double), ncclUint8, 0, h, stream()));
  CF_NCCL(api.GroupStart());
  CF_NCCL(api.Broadcast(da.p, da.p, K * sizeof(double), ncclUint8, 0, h, stream()));
  CF_NCCL(api.Broadcast(db.p, db.p, K * sizeof(double), ncclUint8, 0, h, stream()));
  CF_NCCL(api.GroupEnd());
  CF_CUDA(cudaMemsetAsync(dc.p, 0, K * sizeof(double), stream()));
  CF_NCCL(api.GroupStart());  // the halo exchange's pattern, with this rank as its own neighbour
  CF_NCCL(api.Send(da.p, K * sizeof(double), ncclUint8, 0, h, stream()));
  CF_NCCL(api.Recv(dc.p, K * sizeof(double), ncclUint8, 0, h, stream()));
  CF_NCCL(api.GroupEnd());
  std::fill(b.begin(), b.end(), -1.0);
  CF_CUDA(cudaMemcpyAsync(b.data(), dc.p, K * sizeof(double), cudaMemcpyDeviceToHost, stream()));
  CF_CUDA(cudaStreamSynchronize(stream()));
  bad += std::memcmp(a.data(), b.data(), K * sizeof(double)) != 0;
  CF_NCCL(api.CommDestroy(h));
  return bad;
}

std::unique_ptr<Comm> comm_create_host(int rank, int size, const cf_host_transport& t) {
  if (size < 1 || rank < 0 || rank >= size) fail(CF_ERR_INVALID_ARGUMENT, "comm_create_host: bad rank / size");
  if (!t.allgather_f64 || !t.allreduce_i64 || !t.sendrecv || !t.bcast)
    fail(CF_ERR_INVALID_ARGUMENT, "comm_create_host: missing callback");
  auto c = std::make_unique<Comm>();
  c->rank = rank;
  c->size = size;
  c->host = true;
  c->ht = t;
  return c;
}

namespace {
void host_check(int rc, const char* what) {
  if (rc != 0) fail(CF_ERR_COMM, std::string("host transport: ") + what + " failed");
}
void d2h(void* h, const void* d, size_t bytes) {
  if (bytes) CF_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, stream()));
}
void h2d(void* d, const void* h, size_t bytes) {
  if (bytes) CF_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, stream()));
}
void sync() { CF_CUDA(cudaStreamSynchronize(stream())); }
}  // namespace

Comm::~Comm() {
  if (nccl) {
    cudaStreamSynchronize(stream());
    ::cfb::nccl().CommDestroy(H(nccl));
  }
}

void Comm::sum_ordered(double* dev, int k) const {
  if (size == 1 || k <= 0) return;
  if (gather.n < i64(size) * k) gather.alloc(i64(size) * k);
  if (host) {
    std::vector<double> mine(static_cast<size_t>(k)), all(static_cast<size_t>(size) * k);
    d2h(mine.data(), dev, size_t(k) * sizeof(double));
    sync();
    host_check(ht.allgather_f64(ht.ctx, mine.data(), all.data(), k), "allgather");
    h2d(gather.p, all.data(), all.size() * sizeof(double));
  } else {
    CF_NCCL(::cfb::nccl().AllGather(dev, gather.p, size_t(k), ncclFloat64, H(nccl), stream()));
  }
  k_rank_sum<<<(k + 127) / 128, 128, 0, stream()>>>(gather.p, size, k, dev);
  CF_LAUNCHED();
}

void Comm::allgather(const double* dev, int k, double* out) const {
  if (k <= 0) return;
  if (size == 1) {
    if (out != dev) CF_CUDA(cudaMemcpyAsync(out, dev, size_t(k) * sizeof(double), cudaMemcpyDeviceToDevice, stream()));
    return;
  }
  if (host) {
    std::vector<double> mine(static_cast<size_t>(k)), all(static_cast<size_t>(size) * k);
    d2h(mine.data(), dev, size_t(k) * sizeof(double));
    sync();
    host_check(ht.allgather_f64(ht.ctx, mine.data(), all.data(), k), "allgather");
    h2d(out, all.data(), all.size() * sizeof(double));
    sync();
    return;
  }
  CF_NCCL(::cfb::nccl().AllGather(dev, out, size_t(k), ncclFloat64, H(nccl), stream()));
}

void Comm::allgather_inplace(double* buf, i64 k) const {
  if (size == 1 || k <= 0) return;
  if (host) {
    std::vector<double> mine(static_cast<size_t>(k)), all(static_cast<size_t>(size) * k);
    d2h(mine.data(), buf + i64(rank) * k, size_t(k) * sizeof(double));
    sync();
    host_check(ht.allgather_f64(ht.ctx, mine.data(), all.data(), int(k)), "allgather");
    h2d(buf, all.data(), all.size() * sizeof(double));
    sync();
    return;
  }
  CF_NCCL(::cfb::nccl().AllGather(buf + i64(rank) * k, buf, size_t(k), ncclFloat64, H(nccl), stream()));
}

void Comm::sum_i64(long long* host, int k) const {
  if (size == 1 || k <= 0) return;
  if (this->host) {
    sync();
    host_check(ht.allreduce_i64(ht.ctx, host, k, 0), "allreduce");
    return;
  }
  if (ibuf.n < k) ibuf.alloc(k);
  CF_CUDA(cudaMemcpyAsync(ibuf.p, host, size_t(k) * sizeof(long long), cudaMemcpyHostToDevice, stream()));
  CF_NCCL(::cfb::nccl().AllReduce(ibuf.p, ibuf.p, size_t(k), ncclInt64, ncclSum, H(nccl), stream()));
  CF_CUDA(cudaMemcpyAsync(host, ibuf.p, size_t(k) * sizeof(long long), cudaMemcpyDeviceToHost, stream()));
  CF_CUDA(cudaStreamSynchronize(stream()));
}

void Comm::max_i64(long long* host, int k) const {
  if (size == 1 || k <= 0) return;
  if (this->host) {
    sync();
    host_check(ht.allreduce_i64(ht.ctx, host, k, 1), "allreduce");
    return;
  }
  if (ibuf.n < k) ibuf.alloc(k);
  CF_CUDA(cudaMemcpyAsync(ibuf.p, host, size_t(k) * sizeof(long long), cudaMemcpyHostToDevice, stream()));
  CF_NCCL(::cfb::nccl().AllReduce(ibuf.p, ibuf.p, size_t(k), ncclInt64, ncclMax, H(nccl), stream()));
  CF_CUDA(cudaMemcpyAsync(host, ibuf.p, size_t(k) * sizeof(long long), cudaMemcpyDeviceToHost, stream()));
  CF_CUDA(cudaStreamSynchronize(stream()));
}

void Comm::sendrecv(const std::vector<HaloOp>& ops) const {
  if (size == 1 || ops.empty()) return;
  if (host) {
    std::vector<std::vector<unsigned char>> sb(ops.size()), rb(ops.size());
    std::vector<const void*> sp(ops.size(), nullptr);
    std::vector<void*> rp(ops.size(), nullptr);
    std::vector<size_t> by(ops.size());
    std::vector<int> pe(ops.size());
    for (size_t i = 0; i < ops.size(); ++i) {
      by[i] = ops[i].bytes;
      pe[i] = ops[i].peer;
      if (ops[i].send) {
        sb[i].resize(ops[i].bytes);
        d2h(sb[i].data(), ops[i].send, ops[i].bytes);
        sp[i] = sb[i].data();
      }
      if (ops[i].recv) {
        rb[i].resize(ops[i].bytes);
        rp[i] = rb[i].data();
      }
    }
    sync();
    host_check(ht.sendrecv(ht.ctx, int(ops.size()), sp.data(), rp.data(), by.data(), pe.data()), "sendrecv");
    for (size_t i = 0; i < ops.size(); ++i)
      if (ops[i].recv) h2d(ops[i].recv, rb[i].data(), ops[i].bytes);
    sync();
    return;
  }
  const NcclApi& api = ::cfb::nccl();
  CF_NCCL(api.GroupStart());
  for (const HaloOp& o : ops) {
    if (o.bytes == 0) continue;
    if (o.send) CF_NCCL(api.Send(o.send, o.bytes, ncclUint8, o.peer, H(nccl), stream()));
    if (o.recv) CF_NCCL(api.Recv(o.recv, o.bytes, ncclUint8, o.peer, H(nccl), stream()));
  }
  CF_NCCL(api.GroupEnd());
}

void Comm::bcast(void* buf, size_t bytes, int root) const {
  if (size == 1 || bytes == 0) return;
  if (host) {
    std::vector<unsigned char> hb(bytes);
    if (rank == root) d2h(hb.data(), buf, bytes);
    sync();
    host_check(ht.bcast(ht.ctx, hb.data(), bytes, root), "bcast");
    if (rank != root) h2d(buf, hb.data(), bytes);
    sync();
    return;
  }
  CF_NCCL(::cfb::nccl().Broadcast(buf, buf, bytes, ncclUint8, root, H(nccl), stream()));
}

void Comm::bcast_many(const std::vector<HaloOp>& ops) const {
  if (size == 1 || ops.empty()) return;
  if (host) {
    for (const HaloOp& o : ops) bcast(o.recv, o.bytes, o.peer);
    return;
  }
  const NcclApi& api = ::cfb::nccl();
  CF_NCCL(api.GroupStart());
  for (const HaloOp& o : ops)
    if (o.bytes) CF_NCCL(api.Broadcast(o.recv, o.recv, o.bytes, ncclUint8, o.peer, H(nccl), stream()));
  CF_NCCL(api.GroupEnd());
}

void Comm::barrier() const {
  if (size == 1) return;
  long long one = 1;
  sum_i64(&one, 1);
}

}  // namespace cfb

// Inter-GPU communicator of the slab-decomposed Newton step: one process per GPU,
// NCCL over NVLink / NVSwitch, every call enqueued on the library stream.  Reductions that feed
// control flow or Krylov coefficients are rank-ordered (all-gather of the per-rank partials, then
// the same left-to-right sum on every rank), so all ranks hold bitwise identical scalars and a
// run is reproducible for a fixed rank count.
#pragma once

#include <vector>

#include "cf_types.hpp"

namespace cfb {

struct HaloOp {
  const void* send;  // bytes sent to peer (nullptr: receive only)
  void* recv;        // bytes received from peer (nullptr: send only)
  size_t bytes;
  int peer;
};

struct Comm {
  int rank = 0, size = 1;
  void* nccl = nullptr;  // ncclComm_t
  bool host = false;     // host-staged test transport (cf_host_transport) instead of NCCL
  cf_host_transport ht{};
  mutable DevBuf<double> gather;
  mutable DevBuf<long long> ibuf;
  ~Comm();
  bool distributed() const { return size > 1; }
  // dev[0..k) := sum over ranks (rank order) of every rank's dev[0..k)
  void sum_ordered(double* dev, int k) const;
  // out[r*k .. (r+1)*k) := rank r's dev[0..k) (out: size*k device doubles)
  void allgather(const double* dev, int k, double* out) const;
  // buf[r*k .. (r+1)*k) := rank r's own chunk of buf, in place (buf: size*k device doubles)
  void allgather_inplace(double* buf, i64 k) const;
  // exact integer sums / maxima of host values
  void sum_i64(long long* host, int k) const;
  void max_i64(long long* host, int k) const;
  // grouped point-to-point transfers (halo planes)
  void sendrecv(const std::vector<HaloOp>& ops) const;
  // in-place broadcast of bytes [buf, buf + bytes) from root; bcast_many: one NCCL group
  void bcast(void* buf, size_t bytes, int root) const;
  void bcast_many(const std::vector<HaloOp>& ops) const;  // op.recv = buffer, op.peer = root
  void barrier() const;
};

void comm_unique_id(unsigned char out[128]);
int comm_selftest();  // every NCCL entry point on a one-rank communicator; failed checks
std::unique_ptr<Comm> comm_create(const unsigned char id[128], int rank, int size);
std::unique_ptr<Comm> comm_create_host(int rank, int size, const cf_host_transport& t);

}  // namespace cfb

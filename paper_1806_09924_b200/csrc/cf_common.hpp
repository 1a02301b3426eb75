// Shared runtime pieces of the crackfield_b200 library: errors, the library stream, a
// stream-ordered device buffer and launch accounting.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>

#include "crackfield_b200.h"

namespace cfb {

using i64 = std::int64_t;

// Exception carrying a CF_ERR_* code; converted to a status at the C ABI.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    char buf[512];
    std::snprintf(buf, sizeof(buf), "%s: %s (%s:%d)", what, cudaGetErrorString(e), file, line);
    fail(e == cudaErrorMemoryAllocation ? CF_ERR_OUT_OF_MEMORY : CF_ERR_CUDA, buf);
  }
}
#define CF_CUDA(x) ::cfb::cuda_check((x), #x, __FILE__, __LINE__)

// Library-wide state: the stream all device work is ordered on, the device's SM count and the
// kernel-launch counter (bench.py's gpu_launches).
struct Runtime {
  cudaStream_t stream = nullptr;
  int device = -1;
  int sm_count = 0;
  i64 launches = 0;
  bool ready = false;
  // a second stream for independent work forked from and joined back into `stream` by events
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};
Runtime& rt();
void ensure_device();  // throws CF_ERR_CUDA when no device is usable (no CPU fallback)
inline cudaStream_t stream() { return rt().stream; }
// Enqueue f's kernels on the auxiliary stream, forked from the library stream at this point (f
// must not allocate: the caching allocator relies on one stream order); aux_join() makes the
// library stream wait for them.  Independent outputs only: the results are those of running f
// in sequence.
template <class F>
void on_aux(F&& f) {
  Runtime& R = rt();
  if (!R.aux) {
    CF_CUDA(cudaStreamCreateWithFlags(&R.aux, cudaStreamNonBlocking));
    CF_CUDA(cudaEventCreateWithFlags(&R.ev_fork, cudaEventDisableTiming));
    CF_CUDA(cudaEventCreateWithFlags(&R.ev_join, cudaEventDisableTiming));
  }
  const cudaStream_t main = R.stream;
  CF_CUDA(cudaEventRecord(R.ev_fork, main));
  CF_CUDA(cudaStreamWaitEvent(R.aux, R.ev_fork, 0));
  R.stream = R.aux;
  try {
    f();
  } catch (...) {
    R.stream = main;
    throw;
  }
  R.stream = main;
  CF_CUDA(cudaEventRecord(R.ev_join, R.aux));
}
inline void aux_join() { CF_CUDA(cudaStreamWaitEvent(rt().stream, rt().ev_join, 0)); }

// host round trips of the library stream (diagnostics: CF_TIMING prints them per AMG build)
inline long& host_sync_count() {
  static long n = 0;
  return n;
}
// Small device -> host read, ordered on the library stream and complete on return: the bytes go
// through a pinned staging slot (a pageable destination makes the driver stage and block inside
// cudaMemcpyAsync, about twice the latency of a pinned copy + stream sync).  Counts one host sync.
void read_small(void* dst, const void* src, size_t bytes);
inline void count_launch(i64 n = 1) { rt().launches += n; }
#define CF_LAUNCHED() ::cfb::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__), ::cfb::count_launch()

// Caching device allocator: freed blocks are kept in a best-fit free list and reused in stream
// order (all library work is ordered on one stream, so a block freed by an earlier operation is
// safe to hand to a later one).  Per-Newton-iteration reallocation of multi-GB buffers (J, AMG
// temporaries, Krylov basis) then costs nothing; cached blocks are released only on OOM.
void* dev_alloc(size_t bytes);
void dev_free(void* p, size_t bytes);
size_t dev_cached_bytes();

template <class T>
struct DevBuf {
  T* p = nullptr;
  i64 n = 0;
  DevBuf() = default;
  explicit DevBuf(i64 count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(i64 count) {
    release();
    n = count;
    if (count > 0) p = static_cast<T*>(dev_alloc(size_t(count) * sizeof(T)));
  }
  void release() {
    if (p) dev_free(p, size_t(n) * sizeof(T));
    p = nullptr;
    n = 0;
  }
  void zero() {
    if (n) CF_CUDA(cudaMemsetAsync(p, 0, size_t(n) * sizeof(T), stream()));
  }
  T* get() const { return p; }
  i64 size() const { return n; }
};

// Host-or-device argument staging for the ABI: device pointers pass through, host arrays are
// copied in (and, for outputs, back out at the end of the call).
bool is_device_ptr(const void* p);

template <class T>
struct InArg {
  const T* dev = nullptr;
  DevBuf<T> staged;
  InArg(const T* p, i64 n) {
    if (n == 0 || p == nullptr) { dev = p; return; }
    if (is_device_ptr(p)) { dev = p; return; }
    staged.alloc(n);
    CF_CUDA(cudaMemcpyAsync(staged.p, p, size_t(n) * sizeof(T), cudaMemcpyHostToDevice, stream()));
    dev = staged.p;
  }
};

template <class T>
struct OutArg {
  T* host = nullptr;
  T* dev = nullptr;
  i64 n = 0;
  DevBuf<T> staged;
  OutArg(T* p, i64 count, bool copy_in = false) : n(count) {
    if (count == 0 || p == nullptr) { dev = p; return; }
    if (is_device_ptr(p)) { dev = p; return; }
    host = p;
    staged.alloc(count);
    dev = staged.p;
    if (copy_in) CF_CUDA(cudaMemcpyAsync(dev, p, size_t(count) * sizeof(T), cudaMemcpyHostToDevice, stream()));
  }
  // copy back (synchronous) when the caller passed host memory
  void finish() {
    if (host) {
      CF_CUDA(cudaMemcpyAsync(host, dev, size_t(n) * sizeof(T), cudaMemcpyDeviceToHost, stream()));
      CF_CUDA(cudaStreamSynchronize(stream()));
    }
  }
};

// at least one block, so empty inputs launch a no-op grid instead of an invalid configuration
inline unsigned grid_for(i64 n, int block) { return unsigned(n > 0 ? (n + block - 1) / block : 1); }

}  // namespace cfb

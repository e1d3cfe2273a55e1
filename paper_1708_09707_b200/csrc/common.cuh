// common.cuh -- error handling, device buffers and small device helpers.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <memory>
#include <cstdint>
#include <new>
#include <thread>
#include <vector>
#include <stdexcept>
#include <string>
#include <utility>

namespace hmb {

// Status codes of the C ABI (include/hmat_b200.h); thrown internally and mapped
// at the boundary like the reference's exception kinds.
enum Status : int {
  kOk = 0,
  kEinval = 1,      // std::invalid_argument
  kErange = 2,      // std::out_of_range
  kEnomem = 3,      // allocation failure (device or host)
  kEcuda = 4,       // CUDA runtime error
  kEnccl = 5,       // NCCL error
  kEnonfinite = 6,  // non-finite value (cg_solve, solver.cpp:51-54)
  kElogic = 7,      // std::logic_error / internal invariant
  kEio = 8,         // std::runtime_error from file output
};

struct Error : std::runtime_error {
  Status status;
  Error(Status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void raise(Status s, const std::string& m) { throw Error(s, m); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    const Status s = (e == cudaErrorMemoryAllocation) ? kEnomem : kEcuda;
    raise(s, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" + std::to_string(line) + ")");
  }
}
#define HM_CUDA(x) ::hmb::cuda_check((x), #x, __FILE__, __LINE__)
#define HM_LAUNCH_CHECK() ::hmb::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

// Owning device allocation (cudaMallocAsync on the handle's stream).
template <class T>
class DevBuf {
 public:
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept { swap(o); }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      reset();
      swap(o);
    }
    return *this;
  }
  ~DevBuf() { reset(); }

  // Large buffers (the stored operator: tens of GB) bypass the stream-ordered pool:
  // measured on B200, cudaMallocAsync of 64 GB takes ~2 s and its free 2-9 s, while
  // cudaMalloc maps the same in ~6 ms.  cudaFree synchronises the device, so a large
  // buffer is never released under in-flight work.
  static constexpr size_t kDirectBytes = size_t(256) << 20;
  void alloc(size_t count, cudaStream_t s) {
    reset();
    stream_ = s;
    n_ = count;
    direct_ = count * sizeof(T) >= kDirectBytes;
    if (!count) return;
    if (direct_) HM_CUDA(cudaMalloc(reinterpret_cast<void**>(&p_), count * sizeof(T)));
    else HM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p_), count * sizeof(T), s));
  }
  void reset() {
    if (p_) {
      if (direct_) cudaFree(p_);
      else cudaFreeAsync(p_, stream_);
    }
    p_ = nullptr;
    n_ = 0;
    direct_ = false;
  }
  void zero(cudaStream_t s) {
    if (n_) HM_CUDA(cudaMemsetAsync(p_, 0, n_ * sizeof(T), s));
  }
  void fill_bytes(int v, cudaStream_t s) {
    if (n_) HM_CUDA(cudaMemsetAsync(p_, v, n_ * sizeof(T), s));
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }
  size_t bytes() const { return n_ * sizeof(T); }

 private:
  void swap(DevBuf& o) {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    std::swap(stream_, o.stream_);
    std::swap(direct_, o.direct_);
  }
  T* p_ = nullptr;
  size_t n_ = 0;
  cudaStream_t stream_ = nullptr;
  bool direct_ = false;
};

// Host mirrors of device arrays: default-initialising resize (no serial zero-fill of
// hundreds of MB before the copy overwrites them).  Pageable on purpose: measured at
// config-4 geometry, page-locking the 2-4 GB of mirrors costs more than it saves on the
// device-to-host copies.
template <class T>
struct DefaultInitAlloc : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = DefaultInitAlloc<U>;
  };
  DefaultInitAlloc() = default;
  template <class U>
  DefaultInitAlloc(const DefaultInitAlloc<U>&) {}
  template <class U, class... A>
  void construct(U* p, A&&... a) {
    if constexpr (sizeof...(A) == 0) ::new (static_cast<void*>(p)) U;  // default-init: no zeroing
    else ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
  }
};
template <class T>
using HostVec = std::vector<T, DefaultInitAlloc<T>>;

// f(begin, end) over [0, n) in contiguous blocks on up to `threads` host threads
template <class F>
void parallel_blocks(long long n, F&& f, int threads = 16) {
  if (n <= 0) return;
  const long long nt = std::max<long long>(1, std::min<long long>(threads, n / 65536 + 1));
  if (nt == 1) {
    f(0ll, n);
    return;
  }
  std::vector<std::thread> pool;
  const long long per = (n + nt - 1) / nt;
  for (long long t = 1; t < nt; ++t) {
    const long long b = t * per, e = std::min(n, b + per);
    if (b < e) pool.emplace_back([&f, b, e] { f(b, e); });
  }
  f(0ll, std::min(n, per));
  for (auto& th : pool) th.join();
}

// f(task) for task in [0, n), one host thread per task (coarse tasks, n small)
template <class F>
void parallel_tasks(int n, F&& f) {
  std::vector<std::thread> pool;
  for (int q = 1; q < n; ++q) pool.emplace_back([&f, q] { f(q); });
  if (n > 0) f(0);
  for (auto& th : pool) th.join();
}

inline unsigned grid_for(long long n, int threads, long long cap = 1ll << 30) {
  long long g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<unsigned>(g);
}

}  // namespace hmb

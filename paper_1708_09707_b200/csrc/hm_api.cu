// hm_api.cu -- the C ABI (include/hmat_b200.h): host orchestration in C++,
// exceptions mapped to hm_status at the boundary.

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <atomic>
#include <type_traits>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/hmat_b200.h"
#include "hmatrix.h"
#include "nccl_shim.h"
#include "primitives.h"

namespace hmb {
void plan_far_field(HMatrix& h, cudaStream_t s);
}

using namespace hmb;

struct hm_handle {
  HMatrix h;
  std::mutex mu;
  ncclComm_t comm = nullptr;
  std::vector<long long> rank_bounds;  // Morton row slice [b[r], b[r+1]) of every rank
  bool equal_slices = false;           // all slices the same size: one ncclAllGather
  // pinned staging of hm_mvp's host vectors (H2D / D2H at full PCIe rate)
  double* pin_x = nullptr;
  double* pin_z = nullptr;
  // CG scalars read back once per iteration
  double* pin_scal = nullptr;
  size_t pin_scal_n = 0;
  ~hm_handle() {
    if (comm) hmb::NcclApi::get().CommDestroy(comm);
    if (pin_x) cudaFreeHost(pin_x);
    if (pin_z) cudaFreeHost(pin_z);
    if (pin_scal) cudaFreeHost(pin_scal);
  }
};

namespace {

thread_local std::string g_err;

template <class F>
hm_status guarded(F&& f) {
  try {
    f();
    return HM_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return static_cast<hm_status>(e.status);
  } catch (const std::bad_alloc& e) {
    g_err = "host allocation failed";
    return HM_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HM_ELOGIC;
  } catch (...) {
    g_err = "unknown exception";
    return HM_ELOGIC;
  }
}

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t) { return std::chrono::duration<double, std::milli>(Clock::now() - t).count(); }

KernelParams make_kernel(int kind, double beta, int d) {
  KernelParams kp{kind, d, 0.0};
  if (kind == kMatern) {
    // effective_beta + matern_normalization (core.cpp:83-95), glibc pow/tgamma on the host
    const double b = beta > 0.0 ? beta : 1.0 + 0.5 * d;
    const double order = b - 0.5 * d;
    if (std::fabs(order - 1.0) > 1e-12)
      raise(kEinval, "Matern kernel: only order beta - d/2 = 1 is supported, got beta = " + std::to_string(b) +
                         " at d = " + std::to_string(d));
    kp.matern_norm = 1.0 / (std::pow(2.0, b - 1.0) * std::tgamma(b));
  } else if (kind != kGaussian) {
    raise(kEinval, "unknown kernel kind");
  }
  return kp;
}

Config to_config(const hm_config* c) {
  hm_config def;
  hm_config_default(&def);
  if (!c) c = &def;
  // validate (hmatrix.cpp:20-26)
  if (c->eta < 0.0) raise(kEinval, "HmatrixConfig: eta must be >= 0");
  if (c->c_leaf < 1) raise(kEinval, "HmatrixConfig: c_leaf must be >= 1");
  if (c->k < 1) raise(kEinval, "HmatrixConfig: k must be >= 1");
  if (c->k > 32) raise(kEinval, "HmatrixConfig: k > 32 is not supported on the device");
  if (c->bs_aca < 0 || c->bs_dense < 0) raise(kEinval, "HmatrixConfig: batch sizes must be >= 0");
  if (c->has_epsilon && c->epsilon <= 0.0) raise(kEinval, "HmatrixConfig: epsilon must be > 0");
  if (c->adm_mode < 0 || c->adm_mode > 2) raise(kEinval, "HmatrixConfig: bad admissibility mode");
  if (c->world < 1 || c->rank < 0 || c->rank >= c->world) raise(kEinval, "HmatrixConfig: bad rank/world");
  Config cfg;
  cfg.eta = c->eta;
  cfg.c_leaf = c->c_leaf;
  cfg.k = c->k;
  cfg.bs_aca = c->bs_aca;
  cfg.bs_dense = c->bs_dense;
  cfg.precompute_aca = c->precompute_aca != 0;
  cfg.has_epsilon = c->has_epsilon != 0;
  cfg.epsilon = c->epsilon;
  cfg.mode = c->adm_mode;
  cfg.near_stored = c->near_stored ? 1 : 0;
  cfg.rank = c->rank;
  cfg.world = c->world;
  cfg.aca_chunk_rows = c->aca_chunk_rows;
  return cfg;
}

void require_device() {
  int nd = 0;
  if (cudaGetDeviceCount(&nd) != cudaSuccess || nd == 0) raise(kEcuda, "no CUDA device available");
}

void setup_common(hm_handle* H, const double* coords_dev, long long n, int d) {
  HMatrix& h = H->h;
  const auto t0 = Clock::now();
  build_hmatrix(h, coords_dev);
  // partition_dense_queue throws when one block exceeds a positive bs_dense (dense_blocks.cpp:44-46)
  if (h.cfg.bs_dense > 0) {
    for (long long b = 0; b < h.dense.count; ++b)
      if (static_cast<long long>(h.dense.h_m[b]) * h.dense.h_n[b] > h.cfg.bs_dense)
        raise(kEinval, "partition_dense_queue: a single block exceeds bs_dense");
  }
  h.xm.alloc(n + 16, h.stream);  // padded: bulk copies round x segments up to 16 bytes
  h.xm.zero(h.stream);
  h.zm.alloc(n, h.stream);
  h.zm.zero(h.stream);
  const auto ta = Clock::now();
  plan_far_field(h, h.stream);
  HM_CUDA(cudaStreamSynchronize(h.stream));
  h.tm.aca_ms = ms_since(ta);
  const auto tn = Clock::now();
  if (h.cfg.near_stored) store_near_field(h, h.stream);
  else plan_near_pairs(h, h.stream);
  HM_CUDA(cudaStreamSynchronize(h.stream));
  h.tm.near_ms = ms_since(tn);
  h.tm.setup_ms = ms_since(t0);
  (void)d;
}

hm_handle* new_handle(const hm_config* cfg, long long n, int d, int kernel, double beta) {
  require_device();
  // validate everything before any CUDA object exists
  const Config c = to_config(cfg);
  if (n < 1) raise(kEinval, "build_block_cluster_tree: empty point set");
  if (d < 1 || d > 20) raise(kEinval, "dimension must be in [1, 20]");
  const KernelParams kp = make_kernel(kernel, beta, d);
  auto H = std::make_unique<hm_handle>();
  H->h.cfg = c;
  H->h.kp = kp;
  H->h.n = n;
  H->h.d = d;
  H->h.create(cfg ? cfg->device : 0);  // streams + events, released by ~HandleStreams
  return H.release();
}

// host pointer in page-locked memory (DMA-able without staging)?
bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// dst <- src (host memory) with up to 4 threads over 1 MB chunks; after each chunk is in
// place, on_chunk(offset, length) is called from the calling thread in order (used to
// queue the chunk's DMA while later chunks are still being copied).
template <class F>
void staged_copy(void* dst, const void* src, size_t bytes, F&& on_chunk) {
  constexpr size_t kChunk = size_t(1) << 20;
  const size_t nchunks = (bytes + kChunk - 1) / kChunk;
  auto copy = [&](size_t c) {
    const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
    std::memcpy(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, len);
  };
  constexpr bool kNotify = !std::is_same<std::decay_t<F>, std::nullptr_t>::value;
  if (nchunks <= 2) {
    for (size_t c = 0; c < nchunks; ++c) {
      copy(c);
      if constexpr (kNotify) on_chunk(c * kChunk, std::min(kChunk, bytes - c * kChunk));
    }
    return;
  }
  const unsigned nthr = 4;
  std::atomic<size_t> next{0};
  std::vector<std::atomic<int>> done(nchunks);
  for (auto& d : done) d.store(0, std::memory_order_relaxed);
  auto worker = [&] {
    for (size_t c; (c = next.fetch_add(1)) < nchunks;) {
      copy(c);
      done[c].store(1, std::memory_order_release);
    }
  };
  std::vector<std::thread> pool;
  for (unsigned i = 1; i < nthr; ++i) pool.emplace_back(worker);
  worker();
  if constexpr (kNotify) {
    for (size_t c = 0; c < nchunks; ++c) {
      while (!done[c].load(std::memory_order_acquire)) std::this_thread::yield();
      on_chunk(c * kChunk, std::min(kChunk, bytes - c * kChunk));
    }
  }
  for (auto& th : pool) th.join();
}

// Runs f(stream) on the handle's stream, ordered after the work already queued on
// `caller` and with `caller` ordered after it (event fork/join: capture-safe, so the
// call can be recorded into a CUDA graph on the caller's stream).  All handle work and
// all workspace allocations stay on h.stream, so products issued from different
// caller streams are serialised on the device, not just on the host mutex.
template <class F>
void on_handle_stream(HMatrix& h, cudaStream_t caller, F&& f) {
  if (caller == h.stream) {
    f(h.stream);
    return;
  }
  if (caller == nullptr) caller = cudaStreamLegacy;  // CUDA convention: 0 = the legacy default stream
  HM_CUDA(cudaEventRecord(h.ev_join, caller));
  HM_CUDA(cudaStreamWaitEvent(h.stream, h.ev_join, 0));
  f(h.stream);
  HM_CUDA(cudaEventRecord(h.ev_last, h.stream));
  HM_CUDA(cudaStreamWaitEvent(caller, h.ev_last, 0));
}

// ---------------------------------------------------------------- small kernels
__global__ void eval_pairs_kernel(KernelParams kp, int d, long long n, const double* y, const double* yp,
                                  double* out) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    double r2 = 0.0;
    for (int a = 0; a < d; ++a) {
      const double dx = hsub(y[a * n + i], yp[a * n + i]);
      r2 = hadd(r2, hmul(dx, dx));
    }
    out[i] = phi_r2(kp, r2);
  }
}

__global__ void exp_port_kernel(long long n, const double* x, double* out, int which) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    out[i] = which == 0 ? glibc_exp(x[i]) : glibc_log(x[i]);
}

// exact product, one thread per Morton row, acc += phi(i,j) * x_m[j] sequentially
// (relative_error hmatrix.cpp:136-143 and oracle.cpp:41-49 order)
__global__ void dense_exact_kernel(const double* __restrict__ coords, long long n, int d, KernelParams kp,
                                   const double* __restrict__ xm, long long row_begin, long long row_end,
                                   double* __restrict__ zm) {
  const long long i = row_begin + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= row_end) return;
  double yi[20];
  for (int a = 0; a < d; ++a) yi[a] = coords[a * n + i];
  double acc = 0.0;
  for (long long j = 0; j < n; ++j) {
    double r2 = 0.0;
    for (int a = 0; a < d; ++a) {
      const double dx = hsub(yi[a], __ldg(coords + a * n + j));
      r2 = hadd(r2, hmul(dx, dx));
    }
    acc = hadd(acc, hmul(phi_r2(kp, r2), __ldg(xm + j)));
  }
  zm[i] = acc;
}

__global__ void gather_kernel(const double* __restrict__ x, const long long* __restrict__ perm, long long n,
                              double* __restrict__ xm) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    xm[i] = x[perm[i]];
}
__global__ void scatter_kernel(const double* __restrict__ zm, const long long* __restrict__ perm, long long n,
                               double* __restrict__ z) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    z[perm[i]] = zm[i];
}

// ---------------------------------------------------------------- CG on the device
// R columns (column r at base + r*n).  Scalars stay on the device; the host reads them
// once per iteration (the stopping rule).  Dots are fixed-order (per-block tree
// partials folded in block order), so every run gives the same bits.
constexpr int kDotBlocks = 296;  // 2 x 148 SMs per column

__global__ void dots_partial_kernel(const double* a, const double* b, long long n, double* part) {
  __shared__ double sm[256];
  const long long off = static_cast<long long>(blockIdx.y) * n;
  double acc = 0.0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    acc = hadd(acc, hmul(a[off + i], b[off + i]));
  sm[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s; s >>= 1) {
    if (threadIdx.x < s) sm[threadIdx.x] = hadd(sm[threadIdx.x], sm[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[static_cast<long long>(blockIdx.y) * gridDim.x + blockIdx.x] = sm[0];
}
// out[r] = fold of column r's partials; op 0: store, 1: alpha = rs / out (active columns),
// 2: beta = out / rs, rs = out
__global__ void dots_final_kernel(const double* part, int nb, int R, double* out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  double acc = 0.0;
  for (int i = 0; i < nb; ++i) acc = hadd(acc, part[static_cast<long long>(r) * nb + i]);
  out[r] = acc;
}
__global__ void cg_alpha_kernel(const double* rs, const double* pap, const int* active, double* alpha, int R) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < R) alpha[r] = active[r] ? __ddiv_rn(rs[r], pap[r]) : 0.0;
}
__global__ void cg_beta_kernel(double* rs, const double* rs_next, const int* active, double* beta, int R) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < R && active[r]) {
    beta[r] = __ddiv_rn(rs_next[r], rs[r]);
    rs[r] = rs_next[r];
  }
}
// CG vector updates (solver.cpp:27-31, 46-49, 59-61), column r = blockIdx.y
__global__ void axpy_sigma_kernel(double* ap, const double* p, double sigma2, long long n) {
  const long long off = static_cast<long long>(blockIdx.y) * n;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    ap[off + i] = hadd(ap[off + i], hmul(sigma2, p[off + i]));
}
__global__ void cg_update_kernel(double* x, double* r, const double* p, const double* ap, const double* alpha,
                                 const int* active, long long n) {
  if (!active[blockIdx.y]) return;
  const double al = alpha[blockIdx.y];
  const long long off = static_cast<long long>(blockIdx.y) * n;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    x[off + i] = hadd(x[off + i], hmul(al, p[off + i]));
    r[off + i] = hsub(r[off + i], hmul(al, ap[off + i]));
  }
}
__global__ void cg_dir_kernel(double* p, const double* r, const double* beta, const int* active, long long n) {
  if (!active[blockIdx.y]) return;
  const double be = beta[blockIdx.y];
  const long long off = static_cast<long long>(blockIdx.y) * n;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    p[off + i] = hadd(r[off + i], hmul(be, p[off + i]));
}
__global__ void sub_kernel(double* d, const double* b, long long total) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    d[i] = hsub(b[i], d[i]);
}

// out[r] = a_r . b_r for R columns (device result)
void device_dots(const double* a, const double* b, long long n, int R, DevBuf<double>& part, double* out,
                 cudaStream_t s) {
  if (part.size() < static_cast<size_t>(kDotBlocks) * R) part.alloc(static_cast<size_t>(kDotBlocks) * R, s);
  dots_partial_kernel<<<dim3(kDotBlocks, R), 256, 0, s>>>(a, b, n, part.get());
  dots_final_kernel<<<(R + 31) / 32, 32, 0, s>>>(part.get(), kDotBlocks, R, out);
  HM_LAUNCH_CHECK();
}

// y allgather: rank r's Morton rows [b[r], b[r+1]) of y are gathered in
// place on every rank.  Equal slices (power-of-two N, the bench configurations): one
// in-place ncclAllGather; otherwise grouped in-place broadcasts (ceil-split slices).
void allgather_y(hm_handle* H, double* y, cudaStream_t s) {
  HMatrix& h = H->h;
  if (!H->comm) raise(kEnccl, "world > 1 but no NCCL communicator attached (hm_attach_nccl)");
  const std::vector<long long>& bounds = H->rank_bounds;
  const NcclApi& nc = NcclApi::get();
  if (H->equal_slices) {
    const size_t cnt = static_cast<size_t>(bounds[1] - bounds[0]);
    if (nc.AllGather(y + bounds[h.cfg.rank], y, cnt, ncclDouble, H->comm, s) != ncclSuccess)
      raise(kEnccl, "ncclAllGather of the y slices failed");
    return;
  }
  if (nc.GroupStart() != ncclSuccess) raise(kEnccl, "ncclGroupStart");
  for (int r = 0; r < h.cfg.world; ++r) {
    double* p = y + bounds[r];
    if (nc.Broadcast(p, p, static_cast<size_t>(bounds[r + 1] - bounds[r]), ncclDouble, r, H->comm, s) != ncclSuccess)
      raise(kEnccl, "ncclBroadcast of the y slice failed");
  }
  if (nc.GroupEnd() != ncclSuccess) raise(kEnccl, "ncclGroupEnd");
}

// z (original order, device) = H x, with the row-sliced allgather when world > 1
void product(hm_handle* H, const double* x_dev, double* z_dev, cudaStream_t s) {
  HMatrix& h = H->h;
  const long long n = h.n;
  h.clk.start(kKGather, s);
  gather_kernel<<<grid_for(n, 256, 1 << 16), 256, 0, s>>>(x_dev, h.perm.get(), n, h.xm.get());
  HM_LAUNCH_CHECK();
  h.clk.stop(kKGather, s);
  mvp_morton(h, s);
  if (h.cfg.world > 1) {
    h.clk.start(kKAllgather, s);
    allgather_y(H, h.zm.get(), s);
    h.clk.stop(kKAllgather, s);
  }
  h.clk.start(kKScatter, s);
  scatter_kernel<<<grid_for(n, 256, 1 << 16), 256, 0, s>>>(h.zm.get(), h.perm.get(), n, z_dev);
  HM_LAUNCH_CHECK();
  h.clk.stop(kKScatter, s);
}

// R right-hand sides per pass (multi.cu); X, Z rhs-major device arrays (original order)
void product_multi(hm_handle* H, const double* X_dev, double* Z_dev, int R, int flags, cudaStream_t s) {
  HMatrix& h = H->h;
  const long long n = h.n;
  ensure_multi(h, R, s);
  gather_multi(h, X_dev, n, R, s);
  mvp_multi_morton(h, R, flags, s);
  if (h.cfg.world > 1)
    for (int r = 0; r < R; ++r) allgather_y(H, h.zmR.get() + static_cast<long long>(r) * n, s);
  scatter_multi(h, Z_dev, n, R, s);
}

// nrhs in passes of at most 16
void product_multi_all(hm_handle* H, const double* X_dev, double* Z_dev, long long nrhs, int flags, cudaStream_t s) {
  const long long n = H->h.n;
  if (H->h.tma_rows && !(flags & 1)) {
    // stored operator on the TMA product: it runs at the HBM roofline per vector, faster
    // than the generic multi-RHS kernels (measured: 16 x 10 ms vs 237 ms at C2); same bits
    for (long long r = 0; r < nrhs; ++r) product(H, X_dev + r * n, Z_dev + r * n, s);
    return;
  }
  for (long long r0 = 0; r0 < nrhs; r0 += 16) {
    const int R = static_cast<int>(std::min<long long>(16, nrhs - r0));
    product_multi(H, X_dev + r0 * n, Z_dev + r0 * n, R, flags, s);
  }
}

}  // namespace

extern "C" {

const char* hm_last_error(void) { return g_err.c_str(); }

void hm_config_default(hm_config* c) {
  std::memset(c, 0, sizeof(*c));
  c->eta = 1.5;
  c->c_leaf = 256;
  c->k = 16;
  c->bs_aca = 1ll << 20;
  c->bs_dense = 1ll << 22;
  c->world = 1;
}

int hm_device_count(void) {
  int nd = 0;
  if (cudaGetDeviceCount(&nd) != cudaSuccess) return 0;
  return nd;
}

hm_status hm_setup(const double* coords, int64_t n, int32_t d, int32_t kernel, double beta, const hm_config* cfg,
                   hm_handle** out) {
  if (!out) {
    g_err = "hm_setup: null output handle";
    return HM_EINVAL;
  }
  *out = nullptr;
  std::unique_ptr<hm_handle> H;
  const hm_status st = guarded([&] {
    if (!coords) raise(kEinval, "coords is null");
    H.reset(new_handle(cfg, n, d, kernel, beta));
    DevBuf<double> c;
    c.alloc(static_cast<size_t>(n) * d, H->h.stream);
    HM_CUDA(cudaMemcpyAsync(c.get(), coords, sizeof(double) * n * d, cudaMemcpyHostToDevice, H->h.stream));
    setup_common(H.get(), c.get(), n, d);
  });
  if (st == HM_OK) *out = H.release();
  return st;
}

hm_status hm_setup_device(const double* coords_dev, int64_t n, int32_t d, int32_t kernel, double beta,
                          const hm_config* cfg, hm_handle** out) {
  if (!out) {
    g_err = "hm_setup_device: null output handle";
    return HM_EINVAL;
  }
  *out = nullptr;
  std::unique_ptr<hm_handle> H;
  const hm_status st = guarded([&] {
    if (!coords_dev) raise(kEinval, "coords is null");
    H.reset(new_handle(cfg, n, d, kernel, beta));
    setup_common(H.get(), coords_dev, n, d);
  });
  if (st == HM_OK) *out = H.release();
  return st;
}

void hm_destroy(hm_handle* H) {
  if (!H) return;
  {
    std::lock_guard<std::mutex> lock(H->mu);  // no call on this handle is in flight
  }
  delete H;  // ~hm_handle: NCCL comm, pinned staging; ~HandleStreams syncs, then destroys streams
}

hm_status hm_mvp(hm_handle* H, const double* x, double* z, hm_timings* t) {
  return guarded([&] {
    if (!H || !x || !z) raise(kEinval, "mvp: null argument");
    std::lock_guard<std::mutex> lock(H->mu);
    HMatrix& h = H->h;
    HM_CUDA(cudaSetDevice(h.device));
    const auto t0 = Clock::now();
    cudaStream_t s = h.stream;
    const size_t bytes = sizeof(double) * h.n;
    if (h.xin.size() < static_cast<size_t>(h.n)) h.xin.alloc(h.n, s);
    if (h.zout.size() < static_cast<size_t>(h.n)) h.zout.alloc(h.n, s);
    // pinned staging: the copies run at full link rate (pageable copies are bounced
    // through a driver buffer at a fraction of it)
    if (!H->pin_x && !is_pinned(x)) HM_CUDA(cudaMallocHost(reinterpret_cast<void**>(&H->pin_x), bytes));
    if (!H->pin_z && !is_pinned(z)) HM_CUDA(cudaMallocHost(reinterpret_cast<void**>(&H->pin_z), bytes));
    // page-locked caller buffers (cudaHostAlloc / cudaHostRegister) are transferred
    // directly; pageable ones go through the handle's pinned staging
    const bool x_pinned = is_pinned(x), z_pinned = is_pinned(z);
    if (x_pinned) {
      HM_CUDA(cudaMemcpyAsync(h.xin.get(), x, bytes, cudaMemcpyHostToDevice, s));
    } else {
      // host copies into the pinned staging run on a few threads, chunk by chunk, and each
      // chunk's DMA is queued as soon as it is staged (copy and transfer overlap)
      staged_copy(H->pin_x, x, bytes, [&](size_t off, size_t len) {
        HM_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(h.xin.get()) + off, reinterpret_cast<char*>(H->pin_x) + off,
                                len, cudaMemcpyHostToDevice, s));
      });
    }
    h.phase_events = true;
    try {
      product(H, h.xin.get(), h.zout.get(), s);
    } catch (...) {
      h.phase_events = false;
      throw;
    }
    h.phase_events = false;
    if (z_pinned) {
      HM_CUDA(cudaMemcpyAsync(z, h.zout.get(), bytes, cudaMemcpyDeviceToHost, s));
      HM_CUDA(cudaStreamSynchronize(s));
    } else {
      HM_CUDA(cudaMemcpyAsync(H->pin_z, h.zout.get(), bytes, cudaMemcpyDeviceToHost, s));
      HM_CUDA(cudaStreamSynchronize(s));
      staged_copy(z, H->pin_z, bytes, nullptr);
    }
    h.tm.mvp_ms = ms_since(t0);
    // MvpTimings (hmatrix.cpp:117-121): dense (near-field) and ACA (far-field) phases
    float dms = 0.f, ams = 0.f;
    HM_CUDA(cudaEventElapsedTime(&dms, h.ev_ph[0], h.ev_ph[1]));
    HM_CUDA(cudaEventElapsedTime(&ams, h.ev_ph[2], h.ev_ph[3]));
    h.tm.mvp_dense_ms = dms;
    h.tm.mvp_aca_ms = ams;
    if (t) hm_get_timings(H, t);
  });
}

hm_status hm_mvp_device(hm_handle* H, const double* x_dev, double* z_dev, void* stream) {
  return guarded([&] {
    if (!H || !x_dev || !z_dev) raise(kEinval, "mvp: null argument");
    std::lock_guard<std::mutex> lock(H->mu);
    HM_CUDA(cudaSetDevice(H->h.device));
    on_handle_stream(H->h, static_cast<cudaStream_t>(stream), [&](cudaStream_t s) { product(H, x_dev, z_dev, s); });
  });
}

hm_status hm_mvp_local(hm_handle* H, const double* x, double* z_slice) {
  return guarded([&] {
    if (!H || !x || !z_slice) raise(kEinval, "mvp_local: null argument");
    std::lock_guard<std::mutex> lock(H->mu);
    HMatrix& h = H->h;
    HM_CUDA(cudaSetDevice(h.device));
    cudaStream_t s = h.stream;
    if (h.xin.size() < static_cast<size_t>(h.n)) h.xin.alloc(h.n, s);
    HM_CUDA(cudaMemcpyAsync(h.xin.get(), x, sizeof(double) * h.n, cudaMemcpyHostToDevice, s));
    gather_kernel<<<grid_for(h.n, 256, 1 << 16), 256, 0, s>>>(h.xin.get(), h.perm.get(), h.n, h.xm.get());
    HM_LAUNCH_CHECK();
    mvp_morton(h, s);
    HM_CUDA(cudaMemcpyAsync(z_slice, h.zm.get() + h.row_begin, sizeof(double) * (h.row_end - h.row_begin),
                            cudaMemcpyDeviceToHost, s));
    HM_CUDA(cudaStreamSynchronize(s));
  });
}

hm_status hm_nccl_unique_id(unsigned char id[128]) {
  return guarded([&] {
    if (!id) raise(kEinval, "nccl_unique_id: null argument");
    ncclUniqueId u;
    if (NcclApi::get().GetUniqueId(&u) != ncclSuccess) raise(kEnccl, "ncclGetUniqueId failed");
    static_assert(sizeof(u) == 128, "ncclUniqueId size");
    std::memcpy(id, &u, 128);
  });
}

hm_status hm_attach_nccl(hm_handle* H, const unsigned char id[128]) {
  return guarded([&] {
    if (!H || !id) raise(kEinval, "attach_nccl: null argument");
    std::lock_guard<std::mutex> lock(H->mu);
    if (H->comm) raise(kEinval, "attach_nccl: a communicator is already attached to this handle");
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    HMatrix& h = H->h;
    HM_CUDA(cudaSetDevice(h.device));
    ncclComm_t comm = nullptr;
    if (NcclApi::get().CommInitRank(&comm, h.cfg.world, u, h.cfg.rank) != ncclSuccess)
      raise(kEnccl, "ncclCommInitRank failed");
    H->comm = comm;
    int g = 0;
    while ((1 << g) < h.cfg.world) ++g;
    H->rank_bounds.assign(h.cfg.world + 1, h.n);
    HM_CUDA(cudaMemcpyAsync(H->rank_bounds.data(), h.slot_lo.get() + h.depth_base[g], sizeof(long long) * h.cfg.world,
                            cudaMemcpyDeviceToHost, h.stream));
    HM_CUDA(cudaStreamSynchronize(h.stream));
    H->equal_slices = true;
    for (int r = 0; r < h.cfg.world; ++r)
      H->equal_slices &= (H->rank_bounds[r + 1] - H->rank_bounds[r]) == (H->rank_bounds[1] - H->rank_bounds[0]);
  });
}

hm_status hm_profile_begin(hm_handle* H) {
  return guarded([&] {
    if (!H) raise(kEinval, "profile_begin: null handle");
    std::lock_guard<std::mutex> lock(H->mu);
    H->h.clk.on = true;
  });
}

hm_status hm_profile_end(hm_handle* H, double* ms, int64_t* counts) {
  return guarded([&] {
    if (!H) raise(kEinval, "profile_end: null handle");
    std::lock_guard<std::mutex> lock(H->mu);
    KClock& c = H->h.clk;
    c.on = false;
    for (int id = 0; id < kKNum; ++id) {
      double acc = 0.0;
      const size_t cnt = std::min(c.ev[id][0].size(), c.ev[id][1].size());
      for (size_t i = 0; i < cnt; ++i) {
        HM_CUDA(cudaEventSynchronize(c.ev[id][1][i]));
        float t = 0.f;
        HM_CUDA(cudaEventElapsedTime(&t, c.ev[id][0][i], c.ev[id][1][i]));
        acc += t;
      }
      if (ms) ms[id] = acc;
      if (counts) counts[id] = static_cast<int64_t>(cnt);
      for (int w = 0; w < 2; ++w) {
        for (cudaEvent_t e : c.ev[id][w]) cudaEventDestroy(e);
        c.ev[id][w].clear();
      }
    }
  });
}

namespace {

// nrhs independent cg_solve runs (solver.cpp:19-73) in lock-step, device-resident: one
// (multi-RHS) product per iteration, scalars on the device, ONE host read per iteration
// for the stopping rule / non-finite check.  Each column keeps its own scalars and
// stopping rule, so with flags = 0 (or R = 1) every column follows the single-RHS
// iteration exactly.
void cg_run(hm_handle* H, const double* B, long long R, double sigma2, double tol, long long max_iter, int flags,
            bool multi, double* X, int64_t* iterations, double* rel_res) {
  if (tol <= 0.0) raise(kEinval, "cg_solve: tol must be > 0");
  if (max_iter < 1) raise(kEinval, "cg_solve: max_iter must be >= 1");
  if (sigma2 < 0.0) raise(kEinval, "cg_solve: sigma2 must be >= 0");
  HMatrix& h = H->h;
  HM_CUDA(cudaSetDevice(h.device));
  cudaStream_t s = h.stream;
  const long long n = h.n;
  const int Ri = static_cast<int>(R);
  DevBuf<double> db, dx, dr, dp, dap, part, scal;
  DevBuf<int> act;
  db.alloc(n * R, s);
  dx.alloc(n * R, s);
  dr.alloc(n * R, s);
  dp.alloc(n * R, s);
  dap.alloc(n * R, s);
  scal.alloc(6 * R, s);  // bn2 | rs | pap | rs_next | alpha | beta
  act.alloc(R, s);
  double* bn2 = scal.get();
  double* rs = bn2 + R;
  double* pap = rs + R;
  double* rsn = pap + R;
  double* alpha = rsn + R;
  double* beta = alpha + R;
  const size_t need = static_cast<size_t>(3 * R);
  if (H->pin_scal_n < need) {
    if (H->pin_scal) cudaFreeHost(H->pin_scal);
    H->pin_scal = nullptr;
    H->pin_scal_n = 0;
    HM_CUDA(cudaMallocHost(reinterpret_cast<void**>(&H->pin_scal), need * sizeof(double)));
    H->pin_scal_n = need;
  }
  double* hs = H->pin_scal;  // [0,R) rs_next, [R,2R) alpha, [2R,3R) scratch
  HM_CUDA(cudaMemcpyAsync(db.get(), B, sizeof(double) * n * R, cudaMemcpyHostToDevice, s));
  dx.zero(s);
  HM_CUDA(cudaMemcpyAsync(dr.get(), db.get(), sizeof(double) * n * R, cudaMemcpyDeviceToDevice, s));
  HM_CUDA(cudaMemcpyAsync(dp.get(), db.get(), sizeof(double) * n * R, cudaMemcpyDeviceToDevice, s));
  device_dots(db.get(), db.get(), n, Ri, part, bn2, s);
  device_dots(dr.get(), dr.get(), n, Ri, part, rs, s);
  std::vector<double> bn(R), rs_host(R);
  std::vector<int> active(R, 1);
  HM_CUDA(cudaMemcpyAsync(hs, bn2, sizeof(double) * R, cudaMemcpyDeviceToHost, s));
  HM_CUDA(cudaMemcpyAsync(hs + R, rs, sizeof(double) * R, cudaMemcpyDeviceToHost, s));
  HM_CUDA(cudaStreamSynchronize(s));
  for (long long r = 0; r < R; ++r) {
    iterations[r] = 0;
    rel_res[r] = 0.0;
    bn[r] = std::sqrt(hs[r]);
    rs_host[r] = hs[R + r];
    if (bn[r] == 0.0) active[r] = 0;  // zero rhs: zero solution, no iterations
  }
  HM_CUDA(cudaMemcpyAsync(act.get(), active.data(), sizeof(int) * R, cudaMemcpyHostToDevice, s));
  const unsigned gx = grid_for(n, 256, 4096);
  const dim3 grid(gx, static_cast<unsigned>(R));
  auto apply = [&](double* in, double* out) {
    if (multi) product_multi_all(H, in, out, R, flags, s);
    else product(H, in, out, s);
    axpy_sigma_kernel<<<grid, 256, 0, s>>>(out, in, sigma2, n);
    HM_LAUNCH_CHECK();
  };
  bool any = std::any_of(active.begin(), active.end(), [](int c) { return c != 0; });
  for (long long iter = 1; iter <= max_iter && any; ++iter) {
    apply(dp.get(), dap.get());
    device_dots(dp.get(), dap.get(), n, Ri, part, pap, s);
    cg_alpha_kernel<<<(Ri + 31) / 32, 32, 0, s>>>(rs, pap, act.get(), alpha, Ri);
    cg_update_kernel<<<grid, 256, 0, s>>>(dx.get(), dr.get(), dp.get(), dap.get(), alpha, act.get(), n);
    HM_LAUNCH_CHECK();
    device_dots(dr.get(), dr.get(), n, Ri, part, rsn, s);
    HM_CUDA(cudaMemcpyAsync(hs, rsn, sizeof(double) * R, cudaMemcpyDeviceToHost, s));
    HM_CUDA(cudaMemcpyAsync(hs + R, alpha, sizeof(double) * R, cudaMemcpyDeviceToHost, s));
    HM_CUDA(cudaStreamSynchronize(s));
    any = false;
    bool changed = false;
    for (long long r = 0; r < R; ++r) {
      if (!active[r]) continue;
      const double rs_next = hs[r], a = hs[R + r];
      if (!std::isfinite(rs_next) || !std::isfinite(a))
        raise(kEnonfinite, "cg_solve: non-finite value at iteration " + std::to_string(iter) +
                               (R > 1 ? " (rhs " + std::to_string(r) + ")" : std::string()) + " (residual " +
                               std::to_string(std::sqrt(std::fabs(rs_host[r])) / bn[r]) + ")");
      iterations[r] = iter;
      if (std::sqrt(rs_next) <= tol * bn[r]) {
        active[r] = 0;
        changed = true;
        continue;
      }
      rs_host[r] = rs_next;
      any = true;
    }
    if (changed) HM_CUDA(cudaMemcpyAsync(act.get(), active.data(), sizeof(int) * R, cudaMemcpyHostToDevice, s));
    if (!any) break;
    cg_beta_kernel<<<(Ri + 31) / 32, 32, 0, s>>>(rs, rsn, act.get(), beta, Ri);
    cg_dir_kernel<<<grid, 256, 0, s>>>(dp.get(), dr.get(), beta, act.get(), n);
    HM_LAUNCH_CHECK();
  }
  // true residual of the returned iterates (solver.cpp:64-71), on the device
  apply(dx.get(), dap.get());
  sub_kernel<<<grid_for(n * R, 256, 1 << 16), 256, 0, s>>>(dap.get(), db.get(), n * R);  // dap = b - A x
  HM_LAUNCH_CHECK();
  device_dots(dap.get(), dap.get(), n, Ri, part, pap, s);
  HM_CUDA(cudaMemcpyAsync(hs, pap, sizeof(double) * R, cudaMemcpyDeviceToHost, s));
  HM_CUDA(cudaMemcpyAsync(X, dx.get(), sizeof(double) * n * R, cudaMemcpyDeviceToHost, s));
  HM_CUDA(cudaStreamSynchronize(s));
  for (long long r = 0; r < R; ++r) {
    if (bn[r] == 0.0) {
      std::memset(X + r * n, 0, sizeof(double) * n);
      continue;
    }
    rel_res[r] = std::sqrt(hs[r]) / bn[r];
  }
}

}  // namespace

hm_status hm_cg_solve(hm_handle* H, const double* b, double sigma2, double tol, int64_t max_iter, double* x,
                      int64_t* iterations, double* rel_res) {
  return guarded([&] {
    if (!H || !b || !x || !iterations || !rel_res) raise(kEinval, "cg_solve: null argument");
    std::lock_guard<std::mutex> lock(H->mu);
    cg_run(H, b, 1, sigma2, tol, max_iter, 0, false, x, iterations, rel_res);
  });
}

hm_status hm_mvp_multi(hm_handle* H, const double* X, double* Z, int64_t nrhs, int32_t flags) {
  return guarded([&] {
    if (!H || !X || !Z) raise(kEinval, "mvp_multi: null argument");
    if (nrhs < 1) raise(kEinval, "mvp_multi: nrhs must be >= 1");
    std::lock_guard<std::mutex> lock(H->mu);
    HMatrix& h = H->h;
    HM_CUDA(cudaSetDevice(h.device));
    cudaStream_t s = h.stream;
    const size_t tot = static_cast<size_t>(h.n) * nrhs;
    if (h.xinR.size() < tot) h.xinR.alloc(tot, s);
    if (h.zoutR.size() < tot) h.zoutR.alloc(tot, s);
    HM_CUDA(cudaMemcpyAsync(h.xinR.get(), X, sizeof(double) * tot, cudaMemcpyHostToDevice, s));
    product_multi_all(H, h.xinR.get(), h.zoutR.get(), nrhs, flags, s);
    HM_CUDA(cudaMemcpyAsync(Z, h.zoutR.get(), sizeof(double) * tot, cudaMemcpyDeviceToHost, s));
    HM_CUDA(cudaStreamSynchronize(s));
  });
}

hm_status hm_mvp_multi_device(hm_handle* H, const double* X_dev, double* Z_dev, int64_t nrhs, int32_t flags,
                              void* stream) {
  return guarded([&] {
    if (!H || !X_dev || !Z_dev) raise(kEinval, "mvp_multi: null argument");
    if (nrhs < 1) raise(kEinval, "mvp_multi: nrhs must be >= 1");
    std::lock_guard<std::mutex> lock(H->mu);
    HM_CUDA(cudaSetDevice(H->h.device));
    on_handle_stream(H->h, static_cast<cudaStream_t>(stream),
                     [&](cudaStream_t s) { product_multi_all(H, X_dev, Z_dev, nrhs, flags, s); });
  });
}

hm_status hm_cg_solve_multi(hm_handle* H, const double* B, int64_t nrhs, double sigma2, double tol, int64_t max_iter,
                            int32_t flags, double* X, int64_t* iterations, double* rel_res) {
  return guarded([&] {
    if (!H || !B || !X || !iterations || !rel_res) raise(kEinval, "cg_solve_multi: null argument");
    if (nrhs < 1) raise(kEinval, "cg_solve_multi: nrhs must be >= 1");
    std::lock_guard<std::mutex> lock(H->mu);
    cg_run(H, B, nrhs, sigma2, tol, max_iter, flags, true, X, iterations, rel_res);
  });
}

// dump_leaves_csv (tree.cpp:197-205): every leaf in canonical order (tree.cpp:189-194),
// the dense and admissible lists merged back, with the reference's header and format
hm_status hm_dump_leaves_csv(hm_handle* H, const char* path) {
  return guarded([&] {
    if (!H || !path) raise(kEinval, "dump_leaves_csv: null argument");
    std::lock_guard<std::mutex> lock(H->mu);
    const HMatrix& h = H->h;
    FILE* f = std::fopen(path, "w");
    if (!f) raise(kEio, std::string("dump_leaves_csv: cannot open ") + path);
    std::fputs("row_lower,row_upper,col_lower,col_upper,admissible\n", f);
    const LeafList& D = h.dense;
    const LeafList& A = h.aca;
    long long i = 0, j = 0;
    auto key = [](const LeafList& l, long long q) {
      return std::make_tuple(l.h_rl[q], l.h_rl[q] + l.h_m[q], l.h_cl[q], l.h_cl[q] + l.h_n[q]);
    };
    while (i < D.count || j < A.count) {
      const bool take_d = j >= A.count || (i < D.count && key(D, i) < key(A, j));
      const LeafList& l = take_d ? D : A;
      const long long q = take_d ? i++ : j++;
      std::fprintf(f, "%d,%d,%d,%d,%d\n", l.h_rl[q], l.h_rl[q] + l.h_m[q], l.h_cl[q], l.h_cl[q] + l.h_n[q],
                   take_d ? 0 : 1);
    }
    if (std::fclose(f) != 0) raise(kEio, std::string("dump_leaves_csv: write failed ") + path);
  });
}

hm_status hm_dense_mvp(hm_handle* H, const double* x, double* z) {
  return guarded([&] {
    if (!H || !x || !z) raise(kEinval, "dense_mvp: null argument");
    std::lock_guard<std::mutex> lock(H->mu);
    HMatrix& h = H->h;
    HM_CUDA(cudaSetDevice(h.device));
    cudaStream_t s = h.stream;
    const long long n = h.n;
    DevBuf<double> dx, dz, dzm;
    dx.alloc(n, s);
    dz.alloc(n, s);
    dzm.alloc(n, s);
    HM_CUDA(cudaMemcpyAsync(dx.get(), x, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    gather_kernel<<<grid_for(n, 256, 1 << 16), 256, 0, s>>>(dx.get(), h.perm.get(), n, h.xm.get());
    dense_exact_kernel<<<grid_for(n, 128), 128, 0, s>>>(h.coords.get(), n, h.d, h.kp, h.xm.get(), 0, n, dzm.get());
    scatter_kernel<<<grid_for(n, 256, 1 << 16), 256, 0, s>>>(dzm.get(), h.perm.get(), n, dz.get());
    HM_LAUNCH_CHECK();
    HM_CUDA(cudaMemcpyAsync(z, dz.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    HM_CUDA(cudaStreamSynchronize(s));
  });
}

hm_status hm_relative_error(hm_handle* H, const double* x, double* out) {
  // hmatrix.cpp:125-153 without the N limit (the exact product runs on the device)
  if (!H || !x || !out) {
    g_err = "relative_error: null argument";
    return HM_EINVAL;
  }
  std::vector<double> zh, ze;
  hm_status st = guarded([&] {
    zh.resize(H->h.n);
    ze.resize(H->h.n);
  });
  if (st != HM_OK) return st;
  st = hm_mvp(H, x, zh.data(), nullptr);
  if (st != HM_OK) return st;
  st = hm_dense_mvp(H, x, ze.data());
  if (st != HM_OK) return st;
  double diff_sq = 0.0, ref_sq = 0.0;
  for (size_t i = 0; i < zh.size(); ++i) {
    const double d = zh[i] - ze[i];
    diff_sq += d * d;
    ref_sq += ze[i] * ze[i];
  }
  *out = std::sqrt(diff_sq) / std::sqrt(ref_sq);
  return HM_OK;
}

hm_status hm_get_timings(hm_handle* H, hm_timings* t) {
  return guarded([&] {
    if (!H || !t) raise(kEinval, "get_timings: null argument");
    const Timings& tm = H->h.tm;
    t->setup_ms = tm.setup_ms;
    t->morton_ms = tm.morton_ms;
    t->tree_ms = tm.tree_ms;
    t->aca_ms = tm.aca_ms;
    t->near_ms = tm.near_ms;
    t->mvp_ms = tm.mvp_ms;
    t->mvp_dense_ms = tm.mvp_dense_ms;
    t->mvp_aca_ms = tm.mvp_aca_ms;
  });
}

hm_status hm_get_stats(hm_handle* H, hm_stats* st) {
  return guarded([&] {
    if (!H || !st) raise(kEinval, "get_stats: null argument");
    std::lock_guard<std::mutex> lock(H->mu);
    HMatrix& h = H->h;
    unsigned long long rej[2] = {0, 0};
    HM_CUDA(cudaSetDevice(h.device));
    if (h.aca_rej.size() >= 2)
      HM_CUDA(cudaMemcpyAsync(rej, h.aca_rej.get(), sizeof(rej), cudaMemcpyDeviceToHost, h.stream));
    HM_CUDA(cudaStreamSynchronize(h.stream));
    if (!h.cfg.precompute_aca && h.keff_known) {
      // recompute mode: ranks of the factorisation inside the last product
      long long lo = 0, hi = 0;
      if (!h.chunks.empty()) {
        lo = h.chunks.front().c0;
        hi = h.chunks.back().c1;
      }
      std::vector<int> ke(std::max(hi - lo, 0ll));
      if (hi > lo) {
        HM_CUDA(cudaMemcpyAsync(ke.data(), h.k_eff.get() + lo, sizeof(int) * (hi - lo), cudaMemcpyDeviceToHost,
                                h.stream));
        HM_CUDA(cudaStreamSynchronize(h.stream));
      }
      rank_sums(h, ke.data(), lo, hi);
    }
    st->n_dense = h.dense.count;
    st->n_aca = h.aca.count;
    st->S_d = h.S_d;
    st->S_l = h.S_l;
    st->sum_m_adm = h.sum_m_adm;
    st->sum_n_adm = h.sum_n_adm;
    st->S_lm = h.S_lm;
    st->S_ln = h.S_ln;
    st->S_d_own = h.S_d_own;
    st->aca_rejections = static_cast<int64_t>(rej[0]);
    st->aca_rejected_entries = static_cast<int64_t>(rej[1]);
    st->S_chain = h.S_chain;
    st->near_pairs = h.n_pairs;
    st->near_sym_rc = h.near_sym_rc ? 1 : 0;
    st->dmax_leaf = h.dmax_leaf;
    st->row_begin = h.row_begin;
    st->row_end = h.row_end;
    st->device_bytes = static_cast<double>(h.dense_vals.bytes() + h.U.bytes() + h.V.bytes() + h.U2.bytes() + h.V2.bytes() + h.coords.bytes());
    st->S_d_stored = h.S_d_stored;
    st->near_sym = h.near_sym ? 1 : 0;
    st->n_aca_batches = h.n_batches;
    st->n_aca_chunks = static_cast<int64_t>(h.chunks.size());
  });
}

hm_status hm_get_points(hm_handle* H, double* coords, int64_t* perm) {
  return guarded([&] {
    if (!H || !coords || !perm) raise(kEinval, "get_points: null argument");
    std::lock_guard<std::mutex> lock(H->mu);
    HMatrix& h = H->h;
    HM_CUDA(cudaSetDevice(h.device));
    HM_CUDA(cudaMemcpyAsync(coords, h.coords.get(), sizeof(double) * h.n * h.d, cudaMemcpyDeviceToHost, h.stream));
    HM_CUDA(cudaMemcpyAsync(perm, h.perm.get(), sizeof(long long) * h.n, cudaMemcpyDeviceToHost, h.stream));
    HM_CUDA(cudaStreamSynchronize(h.stream));
  });
}

hm_status hm_get_codes(hm_handle* H, uint64_t* codes) {
  return guarded([&] {
    if (!H || !codes) raise(kEinval, "get_codes: null argument");
    std::lock_guard<std::mutex> lock(H->mu);
    HMatrix& h = H->h;
    HM_CUDA(cudaSetDevice(h.device));
    HM_CUDA(cudaMemcpyAsync(codes, h.codes.get(), sizeof(uint64_t) * h.n, cudaMemcpyDeviceToHost, h.stream));
    HM_CUDA(cudaStreamSynchronize(h.stream));
  });
}

hm_status hm_get_leaves(hm_handle* H, int32_t which, int64_t* rows4, double* boxes) {
  return guarded([&] {
    if (!H || !rows4) raise(kEinval, "get_leaves: null argument");
    std::lock_guard<std::mutex> lock(H->mu);
    HMatrix& h = H->h;
    HM_CUDA(cudaSetDevice(h.device));
    const LeafList& l = which == 0 ? h.dense : h.aca;
    const long long cnt = l.count;
    for (long long i = 0; i < cnt; ++i) {
      rows4[4 * i + 0] = l.h_rl[i];
      rows4[4 * i + 1] = static_cast<long long>(l.h_rl[i]) + l.h_m[i];
      rows4[4 * i + 2] = l.h_cl[i];
      rows4[4 * i + 3] = static_cast<long long>(l.h_cl[i]) + l.h_n[i];
    }
    if (boxes && cnt) {
      const int d = h.d;
      std::vector<int> ts(cnt), ss(cnt);
      std::vector<double> tab(static_cast<size_t>(h.nslots) * 2 * d);
      HM_CUDA(cudaMemcpyAsync(ts.data(), l.tau_slot.get(), sizeof(int) * cnt, cudaMemcpyDeviceToHost, h.stream));
      HM_CUDA(cudaMemcpyAsync(ss.data(), l.sigma_slot.get(), sizeof(int) * cnt, cudaMemcpyDeviceToHost, h.stream));
      HM_CUDA(cudaMemcpyAsync(tab.data(), h.boxes.get(), sizeof(double) * tab.size(), cudaMemcpyDeviceToHost,
                              h.stream));
      HM_CUDA(cudaStreamSynchronize(h.stream));
      for (long long i = 0; i < cnt; ++i) {
        std::memcpy(boxes + 4 * d * i, tab.data() + static_cast<size_t>(ts[i]) * 2 * d, sizeof(double) * 2 * d);
        std::memcpy(boxes + 4 * d * i + 2 * d, tab.data() + static_cast<size_t>(ss[i]) * 2 * d, sizeof(double) * 2 * d);
      }
    }
  });
}

hm_status hm_get_aca(hm_handle* H, int64_t* k_eff, int64_t* row_piv, int64_t* col_piv, double* u, double* v) {
  return guarded([&] {
    if (!H || !k_eff || !row_piv || !col_piv) raise(kEinval, "get_aca: null argument");
    std::lock_guard<std::mutex> lock(H->mu);
    HMatrix& h = H->h;
    HM_CUDA(cudaSetDevice(h.device));
    cudaStream_t s = h.stream;
    const long long cnt = h.aca.count, kmax = h.cfg.k;
    if (h.cfg.world > 1) raise(kEinval, "hm_get_aca: single-rank handles only");
    const auto& uo = h.h_uoff;
    const auto& vo = h.h_voff;
    std::vector<double> hu, hv;
    if (u || v) {
      hu.resize(uo[cnt]);
      hv.resize(vo[cnt]);
    }
    if (!h.factors_valid) {
      // recompute mode: factorise into the product's chunk workspace chunk by chunk
      // (introspection only); the same plan as the product, so any N that runs factorises
      reset_aca_rejections(h, s);
      for (const AcaChunk& c : h.chunks) {
        if (h.U.size() < static_cast<size_t>(c.ue - c.ub)) h.U.alloc(c.ue - c.ub, s);
        if (h.V.size() < static_cast<size_t>(c.ve - c.vb)) h.V.alloc(c.ve - c.vb, s);
        compute_aca(h, c, s);
        h.keff_known = true;
        if (u || v) {
          HM_CUDA(cudaMemcpyAsync(hu.data() + c.ub, h.U.get(), sizeof(double) * (c.ue - c.ub), cudaMemcpyDeviceToHost, s));
          HM_CUDA(cudaMemcpyAsync(hv.data() + c.vb, h.V.get(), sizeof(double) * (c.ve - c.vb), cudaMemcpyDeviceToHost, s));
          HM_CUDA(cudaStreamSynchronize(s));
        }
      }
    } else if ((u || v) && cnt) {
      HM_CUDA(cudaMemcpyAsync(hu.data(), h.U.get(), sizeof(double) * uo[cnt], cudaMemcpyDeviceToHost, s));
      HM_CUDA(cudaMemcpyAsync(hv.data(), h.V.get(), sizeof(double) * vo[cnt], cudaMemcpyDeviceToHost, s));
    }
    std::vector<int> hk(cnt), hrp(cnt * kmax), hcp(cnt * kmax);
    if (cnt) {
      HM_CUDA(cudaMemcpyAsync(hk.data(), h.k_eff.get(), sizeof(int) * cnt, cudaMemcpyDeviceToHost, s));
      HM_CUDA(cudaMemcpyAsync(hrp.data(), h.row_piv.get(), sizeof(int) * cnt * kmax, cudaMemcpyDeviceToHost, s));
      HM_CUDA(cudaMemcpyAsync(hcp.data(), h.col_piv.get(), sizeof(int) * cnt * kmax, cudaMemcpyDeviceToHost, s));
    }
    HM_CUDA(cudaStreamSynchronize(s));
    long long ou = 0, ov = 0;  // output offsets: k x m and k x n per leaf, rank-major
    for (long long b = 0; b < cnt; ++b) {
      k_eff[b] = hk[b];
      const long long m = h.aca.h_m[b], n = h.aca.h_n[b];
      // device layout: stride kmax, or ke2 = k_eff rounded to even (compacted stored factors)
      const long long ks = h.compact ? ((hk[b] + 1) & ~1) : kmax;
      for (long long l = 0; l < kmax; ++l) {
        row_piv[b * kmax + l] = hrp[b * kmax + l];
        col_piv[b * kmax + l] = hcp[b * kmax + l];
        const bool live = l < hk[b];
        const int sh = h.u_tile_shift;
        if (u)
          for (long long i = 0; i < m; ++i) {
            const long long src = sh < 0 ? l * m + i : ((((i >> sh) * ks) + l) << sh) + (i & ((1ll << sh) - 1));
            u[ou + l * m + i] = live ? hu[uo[b] + src] : 0.0;
          }
        if (v)
          for (long long j = 0; j < n; ++j) v[ov + l * n + j] = live ? hv[vo[b] + j * ks + l] : 0.0;
      }
      ou += kmax * m;
      ov += kmax * n;
    }
  });
}

hm_status hm_morton_codes(const double* coords, int64_t n, int32_t d, uint64_t* codes) {
  return guarded([&] {
    require_device();
    if (d < 1 || d > 20) raise(kEinval, "morton_bits_per_dim: dimension out of range");
    cudaStream_t s = nullptr;
    DevBuf<double> c;
    DevBuf<unsigned long long> k;
    c.alloc(static_cast<size_t>(n) * d, s);
    k.alloc(n, s);
    HM_CUDA(cudaMemcpyAsync(c.get(), coords, sizeof(double) * n * d, cudaMemcpyHostToDevice, s));
    if (n) morton_codes_device(c.get(), n, d, k.get(), s);
    HM_CUDA(cudaMemcpyAsync(codes, k.get(), sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, s));
    HM_CUDA(cudaStreamSynchronize(s));
  });
}

hm_status hm_morton_order(const double* coords, int64_t n, int32_t d, const int64_t* perm_in, double* coords_out,
                          int64_t* perm_out) {
  return guarded([&] {
    require_device();
    if (d < 1 || d > 20) raise(kEinval, "morton_bits_per_dim: dimension out of range");
    if (n < 1) return;
    cudaStream_t s = nullptr;
    DevBuf<double> c, co;
    DevBuf<unsigned long long> k;
    DevBuf<unsigned> ord;
    c.alloc(static_cast<size_t>(n) * d, s);
    co.alloc(static_cast<size_t>(n) * d, s);
    k.alloc(n, s);
    ord.alloc(n, s);
    HM_CUDA(cudaMemcpyAsync(c.get(), coords, sizeof(double) * n * d, cudaMemcpyHostToDevice, s));
    morton_codes_device(c.get(), n, d, k.get(), s);
    iota_u32(ord.get(), n, s);
    radix_sort_pairs(k.get(), ord.get(), n, s);
    std::vector<unsigned> ho(n);
    std::vector<double> hc(static_cast<size_t>(n) * d);
    HM_CUDA(cudaMemcpyAsync(ho.data(), ord.get(), sizeof(unsigned) * n, cudaMemcpyDeviceToHost, s));
    HM_CUDA(cudaStreamSynchronize(s));
    for (long long i = 0; i < n; ++i) {
      const long long src = ho[i];
      for (int a = 0; a < d; ++a) coords_out[a * n + i] = coords[a * n + src];
      perm_out[i] = perm_in ? perm_in[src] : src;
    }
  });
}

hm_status hm_aca_dense(int64_t nb, const int64_t* shapes, const double* entries, int64_t kmax, int32_t has_eps,
                       double eps, double eta, int64_t* k_eff, int64_t* row_piv, int64_t* col_piv, double* u,
                       double* v) {
  return guarded([&] {
    require_device();
    if (nb <= 0) return;
    aca_dense_blocks(nb, reinterpret_cast<const long long*>(shapes), entries, kmax, has_eps != 0, eps, eta,
                     reinterpret_cast<long long*>(k_eff), reinterpret_cast<long long*>(row_piv),
                     reinterpret_cast<long long*>(col_piv), u, v, nullptr);
  });
}

hm_status hm_eval_kernel(int32_t kernel, double beta, int32_t d, int64_t n, const double* y, const double* yp,
                         double* out) {
  return guarded([&] {
    require_device();
    const KernelParams kp = make_kernel(kernel, beta, d);
    if (n <= 0) return;
    cudaStream_t s = nullptr;
    DevBuf<double> a, b, o;
    a.alloc(static_cast<size_t>(n) * d, s);
    b.alloc(static_cast<size_t>(n) * d, s);
    o.alloc(n, s);
    HM_CUDA(cudaMemcpyAsync(a.get(), y, sizeof(double) * n * d, cudaMemcpyHostToDevice, s));
    HM_CUDA(cudaMemcpyAsync(b.get(), yp, sizeof(double) * n * d, cudaMemcpyHostToDevice, s));
    eval_pairs_kernel<<<grid_for(n, 256, 1 << 16), 256, 0, s>>>(kp, d, n, a.get(), b.get(), o.get());
    HM_LAUNCH_CHECK();
    HM_CUDA(cudaMemcpyAsync(out, o.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    HM_CUDA(cudaStreamSynchronize(s));
  });
}

void hm_exp_port_host(int64_t n, const double* x, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = glibc_exp(x[i]);
}

void hm_log_port_host(int64_t n, const double* x, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = glibc_log(x[i]);
}

static hm_status libm_port_device(int which, int64_t n, const double* x, double* out);

hm_status hm_exp_port_device(int64_t n, const double* x, double* out) { return libm_port_device(0, n, x, out); }
hm_status hm_log_port_device(int64_t n, const double* x, double* out) { return libm_port_device(1, n, x, out); }

static hm_status libm_port_device(int which, int64_t n, const double* x, double* out) {
  return guarded([&] {
    require_device();
    if (n <= 0) return;
    cudaStream_t s = nullptr;
    DevBuf<double> a, o;
    a.alloc(n, s);
    o.alloc(n, s);
    HM_CUDA(cudaMemcpyAsync(a.get(), x, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    exp_port_kernel<<<grid_for(n, 256, 1 << 16), 256, 0, s>>>(n, a.get(), o.get(), which);
    HM_LAUNCH_CHECK();
    HM_CUDA(cudaMemcpyAsync(out, o.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    HM_CUDA(cudaStreamSynchronize(s));
  });
}

}  // extern "C"

// setup.cu -- Morton order, cluster-box pyramid, level-synchronous block-tree
// traversal and canonical leaf lists (reference setup(), hmatrix.cpp:38-56).
//
//   K1 morton codes           morton.cpp:11-48       1 thread / point
//   K2 stable sort + gather   morton.cpp:50-71       LSD radix (primitives.cu)
//   K3 box pyramid            tree.cpp:59-136        replaces per-level Alg. 7/8
//   K4 traversal              tree.cpp:140-187       per-level classify + scan + emit
//   K5 canonical order+split  tree.cpp:189-194, hmatrix.cpp:51-53
#include <mutex>
#include <cstring>
#include <algorithm>
#include <chrono>
#include <cmath>

#include <math_constants.h>

#include "hmatrix.h"
#include "primitives.h"

namespace hmb {

namespace {

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t) { return std::chrono::duration<double, std::milli>(Clock::now() - t).count(); }

// morton.cpp:17-23
__device__ __forceinline__ unsigned long long fixed_point(double c, int bits) {
  const double scaled = floor(hmul(c, static_cast<double>(1ull << bits)));
  if (!(scaled > 0.0)) return 0ull;
  const unsigned long long maxv = (1ull << bits) - 1ull;
  if (scaled >= static_cast<double>(maxv)) return maxv;
  return static_cast<unsigned long long>(scaled);
}

__device__ __forceinline__ unsigned long long spread2(unsigned long long v) {  // 32 -> 64 bits, even slots
  v &= 0xffffffffull;
  v = (v | (v << 16)) & 0x0000ffff0000ffffull;
  v = (v | (v << 8)) & 0x00ff00ff00ff00ffull;
  v = (v | (v << 4)) & 0x0f0f0f0f0f0f0f0full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}
__device__ __forceinline__ unsigned long long spread3(unsigned long long v) {  // 21 -> 63 bits, every 3rd
  v &= 0x1fffffull;
  v = (v | (v << 32)) & 0x1f00000000ffffull;
  v = (v | (v << 16)) & 0x1f0000ff0000ffull;
  v = (v | (v << 8)) & 0x100f00f00f00f00full;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}

// morton.cpp:25-48: bit b of axis a -> position b*d + a
__global__ void morton_kernel(const double* __restrict__ coords, long long n, int d,
                              unsigned long long* __restrict__ codes) {
  const int bits = 64 / d > 52 ? 52 : 64 / d;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    unsigned long long code = 0;
    if (d == 2) {
      code = spread2(fixed_point(coords[i], bits)) | (spread2(fixed_point(coords[n + i], bits)) << 1);
    } else if (d == 3) {
      code = spread3(fixed_point(coords[i], bits)) | (spread3(fixed_point(coords[n + i], bits)) << 1) |
             (spread3(fixed_point(coords[2 * n + i], bits)) << 2);
    } else {
      for (int a = 0; a < d; ++a) {
        const unsigned long long v = fixed_point(coords[a * n + i], bits);
        for (int b = 0; b < bits; ++b) code |= ((v >> b) & 1ull) << (b * d + a);
      }
    }
    codes[i] = code;
  }
}

__global__ void nonfinite_kernel(const double* __restrict__ c, long long total, int* flag) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    if (!isfinite(c[i])) *flag = 1;
}

// gather coords into Morton order and compose the permutation (morton.cpp:62-69)
__global__ void gather_points_kernel(const double* __restrict__ src, const unsigned* __restrict__ order, long long n,
                                     int d, const long long* __restrict__ perm_in, double* __restrict__ dst,
                                     long long* __restrict__ perm) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long s = order[i];
    for (int a = 0; a < d; ++a) dst[a * n + i] = src[a * n + s];
    perm[i] = perm_in ? perm_in[s] : s;
  }
}

// cluster ranges of every slot (depth e, index idx): descend the ceil-half splits (tree.cpp:120-123)
__global__ void slot_ranges_kernel(long long n, int dcap, long long nslots, long long* __restrict__ lo_out,
                                   long long* __restrict__ hi_out) {
  for (long long s = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; s < nslots;
       s += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int e = 63 - __clzll(static_cast<unsigned long long>(s + 1));  // depth: 2^e - 1 <= s < 2^(e+1) - 1
    const long long idx = s - ((1ll << e) - 1);
    long long lo = 0, hi = n;
    for (int b = e - 1; b >= 0; --b) {
      const long long mid = lo + (hi - lo + 1) / 2;
      if ((idx >> b) & 1) lo = mid;
      else hi = mid;
    }
    lo_out[s] = lo;
    hi_out[s] = hi;
  }
  (void)dcap;
}

// keep-first MinOp/MaxOp (parallel.hpp:68-75): min(acc, x) = x < acc ? x : acc
__device__ __forceinline__ double kmin(double acc, double x) { return x < acc ? x : acc; }
__device__ __forceinline__ double kmax(double acc, double x) { return acc < x ? x : acc; }

// deepest level: one warp per cluster, each lane folds a contiguous chunk, then an
// order-preserving shuffle tree (exact for finite data: the result is the first
// element attaining the extreme, as in the reference's left fold, tree.cpp:76-89).
__global__ void leaf_boxes_kernel(const double* __restrict__ coords, long long n, int d, long long first_slot,
                                  long long count, const long long* __restrict__ slot_lo,
                                  const long long* __restrict__ slot_hi, double* __restrict__ boxes) {
  const long long warp = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= count) return;
  const long long slot = first_slot + warp;
  const long long lo = slot_lo[slot], hi = slot_hi[slot];
  const long long len = hi - lo;
  const long long chunk = (len + 31) / 32;
  const long long a0 = lo + lane * chunk;
  const long long a1 = min(hi, a0 + chunk);
  for (int a = 0; a < d; ++a) {
    const double* c = coords + a * n;
    double mn = CUDART_INF, mx = -CUDART_INF;
    int have = 0;
    for (long long i = a0; i < a1; ++i) {
      const double v = c[i];
      if (!have) {
        mn = mx = v;
        have = 1;
      } else {
        mn = kmin(mn, v);
        mx = kmax(mx, v);
      }
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double omn = __shfl_down_sync(0xffffffffu, mn, o);
      const double omx = __shfl_down_sync(0xffffffffu, mx, o);
      const int ohave = __shfl_down_sync(0xffffffffu, have, o);
      if ((lane & (2 * o - 1)) == 0 && lane + o < 32 && ohave) {
        if (!have) {
          mn = omn;
          mx = omx;
          have = 1;
        } else {
          mn = kmin(mn, omn);
          mx = kmax(mx, omx);
        }
      }
    }
    if (lane == 0) {
      boxes[slot * 2 * d + a] = mn;       // empty cluster -> (+inf, -inf): neutral
      boxes[slot * 2 * d + d + a] = mx;
    }
  }
}

// parent = combine(left child, right child), left first (same keep-first semantics)
__global__ void parent_boxes_kernel(int d, long long first_slot, long long count, long long child_first,
                                    double* __restrict__ boxes) {
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < count * d;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long j = t / d;
    const int a = static_cast<int>(t % d);
    const long long s = first_slot + j;
    const long long l = child_first + 2 * j, r = l + 1;
    boxes[s * 2 * d + a] = kmin(boxes[l * 2 * d + a], boxes[r * 2 * d + a]);
    boxes[s * 2 * d + d + a] = kmax(boxes[l * 2 * d + d + a], boxes[r * 2 * d + d + a]);
  }
}

// tree.cpp:11-32 with the reference's operation order, no contraction
__device__ __forceinline__ double box_diam(const double* box, int d) {
  double sum = 0.0;
  for (int i = 0; i < d; ++i) {
    const double side = hsub(box[d + i], box[i]);
    sum = hadd(sum, hmul(side, side));
  }
  return __dsqrt_rn(sum);
}
__device__ __forceinline__ double stdmax0(double v) { return 0.0 < v ? v : 0.0; }  // std::max(0.0, v)
__device__ __forceinline__ double box_dist(const double* t, const double* s, int d) {
  double sum = 0.0;
  for (int i = 0; i < d; ++i) {
    const double g1 = stdmax0(hsub(t[i], s[d + i]));
    const double g2 = stdmax0(hsub(s[i], t[d + i]));
    sum = hadd(sum, hadd(hmul(g1, g1), hmul(g2, g2)));
  }
  return __dsqrt_rn(sum);
}
__device__ __forceinline__ bool box_admissible(const double* t, const double* s, int d, double eta) {
  const double dt = box_diam(t, d), ds = box_diam(s, d);
  const double mn = ds < dt ? ds : dt;  // std::min
  return mn <= hmul(eta, box_dist(t, s, d));
}

struct LevelArgs {
  const unsigned* tau;
  const unsigned* sigma;
  long long width;
  long long base;  // depth_base[level]
  const long long* slot_lo;
  const long long* slot_hi;
  const double* boxes;
  int d;
  double eta;
  long long c_leaf;
  int mode;
};

// count_children / is_leaf (tree.cpp:153-169): packed (children << 32) | leaf
__global__ void classify_kernel(LevelArgs a, long long* __restrict__ packed, unsigned char* __restrict__ adm_out) {
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < a.width;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long st = a.base + a.tau[k], ss = a.base + a.sigma[k];
    bool adm;
    if (a.mode == 1) adm = false;
    else if (a.mode == 2) adm = true;
    else adm = box_admissible(a.boxes + st * 2 * a.d, a.boxes + ss * 2 * a.d, a.d, a.eta);
    const bool leaf = adm || (a.slot_hi[st] - a.slot_lo[st]) <= a.c_leaf || (a.slot_hi[ss] - a.slot_lo[ss]) <= a.c_leaf;
    packed[k] = leaf ? 1ll : (4ll << 32);
    adm_out[k] = adm ? 1 : 0;
  }
}

// emit_children (tree.cpp:170-183) + leaf records with the canonical sort key
__global__ void emit_kernel(LevelArgs a, int level, const long long* __restrict__ offs,
                            const unsigned char* __restrict__ adm, unsigned* __restrict__ ntau,
                            unsigned* __restrict__ nsigma, long long leaf_base, unsigned long long* __restrict__ lkey,
                            unsigned* __restrict__ ltau, unsigned* __restrict__ lsigma,
                            unsigned char* __restrict__ ldepth, unsigned char* __restrict__ ladm) {
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < a.width;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long o = offs[k];
    const unsigned t = a.tau[k], s = a.sigma[k];
    const long long co = o >> 32, lo = o & 0xffffffffll;
    // same leaf rule as classify_kernel (adm was stored there)
    const long long st = a.base + t, ss = a.base + s;
    const bool is_leaf = adm[k] || (a.slot_hi[st] - a.slot_lo[st]) <= a.c_leaf ||
                         (a.slot_hi[ss] - a.slot_lo[ss]) <= a.c_leaf;
    if (is_leaf) {
      const long long li = leaf_base + lo;
      const unsigned long long rl = static_cast<unsigned long long>(a.slot_lo[st]);
      // canonical order (row.lower, row.upper, col.lower, col.upper) == (row.lower, -depth, sigma index)
      lkey[li] = (rl << 32) | (static_cast<unsigned long long>(31 - level) << 27) | s;
      ltau[li] = t;
      lsigma[li] = s;
      ldepth[li] = static_cast<unsigned char>(level);
      ladm[li] = adm[k];
    } else {
      ntau[co + 0] = 2 * t;      nsigma[co + 0] = 2 * s;
      ntau[co + 1] = 2 * t;      nsigma[co + 1] = 2 * s + 1;
      ntau[co + 2] = 2 * t + 1;  nsigma[co + 2] = 2 * s;
      ntau[co + 3] = 2 * t + 1;  nsigma[co + 3] = 2 * s + 1;
    }
  }
}

__global__ void permute_leaves_kernel(const unsigned* __restrict__ order, long long L,
                                      const unsigned* __restrict__ tau, const unsigned* __restrict__ sigma,
                                      const unsigned char* __restrict__ depth, const unsigned char* __restrict__ adm,
                                      unsigned* __restrict__ otau, unsigned* __restrict__ osigma,
                                      unsigned char* __restrict__ odepth, long long* __restrict__ split_packed) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < L;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const unsigned s = order[i];
    otau[i] = tau[s];
    osigma[i] = sigma[s];
    odepth[i] = depth[s];
    split_packed[i] = adm[s] ? (1ll << 32) : 1ll;  // high: aca, low: dense
  }
}

__global__ void split_kernel(long long L, const long long* __restrict__ offs, const long long* __restrict__ packed_in,
                             const unsigned* __restrict__ tau, const unsigned* __restrict__ sigma,
                             const unsigned char* __restrict__ depth, const long long* __restrict__ depth_base,
                             const long long* __restrict__ slot_lo, const long long* __restrict__ slot_hi,
                             int* d_rl, int* d_m, int* d_cl, int* d_n, int* d_ts, int* d_ss, unsigned char* d_dep,
                             int* a_rl, int* a_m, int* a_cl, int* a_n, int* a_ts, int* a_ss, unsigned char* a_dep) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < L;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const bool is_aca = packed_in[i] >> 32;
    const long long o = is_aca ? (offs[i] >> 32) : (offs[i] & 0xffffffffll);
    const int e = depth[i];
    const long long st = depth_base[e] + tau[i], ss = depth_base[e] + sigma[i];
    const int rl = static_cast<int>(slot_lo[st]), m = static_cast<int>(slot_hi[st] - slot_lo[st]);
    const int cl = static_cast<int>(slot_lo[ss]), nn = static_cast<int>(slot_hi[ss] - slot_lo[ss]);
    if (is_aca) {
      a_rl[o] = rl; a_m[o] = m; a_cl[o] = cl; a_n[o] = nn; a_ts[o] = static_cast<int>(st);
      a_ss[o] = static_cast<int>(ss); a_dep[o] = static_cast<unsigned char>(e);
    } else {
      d_rl[o] = rl; d_m[o] = m; d_cl[o] = cl; d_n[o] = nn; d_ts[o] = static_cast<int>(st);
      d_ss[o] = static_cast<int>(ss); d_dep[o] = static_cast<unsigned char>(e);
    }
  }
}

__global__ void runs_kernel(long long cnt, const int* __restrict__ ts, int* __restrict__ rs, int* __restrict__ re) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < cnt;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int s = ts[i];
    if (i == 0 || ts[i - 1] != s) rs[s] = static_cast<int>(i);
    if (i == cnt - 1 || ts[i + 1] != s) re[s] = static_cast<int>(i + 1);
  }
}

// Spans of the canonical chain of deepest cluster c: groups of equal row.lower
// ascending, inside a group the deeper cluster first (smaller row.upper).
// mode 0: count, mode 1: fill.
__global__ void chain_spans_kernel(int D, long long ncl, const long long* __restrict__ slot_lo,
                                   const int* __restrict__ rs, const int* __restrict__ re, int* __restrict__ cnt,
                                   const int* __restrict__ ptr, int* __restrict__ spans, int mode) {
  for (long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; c < ncl;
       c += static_cast<long long>(gridDim.x) * blockDim.x) {
    int k = 0;
    int o = mode ? ptr[c] : 0;
    for (int e0 = 0; e0 <= D;) {
      const long long lo0 = slot_lo[((1ll << e0) - 1) + (c >> (D - e0))];
      int e1 = e0;
      while (e1 + 1 <= D && slot_lo[((1ll << (e1 + 1)) - 1) + (c >> (D - e1 - 1))] == lo0) ++e1;
      for (int e = e1; e >= e0; --e) {
        const long long s = ((1ll << e) - 1) + (c >> (D - e));
        if (rs[s] < 0) continue;
        if (mode) {
          spans[2 * (o + k)] = rs[s];
          spans[2 * (o + k) + 1] = re[s];
        }
        ++k;
      }
      e0 = e1 + 1;
    }
    if (!mode) cnt[c] = k;
  }
}

// Morton row -> index of its cluster at depth D
__global__ void row_cluster_kernel(int D, long long n, const long long* __restrict__ slot_lo,
                                   const long long* __restrict__ slot_hi, int* __restrict__ rc) {
  const long long first = (1ll << D) - 1;
  for (long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; c < (1ll << D);
       c += static_cast<long long>(gridDim.x) * blockDim.x) {
    for (long long i = slot_lo[first + c]; i < slot_hi[first + c]; ++i) rc[i] = static_cast<int>(c);
  }
  (void)n;
}

void build_spans(HMatrix& h, cudaStream_t s) {
  const int D = h.dmax_leaf;
  const long long ncl = 1ll << D;
  h.row_cluster.alloc(h.n, s);
  row_cluster_kernel<<<grid_for(ncl, 128, 1 << 16), 128, 0, s>>>(D, h.n, h.slot_lo.get(), h.slot_hi.get(),
                                                                 h.row_cluster.get());
  HM_LAUNCH_CHECK();
  struct Side {
    LeafList* l;
    DevBuf<int>* ptr;
    DevBuf<int>* spans;
  } sides[2] = {{&h.dense, &h.dspan_ptr, &h.dspans}, {&h.aca, &h.aspan_ptr, &h.aspans}};
  for (const Side& sd : sides) {
    DevBuf<int> cnt;
    cnt.alloc(ncl, s);
    chain_spans_kernel<<<grid_for(ncl, 128, 1 << 16), 128, 0, s>>>(D, ncl, h.slot_lo.get(), sd.l->run_start.get(),
                                                                   sd.l->run_end.get(), cnt.get(), nullptr, nullptr,
                                                                   0);
    HM_LAUNCH_CHECK();
    DevBuf<long long> c64;
    c64.alloc(ncl + 1, s);
    // widen + scan (int64 scan primitive)
    std::vector<int> hc(ncl);
    HM_CUDA(cudaMemcpyAsync(hc.data(), cnt.get(), sizeof(int) * ncl, cudaMemcpyDeviceToHost, s));
    HM_CUDA(cudaStreamSynchronize(s));
    std::vector<int> hp(ncl + 1, 0);
    for (long long c = 0; c < ncl; ++c) hp[c + 1] = hp[c] + hc[c];
    sd.ptr->alloc(ncl + 1, s);
    HM_CUDA(cudaMemcpyAsync(sd.ptr->get(), hp.data(), sizeof(int) * (ncl + 1), cudaMemcpyHostToDevice, s));
    sd.spans->alloc(2 * std::max(hp[ncl], 1), s);
    chain_spans_kernel<<<grid_for(ncl, 128, 1 << 16), 128, 0, s>>>(D, ncl, h.slot_lo.get(), sd.l->run_start.get(),
                                                                   sd.l->run_end.get(), nullptr, sd.ptr->get(),
                                                                   sd.spans->get(), 1);
    HM_LAUNCH_CHECK();
    HM_CUDA(cudaStreamSynchronize(s));
  }
}

// Host <-> device copies of large arrays through a process-wide page-locked staging ring:
// each 32 MB piece is DMA'd at full link rate while the host threads copy the neighbouring
// piece (and take the first-touch page faults of a fresh host array in parallel).  Small
// copies go direct.
namespace {
struct StagingRing {
  static constexpr size_t kPiece = size_t(32) << 20;
  std::mutex mu;
  char* ring[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  void ready() {
    for (int q = 0; q < 2; ++q) {
      if (!ring[q]) HM_CUDA(cudaMallocHost(reinterpret_cast<void**>(&ring[q]), kPiece));
      if (!done[q]) HM_CUDA(cudaEventCreateWithFlags(&done[q], cudaEventDisableTiming));
    }
  }
  static void host_copy(char* to, const char* from, size_t len) {
    parallel_blocks(static_cast<long long>(len), [&](long long b0, long long b1) {
      std::memcpy(to + b0, from + b0, static_cast<size_t>(b1 - b0));
    }, 8);
  }
  void to_host(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    std::lock_guard<std::mutex> lk(mu);
    ready();
    const size_t np = (bytes + kPiece - 1) / kPiece;
    auto issue = [&](size_t p) {
      const size_t off = p * kPiece, len = std::min(kPiece, bytes - off);
      HM_CUDA(cudaMemcpyAsync(ring[p & 1], static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost, s));
      HM_CUDA(cudaEventRecord(done[p & 1], s));
    };
    issue(0);
    for (size_t p = 0; p < np; ++p) {
      if (p + 1 < np) issue(p + 1);
      HM_CUDA(cudaEventSynchronize(done[p & 1]));
      const size_t off = p * kPiece, len = std::min(kPiece, bytes - off);
      host_copy(static_cast<char*>(dst) + off, ring[p & 1], len);
    }
  }
  void to_device(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    std::lock_guard<std::mutex> lk(mu);
    ready();
    const size_t np = (bytes + kPiece - 1) / kPiece;
    for (size_t p = 0; p < np; ++p) {
      const size_t off = p * kPiece, len = std::min(kPiece, bytes - off);
      if (p >= 2) HM_CUDA(cudaEventSynchronize(done[p & 1]));  // this buffer's previous DMA is done
      host_copy(ring[p & 1], static_cast<const char*>(src) + off, len);
      HM_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, ring[p & 1], len, cudaMemcpyHostToDevice, s));
      HM_CUDA(cudaEventRecord(done[p & 1], s));
    }
    HM_CUDA(cudaStreamSynchronize(s));
  }
};
StagingRing& staging() {
  static StagingRing r;
  return r;
}
}  // namespace

void mirror_to_host(int* dst, const int* src, long long cnt, cudaStream_t s) {
  if (cnt <= 0) return;
  const size_t bytes = sizeof(int) * static_cast<size_t>(cnt);
  if (bytes < (size_t(8) << 20)) {
    HM_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    HM_CUDA(cudaStreamSynchronize(s));
    return;
  }
  staging().to_host(dst, src, bytes, s);
}


void alloc_list(LeafList& l, long long cnt, long long nslots, cudaStream_t s) {
  l.count = cnt;
  l.rl.alloc(cnt, s);
  l.m.alloc(cnt, s);
  l.cl.alloc(cnt, s);
  l.n.alloc(cnt, s);
  l.tau_slot.alloc(cnt, s);
  l.sigma_slot.alloc(cnt, s);
  l.depth.alloc(cnt, s);
  l.run_start.alloc(nslots, s);
  l.run_end.alloc(nslots, s);
  l.run_start.fill_bytes(0xff, s);  // -1: no run
  l.run_end.fill_bytes(0xff, s);
}

template <class T>
void grow(DevBuf<T>& b, size_t need, size_t keep, cudaStream_t s) {
  if (b.size() >= need) return;
  DevBuf<T> nb;
  nb.alloc(std::max(need, b.size() * 2), s);
  if (keep) HM_CUDA(cudaMemcpyAsync(nb.get(), b.get(), keep * sizeof(T), cudaMemcpyDeviceToDevice, s));
  b = std::move(nb);
}

}  // namespace

void upload_staged(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes < (size_t(8) << 20)) {
    HM_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    HM_CUDA(cudaStreamSynchronize(s));  // pageable source: completes before return anyway
    return;
  }
  staging().to_device(dst, src, bytes, s);
}

void morton_codes_device(const double* coords, long long n, int d, unsigned long long* codes, cudaStream_t s) {
  morton_kernel<<<grid_for(n, 256, 1 << 16), 256, 0, s>>>(coords, n, d, codes);
  HM_LAUNCH_CHECK();
}

void HandleStreams::create(int dev) {
  device = dev;
  HM_CUDA(cudaSetDevice(dev));
  HM_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  HM_CUDA(cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking));
  HM_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
  HM_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
  HM_CUDA(cudaEventCreateWithFlags(&ev_last, cudaEventDisableTiming));
  for (cudaEvent_t& e : ev_ph) HM_CUDA(cudaEventCreate(&e));
  for (cudaEvent_t& e : ev_chunk) HM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

HandleStreams::~HandleStreams() {
  cudaSetDevice(device);
  if (stream) cudaStreamSynchronize(stream);
  if (aux) cudaStreamSynchronize(aux);
  if (stream) cudaStreamDestroy(stream);
  if (aux) cudaStreamDestroy(aux);
  for (cudaEvent_t e : {ev_fork, ev_join, ev_last, ev_ph[0], ev_ph[1], ev_ph[2], ev_ph[3]})
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : ev_chunk)
    if (e) cudaEventDestroy(e);
}

HMatrix::~HMatrix() {
  cudaSetDevice(device);
  if (stream) cudaStreamSynchronize(stream);
  if (aux) cudaStreamSynchronize(aux);
}

void build_hmatrix(HMatrix& h, const double* coords_in) {
  cudaStream_t s = h.stream;
  const long long n = h.n;
  const int d = h.d;
  const Config& cfg = h.cfg;
  if (n < 1) raise(kEinval, "build_block_cluster_tree: empty point set");
  if (d < 1 || d > 20) raise(kEinval, "dimension must be in [1, 20]");
  if (n > (1ll << 27)) raise(kErange, "N > 2^27 points is not supported by the packed leaf key");
  const auto t_setup = Clock::now();

  // ---- K1/K2: Morton codes, stable sort, gather (morton.cpp:50-71)
  const auto t0 = Clock::now();
  {
    DevBuf<int> flag;
    flag.alloc(1, s);
    flag.zero(s);
    nonfinite_kernel<<<grid_for(n * d, 256, 1 << 16), 256, 0, s>>>(coords_in, n * d, flag.get());
    HM_LAUNCH_CHECK();
    int hflag = 0;
    HM_CUDA(cudaMemcpyAsync(&hflag, flag.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    HM_CUDA(cudaStreamSynchronize(s));
    if (hflag) raise(kEinval, "setup: non-finite coordinate");
  }
  h.codes.alloc(n, s);
  morton_codes_device(coords_in, n, d, h.codes.get(), s);
  DevBuf<unsigned long long> keys;
  DevBuf<unsigned> order;
  keys.alloc(n, s);
  order.alloc(n, s);
  HM_CUDA(cudaMemcpyAsync(keys.get(), h.codes.get(), sizeof(unsigned long long) * n, cudaMemcpyDeviceToDevice, s));
  iota_u32(order.get(), n, s);
  radix_sort_pairs(keys.get(), order.get(), n, s);
  h.coords.alloc(static_cast<size_t>(n) * d, s);
  h.perm.alloc(n, s);
  gather_points_kernel<<<grid_for(n, 256, 1 << 16), 256, 0, s>>>(coords_in, order.get(), n, d, nullptr,
                                                                 h.coords.get(), h.perm.get());
  HM_LAUNCH_CHECK();
  keys.reset();
  order.reset();
  HM_CUDA(cudaStreamSynchronize(s));
  h.tm.morton_ms = ms_since(t0);

  // ---- K3: cluster table + box pyramid
  const auto t1 = Clock::now();
  int dcap = 0;
  while (dcap < 62 && (((n - 1) >> dcap) + 1) > cfg.c_leaf) ++dcap;  // ceil(n/2^dcap) <= c_leaf
  h.dcap = dcap;
  h.depth_base.resize(dcap + 2);
  for (int e = 0; e <= dcap + 1; ++e) h.depth_base[e] = (1ll << e) - 1;
  h.nslots = h.depth_base[dcap + 1];
  if (h.nslots > (1ll << 31) - 1) raise(kErange, "cluster table too large (c_leaf too small for N)");
  h.slot_lo.alloc(h.nslots, s);
  h.slot_hi.alloc(h.nslots, s);
  slot_ranges_kernel<<<grid_for(h.nslots, 256, 1 << 16), 256, 0, s>>>(n, dcap, h.nslots, h.slot_lo.get(),
                                                                      h.slot_hi.get());
  HM_LAUNCH_CHECK();
  h.boxes.alloc(static_cast<size_t>(h.nslots) * 2 * d, s);
  {
    const long long cnt = 1ll << dcap;
    leaf_boxes_kernel<<<grid_for(cnt * 32, 256), 256, 0, s>>>(h.coords.get(), n, d, h.depth_base[dcap], cnt,
                                                              h.slot_lo.get(), h.slot_hi.get(), h.boxes.get());
    HM_LAUNCH_CHECK();
    for (int e = dcap - 1; e >= 0; --e) {
      const long long c = 1ll << e;
      parent_boxes_kernel<<<grid_for(c * d, 256, 1 << 16), 256, 0, s>>>(d, h.depth_base[e], c, h.depth_base[e + 1],
                                                                       h.boxes.get());
      HM_LAUNCH_CHECK();
    }
  }

  // ---- K4: level-synchronous traversal (tree.hpp:44-62)
  DevBuf<unsigned> tau, sigma, ntau, nsigma;
  tau.alloc(1, s);
  sigma.alloc(1, s);
  tau.zero(s);
  sigma.zero(s);
  long long width = 1;
  DevBuf<unsigned long long> lkey;
  DevBuf<unsigned> ltau, lsigma;
  DevBuf<unsigned char> ldepth, ladm;
  long long L = 0;
  DevBuf<long long> packed;
  DevBuf<unsigned char> adm;
  int level = 0;
  int dmax_leaf = 0;
  while (width > 0) {
    if (level > dcap) raise(kElogic, "traversal deeper than the cluster table");
    packed.alloc(width + 1, s);
    adm.alloc(width, s);
    LevelArgs a{tau.get(), sigma.get(), width, h.depth_base[level], h.slot_lo.get(), h.slot_hi.get(),
                h.boxes.get(), d, cfg.eta, cfg.c_leaf, cfg.mode};
    classify_kernel<<<grid_for(width, 256, 1 << 16), 256, 0, s>>>(a, packed.get(), adm.get());
    HM_LAUNCH_CHECK();
    const long long tot = exclusive_scan_i64(packed.get(), packed.get(), width, s);
    const long long nchild = tot >> 32, nleaf = tot & 0xffffffffll;
    if (nleaf) dmax_leaf = level;
    if (nchild > (1ll << 32) - 1) raise(kErange, "tree level too wide");
    grow(lkey, L + nleaf, L, s);
    grow(ltau, L + nleaf, L, s);
    grow(lsigma, L + nleaf, L, s);
    grow(ldepth, L + nleaf, L, s);
    grow(ladm, L + nleaf, L, s);
    ntau.alloc(std::max(nchild, 1ll), s);
    nsigma.alloc(std::max(nchild, 1ll), s);
    emit_kernel<<<grid_for(width, 256, 1 << 16), 256, 0, s>>>(a, level, packed.get(), adm.get(), ntau.get(),
                                                              nsigma.get(), L, lkey.get(), ltau.get(), lsigma.get(),
                                                              ldepth.get(), ladm.get());
    HM_LAUNCH_CHECK();
    L += nleaf;
    tau = std::move(ntau);
    sigma = std::move(nsigma);
    width = nchild;
    ++level;
  }
  h.dmax_leaf = dmax_leaf;
  tau.reset();
  sigma.reset();
  packed.reset();
  adm.reset();

  // ---- K5: canonical order (radix sort on the packed key) + stable split by flag
  DevBuf<unsigned> lorder;
  lorder.alloc(L, s);
  iota_u32(lorder.get(), L, s);
  radix_sort_pairs(lkey.get(), lorder.get(), L, s);
  lkey.reset();
  DevBuf<unsigned> stau, ssigma;
  DevBuf<unsigned char> sdepth;
  DevBuf<long long> split_in, split_off;
  stau.alloc(L, s);
  ssigma.alloc(L, s);
  sdepth.alloc(L, s);
  split_in.alloc(L, s);
  split_off.alloc(L, s);
  permute_leaves_kernel<<<grid_for(L, 256, 1 << 16), 256, 0, s>>>(lorder.get(), L, ltau.get(), lsigma.get(),
                                                                  ldepth.get(), ladm.get(), stau.get(),
                                                                  ssigma.get(), sdepth.get(), split_in.get());
  HM_LAUNCH_CHECK();
  const long long stot = exclusive_scan_i64(split_in.get(), split_off.get(), L, s);
  const long long n_aca = stot >> 32, n_dense = stot & 0xffffffffll;
  alloc_list(h.dense, n_dense, h.nslots, s);
  alloc_list(h.aca, n_aca, h.nslots, s);
  DevBuf<long long> dbase;
  dbase.alloc(h.depth_base.size(), s);
  HM_CUDA(cudaMemcpyAsync(dbase.get(), h.depth_base.data(), sizeof(long long) * h.depth_base.size(),
                          cudaMemcpyHostToDevice, s));
  split_kernel<<<grid_for(L, 256, 1 << 16), 256, 0, s>>>(
      L, split_off.get(), split_in.get(), stau.get(), ssigma.get(), sdepth.get(), dbase.get(), h.slot_lo.get(),
      h.slot_hi.get(), h.dense.rl.get(), h.dense.m.get(), h.dense.cl.get(), h.dense.n.get(), h.dense.tau_slot.get(),
      h.dense.sigma_slot.get(), h.dense.depth.get(), h.aca.rl.get(), h.aca.m.get(), h.aca.cl.get(), h.aca.n.get(),
      h.aca.tau_slot.get(), h.aca.sigma_slot.get(), h.aca.depth.get());
  HM_LAUNCH_CHECK();
  for (LeafList* l : {&h.dense, &h.aca}) {
    if (l->count) {
      runs_kernel<<<grid_for(l->count, 256, 1 << 16), 256, 0, s>>>(l->count, l->tau_slot.get(), l->run_start.get(),
                                                                    l->run_end.get());
      HM_LAUNCH_CHECK();
    }
    l->h_rl.resize(l->count);
    l->h_m.resize(l->count);
    l->h_cl.resize(l->count);
    l->h_n.resize(l->count);
    mirror_to_host(l->h_rl.data(), l->rl.get(), l->count, s);
    mirror_to_host(l->h_m.data(), l->m.get(), l->count, s);
    mirror_to_host(l->h_cl.data(), l->cl.get(), l->count, s);
    mirror_to_host(l->h_n.data(), l->n.get(), l->count, s);
  }
  HM_CUDA(cudaStreamSynchronize(s));
  build_spans(h, s);
  h.tm.tree_ms = ms_since(t1);

  // algorithmic sizes (host threads over the mirrors; integer partial sums, exact)
  {
    std::mutex mu;
    long long sd = 0, sm = 0, sn = 0;
    parallel_blocks(h.dense.count, [&](long long b0, long long b1) {
      long long a = 0;
      for (long long i = b0; i < b1; ++i) a += static_cast<long long>(h.dense.h_m[i]) * h.dense.h_n[i];
      std::lock_guard<std::mutex> lk(mu);
      sd += a;
    });
    parallel_blocks(h.aca.count, [&](long long b0, long long b1) {
      long long a = 0, b = 0;
      for (long long i = b0; i < b1; ++i) {
        a += h.aca.h_m[i];
        b += h.aca.h_n[i];
      }
      std::lock_guard<std::mutex> lk(mu);
      sm += a;
      sn += b;
    });
    h.S_d = static_cast<double>(sd);
    h.sum_m_adm = static_cast<double>(sm);
    h.sum_n_adm = static_cast<double>(sn);
  }

  // ---- row ownership: rank g owns the depth-log2(world) cluster g
  if (cfg.world > 1) {
    int g = 0;
    while ((1 << g) < cfg.world) ++g;
    if ((1 << g) != cfg.world) raise(kEinval, "world size must be a power of two");
    if (g > dcap) raise(kErange, "too many ranks for the cluster tree depth");
    const long long slot = h.depth_base[g] + cfg.rank;
    long long lo, hi;
    HM_CUDA(cudaMemcpy(&lo, h.slot_lo.get() + slot, sizeof(long long), cudaMemcpyDeviceToHost));
    HM_CUDA(cudaMemcpy(&hi, h.slot_hi.get() + slot, sizeof(long long), cudaMemcpyDeviceToHost));
    h.row_begin = lo;
    h.row_end = hi;
    for (LeafList* l : {&h.dense, &h.aca})
      for (long long i = 0; i < l->count; ++i)
        if (l->h_rl[i] < hi && lo < l->h_rl[i] + l->h_m[i] && (l->h_rl[i] < lo || l->h_rl[i] + l->h_m[i] > hi))
          raise(kErange, "a leaf straddles the row partition (leaf above the partition depth)");
  } else {
    h.row_begin = 0;
    h.row_end = n;
  }
  {
    std::mutex mu;
    long long own = 0;
    parallel_blocks(h.dense.count, [&](long long b0, long long b1) {
      long long a = 0;
      for (long long i = b0; i < b1; ++i)
        if (h.dense.h_rl[i] >= h.row_begin && h.dense.h_rl[i] < h.row_end)
          a += static_cast<long long>(h.dense.h_m[i]) * h.dense.h_n[i];
      std::lock_guard<std::mutex> lk(mu);
      own += a;
    });
    h.S_d_own = static_cast<double>(own);
  }
  h.tm.setup_ms = ms_since(t_setup);
}

}  // namespace hmb

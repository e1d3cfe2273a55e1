// aca.cu -- K7: batched adaptive cross approximation on sm_100a.
//
// Semantics: aca_batched_impl (proj/src/aca.cpp:268-544) per block, which is
// independent of batch composition: for r < k
//   (i)   candidate = first unused column                          aca.cpp:333
//   (ii)  u_hat = A(:,j) - sum_{l<r} u_l * v_l[j]   (l ascending, mul then sub)  :363-364
//   (iii) norm2 = left fold of u_hat^2; argmax |u_hat| over unused rows, first wins :373-376
//   (iv)  qualified <=> best > 0 && (first cross || norm2 > 1e-28 * scale2)       :381-383
//   (v)   else the column is consumed and later columns are scanned               :400-444
//   (vi)  u_r = u_hat / u_hat[p]                                                  :466-470
//   (vii) v_r = A(p,:) - sum_l u_l[p] * v_l                                       :474-481
//   (viii) pivots, scale2 = norm2 of the first accepted column                    :485-494
//   (ix)  optional epsilon criterion                                              :497-538
// Every rejected column is consumed, so the consumed columns always form a
// prefix: the per-block state is a single "next column" pointer.
//
// B200 mapping: blocks are binned by max(m, n) and each bin runs its own persistent
// kernel over a largest-first queue (compute_aca):
//   <= 64 .. 1024 rows   aca_win_kernel     team of NW = 1..16 warps per block, rows in
//                                           registers, shared-memory window of candidate
//                                           columns (speculative, nothing re-evaluated)
//   <= 2048 / 4096       aca_cluster_kernel thread-block cluster of 4 / 8 CTAs, partials
//                                           and pivots exchanged through distributed
//                                           shared memory
//   larger               aca_big_kernel     one CTA, L2-resident window column scratch
//   epsilon, k > 32      aca_kernel         the general CTA-per-block path
// Entries are bit-identical to the host (glibc exp/log ports, no FMA contraction), the
// residual chains run in the reference's order (aca_chain.cuh), so u/v and the pivots
// are bitwise the reference's.  The only order-sensitive quantities, norm2 and scale2,
// are summed in parallel with a rigorous error bound; decisions inside the bound fall
// back to the reference's sequential folds.
#pragma once
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "hmatrix.h"
#include "primitives.h"
#include "aca_chain.cuh"

namespace hmb {

namespace aca_detail {

// HM_TRACE=1: per-phase device times of the factorisation on stderr (development aid)
struct PhaseTrace {
  bool on = std::getenv("HM_TRACE") != nullptr;
  cudaEvent_t e[16];
  const char* name[16];
  int k = 0;
  void mark(const char* nm, cudaStream_t s) {
    if (!on || k >= 16) return;
    cudaEventCreate(&e[k]);
    cudaEventRecord(e[k], s);
    name[k++] = nm;
  }
  void dump() {
    if (!on || k == 0) return;
    cudaEventSynchronize(e[k - 1]);
    for (int i = 1; i < k; ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, e[i - 1], e[i]);
      std::fprintf(stderr, "[hm_trace] %-24s %9.3f ms\n", name[i], ms);
    }
    for (int i = 0; i < k; ++i) cudaEventDestroy(e[i]);
    k = 0;
  }
};

constexpr int kAcaThreads = 256;
constexpr int kKmax = 64;        // compile-time cap on the rank
constexpr int kColBuf = 2048;    // doubles of shared column buffer

// entry sources ---------------------------------------------------------------
// KIND: -1 runtime kernel kind, 0 Gaussian, 1 Matern (compile-time specialisation
// keeps the Bessel code out of the Gaussian kernels' registers).
template <int KIND>
__device__ __forceinline__ double phi_kind(const KernelParams& kp, double r2) {
  if constexpr (KIND == 0) return glibc_exp(-r2);
  else if constexpr (KIND == 1) {
    if (r2 == 0.0) return kp.matern_norm;
    const double r = hm_sqrt(r2);
    return hmul(hmul(bessel_k1(r), r), kp.matern_norm);
  } else {
    return phi_r2(kp, r2);
  }
}

template <int DIM, int KIND = -1>
struct KernelEntry {
  const double* coords;
  long long n;
  int d;
  KernelParams kp;
  // point coordinates of row (absolute) i into registers
  __device__ __forceinline__ void load(long long i, double* y) const {
    if constexpr (DIM > 0) {
#pragma unroll
      for (int a = 0; a < DIM; ++a) y[a] = __ldg(coords + a * n + i);
    } else {
      for (int a = 0; a < d; ++a) y[a] = __ldg(coords + a * n + i);
    }
  }
  // phi(y_row, point j): r2 = ((0 + dx0^2) + dx1^2) + ..., dx = row - col
  __device__ __forceinline__ double eval(const double* y, long long j) const {
    double r2 = 0.0;
    if constexpr (DIM > 0) {
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        const double dx = hsub(y[a], __ldg(coords + a * n + j));
        r2 = hadd(r2, hmul(dx, dx));
      }
    } else {
      for (int a = 0; a < d; ++a) {
        const double dx = hsub(y[a], __ldg(coords + a * n + j));
        r2 = hadd(r2, hmul(dx, dx));
      }
    }
    return phi_kind<KIND>(kp, r2);
  }
  __device__ __forceinline__ double r2_of(const double* y, long long j) const {
    double r2 = 0.0;
    if constexpr (DIM > 0) {
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        const double dx = hsub(y[a], __ldg(coords + a * n + j));
        r2 = hadd(r2, hmul(dx, dx));
      }
    } else {
      for (int a = 0; a < d; ++a) {
        const double dx = hsub(y[a], __ldg(coords + a * n + j));
        r2 = hadd(r2, hmul(dx, dx));
      }
    }
    return r2;
  }
  // two entries with overlapped dependency chains (kernel_math.cuh phi_x2), bitwise equal
  // to two eval() calls: rows y0, y1 against point j, or row y against points j0, j1
  __device__ __forceinline__ void eval2(const double* y0, const double* y1, long long j, double& a0,
                                        double& a1) const {
    if constexpr (KIND >= 0) {
      phi_x2<KIND>(kp, r2_of(y0, j), r2_of(y1, j), a0, a1);
    } else {
      a0 = eval(y0, j);
      a1 = eval(y1, j);
    }
  }
  // r2 between two points held in registers / shared memory (no global loads)
  __device__ __forceinline__ static double r2_pts(const double* y, const double* z) {
    double r2 = 0.0;
#pragma unroll
    for (int a = 0; a < (DIM > 0 ? DIM : 1); ++a) {
      const double dx = hsub(y[a], z[a]);
      r2 = hadd(r2, hmul(dx, dx));
    }
    return r2;
  }
  __device__ __forceinline__ void phi2(double r2a, double r2b, double& a0, double& a1) const {
    if constexpr (KIND >= 0) {
      phi_x2<KIND>(kp, r2a, r2b, a0, a1);
    } else {
      a0 = phi_r2(kp, r2a);
      a1 = phi_r2(kp, r2b);
    }
  }
  // three entries from squared distances (bitwise three scalar evaluations)
  __device__ __forceinline__ void phi3(double r2a, double r2b, double r2c, double& a0, double& a1,
                                       double& a2) const {
    if constexpr (KIND >= 0) {
      const double r2[3] = {r2a, r2b, r2c};
      double f[3];
      phi_xv<KIND, 3>(kp, r2, f);
      a0 = f[0];
      a1 = f[1];
      a2 = f[2];
    } else {
      a0 = phi_r2(kp, r2a);
      a1 = phi_r2(kp, r2b);
      a2 = phi_r2(kp, r2c);
    }
  }
  // four entries: row y against points j0, j1 and rows z0, z1 against point jc
  __device__ __forceinline__ void eval4(const double* y, long long j0, long long j1, const double* z0,
                                        const double* z1, long long jc, double& a0, double& a1, double& c0,
                                        double& c1) const {
    if constexpr (KIND >= 0) {
      const double r2[4] = {r2_of(y, j0), r2_of(y, j1), r2_of(z0, jc), r2_of(z1, jc)};
      double f[4];
      phi_xv<KIND, 4>(kp, r2, f);
      a0 = f[0];
      a1 = f[1];
      c0 = f[2];
      c1 = f[3];
    } else {
      a0 = eval(y, j0);
      a1 = eval(y, j1);
      c0 = eval(z0, jc);
      c1 = eval(z1, jc);
    }
  }
  // row y against four points (bitwise four eval() calls)
  __device__ __forceinline__ void eval4c(const double* y, long long j0, long long j1, long long j2, long long j3,
                                         double& a0, double& a1, double& a2, double& a3) const {
    if constexpr (KIND >= 0) {
      const double r2[4] = {r2_of(y, j0), r2_of(y, j1), r2_of(y, j2), r2_of(y, j3)};
      double f[4];
      phi_xv<KIND, 4>(kp, r2, f);
      a0 = f[0];
      a1 = f[1];
      a2 = f[2];
      a3 = f[3];
    } else {
      a0 = eval(y, j0);
      a1 = eval(y, j1);
      a2 = eval(y, j2);
      a3 = eval(y, j3);
    }
  }
  __device__ __forceinline__ void eval2c(const double* y, long long j0, long long j1, double& a0, double& a1) const {
    if constexpr (KIND >= 0) {
      phi_x2<KIND>(kp, r2_of(y, j0), r2_of(y, j1), a0, a1);
    } else {
      a0 = eval(y, j0);
      a1 = eval(y, j1);
    }
  }
};

struct AcaJob {
  // leaf arrays (absolute leaf index)
  const int* rl;
  const int* m;
  const int* cl;
  const int* nn;
  const int* order;         // leaf indices to process
  long long njobs;
  const long long* u_off;   // absolute offsets; minus u_base / v_base
  const long long* v_off;
  long long u_base, v_base;
  double* U;
  double* V;
  int* k_eff;               // per absolute leaf
  int* row_piv;             // per absolute leaf x kmax
  int* col_piv;
  int kmax;
  int has_eps;
  double eps_factor;        // eps (1 - eta) / (1 + eps), aca.cpp:49
  int* counter;
  unsigned long long* rejections;
  unsigned long long* evals;  // optional (HM_TRACE): [0] column-scan entries, [1] pivot-row entries, [2] blocks
  int tile_shift;           // -1: U rank-major; else log2(S), U row-tiled by S rows
  const int* njobs_dev = nullptr;  // job count on the device (fallback lists), overrides njobs
  int* fb_list = nullptr;   // smooth kernel: blocks that hit a rejection are appended here
  int* fb_count = nullptr;
  int win_one = 0;          // window kernels: one fresh column per rank until a rejection (d >= 3)
  // explicit-matrix seam: block b entries at dense + dense_off[b], row-major m x n
  const double* dense;
  const long long* dense_off;
};

// u_hat[i] / pivot (aca.cpp:466-470), correctly rounded: the pivot's correctly rounded
// reciprocal y and one Markstein correction, q = a*y, r = fma(-q, p, a) (exact),
// q' = fma(r, y, q) -- the IEEE quotient for operands in [2^-500, 2^500] (checked bit for
// bit by tests/cpp/div_const_check.c); a zero numerator gives the signed zero, other
// out-of-range operands take the IEEE division.  One reciprocal per rank instead of m
// full divisions.
static __device__ __noinline__ double ieee_div_slow(double a, double p) { return __ddiv_rn(a, p); }

struct PivotDiv {
  double p, y;
  bool fast;
  __device__ __forceinline__ explicit PivotDiv(double pv) : p(pv) {
    const double ap = fabs(pv);
    fast = ap >= 0x1p-500 && ap <= 0x1p500;
    y = fast ? __drcp_rn(pv) : 0.0;
  }
  __device__ __forceinline__ double operator()(double a) const {
    const double aa = fabs(a);
    // a == 0 is the common case off the fast range: every earlier pivot row's residual is
    // exactly +0 (its fold repeats v_l's), so each rank would otherwise send a few lanes of
    // every warp down the out-of-line division.  0 / p is the zero with the xor'ed sign.
    if (fast && (aa == 0.0 || (aa >= 0x1p-500 && aa <= 0x1p500))) {
      const double q = __dmul_rn(a, y);
      const double r = __fma_rn(-q, p, a);
      const double z = __longlong_as_double((__double_as_longlong(a) ^ __double_as_longlong(p)) &
                                            static_cast<long long>(0x8000000000000000ull));
      return aa == 0.0 ? z : __fma_rn(r, y, q);
    }
    return ieee_div_slow(a, p);  // out of line: keeps the hot loops' register footprint
  }
};

// L1 prefetch of one line (a column's interleaved V row, k = 16 doubles = 128 B): issued
// before an entry evaluation so the residual chain that follows finds v_l in L1
__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

__device__ __forceinline__ void argmax_combine(double& bv, int& bi, double ov, int oi) {
  if (ov > bv || (ov == bv && oi < bi)) {
    bv = ov;
    bi = oi;
  }
}

// Warp argmax of non-negative finite values, first (smallest) index on ties, with three
// redux.sync instructions instead of five shuffle rounds: non-negative doubles order like
// their bit patterns, so the maximum is (max high word, max low word among those lanes).
// "No candidate" is (+0, INT_MAX); a zero maximum is rejected by the caller anyway.
__device__ __forceinline__ void warp_argmax_nonneg(double& bv, int& bi) {
  const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(bv));
  const unsigned hi = static_cast<unsigned>(u >> 32), lo = static_cast<unsigned>(u);
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  const bool top = hi == mhi && lo == mlo;
  bi = static_cast<int>(__reduce_min_sync(0xffffffffu, top ? static_cast<unsigned>(bi) : 0x7fffffffu));
  bv = __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(mhi) << 32) | mlo));
}

template <int DIM, bool DENSE>
__global__ void __launch_bounds__(kAcaThreads) aca_kernel(AcaJob J, KernelEntry<DIM> E) {
  __shared__ double s_col[kColBuf];
  __shared__ double s_vj[8][kKmax];   // v_l[cand] per wave column (W <= 8)
  __shared__ double s_upiv[kKmax];
  __shared__ int s_piv[kKmax];
  __shared__ double s_wsum[kAcaThreads / 32];
  __shared__ double s_wbv[kAcaThreads / 32];
  __shared__ int s_wbi[kAcaThreads / 32];
  __shared__ int s_job, s_next, s_acc, s_prow, s_stop;
  __shared__ double s_scale, s_frob;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double kEps0sq = 1e-14 * 1e-14;  // aca.cpp:32, kEps0 * kEps0

  for (;;) {
    if (tid == 0) s_job = atomicAdd(J.counter, 1);
    __syncthreads();
    const int job = s_job;
    if (job >= J.njobs) return;
    const int b = J.order[job];
    const int rl = J.rl[b], m = J.m[b], cl = J.cl[b], n = J.nn[b];
    const int kmax = J.kmax;
    double* U = J.U + (J.u_off[b] - J.u_base);  // kmax x m: rank-major, or row-tiled (tile_shift >= 0)
    double* V = J.V + (J.v_off[b] - J.v_base);  // n x kmax, interleaved
    const double* A = DENSE ? J.dense + J.dense_off[b] : nullptr;
    // U element (l, i): rank-major l*m + i, or tiled [i / S][l][i % S] so that the
    // k x S slice of one row tile is contiguous for the product's bulk copies
    const int tsh = J.tile_shift;
    auto uix = [&](int l, int i) -> long long {
      if (tsh < 0) return static_cast<long long>(l) * m + i;
      return ((static_cast<long long>(i >> tsh) * kmax + l) << tsh) + (i & ((1 << tsh) - 1));
    };

    int G = 32;
    while (G < m && G < kAcaThreads) G <<= 1;
    const int W = kAcaThreads / G;
    const int g = tid / G, lt = tid % G;
    const bool col_in_smem = static_cast<long long>(W) * m <= kColBuf;

    if (tid == 0) {
      s_next = 0;
      s_stop = 0;
      s_scale = -1.0;
      s_frob = 0.0;
    }
    for (int l = tid; l < kmax; l += kAcaThreads) {
      J.row_piv[static_cast<long long>(b) * kmax + l] = -1;
      J.col_piv[static_cast<long long>(b) * kmax + l] = -1;
    }
    __syncthreads();
    int k_eff = 0;
    unsigned long long rejections = 0;

    for (int r = 0; r < kmax; ++r) {
      // ---------------- column search: waves of W candidate columns
      bool accepted = false;
      while (!accepted) {
        const int next = s_next;
        if (next >= n) break;
        // v_l[cand] of every wave column (aca.cpp:349-352)
        for (int q = tid; q < W * r; q += kAcaThreads) {
          const int gg = q / r, l = q % r;
          const int c = next + gg;
          s_vj[gg][l] = c < n ? V[static_cast<long long>(c) * kmax + l] : 0.0;
        }
        __syncthreads();
        const int c = next + g;
        const bool valid = c < n;
        double sum = 0.0, bv = -1.0;
        int bi = 0x7fffffff;
        if (valid) {
          for (int i = lt; i < m; i += G) {
            double a;
            if constexpr (DENSE) {
              a = A[static_cast<long long>(i) * n + c];
            } else {
              double y[DIM > 0 ? DIM : 20];
              E.load(rl + i, y);
              a = E.eval(y, cl + c);
            }
            for (int l = 0; l < r; ++l) a = hsub(a, hmul(U[uix(l, i)], s_vj[g][l]));
            if (col_in_smem) s_col[g * m + i] = a;
            else U[uix(r, i)] = a;
            sum = hadd(sum, hmul(a, a));
            bool used = false;
            for (int l = 0; l < r; ++l) used |= (s_piv[l] == i);
            const double av = fabs(a);
            if (!used && av > bv) {
              bv = av;
              bi = i;
            }
          }
        }
        // group reduction: warp shuffles, then across the G/32 warps of the group
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          sum = hadd(sum, __shfl_xor_sync(0xffffffffu, sum, o));
          const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          argmax_combine(bv, bi, ov, oi);
        }
        if (lane == 0) {
          s_wsum[warp] = sum;
          s_wbv[warp] = bv;
          s_wbi[warp] = bi;
        }
        __syncthreads();
        if (tid == 0) {
          const int wpg = G / 32;
          int acc = -1, consumed = 0;
          for (int gg = 0; gg < W && next + gg < n; ++gg) {
            double gs = 0.0, gbv = -1.0;
            int gbi = 0x7fffffff;
            for (int w = gg * wpg; w < (gg + 1) * wpg; ++w) {
              gs = hadd(gs, s_wsum[w]);
              argmax_combine(gbv, gbi, s_wbv[w], s_wbi[w]);
            }
            bool q = false;
            if (gbv > 0.0) {
              if (s_scale < 0.0) {
                q = true;
              } else {
                // parallel sum vs the reference's left fold: both within gamma_m * S of
                // the exact sum S of the (bitwise identical) squares
                const double T = hmul(kEps0sq, s_scale);
                const double gm = static_cast<double>(m) * 1.2e-16;
                const double lo = hmul(gs, 1.0 - 4.0 * gm), hi = hmul(gs, 1.0 + 4.0 * gm);
                if (lo > T) {
                  q = true;
                } else if (hi <= T) {
                  q = false;
                } else {  // ambiguous: the reference's sequential fold (aca.cpp:373-374 / 414-415)
                  auto cbv = [&](int i) { return col_in_smem ? s_col[gg * m + i] : U[uix(r, i)]; };
                  double f = hmul(cbv(0), cbv(0));
                  for (int i = 1; i < m; ++i) f = hadd(f, hmul(cbv(i), cbv(i)));
                  q = f > T;
                }
              }
            }
            if (q) {
              acc = gg;
              s_prow = gbi;
              break;
            }
            ++consumed;
          }
          rejections += consumed;
          if (acc >= 0) {
            s_acc = acc;
            s_next = next + acc;  // accepted column index (advanced after bookkeeping)
          } else {
            s_acc = -1;
            s_next = next + consumed;
          }
        }
        __syncthreads();
        accepted = s_acc >= 0;
      }
      if (!accepted) break;  // no usable column left: converged at rank r (aca.cpp:442-443)

      // ---------------- accepted column: pivot, normalise, pivot-row pass
      const int ga = s_acc, cstar = s_next, p = s_prow;
      auto cbv = [&](int i) { return col_in_smem ? s_col[ga * m + i] : U[uix(r, i)]; };
      if (r == 0 && tid == 0) {
        // scale2 = exact left fold of the first accepted column (aca.cpp:491)
        double f = hmul(cbv(0), cbv(0));
        for (int i = 1; i < m; ++i) f = hadd(f, hmul(cbv(i), cbv(i)));
        s_scale = f;
      }
      const double pivot_val = cbv(p);
      for (int l = tid; l < r; l += kAcaThreads) s_upiv[l] = U[uix(l, p)];
      __syncthreads();
      const PivotDiv pdiv(pivot_val);
      for (int i = tid; i < m; i += kAcaThreads) U[uix(r, i)] = pdiv(cbv(i));
      {
        double yp[DIM > 0 ? DIM : 20];
        if constexpr (!DENSE) E.load(rl + p, yp);
        for (int j = tid; j < n; j += kAcaThreads) {
          double a;
          if constexpr (DENSE) a = A[static_cast<long long>(p) * n + j];
          else a = E.eval(yp, cl + j);
          const double* vrow = V + static_cast<long long>(j) * kmax;
          for (int l = 0; l < r; ++l) a = hsub(a, hmul(s_upiv[l], vrow[l]));
          V[static_cast<long long>(j) * kmax + r] = a;
        }
      }
      if (tid == 0) {
        s_piv[r] = p;
        J.row_piv[static_cast<long long>(b) * kmax + r] = p;
        J.col_piv[static_cast<long long>(b) * kmax + r] = cstar;
        s_next = cstar + 1;
      }
      k_eff = r + 1;
      __syncthreads();
      if (J.has_eps) {
        // epsilon criterion with the reference's exact left folds (aca.cpp:497-538); test path
        if (tid == 0) {
          auto ur = [&](int i) { return U[uix(r, i)]; };
          double nu = hmul(ur(0), ur(0));
          for (int i = 1; i < m; ++i) nu = hadd(nu, hmul(ur(i), ur(i)));
          double nv = hmul(V[r], V[r]);
          for (int j = 1; j < n; ++j) nv = hadd(nv, hmul(V[static_cast<long long>(j) * kmax + r], V[static_cast<long long>(j) * kmax + r]));
          double cross = 0.0;
          for (int l = 0; l < r; ++l) {
            double du = hmul(U[uix(l, 0)], ur(0));
            for (int i = 1; i < m; ++i) du = hadd(du, hmul(U[uix(l, i)], ur(i)));
            double dv = hmul(V[l], V[r]);
            for (int j = 1; j < n; ++j)
              dv = hadd(dv, hmul(V[static_cast<long long>(j) * kmax + l], V[static_cast<long long>(j) * kmax + r]));
            cross = hadd(cross, hmul(du, dv));
          }
          s_frob = hadd(s_frob, hadd(hmul(2.0, cross), hmul(nu, nv)));
          const double bound = hmul(J.eps_factor, __dsqrt_rn(s_frob));
          s_stop = hmul(__dsqrt_rn(nu), __dsqrt_rn(nv)) <= bound ? 1 : 0;
        }
        __syncthreads();
        if (s_stop) break;
      }
    }
    if (tid == 0) {
      J.k_eff[b] = k_eff;
      if (J.rejections && rejections) {
        atomicAdd(J.rejections, rejections);  // [0] columns, [1] their entries (sum of m)
        atomicAdd(J.rejections + 1, rejections * static_cast<unsigned long long>(m));
      }
    }
    __syncthreads();
  }
}

template <int DIM>
void launch_kernel_aca(const AcaJob& J, const KernelEntry<DIM>& E, int sms, cudaStream_t s) {
  int occ = 0;
  HM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, aca_kernel<DIM, false>, kAcaThreads, 0));
  const long long grid = std::min<long long>(J.njobs, static_cast<long long>(std::max(occ, 1)) * sms);
  aca_kernel<DIM, false><<<static_cast<unsigned>(std::max(grid, 1ll)), kAcaThreads, 0, s>>>(J, E);
  HM_LAUNCH_CHECK();
}

// Window columns receive the new cross: dst_c[i] -= u_r[i] * v_r[c] for the `filled`
// window columns c.  Batches of 4 columns: the v_r values and the window entries of a
// batch are loaded before any store, so the loads overlap (the compiler cannot hoist
// them across the stores of a plain loop: same array).
template <int RPL, class VAT, class DST>
__device__ __forceinline__ void window_cross(int filled, int next, const double (&ur)[RPL], const bool (&rv)[RPL],
                                             int t, int TT, VAT vat_r, DST dst_of) {
  for (int c0 = 0; c0 < filled; c0 += 4) {
    double vr[4], a[4][RPL];
#pragma unroll
    for (int c = 0; c < 4; ++c) vr[c] = c0 + c < filled ? vat_r(next + c0 + c) : 0.0;
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int q = 0; q < RPL; ++q)
        a[c][q] = (c0 + c < filled && rv[q]) ? dst_of(next + c0 + c)[t + q * TT] : 0.0;
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int q = 0; q < RPL; ++q)
        if (c0 + c < filled && rv[q]) dst_of(next + c0 + c)[t + q * TT] = hsub(a[c][q], hmul(ur[q], vr[c]));
  }
}

// Team barrier: a warp (NW = 1) or a named barrier over the team's NW warps.
template <int NW>
__device__ __forceinline__ void team_sync(int team) {
  if constexpr (NW == 1) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(team + 1), "r"(NW * 32) : "memory");
  }
}

// ---------------------------------------------------------------------------
// Window kernel: the team kernel's row-in-register layout with a SHARED-memory
// window of W candidate columns (ring slots col % W, padded stride).  Columns are
// evaluated W at a time by all threads of the team (fill), their qualification is
// decided by G = TT/W threads per column (partial sums + the rigorous bound, the
// reference's sequential fold when ambiguous), and the unconsumed columns stay in
// the window, receiving each accepted cross as the next step of their chain.  In
// the noise-floor regime (most columns rejected) this turns the scan
// into dense, barrier-amortised evaluation.  v_l lives in shared memory (VSM) or
// directly in the interleaved V factor.
template <int NW, int KC, int W, bool VSM>
__host__ __device__ constexpr size_t win_stride() {
  return static_cast<size_t>(W) * (NW * 64 + 1) + (VSM ? static_cast<size_t>(KC) * NW * 64 : 0) + KC + 2 * NW + W +
         NW * 64 / 8 + 8 + 2 * NW;
}

template <int DIM, int KIND, int NW, int KC, int W, bool VSM, int MINB>
__global__ void __launch_bounds__(NW * 32 < 128 ? 128 : NW * 32, MINB)
    aca_win_kernel(AcaJob J, KernelEntry<DIM, KIND> E, int teams_per_cta) {
  constexpr int RPL = 2;
  constexpr int TT = NW * 32;
  constexpr int NCAP = TT * RPL;
  constexpr int PS = NCAP + 1;  // padded slot stride (bank spread for the per-column folds)
  constexpr int G = TT / W;     // threads per column in the qualification pass
  static_assert(TT % W == 0 && G >= 1 && (G <= 32 || G % 32 == 0), "window / team shape");
  constexpr int GL = G < 32 ? G : 32;  // lanes of one column inside a warp
  constexpr int YD = DIM > 0 ? DIM : 1;
  extern __shared__ double smem[];
  const int team = threadIdx.x / TT, t = threadIdx.x % TT, lane = t & 31, wib = t >> 5;
  if (team >= teams_per_cta) return;
  double* base = smem + static_cast<size_t>(team) * win_stride<NW, KC, W, VSM>();
  double* s_win = base;
  double* s_v = s_win + W * PS;
  double* s_up = s_v + (VSM ? KC * NCAP : 0);
  double* s_rbv = s_up + KC;
  int* s_rbi = reinterpret_cast<int*>(s_rbv + NW);
  int* s_state = reinterpret_cast<int*>(s_rbv + 2 * NW);
  unsigned char* s_used = reinterpret_cast<unsigned char*>(s_rbv + 2 * NW + W);
  double* s_misc = s_rbv + 2 * NW + W + NCAP / 8;  // [0] job, [1] scale, [2] exact-fold verdict
  double* s_fbv = s_misc + 8;                       // NW: fused fast-path argmax (value, index)
  int* s_fbi = reinterpret_cast<int*>(s_fbv + NW);
  const double kEps0sq = 1e-14 * 1e-14;
  const int kmax = J.kmax;
  const bool kpow2 = (kmax & (kmax - 1)) == 0;
  const int kshift = __popc(kmax - 1);

  for (;;) {
    if (t == 0) s_misc[0] = static_cast<double>(atomicAdd(J.counter, 1));
    for (int i = t; i < NCAP; i += TT) s_used[i] = 0;
    team_sync<NW>(team);
    const long long job = static_cast<long long>(s_misc[0]);
    team_sync<NW>(team);
    if (job >= (J.njobs_dev ? static_cast<long long>(*J.njobs_dev) : J.njobs)) return;
    const int b = J.order[job];
    const int rl = J.rl[b], m = J.m[b], cl = J.cl[b], n = J.nn[b];
    double* U = J.U + (J.u_off[b] - J.u_base);
    double* V = J.V + (J.v_off[b] - J.v_base);
    const int tsh = J.tile_shift;
    auto uix = [&](int l, int i) -> long long {
      if (tsh < 0) return static_cast<long long>(l) * m + i;
      return ((static_cast<long long>(i >> tsh) * kmax + l) << tsh) + (i & ((1 << tsh) - 1));
    };
    auto vat = [&](int l, int j) -> double& {
      if constexpr (VSM) return s_v[l * NCAP + j];
      else return V[static_cast<long long>(j) * kmax + l];
    };

    double y[RPL][YD];
    bool rv[RPL];
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
      const int i = t + q * TT;
      rv[q] = i < m;
      if constexpr (DIM > 0) {
#pragma unroll
        for (int a = 0; a < DIM; ++a) y[q][a] = rv[q] ? __ldg(E.coords + a * E.n + rl + i) : 0.0;
      }
    }
    auto entry = [&](int q, long long colpt) -> double {
      if constexpr (DIM > 0) {
        return E.eval(y[q], colpt);
      } else {
        double yy[20];
        E.load(rl + t + q * TT, yy);
        return E.eval(yy, colpt);
      }
    };
    double uR[RPL][KC];  // right-aligned u_l of the own rows (aca_chain.cuh)
#pragma unroll
    for (int q = 0; q < RPL; ++q)
#pragma unroll
      for (int j = 0; j < KC; ++j) uR[q][j] = 0.0;
    int next = 0, filled = 0, k_eff = 0;
    unsigned long long rejections = 0, ev_col = 0, ev_row = 0;
    double scale = -1.0;
    const double gm = static_cast<double>(m) * 1.2e-16;

    for (int r = 0; r < kmax; ++r) {
      int acc_w = -1;
      // fast path: the first window column's norm2, nonzero flag and argmax over unused
      // rows in ONE reduction (the argmax is the pivot when the column qualifies)
      bool fast_ok = false;
      double fbv = 0.0;
      int fbi = 0x7fffffff;
      while (next < n) {
        // speculation depth: while no column was rejected, at most kmax - r more can be
        // accepted (smooth blocks, d >= 3: no noise floor), so do not evaluate past them
        // (win_one, d >= 3: one fresh column per rank, no speculative columns to cross-update)
        const int lim = rejections ? W : (J.win_one ? 1 : max(kmax - r, 1));
        const int wcols = max(filled, min(min(W, lim), n - next));
        ev_col += static_cast<unsigned long long>(wcols - filled) * m;
        // fill: fresh window columns, entry then the reference chain over l < r
        for (int co = filled; co < wcols; ++co) {
          const int col = next + co;
          double* dst = s_win + (col % W) * PS;
          const double* vb;
          int vs;
          if constexpr (VSM) {
            vb = s_v + static_cast<long long>(r - KC) * NCAP + col;
            vs = NCAP;
          } else {
            vb = V + static_cast<long long>(col) * kmax + (r - KC);
            vs = 1;
          }
          double a0, a1;
          if constexpr (DIM > 0) {
            E.eval2(y[0], y[1], cl + col, a0, a1);  // invalid rows: finite dummies, never stored
          } else {
            a0 = rv[0] ? entry(0, cl + col) : 0.0;
            a1 = rv[1] ? entry(1, cl + col) : 0.0;
          }
          Chain<KC>::run2(a0, a1, uR[0], uR[1], r, vb, vs);
          if (rv[0]) dst[t] = a0;
          if (rv[1]) dst[t + TT] = a1;
        }
        filled = wcols;
        team_sync<NW>(team);
        // fast path while the block has rejected nothing (smooth blocks accept the first
        // candidate of every rank): the first window column with all team threads
        int first_state = -1;
        if (rejections == 0) {
          const double* src = s_win + (next % W) * PS;
          double sum = 0.0;
          fbv = 0.0;
          fbi = 0x7fffffff;
#pragma unroll
          for (int q = 0; q < RPL; ++q) {  // rows in increasing order, strict >: first index on ties
            const int i = t + q * TT;
            if (i < m) {
              const double a = src[i];
              sum = hadd(sum, hmul(a, a));
              if (!s_used[i] && fabs(a) > fbv) {
                fbv = fabs(a);
                fbi = i;
              }
            }
          }
#pragma unroll
          for (int o = 16; o; o >>= 1) sum = hadd(sum, __shfl_xor_sync(0xffffffffu, sum, o));
          warp_argmax_nonneg(fbv, fbi);
          if constexpr (NW > 1) {
            // published in s_rbv / s_fbv, read after ONE barrier; the next writer of these
            // slots is the next rank's fast path, several barriers later
            if (lane == 0) {
              s_rbv[wib] = sum;
              s_fbv[wib] = fbv;
              s_fbi[wib] = fbi;
            }
            team_sync<NW>(team);
            sum = s_rbv[0];
            fbv = s_fbv[0];
            fbi = s_fbi[0];
            for (int k2 = 1; k2 < NW; ++k2) {
              sum = hadd(sum, s_rbv[k2]);
              argmax_combine(fbv, fbi, s_fbv[k2], s_fbi[k2]);
            }
          }
          const int nz = fbv > 0.0 ? 1 : 0;
          first_state = 0;
          if (nz) {
            if (scale < 0.0) {
              first_state = 1;
            } else {
              const double T = hmul(kEps0sq, scale);
              const double lo = hmul(sum, 1.0 - 4.0 * gm), hi = hmul(sum, 1.0 + 4.0 * gm);
              first_state = lo > T ? 1 : (hi <= T ? 0 : 2);
            }
          }
        }
        if (first_state == 1) {
          acc_w = 0;
          fast_ok = true;
        } else {
          if constexpr (NW > 1) {
            if (first_state >= 0) team_sync<NW>(team);  // s_rbv is rewritten below
          }
          // qualification: G threads per column; state 0 no, 1 yes, 2 ambiguous
          {
            const int w = t / G, g = t % G;
            double sum = 0.0;
            int nz = 0;
            if (w < wcols) {
              const double* src = s_win + ((next + w) % W) * PS;
              for (int i = g; i < m; i += G) {
                const double a = src[i];
                sum = hadd(sum, hmul(a, a));
                nz |= (!s_used[i] && fabs(a) > 0.0) ? 1 : 0;
              }
            }
  #pragma unroll
            for (int o = GL / 2; o; o >>= 1) {
              sum = hadd(sum, __shfl_xor_sync(0xffffffffu, sum, o));
              nz |= __shfl_xor_sync(0xffffffffu, nz, o);
            }
            if constexpr (G > 32) {  // a column spans G/32 warps: combine their partials in warp order
              if (lane == 0) {
                s_rbv[wib] = sum;
                s_rbi[wib] = nz;
              }
              team_sync<NW>(team);
              if (g == 0 && w < wcols) {
                sum = s_rbv[wib];
                nz = s_rbi[wib];
                for (int k2 = 1; k2 < G / 32; ++k2) {
                  sum = hadd(sum, s_rbv[wib + k2]);
                  nz |= s_rbi[wib + k2];
                }
              }
            }
            if (g == 0 && w < wcols) {
              int st = 0;
              if (nz) {
                if (scale < 0.0) {
                  st = 1;
                } else {
                  const double T = hmul(kEps0sq, scale);
                  const double lo = hmul(sum, 1.0 - 4.0 * gm), hi = hmul(sum, 1.0 + 4.0 * gm);
                  st = lo > T ? 1 : (hi <= T ? 0 : 2);
                }
              }
              s_state[w] = st;
            }
          }
          team_sync<NW>(team);
          for (int w = 0; w < wcols; ++w) {
            int st = s_state[w];
            if (st == 2) {  // the reference's sequential left fold (aca.cpp:373-374 / 414-415)
              if (t == 0) {
                const double* src = s_win + ((next + w) % W) * PS;
                double f = hmul(src[0], src[0]);
                for (int i = 1; i < m; ++i) f = hadd(f, hmul(src[i], src[i]));
                s_misc[2] = f > hmul(kEps0sq, scale) ? 1.0 : 0.0;
              }
              team_sync<NW>(team);
              st = s_misc[2] != 0.0 ? 1 : 0;
              team_sync<NW>(team);
            }
            if (st == 1) {
              acc_w = w;
              break;
            }
          }
        }
        const int consumed = acc_w >= 0 ? acc_w + 1 : wcols;
        rejections += static_cast<unsigned long long>(acc_w >= 0 ? acc_w : wcols);
        next += consumed;
        filled = acc_w >= 0 ? wcols - consumed : 0;
        if (acc_w >= 0) break;
      }
      if (acc_w < 0) break;  // no usable column left (aca.cpp:442-443)
      const int cstar = next - 1;
      const double* acol = s_win + (cstar % W) * PS;

      // pivot row: argmax |u_hat| over unused rows, first index wins (aca.cpp:367, 375-376);
      // the column qualified, so the maximum is > 0 and zero rows never matter
      double bv = fbv;
      int bi = fbi;
      if (!fast_ok) {
        bv = 0.0;
        bi = 0x7fffffff;
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
          const int i = t + q * TT;
          if (rv[q] && !s_used[i]) {
            const double av = fabs(acol[i]);
            if (av > bv) {
              bv = av;
              bi = i;
            }
          }
        }
        warp_argmax_nonneg(bv, bi);
        if constexpr (NW > 1) {
          if (lane == 0) {
            s_rbv[wib] = bv;
            s_rbi[wib] = bi;
          }
          team_sync<NW>(team);
          bv = s_rbv[0];
          bi = s_rbi[0];
          for (int g = 1; g < NW; ++g) argmax_combine(bv, bi, s_rbv[g], s_rbi[g]);
        }
      }
      const int p = bi;
      if (r == 0 && t == 0) {  // scale2 = exact left fold of the first accepted column (aca.cpp:491)
        double f = hmul(acol[0], acol[0]);
        for (int i = 1; i < m; ++i) f = hadd(f, hmul(acol[i], acol[i]));
        s_misc[1] = f;
      }
      const int pt = p % TT, pq = p / TT;
      if (t == pt) {
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
          if (q == pq) {
#pragma unroll
            for (int j = 0; j < KC; ++j)
              if (j >= KC - r) s_up[j - (KC - r)] = uR[q][j];
            if constexpr (DIM > 0) {  // the pivot row's point, from the owner's registers
#pragma unroll
              for (int a = 0; a < DIM; ++a) s_misc[4 + a] = y[q][a];
            }
          }
        }
      }
      team_sync<NW>(team);
      if (r == 0) scale = s_misc[1];
      const PivotDiv pdiv(acol[p]);
      // u_r = u_hat / pivot (aca.cpp:466-470), appended right-aligned
#pragma unroll
      for (int q = 0; q < RPL; ++q) {
        const double nu = rv[q] ? pdiv(acol[t + q * TT]) : 0.0;
#pragma unroll
        for (int j = 0; j + 1 < KC; ++j) uR[q][j] = uR[q][j + 1];
        uR[q][KC - 1] = nu;
      }
      // v_r = A(p,:) - sum_l u_l[p] v_l (aca.cpp:474-481); window columns already hold it
      ev_row += n;
      {
        double yp[DIM > 0 ? DIM : 20];
        if constexpr (DIM > 0) {
#pragma unroll
          for (int a = 0; a < DIM; ++a) yp[a] = s_misc[4 + a];
        } else {
          E.load(rl + p, yp);
        }
        double uP[KC];  // u_l[p], right-aligned (aca_chain.cuh)
#pragma unroll
        for (int j = 0; j < KC; ++j) uP[j] = j >= KC - r ? s_up[j - (KC - r)] : 0.0;
        // two columns per step (j, j + TT): their entry evaluations and chains overlap
        auto vbase = [&](int j) -> const double* {
          if constexpr (VSM) return s_v + static_cast<long long>(r - KC) * NCAP + j;
          else return V + static_cast<long long>(j) * kmax + (r - KC);
        };
        constexpr int VS = VSM ? NCAP : 1;
        for (int j = t; j < n; j += 2 * TT) {
          const int j1 = j + TT;
          const bool in0 = j >= next && j < next + filled;
          const bool ok1 = j1 < n, in1 = ok1 && j1 >= next && j1 < next + filled;
          double a0, a1;
          if (in0 && (in1 || !ok1)) {
            a0 = s_win[(j % W) * PS + p];
            a1 = ok1 ? s_win[(j1 % W) * PS + p] : 0.0;
          } else {
            E.eval2c(yp, cl + j, cl + (ok1 ? j1 : j), a0, a1);
            Chain<KC>::run2v(a0, a1, uP, r, vbase(j), vbase(ok1 ? j1 : j), VS);
            if (in0) a0 = s_win[(j % W) * PS + p];
            if (in1) a1 = s_win[(j1 % W) * PS + p];
          }
          vat(r, j) = a0;
          if (ok1) vat(r, j1) = a1;
        }
      }
      team_sync<NW>(team);
      if (t == pt) s_used[p] = 1;  // after every reader of the old flag (argmax above)
      // window columns receive this cross (next step of their chain)
      {
        double ur[RPL];
#pragma unroll
        for (int q = 0; q < RPL; ++q) ur[q] = uR[q][KC - 1];
        window_cross<RPL>(filled, next, ur, rv, t, TT, [&](int col) { return vat(r, col); },
                          [&](int col) { return s_win + (col % W) * PS; });
      }
      if (t == 0) {
        J.row_piv[static_cast<long long>(b) * kmax + r] = p;
        J.col_piv[static_cast<long long>(b) * kmax + r] = cstar;
      }
      k_eff = r + 1;
    }
    // factors: U (layout uix), V interleaved n x kmax, zero past k_eff
#pragma unroll
    for (int j = 0; j < KC; ++j) {
      const int l = j - (KC - k_eff);
      if (l >= 0) {
#pragma unroll
        for (int q = 0; q < RPL; ++q)
          if (rv[q]) U[uix(l, t + q * TT)] = uR[q][j];
      }
    }
    for (int l = k_eff; l < kmax; ++l)
#pragma unroll
      for (int q = 0; q < RPL; ++q)
        if (rv[q]) U[uix(l, t + q * TT)] = 0.0;
    if constexpr (VSM) {
      team_sync<NW>(team);
      for (int idx = t; idx < n * kmax; idx += TT) {
        // kmax is a power of two in practice (k = 16): shift instead of an integer division
        const int j = kpow2 ? idx >> kshift : idx / kmax, l = idx - j * kmax;
        V[idx] = l < k_eff ? s_v[l * NCAP + j] : 0.0;
      }
    } else {
      for (int idx = t; idx < n * (kmax - k_eff); idx += TT) {
        const int j = idx / (kmax - k_eff), l = k_eff + idx % (kmax - k_eff);
        V[static_cast<long long>(j) * kmax + l] = 0.0;
      }
    }
    for (int l = k_eff + t; l < kmax; l += TT) {
      J.row_piv[static_cast<long long>(b) * kmax + l] = -1;
      J.col_piv[static_cast<long long>(b) * kmax + l] = -1;
    }
    if (t == 0) {
      J.k_eff[b] = k_eff;
      if (J.rejections && rejections) {
        atomicAdd(J.rejections, rejections);  // [0] columns, [1] their entries (sum of m)
        atomicAdd(J.rejections + 1, rejections * static_cast<unsigned long long>(m));
      }
      if (J.evals) {
        atomicAdd(J.evals, ev_col);
        atomicAdd(J.evals + 1, ev_row);
        atomicAdd(J.evals + 2, 1ull);
      }
    }
    team_sync<NW>(team);
  }
}

template <int DIM, int KIND, int NW, int KC, int W, bool VSM, int MINB = 1>
void launch_win(const AcaJob& J, const KernelEntry<DIM, KIND>& E, int sms, cudaStream_t s) {
  if (J.njobs <= 0) return;
  constexpr int teams = NW >= 4 ? 1 : 4 / NW;
  const size_t smem = teams * win_stride<NW, KC, W, VSM>() * sizeof(double);
  auto kfn = aca_win_kernel<DIM, KIND, NW, KC, W, VSM, MINB>;
  HM_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int occ = 0;
  HM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, teams * NW * 32, smem));
  const long long ctas = std::min<long long>((J.njobs + teams - 1) / teams, static_cast<long long>(std::max(occ, 1)) * sms);
  kfn<<<static_cast<unsigned>(std::max(ctas, 1ll)), teams * NW * 32, smem, s>>>(J, E, teams);
  HM_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// Smooth-path kernel (max(m, n) <= 64 NW, k = 16): the regime of every block in d >= 3
// (no candidate column is ever rejected), where the batched ACA is
// a fixed schedule -- the candidate column at rank r is column r.  A team of NW warps
// per block, lane-owned rows i = t, t + 64 NW/2 (u_l of its rows LEFT-aligned in
// registers: no per-rank shifting) and columns j = t, t + 32 NW.
//   * the k raw candidate columns A(:, c) are evaluated up front, all rows at once
//     (independent evaluations, off the per-rank critical path), into shared memory;
//   * per rank: the column's residual chain, ONE fused reduction (norm2 for the
//     qualification test, nonzero flag, argmax over unused rows), the pivot export,
//     u_r, then the pivot row's entries and chain for two columns per thread;
//   * scale2 is a bracket of the parallel norm until a decision needs it exactly.
// If a candidate column is not qualified (a rejection: noise floor, zero column) the
// block is handed to the general window kernel through a fallback list and recomputed
// there from scratch, so every block's factors are bitwise the reference's either way.
// PRE: the k raw candidate columns are evaluated up front into shared memory (more
// shared memory per team, fewer teams per SM) or each rank's column is evaluated in place.
// Compact residual chains of the smooth kernels (HM_SMOOTH_ROLLED): the same
// left folds as SmoothChain (l = 0 .. r-1 in order: bitwise identical), as a loop of four
// predicated steps whose loads issue together, instead of a straight-line case per r --
// O(k) instead of O(k^2) code in the kernels' hot loop (instruction-cache misses were
// 16-21% of the smooth kernels' stall samples).  Indices past r are clamped to k - 1
// (valid shared-memory addresses, results unused).
#ifndef HM_SMOOTH_ROLLED
#define HM_SMOOTH_ROLLED 1
#endif
template <int KC, int US, int VS>
__device__ __forceinline__ void col2_rolled(double& a0, double& a1, const double* u0, const double* u1, int r,
                                            const double* vb) {
#pragma unroll 1
  for (int l0 = 0; l0 < r; l0 += 4) {
    double x0[4], x1[4], w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int l = min(l0 + q, KC - 1);
      x0[q] = u0[l * US];
      x1[q] = u1[l * US];
      w[q] = vb[l * VS];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (l0 + q < r) {
        a0 = hsub(a0, hmul(x0[q], w[q]));
        a1 = hsub(a1, hmul(x1[q], w[q]));
      }
  }
}
template <int KC, int VS, int US>
__device__ __forceinline__ void row2_rolled(double& b0, double& b1, const double* up, const double* vb0,
                                            const double* vb1, int r) {
#pragma unroll 1
  for (int l0 = 0; l0 < r; l0 += 4) {
    double w[4], x0[4], x1[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int l = min(l0 + q, KC - 1);
      w[q] = up[l * US];
      x0[q] = vb0[l * VS];
      x1[q] = vb1[l * VS];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (l0 + q < r) {
        b0 = hsub(b0, hmul(w[q], x0[q]));
        b1 = hsub(b1, hmul(w[q], x1[q]));
      }
  }
}

template <int NW, bool PRE>
__host__ __device__ constexpr size_t smooth_stride() {
  return (PRE ? static_cast<size_t>(16) * (NW * 64 + 1) : static_cast<size_t>(NW * 64 + 1) + 64) +
         static_cast<size_t>(2) * 16 * NW * 64 + 4 + 4 * NW + 8;
}

template <int DIM, int KIND, int NW, bool PRE>
__global__ void __launch_bounds__(128, 3) aca_smooth_kernel(AcaJob J, KernelEntry<DIM, KIND> E, int teams_per_cta) {
  constexpr int KC = 16;
  constexpr int TT = NW * 32, NCAP = 2 * TT, CS = NCAP + 1;
  // compact chains where measured faster (config 3 / config-5 geometry, per class): NW = 1
  // -10% / -11%, NW = 2 Matern -5% (Gaussian +2%), NW = 4 +3% / +8% (straight-line kept)
  constexpr bool kRolled = HM_SMOOTH_ROLLED && (NW == 1 || (NW == 2 && KIND == 1));
  static_assert(DIM > 0, "smooth kernel: compile-time dimension");
  extern __shared__ double smem[];
  const int team = threadIdx.x / TT, t = threadIdx.x % TT, lane = t & 31, wib = t >> 5;
  if (team >= teams_per_cta) return;
  double* base = smem + static_cast<size_t>(team) * smooth_stride<NW, PRE>();
  double* s_col = base;                 // PRE: KC x CS raw candidate columns A(i, c); else 1 x CS scratch
  double* s_v = s_col + (PRE ? KC * CS : CS + 64);  // KC x NCAP: v_l[j]
  double* s_u = s_v + KC * NCAP;        // KC x NCAP: u_l[i] (no dynamic register indexing)
  double* s_yp = s_u + KC * NCAP;       // the pivot row's point
  double* s_cc = s_col + CS;            // (!PRE) points of the k candidate columns, KC x 4
  double* s_red = s_yp + 4;             // NW x 4: per-warp sum, nz, bv, bi
  double* s_misc = s_red + 4 * NW;      // [0] job [1] pivot value [2] exact verdict [3] scale
  const double kEps0sq = 1e-14 * 1e-14;
  const int kmax = J.kmax;

  for (;;) {
    if (t == 0) s_misc[0] = static_cast<double>(atomicAdd(J.counter, 1));
    team_sync<NW>(team);
    const long long job = static_cast<long long>(s_misc[0]);
    team_sync<NW>(team);
    if (job >= J.njobs) return;
    const int b = J.order[job];
    const int rl = J.rl[b], m = J.m[b], cl = J.cl[b], n = J.nn[b];
    const bool rv0 = t < m, rv1 = t + TT < m;
    double y0[DIM], y1[DIM];
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      y0[a] = rv0 ? __ldg(E.coords + a * E.n + rl + t) : 0.0;
      y1[a] = rv1 ? __ldg(E.coords + a * E.n + rl + t + TT) : 0.0;
    }
    // the points of this thread's two columns (row pass) stay in registers; the k candidate
    // columns' points go to shared memory: no global loads on the per-rank critical path
    double yc0[DIM], yc1[DIM];
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      yc0[a] = t < n ? __ldg(E.coords + a * E.n + cl + t) : 0.0;
      yc1[a] = t + TT < n ? __ldg(E.coords + a * E.n + cl + t + TT) : 0.0;
    }
    if constexpr (!PRE) {
      if (t < KC && t < n)
#pragma unroll
        for (int a = 0; a < DIM; ++a) s_cc[t * 4 + a] = yc0[a];
    }
    // raw candidate columns 0 .. min(k, n) - 1, two columns (four entries) at a time
    const int ncol = min(kmax, n);
    for (int c = 0; PRE && c < ncol; c += 2) {
      const int c1 = c + 1 < ncol ? c + 1 : c;
      double a0, a1, b0, b1;
      E.eval2(y0, y1, cl + c, a0, a1);
      E.eval2(y0, y1, cl + c1, b0, b1);
      s_col[c * CS + t] = a0;
      s_col[c * CS + t + TT] = a1;
      s_col[c1 * CS + t] = b0;
      s_col[c1 * CS + t + TT] = b1;
    }
    team_sync<NW>(team);
    bool used0 = false, used1 = false;
    double s_lo = 0.0, s_hi = 0.0, scale = 0.0;
    bool scale_exact = false;
    const double gm = static_cast<double>(m) * 1.2e-16;
    int k_eff = 0;
    bool fallback = false;
    for (int r = 0; r < kmax; ++r) {
      if (r >= n) break;  // no candidate column left: converged (aca.cpp:442-443)
      // column r residual (aca.cpp:363-364), rows of this thread
      double a0, a1;
      if constexpr (PRE) {
        a0 = s_col[r * CS + t];
        a1 = rv1 ? s_col[r * CS + t + TT] : 0.0;
      } else {
        double pc[DIM];
#pragma unroll
        for (int a = 0; a < DIM; ++a) pc[a] = s_cc[r * 4 + a];
        E.phi2(E.r2_pts(y0, pc), E.r2_pts(y1, pc), a0, a1);
        if (!rv1) a1 = 0.0;
      }
      if constexpr (kRolled) col2_rolled<KC, NCAP, NCAP>(a0, a1, s_u + t, s_u + t + TT, r, s_v + r);
      else SmoothChain<KC>::col2s<NCAP>(a0, a1, s_u + t, s_u + t + TT, r, s_v + r);
      // fused reduction: norm2 (any order, bounded), argmax over unused rows; the nonzero
      // flag is "maximum > 0" (|u_hat| >= 0, no candidate = +0)
      double sum = 0.0, bv = 0.0;
      int bi = 0x7fffffff;
      if (rv0) {
        sum = hmul(a0, a0);
        if (!used0) {
          bv = fabs(a0);
          bi = t;
        }
      }
      if (rv1) {
        sum = hadd(sum, hmul(a1, a1));
        if (!used1) argmax_combine(bv, bi, fabs(a1), t + TT);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) sum = hadd(sum, __shfl_xor_sync(0xffffffffu, sum, o));
      warp_argmax_nonneg(bv, bi);
      int nz = bv > 0.0 ? 1 : 0;
      if constexpr (NW > 1) {
        if (lane == 0) {
          s_red[4 * wib] = sum;
          s_red[4 * wib + 1] = static_cast<double>(nz);
          s_red[4 * wib + 2] = bv;
          s_red[4 * wib + 3] = static_cast<double>(bi);
        }
        team_sync<NW>(team);
        sum = s_red[0];
        nz = static_cast<int>(s_red[1]);
        bv = s_red[2];
        bi = static_cast<int>(s_red[3]);
        for (int w = 1; w < NW; ++w) {
          sum = hadd(sum, s_red[4 * w]);
          nz |= static_cast<int>(s_red[4 * w + 1]);
          argmax_combine(bv, bi, s_red[4 * w + 2], static_cast<int>(s_red[4 * w + 3]));
        }
      }
      // qualification (aca.cpp:381-383): best > 0 and (first cross or norm2 > 1e-28 scale2)
      int st = 0;
      if (nz) {
        if (r == 0) {
          st = 1;
        } else {
          const double Tlo = hmul(kEps0sq, scale_exact ? scale : s_lo);
          const double Thi = hmul(kEps0sq, scale_exact ? scale : s_hi);
          const double lo = hmul(sum, 1.0 - 4.0 * gm), hi = hmul(sum, 1.0 + 4.0 * gm);
          st = lo > Thi ? 1 : (hi <= Tlo ? 0 : 2);
        }
      }
      if (st == 2) {  // inside the bound: the reference's sequential left folds
        double* sr = s_col + (PRE ? r * CS : 0);
        if (!scale_exact) {
          // scale2 = left fold of the first accepted column, A(:, 0) (raw: no cross yet)
          double c0, c1;
          if constexpr (PRE) {
            c0 = s_col[t];
            c1 = s_col[t + TT];
          } else {
            E.eval2(y0, y1, cl, c0, c1);
          }
          team_sync<NW>(team);
          if (rv0) sr[t] = c0;
          if (rv1) sr[t + TT] = c1;
          team_sync<NW>(team);
          if (t == 0) {
            double f = hmul(sr[0], sr[0]);
            for (int i = 1; i < m; ++i) f = hadd(f, hmul(sr[i], sr[i]));
            s_misc[3] = f;
          }
          team_sync<NW>(team);
        }
        if (rv0) sr[t] = a0;  // raw column r is no longer needed
        if (rv1) sr[t + TT] = a1;
        team_sync<NW>(team);
        if (t == 0) {
          const double sc = scale_exact ? scale : s_misc[3];
          double f = hmul(sr[0], sr[0]);
          for (int i = 1; i < m; ++i) f = hadd(f, hmul(sr[i], sr[i]));
          s_misc[2] = f > hmul(kEps0sq, sc) ? 1.0 : 0.0;
        }
        team_sync<NW>(team);
        if (!scale_exact) {
          scale = s_misc[3];
          scale_exact = true;
        }
        st = s_misc[2] != 0.0 ? 1 : 0;
        team_sync<NW>(team);
      }
      if (st != 1) {  // a rejection: the general kernel takes the block
        fallback = true;
        break;
      }
      if (r == 0) {  // scale2 (aca.cpp:491) bracketed by the parallel norm of column 0
        s_lo = hmul(sum, 1.0 - 4.0 * gm);
        s_hi = hmul(sum, 1.0 + 4.0 * gm);
      }
      const int p = bi;
      // the pivot row's owner exports the pivot value and its point (u_l[p] is s_u[l][p])
      if (t == (p % TT)) {
        const bool q1 = p >= TT;
        s_misc[1] = q1 ? a1 : a0;
#pragma unroll
        for (int a = 0; a < DIM; ++a) s_yp[a] = q1 ? y1[a] : y0[a];
        if (q1) used1 = true;
        else used0 = true;
      }
      team_sync<NW>(team);
      const PivotDiv pdiv(s_misc[1]);
      s_u[r * NCAP + t] = rv0 ? pdiv(a0) : 0.0;  // u_r = u_hat / pivot (aca.cpp:466-470)
      s_u[r * NCAP + t + TT] = rv1 ? pdiv(a1) : 0.0;
      // pivot row: v_r[j] = A(p, j) - sum_l u_l[p] v_l[j] (aca.cpp:474-481), columns t, t + TT
      {
        double yp[DIM];
#pragma unroll
        for (int a = 0; a < DIM; ++a) yp[a] = s_yp[a];
        const int j0 = t, j1 = t + TT;
        const bool cv0 = j0 < n, cv1 = j1 < n;
        double b0, b1;
        E.phi2(E.r2_pts(yp, yc0), E.r2_pts(yp, yc1), b0, b1);
        if constexpr (kRolled) row2_rolled<KC, NCAP, NCAP>(b0, b1, s_u + p, s_v + j0, s_v + j1, r);
        else SmoothChain<KC>::row2<NCAP, NCAP>(b0, b1, s_u + p, s_v + j0, s_v + j1, r);
        if (cv0) s_v[r * NCAP + j0] = b0;
        if (cv1) s_v[r * NCAP + j1] = b1;
      }
      if (t == 0) {
        J.row_piv[static_cast<long long>(b) * kmax + r] = p;
        J.col_piv[static_cast<long long>(b) * kmax + r] = r;
      }
      k_eff = r + 1;
      team_sync<NW>(team);
    }
    if (fallback) {
      if (t == 0) J.fb_list[atomicAdd(J.fb_count, 1)] = b;
      team_sync<NW>(team);
      continue;
    }
    // factors: U (layout uix, zero past k_eff), V interleaved n x kmax
    double* U = J.U + (J.u_off[b] - J.u_base);
    double* V = J.V + (J.v_off[b] - J.v_base);
    const int tsh = J.tile_shift;
    auto uix = [&](int l, int i) -> long long {
      if (tsh < 0) return static_cast<long long>(l) * m + i;
      return ((static_cast<long long>(i >> tsh) * kmax + l) << tsh) + (i & ((1 << tsh) - 1));
    };
#pragma unroll
    for (int l = 0; l < KC; ++l) {
      if (rv0) U[uix(l, t)] = l < k_eff ? s_u[l * NCAP + t] : 0.0;
      if (rv1) U[uix(l, t + TT)] = l < k_eff ? s_u[l * NCAP + t + TT] : 0.0;
    }
    for (int idx = t; idx < n * KC; idx += TT) {
      const int j = idx >> 4, l = idx & 15;
      V[idx] = l < k_eff ? s_v[l * NCAP + j] : 0.0;
    }
    for (int l = k_eff + t; l < kmax; l += TT) {
      J.row_piv[static_cast<long long>(b) * kmax + l] = -1;
      J.col_piv[static_cast<long long>(b) * kmax + l] = -1;
    }
    if (t == 0) {
      J.k_eff[b] = k_eff;
      if (J.evals) {
        atomicAdd(J.evals, static_cast<unsigned long long>(ncol) * m);
        atomicAdd(J.evals + 1, static_cast<unsigned long long>(k_eff) * n);
        atomicAdd(J.evals + 2, 1ull);
      }
    }
    team_sync<NW>(team);
  }
}

template <int DIM, int KIND, int NW, bool PRE>
void launch_smooth(const AcaJob& J, const KernelEntry<DIM, KIND>& E, int sms, cudaStream_t s) {
  if (J.njobs <= 0) return;
  constexpr int teams = 4 / NW;
  const size_t smem = teams * smooth_stride<NW, PRE>() * sizeof(double);
  auto kfn = aca_smooth_kernel<DIM, KIND, NW, PRE>;
  HM_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int occ = 0;
  HM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, 128, smem));
  const long long ctas = std::min<long long>((J.njobs + teams - 1) / teams, static_cast<long long>(std::max(occ, 1)) * sms);
  kfn<<<static_cast<unsigned>(std::max(ctas, 1ll)), 128, smem, s>>>(J, E, teams);
  HM_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// Big-block kernel (max(m, n) > 1024): one 256-thread CTA per block, rows strided
// over the CTA in pairs.  The window of W candidate columns lives in a per-CTA
// global scratch (L2-resident: W x m doubles); for each row pair a thread loads
// u_l of its two rows from the U factor into right-aligned registers once and
// reuses them for every fresh window column (Chain<KC>::run2), so the chain costs
// one broadcast v load per step as in the window kernels.  Pivot rows are a
// shared bitmask.  Same semantics and bits as the window kernels.
constexpr int kBigThreads = 256;
constexpr int kBigW = 8;

template <int DIM, int KIND, int KC>
__global__ void __launch_bounds__(kBigThreads, 2) aca_big_kernel(AcaJob J, KernelEntry<DIM, KIND> E, double* gscratch,
                                                              long long gstride, int mask_words, int smooth1) {
  constexpr int TT = kBigThreads;
  constexpr int W = kBigW;
  constexpr int G = TT / W;  // 32: one warp per column in the qualification pass
  constexpr int YD = DIM > 0 ? DIM : 20;
  extern __shared__ double smem[];
  unsigned* s_mask = reinterpret_cast<unsigned*>(smem);
  double* s_up = smem + (mask_words + 1) / 2;  // kKmax
  double* s_rbv = s_up + kKmax;                // 8 warps
  int* s_rbi = reinterpret_cast<int*>(s_rbv + 8);
  int* s_state = reinterpret_cast<int*>(s_rbv + 12);
  double* s_misc = s_rbv + 20;  // [0] job [1] scale [2] verdict
  double* s_wsum = s_misc + 4;  // W: parallel norm of each window column
  const int t = threadIdx.x, lane = t & 31, wib = t >> 5;
  const double kEps0sq = 1e-14 * 1e-14;
  const int kmax = J.kmax;
  double* win = gscratch + static_cast<long long>(blockIdx.x) * gstride * W;

  for (;;) {
    if (t == 0) s_misc[0] = static_cast<double>(atomicAdd(J.counter, 1));
    __syncthreads();
    const long long job = static_cast<long long>(s_misc[0]);
    if (job >= J.njobs) return;
    const int b = J.order[job];
    const int rl = J.rl[b], m = J.m[b], cl = J.cl[b], n = J.nn[b];
    double* U = J.U + (J.u_off[b] - J.u_base);
    double* V = J.V + (J.v_off[b] - J.v_base);
    const int tsh = J.tile_shift;
    auto uix = [&](int l, int i) -> long long {
      if (tsh < 0) return static_cast<long long>(l) * m + i;
      return ((static_cast<long long>(i >> tsh) * kmax + l) << tsh) + (i & ((1 << tsh) - 1));
    };
    const long long PS = gstride;
    for (int i = t; i < (m + 31) / 32; i += TT) s_mask[i] = 0u;
    __syncthreads();
    auto is_used = [&](int i) -> bool { return (s_mask[i >> 5] >> (i & 31)) & 1u; };

    int next = 0, filled = 0, k_eff = 0;
    unsigned long long rejections = 0, ev_col = 0, ev_row = 0;
    // scale2 = norm2 of the first accepted column (aca.cpp:491): a bracket [s_lo, s_hi] of
    // its parallel sum until a decision falls inside it, then the exact left fold
    double scale = -1.0, s_lo = 0.0, s_hi = 0.0;
    bool have_scale = false, scale_exact = false;
    int c0col = 0;
    const double gm = static_cast<double>(m) * 1.2e-16;
    auto decide = [&](double sum, int nz) -> int {
      if (!nz) return 0;
      if (!have_scale) return 1;
      const double Tlo = hmul(kEps0sq, scale_exact ? scale : s_lo);
      const double Thi = hmul(kEps0sq, scale_exact ? scale : s_hi);
      const double lo = hmul(sum, 1.0 - 4.0 * gm), hi = hmul(sum, 1.0 + 4.0 * gm);
      return lo > Thi ? 1 : (hi <= Tlo ? 0 : 2);
    };
    // exact scale2 on demand: the first accepted column carried no cross, so its entries are
    // A(:, c0col) -- re-evaluated (bitwise the same) into U's next rank slot, folded in order
    int r_cur = 0;
    auto resolve_exact = [&]() {
      if (scale_exact) return;
      for (int i = t; i < m; i += TT) {
        double y0[YD];
        E.load(rl + i, y0);
        U[uix(r_cur, i)] = E.eval(y0, cl + c0col);
      }
      __syncthreads();
      if (t == 0) {
        double f = hmul(U[uix(r_cur, 0)], U[uix(r_cur, 0)]);
        for (int i = 1; i < m; ++i) f = hadd(f, hmul(U[uix(r_cur, i)], U[uix(r_cur, i)]));
        s_misc[1] = f;
      }
      __syncthreads();
      scale = s_misc[1];
      scale_exact = true;
    };

    // smooth1 (d >= 3): while the block has rejected nothing, the window is ONE column in
    // slot 0 (evaluated when it is needed, no cross updates): the per-CTA scratch actually
    // touched is m doubles, so all resident CTAs' windows stay in L2; the first rejection
    // switches to the W-column speculative window (filled == 0 at that point).
    bool one = false, fused_ok = false;
    int fused_p = 0;
    double* s_fsum = s_wsum + W;  // 8 warps: fused pass partial norms
    auto wslot = [&](int col) -> double* { return win + (one ? 0ll : static_cast<long long>(col % W)) * PS; };
    for (int r = 0; r < kmax; ++r) {
      int acc_w = -1;
      double acc_sum = 0.0;
      r_cur = r;
      while (next < n) {
        one = smooth1 && rejections == 0;
        // speculation depth: while no column was rejected, at most kmax - r more can be
        // accepted (smooth blocks, d >= 3: no noise floor), so do not evaluate past them
        const int lim = rejections ? W : (one ? 1 : max(kmax - r, 1));
        const int wcols = max(filled, min(min(W, lim), n - next));
        ev_col += static_cast<unsigned long long>(wcols - filled) * m;
        // one-column path: the fill also forms the column's norm2 (any order: bounded), the
        // nonzero flag and the argmax over unused rows (rows visited in increasing order,
        // strict >: first index on ties) -- no second and third pass over the column
        const bool fuse = one && filled == 0 && wcols == 1;
        double fsum = 0.0, fbv = 0.0;
        int fbi = 0x7fffffff;
        fused_ok = false;
        // fill: per row pair, u of the two rows into registers once, then every fresh column
        for (int i0 = t; i0 < m; i0 += 2 * TT) {
          const int i1 = i0 + TT;
          const bool ok1 = i1 < m;
          // u_l of the two rows: right-aligned for Chain<KC>, left-aligned (u_l at [l]) for
          // the straight-line SmoothChain cases (k = 16), whose V loads can be issued together
          constexpr bool kLeft = KC == 16;
          double uR[2][KC];
#pragma unroll
          for (int j = 0; j < KC; ++j) {
            const int l = kLeft ? (j < r ? j : -1) : j - (KC - r);
            uR[0][j] = l >= 0 ? U[uix(l, i0)] : 0.0;
            uR[1][j] = (l >= 0 && ok1) ? U[uix(l, i1)] : 0.0;
          }
          double y0[YD], y1[YD];
          E.load(rl + i0, y0);
          E.load(rl + (ok1 ? i1 : i0), y1);
          for (int co = filled; co < wcols; ++co) {
            const int col = next + co;
            double a0, a1;
            E.eval2(y0, y1, cl + col, a0, a1);
            if (!ok1) a1 = 0.0;
            if constexpr (kLeft) SmoothChain<16>::col2<1>(a0, a1, uR[0], uR[1], r, V + static_cast<long long>(col) * kmax);
            else Chain<KC>::run2(a0, a1, uR[0], uR[1], r, V + static_cast<long long>(col) * kmax + (r - KC), 1);
            double* dst = wslot(col);
            dst[i0] = a0;
            if (ok1) dst[i1] = a1;
            if (fuse) {
              fsum = hadd(fsum, hmul(a0, a0));
              if (!is_used(i0) && fabs(a0) > fbv) {
                fbv = fabs(a0);
                fbi = i0;
              }
              if (ok1) {
                fsum = hadd(fsum, hmul(a1, a1));
                if (!is_used(i1) && fabs(a1) > fbv) {
                  fbv = fabs(a1);
                  fbi = i1;
                }
              }
            }
          }
        }
        filled = wcols;
        if (fuse) {
#pragma unroll
          for (int o = 16; o; o >>= 1) fsum = hadd(fsum, __shfl_xor_sync(0xffffffffu, fsum, o));
          warp_argmax_nonneg(fbv, fbi);
          if (lane == 0) {
            s_fsum[wib] = fsum;
            s_rbv[wib] = fbv;
            s_rbi[wib] = fbi;
          }
        }
        __syncthreads();
        if (fuse) {
          double sum = s_fsum[0], bv = s_rbv[0];
          int bi = s_rbi[0];
          for (int g = 1; g < TT / 32; ++g) {
            sum = hadd(sum, s_fsum[g]);
            argmax_combine(bv, bi, s_rbv[g], s_rbi[g]);
          }
          if (decide(sum, bv > 0.0 ? 1 : 0) == 1) {
            acc_w = 0;
            acc_sum = sum;
            fused_ok = true;
            fused_p = bi;
          }
        }
        // qualification.  Fast path while the block has rejected nothing: the first window
        // column with the whole CTA (4 loads in flight per thread); otherwise one warp per
        // window column.  Decisions use the rigorous bound of the parallel sums; scale2 is a
        // bracket until an ambiguous decision needs it exactly (resolve_exact).
        int first_state = -1;
        if (rejections == 0 && !fuse) {
          const double* src = wslot(next);
          double sum = 0.0;
          int nz = 0;
          for (int i = t; i < m; i += 4 * TT) {
            double a[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) a[u] = i + u * TT < m ? src[i + u * TT] : 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (i + u * TT < m) {
                sum = hadd(sum, hmul(a[u], a[u]));
                nz |= (!is_used(i + u * TT) && fabs(a[u]) > 0.0) ? 1 : 0;
              }
          }
#pragma unroll
          for (int o = 16; o; o >>= 1) {
            sum = hadd(sum, __shfl_xor_sync(0xffffffffu, sum, o));
            nz |= __shfl_xor_sync(0xffffffffu, nz, o);
          }
          if (lane == 0) {
            s_rbv[wib] = sum;
            s_rbi[wib] = nz;
          }
          __syncthreads();
          sum = s_rbv[0];
          nz = s_rbi[0];
          for (int g = 1; g < TT / 32; ++g) {
            sum = hadd(sum, s_rbv[g]);
            nz |= s_rbi[g];
          }
          __syncthreads();
          first_state = decide(sum, nz);
          if (first_state == 1) {
            acc_w = 0;
            acc_sum = sum;
          }
        }
        if (acc_w < 0) {
          {
            const int w = wib;  // G == 32: warp w scans window column w
            double sum = 0.0;
            int nz = 0;
            if (w < wcols) {
              const double* src = wslot(next + w);
              for (int i = lane; i < m; i += 4 * 32) {
                double a[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) a[u] = i + 32 * u < m ? src[i + 32 * u] : 0.0;
#pragma unroll
                for (int u = 0; u < 4; ++u)
                  if (i + 32 * u < m) {
                    sum = hadd(sum, hmul(a[u], a[u]));
                    nz |= (!is_used(i + 32 * u) && fabs(a[u]) > 0.0) ? 1 : 0;
                  }
              }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
              sum = hadd(sum, __shfl_xor_sync(0xffffffffu, sum, o));
              nz |= __shfl_xor_sync(0xffffffffu, nz, o);
            }
            if (lane == 0 && w < wcols) {
              s_state[w] = decide(sum, nz);
              s_wsum[w] = sum;
            }
          }
          __syncthreads();
          for (int w = 0; w < wcols; ++w) {
            int st = s_state[w];
            if (st == 2) {
              resolve_exact();
              if (t == 0) {  // the reference's sequential left fold (aca.cpp:373-374 / 414-415)
                const double* src = wslot(next + w);
                double f = hmul(src[0], src[0]);
                for (int i = 1; i < m; ++i) f = hadd(f, hmul(src[i], src[i]));
                s_misc[2] = f > hmul(kEps0sq, scale) ? 1.0 : 0.0;
              }
              __syncthreads();
              st = s_misc[2] != 0.0 ? 1 : 0;
              __syncthreads();
            }
            if (st == 1) {
              acc_w = w;
              acc_sum = s_wsum[w];
              break;
            }
          }
        }
        if (!have_scale && acc_w >= 0) {
          // first cross: scale2 (aca.cpp:491) bracketed by the parallel norm of the column
          s_lo = hmul(acc_sum, 1.0 - 4.0 * gm);
          s_hi = hmul(acc_sum, 1.0 + 4.0 * gm);
          c0col = next + acc_w;
          have_scale = true;
        }
        const int consumed = acc_w >= 0 ? acc_w + 1 : wcols;
        rejections += static_cast<unsigned long long>(acc_w >= 0 ? acc_w : wcols);
        next += consumed;
        filled = acc_w >= 0 ? wcols - consumed : 0;
        if (acc_w >= 0) break;
      }
      if (acc_w < 0) break;
      const int cstar = next - 1;
      const double* acol = wslot(cstar);
      double bv = -1.0;
      int bi = 0x7fffffff;
      for (int i = t; !fused_ok && i < m; i += 4 * TT) {
        double a[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) a[u] = i + u * TT < m ? acol[i + u * TT] : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int ii = i + u * TT;
          if (ii < m && !is_used(ii)) {
            const double av = fabs(a[u]);
            if (av > bv) {
              bv = av;
              bi = ii;
            }
          }
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        argmax_combine(bv, bi, ov, oi);
      }
      if (!fused_ok) {
        if (lane == 0) {
          s_rbv[wib] = bv;
          s_rbi[wib] = bi;
        }
        __syncthreads();
        bv = s_rbv[0];
        bi = s_rbi[0];
        for (int g = 1; g < TT / 32; ++g) argmax_combine(bv, bi, s_rbv[g], s_rbi[g]);
      }
      const int p = fused_ok ? fused_p : bi;
      for (int l = t; l < r; l += TT) s_up[l] = U[uix(l, p)];
      __syncthreads();
      const PivotDiv pdiv(acol[p]);
      ev_row += n;
      {
        double yp[YD];
        E.load(rl + p, yp);
        double uP[KC];  // u_l[p], right-aligned: every V-row load of the chain issues up front
#pragma unroll
        for (int j = 0; j < KC; ++j) uP[j] = j >= KC - r ? s_up[j - (KC - r)] : 0.0;
        // no window columns (the one-column path): four columns per step, one 4-way
        // evaluation (independent K1 / exp chains) and two chains
        const int jstart = (KC == 16 && filled == 0) ? n : t;
        if constexpr (KC == 16) {
          for (int j = t; filled == 0 && j < n; j += 4 * TT) {
            long long jq[4];
            bool okq[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              okq[q] = j + q * TT < n;
              jq[q] = okq[q] ? j + q * TT : j;
            }
            if (r > 0) {
#pragma unroll
              for (int q = 0; q < 4; ++q) prefetch_l1(V + jq[q] * kmax);
            }
            double a[4];
            E.eval4c(yp, cl + jq[0], cl + jq[1], cl + jq[2], cl + jq[3], a[0], a[1], a[2], a[3]);
            SmoothChain<16>::row2<1>(a[0], a[1], s_up, V + jq[0] * kmax, V + jq[1] * kmax, r);
            SmoothChain<16>::row2<1>(a[2], a[3], s_up, V + jq[2] * kmax, V + jq[3] * kmax, r);
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (okq[q]) V[jq[q] * kmax + r] = a[q];
          }
        }
        for (int j = jstart; j < n; j += 2 * TT) {
          const int j1 = j + TT;
          const bool ok1 = j1 < n;
          const int jj = ok1 ? j1 : j;
          const bool in0 = j >= next && j < next + filled, in1 = jj >= next && jj < next + filled;
          double a0, a1;
          if (in0 && in1) {
            a0 = win[static_cast<long long>(j % W) * PS + p];
            a1 = win[static_cast<long long>(jj % W) * PS + p];
          } else {
            E.eval2c(yp, cl + j, cl + jj, a0, a1);
            if constexpr (KC == 16)
              SmoothChain<16>::row2<1>(a0, a1, s_up, V + static_cast<long long>(j) * kmax,
                                       V + static_cast<long long>(jj) * kmax, r);
            else
              Chain<KC>::run2v(a0, a1, uP, r, V + static_cast<long long>(j) * kmax + (r - KC),
                               V + static_cast<long long>(jj) * kmax + (r - KC), 1);
            if (in0) a0 = win[static_cast<long long>(j % W) * PS + p];
            if (in1) a1 = win[static_cast<long long>(jj % W) * PS + p];
          }
          V[static_cast<long long>(j) * kmax + r] = a0;
          if (ok1) V[static_cast<long long>(j1) * kmax + r] = a1;
        }
      }
      // (the used-row mask changes before the barrier: the next rank's fused fill reads it)
      if (t == 0) s_mask[p >> 5] |= 1u << (p & 31);
      __syncthreads();
      {
        // u_r = u_hat / pivot (aca.cpp:466-470) fused with the window cross: per row the
        // accepted column's entry and the W window entries are loaded together, u_r goes
        // to U and straight into the window updates (no reload)
        if (filled == 0) {  // no window left (always so on the one-column path): 4 loads in flight
          for (int i = t; i < m; i += 4 * TT) {
            double a[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) a[u] = i + u * TT < m ? acol[i + u * TT] : 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (i + u * TT < m) U[uix(r, i + u * TT)] = pdiv(a[u]);
          }
        }
        double vr[W];
#pragma unroll
        for (int co = 0; co < W; ++co) vr[co] = co < filled ? V[static_cast<long long>(next + co) * kmax + r] : 0.0;
        for (int i = t; filled > 0 && i < m; i += TT) {
          const double ah = acol[i];
          double a[W];
#pragma unroll
          for (int co = 0; co < W; ++co)
            a[co] = co < filled ? win[static_cast<long long>((next + co) % W) * PS + i] : 0.0;
          const double u = pdiv(ah);
          U[uix(r, i)] = u;
#pragma unroll
          for (int co = 0; co < W; ++co)
            if (co < filled) win[static_cast<long long>((next + co) % W) * PS + i] = hsub(a[co], hmul(u, vr[co]));
        }
      }
      if (t == 0) {
        J.row_piv[static_cast<long long>(b) * kmax + r] = p;
        J.col_piv[static_cast<long long>(b) * kmax + r] = cstar;
      }
      k_eff = r + 1;
    }
    for (int l = k_eff; l < kmax; ++l)
      for (int i = t; i < m; i += TT) U[uix(l, i)] = 0.0;
    if (k_eff < kmax) {
      for (int idx = t; idx < n * (kmax - k_eff); idx += TT) {
        const int j = idx / (kmax - k_eff), l = k_eff + idx % (kmax - k_eff);
        V[static_cast<long long>(j) * kmax + l] = 0.0;
      }
    }
    for (int l = k_eff + t; l < kmax; l += TT) {
      J.row_piv[static_cast<long long>(b) * kmax + l] = -1;
      J.col_piv[static_cast<long long>(b) * kmax + l] = -1;
    }
    if (t == 0) {
      J.k_eff[b] = k_eff;
      if (J.rejections && rejections) {
        atomicAdd(J.rejections, rejections);  // [0] columns, [1] their entries (sum of m)
        atomicAdd(J.rejections + 1, rejections * static_cast<unsigned long long>(m));
      }
      if (J.evals) {
        atomicAdd(J.evals, ev_col);
        atomicAdd(J.evals + 1, ev_row);
        atomicAdd(J.evals + 2, 1ull);
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Cluster kernel (1024 < max(m, n) <= 512 * CL): a THREAD-BLOCK CLUSTER of CL CTAs
// (256 threads each) factorises one block.  CTA c of the cluster owns rows
// [512c, 512c + 512) with u_l right-aligned in registers (exactly the window kernel's
// thread mapping) and keeps its rows of the W-column window in its own shared memory.
// Per-column partial norms, the pivot argmax, the exact folds and the pivot row's u_l
// travel through distributed shared memory (mapa / ld.shared::cluster via
// cluster.map_shared_rank); every CTA combines the CL partials in rank order, so all
// CTAs take identical decisions and the whole factorisation is bitwise the reference's.
// v_l lives in the interleaved V factor (written by the row pass, made visible to the
// cluster by the release/acquire cluster barrier).
template <int DIM, int KIND, int KC, int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(256, 2)
    aca_cluster_kernel(AcaJob J, KernelEntry<DIM, KIND> E) {
  namespace cg = cooperative_groups;
  constexpr int TT = 256, RPL = 2, NCAP = TT * RPL, W = 16, PS = NCAP + 1, G = TT / W;  // G = 16
  constexpr int YD = DIM > 0 ? DIM : 1;
  cg::cluster_group cluster = cg::this_cluster();
  const int cr = static_cast<int>(cluster.block_rank());
  extern __shared__ double smem[];
  double* s_win = smem;                       // W x PS (own rows)
  double* s_up = s_win + W * PS;              // KC: u_l[p] (copied from the owner)
  double* s_csum = s_up + KC;                 // W: this CTA's partial norm per column
  int* s_cnz = reinterpret_cast<int*>(s_csum + W);      // W ints
  double* s_wsum = s_csum + W + W / 2;        // 8 warps x 2 (sum pieces for G=16 groups)
  double* s_rbv = s_wsum + 16;                // 8 warps (argmax)
  int* s_rbi = reinterpret_cast<int*>(s_rbv + 8);       // 8 ints
  double* s_cbv = s_rbv + 12;                 // [0] CTA argmax value, [1] (int) index
  int* s_state = reinterpret_cast<int*>(s_cbv + 2);     // W ints
  unsigned char* s_used = reinterpret_cast<unsigned char*>(s_cbv + 2 + W / 2);  // NCAP bytes
  double* s_misc = s_cbv + 2 + W / 2 + NCAP / 8;  // [0] job [1] scale [2] verdict [3] pivot value
  double* s_tot = s_misc + 8;                     // W: combined norm per window column
  double* s_scr = s_tot + W;                      // NCAP: re-evaluated first column (exact scale2)
  const int t = threadIdx.x, lane = t & 31, wib = t >> 5;
  const double kEps0sq = 1e-14 * 1e-14;
  const int kmax = J.kmax;
  auto rem = [&](double* p, int rank) -> const double* { return cluster.map_shared_rank(p, rank); };

  for (;;) {
    if (cr == 0 && t == 0) s_misc[0] = static_cast<double>(atomicAdd(J.counter, 1));
    for (int i = t; i < NCAP; i += TT) s_used[i] = 0;
    cluster.sync();
    const long long job = static_cast<long long>(*rem(s_misc, 0));
    cluster.sync();  // everyone has read the job before rank 0 may overwrite it
    if (job >= (J.njobs_dev ? static_cast<long long>(*J.njobs_dev) : J.njobs)) return;
    const int b = J.order[job];
    const int rl = J.rl[b], m = J.m[b], cl = J.cl[b], n = J.nn[b];
    double* U = J.U + (J.u_off[b] - J.u_base);
    double* V = J.V + (J.v_off[b] - J.v_base);
    const int tsh = J.tile_shift;
    auto uix = [&](int l, int i) -> long long {
      if (tsh < 0) return static_cast<long long>(l) * m + i;
      return ((static_cast<long long>(i >> tsh) * kmax + l) << tsh) + (i & ((1 << tsh) - 1));
    };
    const int row0 = cr * NCAP;  // first block row of this CTA
    double y[RPL][YD];
    bool rv[RPL];
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
      const int i = row0 + t + q * TT;
      rv[q] = i < m;
      if constexpr (DIM > 0) {
#pragma unroll
        for (int a = 0; a < DIM; ++a) y[q][a] = rv[q] ? __ldg(E.coords + a * E.n + rl + i) : 0.0;
      }
    }
    auto entry = [&](int q, long long colpt) -> double {
      if constexpr (DIM > 0) {
        return E.eval(y[q], colpt);
      } else {
        double yy[20];
        E.load(rl + row0 + t + q * TT, yy);
        return E.eval(yy, colpt);
      }
    };
    double uR[RPL][KC];
#pragma unroll
    for (int q = 0; q < RPL; ++q)
#pragma unroll
      for (int j = 0; j < KC; ++j) uR[q][j] = 0.0;
    int next = 0, filled = 0, k_eff = 0;
    unsigned long long rejections = 0, ev_col = 0, ev_row = 0;
    double scale = -1.0, s_lo = 0.0, s_hi = 0.0;  // scale2: exact (scale_exact) or bracket
    bool have_scale = false, scale_exact = false;
    int c0col = 0;
    const double gm = static_cast<double>(m) * 1.2e-16;
    // exact left fold of a window column over ALL rows (rank order, then row order)
    auto exact_fold = [&](int slot) -> double {
      double f = 0.0;
      bool first = true;
      for (int c = 0; c < CL; ++c) {
        const double* w = rem(s_win, c) + slot * PS;
        const int rows = min(NCAP, m - c * NCAP);
        for (int i = 0; i < rows; ++i) {
          const double a = w[i];
          f = first ? hmul(a, a) : hadd(f, hmul(a, a));
          first = false;
        }
      }
      return f;
    };

    for (int r = 0; r < kmax; ++r) {
      int acc_w = -1;
      while (next < n) {
        const int lim = rejections ? W : max(kmax - r, 1);
        const int wcols = max(filled, min(min(W, lim), n - next));
        ev_col += static_cast<unsigned long long>(wcols - filled) * m;
        for (int co = filled; co < wcols; ++co) {
          const int col = next + co;
          double* dst = s_win + (col % W) * PS;
          double a0, a1;
          if constexpr (DIM > 0) {
            E.eval2(y[0], y[1], cl + col, a0, a1);
          } else {
            a0 = rv[0] ? entry(0, cl + col) : 0.0;
            a1 = rv[1] ? entry(1, cl + col) : 0.0;
          }
          Chain<KC>::run2(a0, a1, uR[0], uR[1], r, V + static_cast<long long>(col) * kmax + (r - KC), 1);
          if (rv[0]) dst[t] = a0;
          if (rv[1]) dst[t + TT] = a1;
        }
        filled = wcols;
        __syncthreads();
        // this CTA's partial norm / nonzero flag per window column (G = 16 threads each)
        {
          const int w = t / G, g = t % G;
          double sum = 0.0;
          int nz = 0;
          if (w < wcols) {
            const double* src = s_win + ((next + w) % W) * PS;
            const int rows = min(NCAP, m - row0);
            for (int i = g; i < rows; i += G) {
              const double a = src[i];
              sum = hadd(sum, hmul(a, a));
              nz |= (!s_used[i] && fabs(a) > 0.0) ? 1 : 0;
            }
          }
#pragma unroll
          for (int o = G / 2; o; o >>= 1) {
            sum = hadd(sum, __shfl_xor_sync(0xffffffffu, sum, o));
            nz |= __shfl_xor_sync(0xffffffffu, nz, o);
          }
          if (g == 0) {
            s_csum[w] = sum;
            s_cnz[w] = nz;
          }
        }
        cluster.sync();
        // identical decision in every CTA: partials combined in rank order.  scale2 is
        // known exactly only on demand (see scale_exact): until then the test uses the
        // bracket [s_lo, s_hi] of the parallel sum, which contains the exact left fold.
        if (t < W) {
          const int w = t;
          int st = 0;
          double sum = 0.0;
          if (w < wcols) {
            double ps[CL];
            int pn[CL];
#pragma unroll
            for (int c = 0; c < CL; ++c) {  // all remote loads issued before the fold
              ps[c] = *rem(s_csum + w, c);
              pn[c] = cluster.map_shared_rank(s_cnz, c)[w];
            }
            int nz = 0;
            sum = ps[0];
#pragma unroll
            for (int c = 0; c < CL; ++c) {
              if (c) sum = hadd(sum, ps[c]);
              nz |= pn[c];
            }
            if (nz) {
              if (!have_scale) {
                st = 1;
              } else {
                const double Tlo = hmul(kEps0sq, scale_exact ? scale : s_lo);
                const double Thi = hmul(kEps0sq, scale_exact ? scale : s_hi);
                const double lo = hmul(sum, 1.0 - 4.0 * gm), hi = hmul(sum, 1.0 + 4.0 * gm);
                st = lo > Thi ? 1 : (hi <= Tlo ? 0 : 2);
              }
            }
          }
          s_state[w] = st;
          s_tot[w] = sum;
        }
        __syncthreads();
        for (int w = 0; w < wcols; ++w) {
          int st = s_state[w];
          if (st == 2) {  // the reference's sequential left folds (aca.cpp:373-374, 491)
            if (!scale_exact) {
              // the first accepted column is A(:, c0col) (no cross subtracted yet):
              // re-evaluate it (bitwise the same entries) and fold it over all rows
#pragma unroll
              for (int q = 0; q < RPL; ++q)
                if (rv[q]) s_scr[t + q * TT] = entry(q, cl + c0col);
              cluster.sync();
              if (t == 0) {
                double f = 0.0;
                bool first = true;
                for (int c = 0; c < CL; ++c) {
                  const double* w2 = rem(s_scr, c);
                  const int rows = min(NCAP, m - c * NCAP);
                  for (int i = 0; i < rows; ++i) {
                    f = first ? hmul(w2[i], w2[i]) : hadd(f, hmul(w2[i], w2[i]));
                    first = false;
                  }
                }
                s_misc[1] = f;
              }
              cluster.sync();
              scale = s_misc[1];
              scale_exact = true;
            }
            if (t == 0) s_misc[2] = exact_fold((next + w) % W) > hmul(kEps0sq, scale) ? 1.0 : 0.0;
            __syncthreads();
            st = s_misc[2] != 0.0 ? 1 : 0;
          }
          if (st == 1) {
            acc_w = w;
            break;
          }
        }
        if (!have_scale && acc_w >= 0) {
          // first cross: bracket of scale2 from the parallel norm of the accepted column
          const double sp = s_tot[acc_w];
          s_lo = hmul(sp, 1.0 - 4.0 * gm);
          s_hi = hmul(sp, 1.0 + 4.0 * gm);
          c0col = next + acc_w;
          have_scale = true;
        }
        cluster.sync();  // partials / windows read by every CTA before they change
        const int consumed = acc_w >= 0 ? acc_w + 1 : wcols;
        rejections += static_cast<unsigned long long>(acc_w >= 0 ? acc_w : wcols);
        next += consumed;
        filled = acc_w >= 0 ? wcols - consumed : 0;
        if (acc_w >= 0) break;
      }
      if (acc_w < 0) break;  // no usable column left (aca.cpp:442-443)
      const int cstar = next - 1;
      const int aslot = cstar % W;
      const double* acol = s_win + aslot * PS;

      // pivot row: argmax over unused rows, first (global) index wins
      double bv = -1.0;
      int bi = 0x7fffffff;
#pragma unroll
      for (int q = 0; q < RPL; ++q) {
        const int il = t + q * TT;
        if (rv[q] && !s_used[il]) {
          const double av = fabs(acol[il]);
          if (av > bv) {
            bv = av;
            bi = row0 + il;
          }
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        argmax_combine(bv, bi, ov, oi);
      }
      if (lane == 0) {
        s_rbv[wib] = bv;
        s_rbi[wib] = bi;
      }
      __syncthreads();
      if (t == 0) {
        double cbv = s_rbv[0];
        int cbi = s_rbi[0];
        for (int g = 1; g < TT / 32; ++g) argmax_combine(cbv, cbi, s_rbv[g], s_rbi[g]);
        s_cbv[0] = cbv;
        reinterpret_cast<int*>(s_cbv + 1)[0] = cbi;
      }
      cluster.sync();
      int p;
      {
        double gbv = -1.0;
        int gbi = 0x7fffffff;
        double cv[CL];
        int ci[CL];
#pragma unroll
        for (int c = 0; c < CL; ++c) {
          const double* rc = rem(s_cbv, c);
          cv[c] = rc[0];
          ci[c] = reinterpret_cast<const int*>(rc + 1)[0];
        }
#pragma unroll
        for (int c = 0; c < CL; ++c) argmax_combine(gbv, gbi, cv[c], ci[c]);
        p = gbi;
      }
      const int po = p / NCAP, pl = p - po * NCAP, pt = pl % TT, pq = pl / TT;
      if (cr == po && t == pt) {
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
          if (q == pq) {
            s_misc[3] = acol[pl];
#pragma unroll
            for (int j = 0; j < KC; ++j)
              if (j >= KC - r) s_up[j - (KC - r)] = uR[q][j];
          }
        }
      }
      cluster.sync();
      // the owner's u_l[p] and pivot value into every CTA
      if (cr != po) {
        const double* ru = rem(s_up, po);
        for (int l = t; l < r; l += TT) s_up[l] = ru[l];
        if (t == 0) s_misc[3] = *rem(s_misc + 3, po);
      }
      __syncthreads();
      const PivotDiv pdiv(s_misc[3]);
#pragma unroll
      for (int q = 0; q < RPL; ++q) {
        const double nu = rv[q] ? pdiv(acol[t + q * TT]) : 0.0;
#pragma unroll
        for (int j = 0; j + 1 < KC; ++j) uR[q][j] = uR[q][j + 1];
        uR[q][KC - 1] = nu;
      }
      // v_r = A(p,:) - sum_l u_l[p] v_l (aca.cpp:474-481), columns split over the cluster
      ev_row += n;
      {
        double yp[DIM > 0 ? DIM : 20];
        E.load(rl + p, yp);
        double uP[KC];
#pragma unroll
        for (int j = 0; j < KC; ++j) uP[j] = j >= KC - r ? s_up[j - (KC - r)] : 0.0;
        for (int j = cr * TT + t; j < n; j += 2 * CL * TT) {
          const int j1 = j + CL * TT;
          const bool ok1 = j1 < n;
          const int jj = ok1 ? j1 : j;
          double a0, a1;
          E.eval2c(yp, cl + j, cl + jj, a0, a1);
          Chain<KC>::run2v(a0, a1, uP, r, V + static_cast<long long>(j) * kmax + (r - KC),
                           V + static_cast<long long>(jj) * kmax + (r - KC), 1);
          V[static_cast<long long>(j) * kmax + r] = a0;
          if (ok1) V[static_cast<long long>(j1) * kmax + r] = a1;
        }
      }
      cluster.sync();  // v_r visible to the whole cluster (release / acquire)
      if (cr == po && t == pt) s_used[pl] = 1;
      {
        double ur[RPL];
#pragma unroll
        for (int q = 0; q < RPL; ++q) ur[q] = uR[q][KC - 1];
        window_cross<RPL>(filled, next, ur, rv, t, TT,
                          [&](int col) { return V[static_cast<long long>(col) * kmax + r]; },
                          [&](int col) { return s_win + (col % W) * PS; });
      }
      if (cr == 0 && t == 0) {
        J.row_piv[static_cast<long long>(b) * kmax + r] = p;
        J.col_piv[static_cast<long long>(b) * kmax + r] = cstar;
      }
      k_eff = r + 1;
      __syncthreads();
    }
    // factors: own rows of U; V past k_eff zeroed (columns split over the cluster)
#pragma unroll
    for (int j = 0; j < KC; ++j) {
      const int l = j - (KC - k_eff);
      if (l >= 0) {
#pragma unroll
        for (int q = 0; q < RPL; ++q)
          if (rv[q]) U[uix(l, row0 + t + q * TT)] = uR[q][j];
      }
    }
    for (int l = k_eff; l < kmax; ++l)
#pragma unroll
      for (int q = 0; q < RPL; ++q)
        if (rv[q]) U[uix(l, row0 + t + q * TT)] = 0.0;
    if (k_eff < kmax)
      for (int j = cr * TT + t; j < n; j += CL * TT)
        for (int l = k_eff; l < kmax; ++l) V[static_cast<long long>(j) * kmax + l] = 0.0;
    if (cr == 0) {
      for (int l = k_eff + t; l < kmax; l += TT) {
        J.row_piv[static_cast<long long>(b) * kmax + l] = -1;
        J.col_piv[static_cast<long long>(b) * kmax + l] = -1;
      }
      if (t == 0) {
        J.k_eff[b] = k_eff;
        if (J.rejections && rejections) {
        atomicAdd(J.rejections, rejections);  // [0] columns, [1] their entries (sum of m)
        atomicAdd(J.rejections + 1, rejections * static_cast<unsigned long long>(m));
      }
        if (J.evals) {
          atomicAdd(J.evals, ev_col);
          atomicAdd(J.evals + 1, ev_row);
          atomicAdd(J.evals + 2, 1ull);
        }
      }
    }
    cluster.sync();
  }
}

template <int DIM, int KIND, int KC, int CL>
void launch_cluster(const AcaJob& J, const KernelEntry<DIM, KIND>& E, int sms, cudaStream_t s) {
  if (J.njobs <= 0) return;
  constexpr int W = 16, NCAP = 512;
  const size_t smem = sizeof(double) * (W * (NCAP + 1) + KC + W + W / 2 + 16 + 12 + 2 + W / 2 + NCAP / 8 + 8 + W + NCAP);
  auto kfn = aca_cluster_kernel<DIM, KIND, KC, CL>;
  HM_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  // one cluster per SM-group: CTAs = CL * min(jobs, SMs / CL * 2)
  const long long clusters = std::min<long long>(J.njobs, std::max(1, 2 * sms / CL));
  kfn<<<static_cast<unsigned>(clusters * CL), 256, smem, s>>>(J, E);
  HM_LAUNCH_CHECK();
}

// Split cluster barrier: arrive (release) ... independent work ... wait (acquire); together
// exactly cluster.sync().
__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acquire() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// ---------------------------------------------------------------------------
// Smooth-path cluster kernel (1024 < max(m, n) <= 512 CL, k = 16): the smooth_kernel
// schedule over a thread-block cluster of CL CTAs, with ONE cluster barrier per rank.
// CTA c owns rows [512c, 512c + 512) (two per thread, u_l of its rows in its shared
// memory) and the row pass's columns [512c, 512c + 512); every CTA also keeps its own
// copy of v_l at the k candidate columns (computed redundantly), so the column chain
// never leaves the CTA.  Per rank each CTA publishes its partial (norm2, nonzero, argmax)
// and its rows' residuals; after the barrier every CTA combines the CL partials in rank
// order (identical decisions everywhere), reads the pivot value and u_l[p] from the
// owner through distributed shared memory, and runs its row pass.  Published buffers
// alternate by rank parity: a CTA rewrites a buffer only after the NEXT barrier, which
// every reader of its previous contents has passed.  A rejection or a decision inside the
// rigorous bound hands the block to the general cluster kernel (fallback list).
template <int DIM, int KIND, int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(256, 2)
    aca_smooth_cluster_kernel(AcaJob J, KernelEntry<DIM, KIND> E) {
  namespace cg = cooperative_groups;
  constexpr int KC = 16, TT = 256, NCAP = 512;
  static_assert(DIM > 0, "smooth cluster kernel: compile-time dimension");
  cg::cluster_group cluster = cg::this_cluster();
  const int cr = static_cast<int>(cluster.block_rank());
  extern __shared__ double smem[];
  double* s_u = smem;                     // KC x NCAP: u_l of the own rows
  double* s_res = s_u + KC * NCAP;        // 2 x NCAP: residuals of the own rows (rank parity)
  double* s_vc = s_res + 2 * NCAP;        // KC x KC: v_l at the candidate columns
  double* s_part = s_vc + KC * KC;        // 2 x 8: CTA partial + its argmax row's point (rank parity)
  double* s_red = s_part + 16;            // 8 warps x 8: warp partial + its argmax row's point
  double* s_up = s_red + 64;              // KC: u_l[p]
  double* s_misc = s_up + KC;             // [0] job [1] pivot value
  double* s_cc = s_misc + 8;              // KC x 4: points of the candidate columns
  const int t = threadIdx.x, lane = t & 31, wib = t >> 5;
  const double kEps0sq = 1e-14 * 1e-14;
  const int kmax = J.kmax;
  auto rem = [&](double* p, int rank) -> const double* { return cluster.map_shared_rank(p, rank); };

  for (;;) {
    if (cr == 0 && t == 0) s_misc[0] = static_cast<double>(atomicAdd(J.counter, 1));
    cluster.sync();
    const long long job = static_cast<long long>(*rem(s_misc, 0));
    cluster.sync();
    if (job >= J.njobs) return;
    const int b = J.order[job];
    const int rl = J.rl[b], m = J.m[b], cl = J.cl[b], n = J.nn[b];
    const int row0 = cr * NCAP;
    const int i0 = row0 + t, i1 = row0 + t + TT;
    const bool rv0 = i0 < m, rv1 = i1 < m;
    double y0[DIM], y1[DIM];
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      y0[a] = rv0 ? __ldg(E.coords + a * E.n + rl + i0) : 0.0;
      y1[a] = rv1 ? __ldg(E.coords + a * E.n + rl + i1) : 0.0;
    }
    double* V = J.V + (J.v_off[b] - J.v_base);
    // the points of this thread's row-pass columns in registers, the candidate columns' in
    // shared memory: no global loads on the per-rank critical path but the pivot's point
    double yc0[DIM], yc1[DIM];
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      yc0[a] = row0 + t < n ? __ldg(E.coords + a * E.n + cl + row0 + t) : 0.0;
      yc1[a] = row0 + t + TT < n ? __ldg(E.coords + a * E.n + cl + row0 + t + TT) : 0.0;
    }
    if (t < KC && t < n)
#pragma unroll
      for (int a = 0; a < DIM; ++a) s_cc[t * 4 + a] = __ldg(E.coords + a * E.n + cl + t);
    __syncthreads();
    bool used0 = false, used1 = false;
    double s_lo = 0.0, s_hi = 0.0;
    const double gm = static_cast<double>(m) * 1.2e-16;
    int k_eff = 0;
    bool fallback = false;
    // raw candidate column entries A(i, r) of the own rows, one rank ahead: column r + 1 is
    // evaluated between the arrive and the wait of rank r's cluster barrier (independent
    // work hiding the barrier); column 0 here
    double na0, na1;
    {
      double pc[DIM];
#pragma unroll
      for (int a = 0; a < DIM; ++a) pc[a] = s_cc[a];
      E.phi2(E.r2_pts(y0, pc), E.r2_pts(y1, pc), na0, na1);
    }
    const int rlast = min(kmax, n);
    for (int r = 0; r < kmax; ++r) {
      if (r >= n) break;
      const int par = r & 1;
      // column r residual of the own rows (candidate column r: no rejection so far)
      double a0 = na0, a1 = na1;
      SmoothChain<KC>::col2s<NCAP, KC>(a0, a1, s_u + t, s_u + t + TT, r, s_vc + r);
      // publish the residuals (the pivot value is read from its owner after the barrier)
      s_res[par * NCAP + t] = a0;
      s_res[par * NCAP + t + TT] = a1;
      double sum = 0.0, bv = 0.0;  // no candidate = +0 (see warp_argmax_nonneg)
      int bi = 0x7fffffff;
      if (rv0) {
        sum = hmul(a0, a0);
        if (!used0) {
          bv = fabs(a0);
          bi = i0;
        }
      }
      if (rv1) {
        sum = hadd(sum, hmul(a1, a1));
        if (!used1) argmax_combine(bv, bi, fabs(a1), i1);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) sum = hadd(sum, __shfl_xor_sync(0xffffffffu, sum, o));
      warp_argmax_nonneg(bv, bi);
      int nz = bv > 0.0 ? 1 : 0;
      if (lane == 0) {
        s_red[8 * wib] = sum;
        s_red[8 * wib + 2] = bv;
        s_red[8 * wib + 3] = static_cast<double>(bi);
      }
      // the warp winner's point, from its owner's registers (published with the partial, so
      // the pivot point needs no dependent global load after the cluster barrier)
      if (bi == i0 || bi == i1) {
#pragma unroll
        for (int a = 0; a < DIM; ++a) s_red[8 * wib + 4 + a] = bi == i0 ? y0[a] : y1[a];
      }
      __syncthreads();
      // CTA partial: warp 0 combines the 8 warps' partials with one butterfly (the norm2's
      // summation order is free -- rigorous bound; argmax and the flag are order-free)
      if (wib == 0) {
        double cs = lane < TT / 32 ? s_red[8 * lane] : 0.0, cb = lane < TT / 32 ? s_red[8 * lane + 2] : 0.0;
        int ci = lane < TT / 32 ? static_cast<int>(s_red[8 * lane + 3]) : 0x7fffffff;
#pragma unroll
        for (int o = TT / 64; o; o >>= 1) cs = hadd(cs, __shfl_xor_sync(0xffffffffu, cs, o));
        warp_argmax_nonneg(cb, ci);
        if (lane == 0) {
          s_part[8 * par] = cs;
          s_part[8 * par + 2] = cb;
          s_part[8 * par + 3] = static_cast<double>(ci);
        }
        if (ci != 0x7fffffff && lane < DIM) {
          const int w = ((ci - row0) % TT) >> 5;  // the warp owning row ci
          s_part[8 * par + 4 + lane] = s_red[8 * w + 4 + lane];
        }
      }
      // the ONE barrier of the rank: partials and residuals published
      cluster_arrive_release();
      if (r + 1 < rlast) {
        double pc[DIM];
#pragma unroll
        for (int a = 0; a < DIM; ++a) pc[a] = s_cc[(r + 1) * 4 + a];
        E.phi2(E.r2_pts(y0, pc), E.r2_pts(y1, pc), na0, na1);
      }
      cluster_wait_acquire();
      // identical decision in every CTA and warp: lane c < CL reads CTA c's partial (CL
      // remote loads per warp instead of CL x 4 per thread), one fixed butterfly combines
      // them (commutative at every node: the same bits in every lane, warp and CTA); the
      // nonzero flag is "maximum > 0" as in the smooth kernel
      {
        double ps = 0.0, pb = 0.0;
        int pi = 0x7fffffff;
        if (lane < CL) {
          const double* q = rem(s_part + 8 * par, lane);
          ps = q[0];
          pb = q[2];
          pi = static_cast<int>(q[3]);
        }
#pragma unroll
        for (int o = CL / 2; o; o >>= 1) ps = hadd(ps, __shfl_xor_sync(0xffffffffu, ps, o));
        warp_argmax_nonneg(pb, pi);
        sum = __shfl_sync(0xffffffffu, ps, 0);  // lanes >= CL folded zeros: lane 0's value for all
        bv = pb;
        bi = pi;
        nz = bv > 0.0 ? 1 : 0;
      }
      int st = 0;
      if (nz) {
        if (r == 0) {
          st = 1;
        } else {
          const double Tlo = hmul(kEps0sq, s_lo), Thi = hmul(kEps0sq, s_hi);
          const double lo = hmul(sum, 1.0 - 4.0 * gm), hi = hmul(sum, 1.0 + 4.0 * gm);
          st = lo > Thi ? 1 : (hi <= Tlo ? 0 : 2);
        }
      }
      if (st != 1) {  // rejection, or a decision the bound cannot settle: general kernel
        fallback = true;
        break;
      }
      if (r == 0) {
        s_lo = hmul(sum, 1.0 - 4.0 * gm);
        s_hi = hmul(sum, 1.0 + 4.0 * gm);
      }
      const int p = bi, po = p / NCAP, pl = p - po * NCAP;
      // u_l[p] (l < r) and the pivot value from the owner CTA
      if (t < r) s_up[t] = *rem(s_u + t * NCAP + pl, po);
      if (t == KC) s_misc[1] = *rem(s_res + par * NCAP + pl, po);
      if (t >= 32 && t < 32 + DIM) s_misc[2 + t - 32] = *rem(s_part + 8 * par + 4 + (t - 32), po);  // pivot point
      if (po == cr && t == (pl % TT)) {
        if (pl >= TT) used1 = true;
        else used0 = true;
      }
      __syncthreads();
      const PivotDiv pdiv(s_misc[1]);
      s_u[r * NCAP + t] = rv0 ? pdiv(a0) : 0.0;  // u_r (aca.cpp:466-470)
      s_u[r * NCAP + t + TT] = rv1 ? pdiv(a1) : 0.0;
      // pivot row: own columns [512 cr, 512 cr + 512), plus the candidate columns c < k
      {
        double yp[DIM];
#pragma unroll
        for (int a = 0; a < DIM; ++a) yp[a] = s_misc[2 + a];
        const int j0 = row0 + t, j1 = row0 + t + TT;
        const bool cv0 = j0 < n, cv1 = j1 < n;
        const int jj0 = cv0 ? j0 : 0, jj1 = cv1 ? j1 : 0;
        // v_r at the candidate columns c < k (this CTA's copy): CTA 0 owns those columns
        // (its lane t < k computes column t below); elsewhere warp 0 evaluates them
        // interleaved with its own two columns (one 3-way evaluation, not two 2-way ones
        // in sequence, so warp 0 does not hold the end-of-rank barrier)
        const bool cand = cr != 0 && wib == 0;
        // (an L1 prefetch of the own columns' V rows here measured 1-4% slower)
        double b0, b1, c0 = 0.0;
        if (cand) {
          double pc[DIM];
          const int tc = (t < KC && t < n) ? t : 0;
#pragma unroll
          for (int a = 0; a < DIM; ++a) pc[a] = s_cc[tc * 4 + a];
          E.phi3(E.r2_pts(yp, yc0), E.r2_pts(yp, yc1), E.r2_pts(yp, pc), b0, b1, c0);
        } else {
          E.phi2(E.r2_pts(yp, yc0), E.r2_pts(yp, yc1), b0, b1);
        }
        SmoothChain<KC>::row2<1>(b0, b1, s_up, V + static_cast<long long>(jj0) * kmax,
                                 V + static_cast<long long>(jj1) * kmax, r);
        if (cv0) V[static_cast<long long>(j0) * kmax + r] = b0;
        if (cv1) V[static_cast<long long>(j1) * kmax + r] = b1;
        if (t < KC && t < n) {
          if (cr == 0) {
            s_vc[r * KC + t] = b0;  // column j0 = t: the same chain over the same v_l values
          } else {
            double c1 = c0;
            SmoothChain<KC>::row2<KC>(c0, c1, s_up, s_vc + t, s_vc + t, r);
            s_vc[r * KC + t] = c0;
          }
        }
      }
      if (cr == 0 && t == 0) {
        J.row_piv[static_cast<long long>(b) * kmax + r] = p;
        J.col_piv[static_cast<long long>(b) * kmax + r] = r;
      }
      k_eff = r + 1;
      __syncthreads();
    }
    if (fallback) {
      if (cr == 0 && t == 0) J.fb_list[atomicAdd(J.fb_count, 1)] = b;
      cluster.sync();  // every CTA is done with this block's shared buffers
      continue;
    }
    double* U = J.U + (J.u_off[b] - J.u_base);
    const int tsh = J.tile_shift;
    auto uix = [&](int l, int i) -> long long {
      if (tsh < 0) return static_cast<long long>(l) * m + i;
      return ((static_cast<long long>(i >> tsh) * kmax + l) << tsh) + (i & ((1 << tsh) - 1));
    };
#pragma unroll
    for (int l = 0; l < KC; ++l) {
      if (rv0) U[uix(l, i0)] = l < k_eff ? s_u[l * NCAP + t] : 0.0;
      if (rv1) U[uix(l, i1)] = l < k_eff ? s_u[l * NCAP + t + TT] : 0.0;
    }
    if (k_eff < kmax)
      for (int j = row0 + t; j < min(n, row0 + NCAP); j += TT)
        for (int l = k_eff; l < kmax; ++l) V[static_cast<long long>(j) * kmax + l] = 0.0;
    if (cr == 0) {
      for (int l = k_eff + t; l < kmax; l += TT) {
        J.row_piv[static_cast<long long>(b) * kmax + l] = -1;
        J.col_piv[static_cast<long long>(b) * kmax + l] = -1;
      }
      if (t == 0) {
        J.k_eff[b] = k_eff;
        if (J.evals) {
          atomicAdd(J.evals, static_cast<unsigned long long>(k_eff) * m);
          atomicAdd(J.evals + 1, static_cast<unsigned long long>(k_eff) * n);
          atomicAdd(J.evals + 2, 1ull);
        }
      }
    }
    cluster.sync();  // shared buffers free for the next block
  }
}

template <int DIM, int KIND, int CL>
void launch_smooth_cluster(const AcaJob& J, const KernelEntry<DIM, KIND>& E, int sms, cudaStream_t s) {
  if (J.njobs <= 0) return;
  const size_t smem = sizeof(double) * (16 * 512 + 2 * 512 + 16 * 16 + 16 + 64 + 16 + 8 + 64);
  auto kfn = aca_smooth_cluster_kernel<DIM, KIND, CL>;
  HM_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const long long clusters = std::min<long long>(J.njobs, std::max(1, 2 * sms / CL));
  kfn<<<static_cast<unsigned>(clusters * CL), 256, smem, s>>>(J, E);
  HM_LAUNCH_CHECK();
}

template <int DIM, int KIND, int KC>
void launch_big(const AcaJob& J, const KernelEntry<DIM, KIND>& E, int max_rows, int sms, DevBuf<double>& scratch,
                cudaStream_t s, bool smooth1) {
  if (J.njobs <= 0) return;
  const int mask_words = (max_rows + 31) / 32;
  const size_t smem = ((mask_words + 1) / 2 + kKmax + 40) * sizeof(double);
  auto kfn = aca_big_kernel<DIM, KIND, KC>;
  HM_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int occ = 0;
  HM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, kBigThreads, smem));
  const long long ctas = std::min<long long>(J.njobs, static_cast<long long>(std::max(occ, 1)) * sms);
  // per-CTA window of kBigW columns (L2-resident); a persistent per-handle workspace,
  // grown on first use (no allocation inside a steady-state product)
  const long long gstride = max_rows + 1;
  const size_t need = static_cast<size_t>(gstride) * kBigW * ctas;
  if (scratch.size() < need) scratch.alloc(need, s);
  kfn<<<static_cast<unsigned>(std::max(ctas, 1ll)), kBigThreads, smem, s>>>(J, E, scratch.get(), gstride, mask_words,
                                                                            smooth1 ? 1 : 0);
  HM_LAUNCH_CHECK();
}

// ACA size classes: team kernels for max(m, n) <= 64 * NW (NW = 1, 2, 4, 8), the
// CTA kernel for larger blocks, for k > 32 and for the epsilon criterion.
constexpr int kAcaCl4 = 5;                // aca_cluster_kernel, 4 CTAs (<= 2048 rows)
constexpr int kAcaCl8 = 6;                // aca_cluster_kernel, 8 CTAs (<= 4096 rows)
constexpr int kAcaBig = 7;                // aca_big_kernel
constexpr int kAcaCta = kAcaClasses - 1;  // the general CTA kernel (epsilon criterion, k > 32)
__host__ __device__ inline int aca_class(int m, int n, long long kmax, bool has_eps, bool clusters = true) {
  if (has_eps || kmax > 32) return kAcaCta;
  const int c = m > n ? m : n;
  if (c <= 1024) return c <= 64 ? 0 : c <= 128 ? 1 : c <= 256 ? 2 : c <= 512 ? 3 : 4;
  if (clusters && c <= 2048) return kAcaCl4;
  if (clusters && c <= 4096) return kAcaCl8;
  return kAcaBig;
}

// Everything one size-class launch sequence needs; the kernels are instantiated per
// point dimension in separate translation units (aca_dim.cu, built once per DIM) so the
// library compiles in parallel.
struct AcaClassLaunch {
  AcaJob J[kAcaClasses];       // per class: job list, count, counter
  int sms = 0;
  int max_rows_big = 0;
  int kind = 0;                // kGaussian / kMatern
  KernelParams kp{};
  const double* coords = nullptr;
  long long n = 0;
  int d = 0;
  int device = 0;
  DevBuf<double>* big_scratch = nullptr;  // persistent window scratch of the big-block kernel
  PhaseTrace* tr = nullptr;
  bool smooth = false;         // smooth-path kernels for the <= 256 classes (fallback lists)
  bool smooth_pre = false;     // ... with the candidate columns evaluated up front
  bool smooth_mid = false;     // smooth cluster kernel also for <= 512 / <= 1024 (CL = 1, 2;
                               // measured slower than the window kernels there: off)
  bool big_one = false;        // big-block kernel: one-column window until a rejection (d >= 3)
  int* fb_list = nullptr;      // per class q at offset first[q]: blocks handed back
  int* fb_count = nullptr;     // kAcaClasses counts
  int* fb_counter = nullptr;   // kAcaClasses job counters of the fallback passes
  long long first[kAcaClasses + 1] = {};
  cudaStream_t s2 = nullptr;   // second stream: cluster / big kernels beside the window kernels
};
void aca_classes_d0(const AcaClassLaunch& L, cudaStream_t s);
void aca_classes_d1(const AcaClassLaunch& L, cudaStream_t s);
void aca_classes_d2(const AcaClassLaunch& L, cudaStream_t s);
void aca_classes_d3(const AcaClassLaunch& L, cudaStream_t s);
void aca_classes_d4(const AcaClassLaunch& L, cudaStream_t s);

}  // namespace aca_detail
}  // namespace hmb

// mvp.cu -- K6 near field, K8 low-rank apply, K9 permutations (sm_100a).
//
// Reference: mvp() hmatrix.cpp:66-123.  z = 0; for every dense leaf in leaf
// order: z[row] += ((0 + a_0 x_0) + a_1 x_1) + ... (dense_blocks.cpp:101-116);
// then for every admissible leaf in leaf order: z[row] += ((0 + u_0 t_0) + u_1 t_1)
// + ... with t_l = ((v_l0 x_0 + v_l1 x_1) + ...) (aca.cpp:597-619).
//
// B200 mapping ("row gather"): one thread per Morton row i walks the chain of
// row clusters containing i in canonical order (row.lower asc, row.upper asc,
// tree.cpp:189-194) and, per cluster, the contiguous run of its leaves.  Each
// leaf contributes with the reference's own summation order, so the product is
// bitwise identical to the single-thread reference -- no atomics, no staging.
// Stored dense blocks are column-major (entry (i,j) at j*m + i) so the threads
// of a row cluster stream each block with fully coalesced 256-B warp loads;
// U is rank-major (coalesced over i), V interleaved n x k (coalesced over l).
#include <algorithm>
#include <chrono>
#include <vector>

#include "hmatrix.h"
#include "primitives.h"

namespace hmb {

namespace {

constexpr int kMaxDepth = 32;

__global__ void gather_x_kernel(const double* __restrict__ x, const long long* __restrict__ perm, long long n,
                                double* __restrict__ xm) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    xm[i] = x[perm[i]];  // permute_vector Forward (core.cpp:167-177)
}

__global__ void scatter_z_kernel(const double* __restrict__ zm, const long long* __restrict__ perm, long long n,
                                 double* __restrict__ z) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    z[perm[i]] = zm[i];  // permute_vector Inverse
}

// stored near field: column-major blocks
template <int DIM>
__global__ void store_dense_kernel(const double* __restrict__ coords, long long n, int d, KernelParams kp,
                                   const int* __restrict__ rl, const int* __restrict__ m, const int* __restrict__ cl,
                                   const int* __restrict__ nn, long long leaf_begin, long long leaf_end,
                                   const long long* __restrict__ off, long long off_base, double* __restrict__ vals) {
  for (long long b = leaf_begin + blockIdx.x; b < leaf_end; b += gridDim.x) {
    const int r0 = rl[b], mb = m[b], c0 = cl[b], nb = nn[b];
    double* out = vals + (off[b] - off_base);
    const long long total = static_cast<long long>(mb) * nb;
    for (long long e = threadIdx.x; e < total; e += blockDim.x) {
      const long long j = e / mb, i = e % mb;
      double r2 = 0.0;
      if constexpr (DIM > 0) {
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
          const double dx = hsub(__ldg(coords + a * n + r0 + i), __ldg(coords + a * n + c0 + j));
          r2 = hadd(r2, hmul(dx, dx));
        }
      } else {
        for (int a = 0; a < d; ++a) {
          const double dx = hsub(__ldg(coords + a * n + r0 + i), __ldg(coords + a * n + c0 + j));
          r2 = hadd(r2, hmul(dx, dx));
        }
      }
      out[e] = phi_r2(kp, r2);
    }
  }
}

// t[b, l] = v_l . x_sigma with the reference's left fold starting at the first product
__global__ void lowrank_t_kernel(const int* __restrict__ order, long long njobs, const int* __restrict__ cl,
                                 const int* __restrict__ nn, const int* __restrict__ k_eff,
                                 const long long* __restrict__ v_off, long long v_base, const double* __restrict__ V,
                                 const double* __restrict__ xm, int kmax, int G, double* __restrict__ t) {
  const long long gtid = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long job = gtid / G;
  const int l = static_cast<int>(gtid % G);
  if (job >= njobs) return;
  const int b = order[job];
  const int ke = k_eff[b];
  if (l >= kmax) return;
  if (l >= ke) {
    t[static_cast<long long>(b) * kmax + l] = 0.0;
    return;
  }
  const int n = nn[b];
  const double* v = V + (v_off[b] - v_base) + l;
  const double* x = xm + cl[b];
  double acc = hmul(v[0], x[0]);
  int j = 1;
  for (; j + 4 <= n; j += 4) {
    const double v0 = v[static_cast<long long>(j) * kmax], v1 = v[static_cast<long long>(j + 1) * kmax];
    const double v2 = v[static_cast<long long>(j + 2) * kmax], v3 = v[static_cast<long long>(j + 3) * kmax];
    const double x0 = x[j], x1 = x[j + 1], x2 = x[j + 2], x3 = x[j + 3];
    acc = hadd(acc, hmul(v0, x0));
    acc = hadd(acc, hmul(v1, x1));
    acc = hadd(acc, hmul(v2, x2));
    acc = hadd(acc, hmul(v3, x3));
  }
  for (; j < n; ++j) acc = hadd(acc, hmul(v[static_cast<long long>(j) * kmax], x[j]));
  t[static_cast<long long>(b) * kmax + l] = acc;
}

struct RowArgs {
  long long n;
  long long row_begin, row_end;
  int dmax;                      // deepest leaf depth
  const double* coords;
  int d;
  KernelParams kp;
  const double* xm;
  const double* z_in;            // nullptr: start from 0
  double* z_out;
  // dense list
  const int* d_rl;
  const int* d_m;
  const int* d_cl;
  const int* d_n;
  const int* d_rs;
  const int* d_re;
  const long long* d_off;        // stored mode
  long long d_off_base;
  const double* d_vals;
  // aca list (window [a_lo, a_hi) of leaves)
  const int* a_rl;
  const int* a_m;
  const int* a_rs;
  const int* a_re;
  const int* a_keff;
  const long long* a_uoff;
  long long a_ubase;
  const double* U;
  const double* t;
  int kmax;
  long long a_lo, a_hi;
};

template <int DIM, int NEAR /*0 none, 1 recompute, 2 stored*/, bool FAR>
__global__ void __launch_bounds__(256) rows_kernel(RowArgs a) {
  const long long i = a.row_begin + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= a.row_end) return;
  // chain of clusters containing row i: slot of depth e = 2^e - 1 + idx_e
  long long lo_e[kMaxDepth];
  long long slot_e[kMaxDepth];
  {
    long long lo = 0, hi = a.n, idx = 0;
    for (int e = 0; e <= a.dmax; ++e) {
      lo_e[e] = lo;
      slot_e[e] = ((1ll << e) - 1) + idx;
      const long long mid = lo + (hi - lo + 1) / 2;
      if (i < mid) {
        hi = mid;
        idx = 2 * idx;
      } else {
        lo = mid;
        idx = 2 * idx + 1;
      }
    }
  }
  double yi[DIM > 0 ? DIM : 20];
  if constexpr (NEAR == 1) {
    if constexpr (DIM > 0) {
#pragma unroll
      for (int q = 0; q < DIM; ++q) yi[q] = a.coords[q * a.n + i];
    } else {
      for (int q = 0; q < a.d; ++q) yi[q] = a.coords[q * a.n + i];
    }
  }
  double z = a.z_in ? a.z_in[i] : 0.0;

  // canonical order of the chain: groups of equal row.lower ascending; inside a group
  // the deeper (smaller row.upper) cluster first
  if constexpr (NEAR != 0) {
    for (int e0 = 0; e0 <= a.dmax;) {
      int e1 = e0;
      while (e1 + 1 <= a.dmax && lo_e[e1 + 1] == lo_e[e0]) ++e1;
      for (int e = e1; e >= e0; --e) {
        const long long s = slot_e[e];
        const int rs = a.d_rs[s];
        if (rs < 0) continue;
        const int re = a.d_re[s];
        for (int L = rs; L < re; ++L) {
          const int r0 = a.d_rl[L], mb = a.d_m[L], c0 = a.d_cl[L], nb = a.d_n[L];
          const double* x = a.xm + c0;
          double y = 0.0;
          if constexpr (NEAR == 2) {
            const double* col = a.d_vals + (a.d_off[L] - a.d_off_base) + (i - r0);
            int j = 0;
            for (; j + 8 <= nb; j += 8) {
              double av[8], xv[8];
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                av[q] = __ldcs(col + static_cast<long long>(j + q) * mb);
                xv[q] = __ldg(x + j + q);
              }
#pragma unroll
              for (int q = 0; q < 8; ++q) y = hadd(y, hmul(av[q], xv[q]));
            }
            for (; j < nb; ++j) y = hadd(y, hmul(__ldcs(col + static_cast<long long>(j) * mb), __ldg(x + j)));
          } else {
            for (int j = 0; j < nb; ++j) {
              double r2 = 0.0;
              if constexpr (DIM > 0) {
#pragma unroll
                for (int q = 0; q < DIM; ++q) {
                  const double dx = hsub(yi[q], __ldg(a.coords + q * a.n + c0 + j));
                  r2 = hadd(r2, hmul(dx, dx));
                }
              } else {
                for (int q = 0; q < a.d; ++q) {
                  const double dx = hsub(yi[q], __ldg(a.coords + q * a.n + c0 + j));
                  r2 = hadd(r2, hmul(dx, dx));
                }
              }
              y = hadd(y, hmul(phi_r2(a.kp, r2), __ldg(x + j)));
            }
          }
          z = hadd(z, y);
        }
      }
      e0 = e1 + 1;
    }
  }
  if constexpr (FAR) {
    for (int e0 = 0; e0 <= a.dmax;) {
      int e1 = e0;
      while (e1 + 1 <= a.dmax && lo_e[e1 + 1] == lo_e[e0]) ++e1;
      for (int e = e1; e >= e0; --e) {
        const long long s = slot_e[e];
        int rs = a.a_rs[s];
        if (rs < 0) continue;
        int re = a.a_re[s];
        rs = static_cast<int>(max(static_cast<long long>(rs), a.a_lo));
        re = static_cast<int>(min(static_cast<long long>(re), a.a_hi));
        for (int L = rs; L < re; ++L) {
          const int r0 = a.a_rl[L], mb = a.a_m[L], ke = a.a_keff[L];
          const double* u = a.U + (a.a_uoff[L] - a.a_ubase) + (i - r0);
          const double* tl = a.t + static_cast<long long>(L) * a.kmax;
          double y = 0.0;
          for (int l = 0; l < ke; ++l) y = hadd(y, hmul(__ldcs(u + static_cast<long long>(l) * mb), __ldg(tl + l)));
          z = hadd(z, y);
        }
      }
      e0 = e1 + 1;
    }
  }
  a.z_out[i] = z;
}

template <int DIM>
void launch_rows(const RowArgs& a, int near, bool far, cudaStream_t s) {
  const long long rows = a.row_end - a.row_begin;
  if (rows <= 0) return;
  const unsigned grid = grid_for(rows, 256);
#define HM_ROWS(NEAR, FAR) rows_kernel<DIM, NEAR, FAR><<<grid, 256, 0, s>>>(a)
  if (near == 2 && far) HM_ROWS(2, true);
  else if (near == 2) HM_ROWS(2, false);
  else if (near == 1 && far) HM_ROWS(1, true);
  else if (near == 1) HM_ROWS(1, false);
  else if (far) HM_ROWS(0, true);
  else HM_ROWS(0, false);
#undef HM_ROWS
  HM_LAUNCH_CHECK();
}

void dispatch_rows(const HMatrix& h, const RowArgs& a, int near, bool far, cudaStream_t s) {
  switch (h.d) {
    case 1: launch_rows<1>(a, near, far, s); break;
    case 2: launch_rows<2>(a, near, far, s); break;
    case 3: launch_rows<3>(a, near, far, s); break;
    case 4: launch_rows<4>(a, near, far, s); break;
    default: launch_rows<0>(a, near, far, s); break;
  }
}

long long lower_bound_rows(const std::vector<int>& rl, long long v) {
  return std::lower_bound(rl.begin(), rl.end(), v, [](int a, long long b) { return a < b; }) - rl.begin();
}

RowArgs base_row_args(HMatrix& h) {
  RowArgs a{};
  a.n = h.n;
  a.row_begin = h.row_begin;
  a.row_end = h.row_end;
  a.dmax = h.dmax_leaf;
  a.coords = h.coords.get();
  a.d = h.d;
  a.kp = h.kp;
  a.xm = h.xm.get();
  a.z_out = h.zm.get();
  a.d_rl = h.dense.rl.get();
  a.d_m = h.dense.m.get();
  a.d_cl = h.dense.cl.get();
  a.d_n = h.dense.n.get();
  a.d_rs = h.dense.run_start.get();
  a.d_re = h.dense.run_end.get();
  a.d_off = h.dense_off.get();
  a.d_vals = h.dense_vals.get();
  a.a_rl = h.aca.rl.get();
  a.a_m = h.aca.m.get();
  a.a_rs = h.aca.run_start.get();
  a.a_re = h.aca.run_end.get();
  a.a_keff = h.k_eff.get();
  a.a_uoff = h.u_off.get();
  a.U = h.U.get();
  a.t = h.t.get();
  a.kmax = static_cast<int>(h.cfg.k);
  return a;
}

void launch_t(HMatrix& h, long long njobs, long long v_base, cudaStream_t s) {
  if (njobs <= 0) return;
  int G = 1;
  while (G < h.cfg.k) G <<= 1;
  if (G > 32) raise(kEinval, "k > 32 not supported by the low-rank apply");
  const long long threads = njobs * G;
  lowrank_t_kernel<<<grid_for(threads, 256), 256, 0, s>>>(h.aca_order.get(), njobs, h.aca.cl.get(), h.aca.n.get(),
                                                          h.k_eff.get(), h.v_off.get(), v_base, h.V.get(),
                                                          h.xm.get(), static_cast<int>(h.cfg.k), G, h.t.get());
  HM_LAUNCH_CHECK();
}

}  // namespace

// own leaf ranges of the two lists (rows [row_begin,row_end))
static void own_range(const LeafList& l, long long rb, long long re, long long& lo, long long& hi) {
  lo = lower_bound_rows(l.h_rl, rb);
  hi = lower_bound_rows(l.h_rl, re);
}

void store_near_field(HMatrix& h, cudaStream_t s) {
  long long lo, hi;
  own_range(h.dense, h.row_begin, h.row_end, lo, hi);
  std::vector<long long> off(h.dense.count + 1, 0);
  for (long long b = 0; b < h.dense.count; ++b)
    off[b + 1] = off[b] + static_cast<long long>(h.dense.h_m[b]) * h.dense.h_n[b];
  h.dense_off.alloc(off.size(), s);
  HM_CUDA(cudaMemcpyAsync(h.dense_off.get(), off.data(), sizeof(long long) * off.size(), cudaMemcpyHostToDevice, s));
  const long long total = off[hi] - off[lo];
  h.dense_vals.alloc(std::max(total, 1ll), s);
  const unsigned grid = static_cast<unsigned>(std::min<long long>(std::max(hi - lo, 1ll), 148ll * 32));
#define HM_STORE(D)                                                                                                   \
  store_dense_kernel<D><<<grid, 256, 0, s>>>(h.coords.get(), h.n, h.d, h.kp, h.dense.rl.get(), h.dense.m.get(),       \
                                             h.dense.cl.get(), h.dense.n.get(), lo, hi, h.dense_off.get(), off[lo],  \
                                             h.dense_vals.get())
  switch (h.d) {
    case 1: HM_STORE(1); break;
    case 2: HM_STORE(2); break;
    case 3: HM_STORE(3); break;
    case 4: HM_STORE(4); break;
    default: HM_STORE(0); break;
  }
#undef HM_STORE
  HM_LAUNCH_CHECK();
}

// Allocates offsets and (precompute mode) computes all factors of the own range.
void plan_far_field(HMatrix& h, cudaStream_t s) {
  const long long kmax = h.cfg.k;
  std::vector<long long> uo(h.aca.count + 1, 0), vo(h.aca.count + 1, 0);
  for (long long b = 0; b < h.aca.count; ++b) {
    uo[b + 1] = uo[b] + kmax * h.aca.h_m[b];
    vo[b + 1] = vo[b] + kmax * h.aca.h_n[b];
  }
  h.u_off.alloc(uo.size(), s);
  h.v_off.alloc(vo.size(), s);
  HM_CUDA(cudaMemcpyAsync(h.u_off.get(), uo.data(), sizeof(long long) * uo.size(), cudaMemcpyHostToDevice, s));
  HM_CUDA(cudaMemcpyAsync(h.v_off.get(), vo.data(), sizeof(long long) * vo.size(), cudaMemcpyHostToDevice, s));
  h.k_eff.alloc(std::max(h.aca.count, 1ll), s);
  h.k_eff.zero(s);
  h.row_piv.alloc(std::max(h.aca.count * kmax, 1ll), s);
  h.col_piv.alloc(std::max(h.aca.count * kmax, 1ll), s);
  h.t.alloc(std::max(h.aca.count * kmax, 1ll), s);
  long long lo, hi;
  own_range(h.aca, h.row_begin, h.row_end, lo, hi);
  if (h.cfg.precompute_aca) {
    h.U.alloc(std::max(uo[hi] - uo[lo], 1ll), s);
    h.V.alloc(std::max(vo[hi] - vo[lo], 1ll), s);
    compute_aca(h, lo, hi, s);
    h.factors_valid = true;
    // S_l with the achieved ranks
    std::vector<int> ke(hi - lo);
    if (hi > lo) HM_CUDA(cudaMemcpyAsync(ke.data(), h.k_eff.get() + lo, sizeof(int) * (hi - lo), cudaMemcpyDeviceToHost, s));
    HM_CUDA(cudaStreamSynchronize(s));
    h.S_l = h.S_lm = h.S_ln = 0;
    for (long long b = lo; b < hi; ++b) {
      h.S_lm += static_cast<double>(ke[b - lo]) * h.aca.h_m[b];
      h.S_ln += static_cast<double>(ke[b - lo]) * h.aca.h_n[b];
    }
    h.S_l = h.S_lm + h.S_ln;
  }
}

void mvp_morton(HMatrix& h, cudaStream_t s) {
  RowArgs a = base_row_args(h);
  const int near = h.cfg.near_stored ? 2 : 1;
  long long alo, ahi, dlo, dhi;
  own_range(h.aca, h.row_begin, h.row_end, alo, ahi);
  own_range(h.dense, h.row_begin, h.row_end, dlo, dhi);
  a.d_off_base = 0;
  if (h.cfg.near_stored) {
    long long ob = 0;
    HM_CUDA(cudaMemcpyAsync(&ob, h.dense_off.get() + dlo, sizeof(long long), cudaMemcpyDeviceToHost, s));
    HM_CUDA(cudaStreamSynchronize(s));
    a.d_off_base = ob;
  }
  if (h.cfg.precompute_aca) {
    long long ub = 0, vb = 0;
    HM_CUDA(cudaMemcpyAsync(&ub, h.u_off.get() + alo, sizeof(long long), cudaMemcpyDeviceToHost, s));
    HM_CUDA(cudaMemcpyAsync(&vb, h.v_off.get() + alo, sizeof(long long), cudaMemcpyDeviceToHost, s));
    HM_CUDA(cudaStreamSynchronize(s));
    // aca_order covers [alo, ahi) from the precompute
    h.clk.start(kKLowrankT, s);
    launch_t(h, ahi - alo, vb, s);
    h.clk.stop(kKLowrankT, s);
    a.a_ubase = ub;
    a.a_lo = alo;
    a.a_hi = ahi;
    h.clk.start(kKRows, s);
    dispatch_rows(h, a, near, true, s);
    h.clk.stop(kKRows, s);
    return;
  }
  // recompute mode (reference default): near field first, then ACA chunk by chunk
  h.clk.start(kKRows, s);
  dispatch_rows(h, a, near, false, s);
  h.clk.stop(kKRows, s);
  const long long kmax = h.cfg.k;
  // chunk budget: U+V bytes
  size_t free_b = 0, total_b = 0;
  HM_CUDA(cudaMemGetInfo(&free_b, &total_b));
  long long budget = h.cfg.aca_chunk_rows > 0 ? h.cfg.aca_chunk_rows * kmax * 16
                                              : std::min<long long>(static_cast<long long>(free_b / 4), 8ll << 30);
  budget = std::max(budget, 1ll << 20);
  long long c0 = alo;
  while (c0 < ahi) {
    long long c1 = c0, bytes = 0;
    while (c1 < ahi) {
      const long long add = 8 * kmax * (h.aca.h_m[c1] + h.aca.h_n[c1]);
      if (c1 > c0 && bytes + add > budget) break;
      bytes += add;
      ++c1;
    }
    long long ub = 0, vb = 0, ue = 0, ve = 0;
    HM_CUDA(cudaMemcpyAsync(&ub, h.u_off.get() + c0, sizeof(long long), cudaMemcpyDeviceToHost, s));
    HM_CUDA(cudaMemcpyAsync(&vb, h.v_off.get() + c0, sizeof(long long), cudaMemcpyDeviceToHost, s));
    HM_CUDA(cudaMemcpyAsync(&ue, h.u_off.get() + c1, sizeof(long long), cudaMemcpyDeviceToHost, s));
    HM_CUDA(cudaMemcpyAsync(&ve, h.v_off.get() + c1, sizeof(long long), cudaMemcpyDeviceToHost, s));
    HM_CUDA(cudaStreamSynchronize(s));
    if (h.U.size() < static_cast<size_t>(ue - ub)) h.U.alloc(ue - ub, s);
    if (h.V.size() < static_cast<size_t>(ve - vb)) h.V.alloc(ve - vb, s);
    h.clk.start(kKAca, s);
    compute_aca(h, c0, c1, s);
    h.clk.stop(kKAca, s);
    h.clk.start(kKLowrankT, s);
    launch_t(h, c1 - c0, vb, s);
    h.clk.stop(kKLowrankT, s);
    RowArgs b = base_row_args(h);
    b.z_in = h.zm.get();
    b.a_ubase = ub;
    b.a_lo = c0;
    b.a_hi = c1;
    h.clk.start(kKRowsFar, s);
    dispatch_rows(h, b, 0, true, s);
    h.clk.stop(kKRowsFar, s);
    c0 = c1;
  }
}

void mvp_device(HMatrix& h, const double* x_dev, double* z_dev, cudaStream_t s) {
  const long long n = h.n;
  gather_x_kernel<<<grid_for(n, 256, 1 << 16), 256, 0, s>>>(x_dev, h.perm.get(), n, h.xm.get());
  HM_LAUNCH_CHECK();
  mvp_morton(h, s);
  scatter_z_kernel<<<grid_for(n, 256, 1 << 16), 256, 0, s>>>(h.zm.get(), h.perm.get(), n, z_dev);
  HM_LAUNCH_CHECK();
}

}  // namespace hmb

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
// B200 mapping: one CTA (256 threads) per block, persistent over a largest-first
// queue.  The CTA is split into W = 256/G column groups of G threads
// (G = clamp(pow2ceil(m), 32, 256)) so small blocks evaluate W candidate
// columns per wave; the lowest qualifying index wins, exactly reproducing the
// sequential scan.  Entries are bit-identical to the host (glibc exp port, no
// FMA contraction), so u/v and the pivots are bitwise the reference's.  The only
// order-sensitive quantity, norm2, is summed in parallel with a rigorous error
// bound; decisions inside the bound fall back to the reference's sequential fold.
#include <algorithm>
#include <vector>

#include "hmatrix.h"
#include "primitives.h"

namespace hmb {

namespace {

constexpr int kAcaThreads = 256;
constexpr int kKmax = 64;        // compile-time cap on the rank
constexpr int kColBuf = 2048;    // doubles of shared column buffer

// entry sources ---------------------------------------------------------------
template <int DIM>
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
    return phi_r2(kp, r2);
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
  int tile_shift;           // -1: U rank-major; else log2(S), U row-tiled by S rows
  // explicit-matrix seam: block b entries at dense + dense_off[b], row-major m x n
  const double* dense;
  const long long* dense_off;
};

__device__ __forceinline__ void argmax_combine(double& bv, int& bi, double ov, int oi) {
  if (ov > bv || (ov == bv && oi < bi)) {
    bv = ov;
    bi = oi;
  }
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
      for (int i = tid; i < m; i += kAcaThreads) U[uix(r, i)] = __ddiv_rn(cbv(i), pivot_val);
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
      if (J.rejections && rejections) atomicAdd(J.rejections, rejections);
    }
    __syncthreads();
  }
}

template <int DIM>
void launch_kernel_aca(const AcaJob& J, const HMatrix& h, cudaStream_t s) {
  KernelEntry<DIM> E{h.coords.get(), h.n, h.d, h.kp};
  int occ = 0;
  HM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, aca_kernel<DIM, false>, kAcaThreads, 0));
  int sms = 0;
  HM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h.device));
  const long long grid = std::min<long long>(J.njobs, static_cast<long long>(std::max(occ, 1)) * sms);
  aca_kernel<DIM, false><<<static_cast<unsigned>(std::max(grid, 1ll)), kAcaThreads, 0, s>>>(J, E);
  HM_LAUNCH_CHECK();
}

__global__ void size_key_kernel(const int* __restrict__ m, const int* __restrict__ nn, long long begin, long long cnt,
                                unsigned long long* __restrict__ keys, unsigned* __restrict__ vals) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < cnt;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long b = begin + i;
    // n descending, then m descending: largest first, and the n >= 2048 blocks of the
    // low-rank apply form a prefix
    keys[i] = ((~static_cast<unsigned long long>(nn[b]) & 0xffffffffull) << 32) |
              (~static_cast<unsigned long long>(m[b]) & 0xffffffffull);
    vals[i] = static_cast<unsigned>(b);
  }
}

}  // namespace

// Factorises aca leaves [leaf_begin, leaf_end) into h.U / h.V at offsets
// h.u_off[b] - h.u_off[leaf_begin] (so a chunk workspace can be reused).
void compute_aca(HMatrix& h, long long leaf_begin, long long leaf_end, cudaStream_t s) {
  const long long cnt = leaf_end - leaf_begin;
  if (cnt <= 0) return;
  if (h.cfg.k > kKmax) raise(kEinval, "k > 64 is not supported by the device ACA");
  // largest-first schedule
  DevBuf<unsigned long long> keys;
  keys.alloc(cnt, s);
  h.aca_order.alloc(cnt, s);
  size_key_kernel<<<grid_for(cnt, 256, 1 << 16), 256, 0, s>>>(h.aca.m.get(), h.aca.n.get(), leaf_begin, cnt,
                                                               keys.get(), reinterpret_cast<unsigned*>(h.aca_order.get()));
  HM_LAUNCH_CHECK();
  radix_sort_pairs(keys.get(), reinterpret_cast<unsigned*>(h.aca_order.get()), cnt, s);
  h.aca_long_jobs = 0;
  for (long long b = leaf_begin; b < leaf_end; ++b) h.aca_long_jobs += h.aca.h_n[b] >= 2048 ? 1 : 0;
  h.counter.alloc(1, s);
  h.counter.zero(s);
  DevBuf<unsigned long long> rej;
  rej.alloc(1, s);
  rej.zero(s);
  long long ub = 0, vb = 0;
  HM_CUDA(cudaMemcpyAsync(&ub, h.u_off.get() + leaf_begin, sizeof(long long), cudaMemcpyDeviceToHost, s));
  HM_CUDA(cudaMemcpyAsync(&vb, h.v_off.get() + leaf_begin, sizeof(long long), cudaMemcpyDeviceToHost, s));
  HM_CUDA(cudaStreamSynchronize(s));
  AcaJob J{};
  J.rl = h.aca.rl.get();
  J.m = h.aca.m.get();
  J.cl = h.aca.cl.get();
  J.nn = h.aca.n.get();
  J.order = h.aca_order.get();
  J.njobs = cnt;
  J.u_off = h.u_off.get();
  J.v_off = h.v_off.get();
  J.u_base = ub;
  J.v_base = vb;
  J.U = h.U.get();
  J.V = h.V.get();
  J.k_eff = h.k_eff.get();
  J.row_piv = h.row_piv.get();
  J.col_piv = h.col_piv.get();
  J.kmax = static_cast<int>(h.cfg.k);
  J.has_eps = h.cfg.has_epsilon ? 1 : 0;
  J.eps_factor = h.cfg.epsilon * (1.0 - h.cfg.eta) / (1.0 + h.cfg.epsilon);
  J.counter = h.counter.get();
  J.rejections = rej.get();
  J.tile_shift = h.u_tile_shift;
  switch (h.d) {
    case 1: launch_kernel_aca<1>(J, h, s); break;
    case 2: launch_kernel_aca<2>(J, h, s); break;
    case 3: launch_kernel_aca<3>(J, h, s); break;
    case 4: launch_kernel_aca<4>(J, h, s); break;
    default: launch_kernel_aca<0>(J, h, s); break;
  }
  unsigned long long hrej = 0;
  HM_CUDA(cudaMemcpyAsync(&hrej, rej.get(), sizeof(hrej), cudaMemcpyDeviceToHost, s));
  HM_CUDA(cudaStreamSynchronize(s));
  h.aca_rejections += static_cast<long long>(hrej);
}

// Explicit-matrix seam (aca.cpp:567-578): host blocks in, host factors out in the
// oracle's layout (u: kmax x m rank-major, v: kmax x n rank-major, zero padded).
void aca_dense_blocks(long long nb, const long long* shapes, const double* entries_host, long long kmax, bool has_eps,
                      double eps, double eta, long long* k_eff_out, long long* row_piv_out, long long* col_piv_out,
                      double* u_host, double* v_host, cudaStream_t s) {
  if (kmax < 1) raise(kEinval, "aca: max_rank must be >= 1");
  if (kmax > kKmax) raise(kEinval, "k > 64 is not supported by the device ACA");
  std::vector<int> hm(nb), hn(nb), hz(nb, 0), hord(nb);
  std::vector<long long> uoff(nb), voff(nb), doff(nb);
  long long su = 0, sv = 0, sd = 0;
  for (long long b = 0; b < nb; ++b) {
    hm[b] = static_cast<int>(shapes[2 * b]);
    hn[b] = static_cast<int>(shapes[2 * b + 1]);
    if (hm[b] < 1 || hn[b] < 1) raise(kEinval, "aca: empty block");
    uoff[b] = su;
    voff[b] = sv;
    doff[b] = sd;
    su += kmax * hm[b];
    sv += kmax * hn[b];
    sd += static_cast<long long>(hm[b]) * hn[b];
    hord[b] = static_cast<int>(b);
  }
  DevBuf<int> dm, dn, dz, dord, dk, drp, dcp, cnt;
  DevBuf<long long> duo, dvo, ddo;
  DevBuf<double> dA, dU, dV;
  auto up = [&](auto& buf, const auto& vec) {
    buf.alloc(vec.size(), s);
    HM_CUDA(cudaMemcpyAsync(buf.get(), vec.data(), vec.size() * sizeof(vec[0]), cudaMemcpyHostToDevice, s));
  };
  up(dm, hm);
  up(dn, hn);
  up(dz, hz);
  up(dord, hord);
  up(duo, uoff);
  up(dvo, voff);
  up(ddo, doff);
  dA.alloc(sd, s);
  HM_CUDA(cudaMemcpyAsync(dA.get(), entries_host, sizeof(double) * sd, cudaMemcpyHostToDevice, s));
  dU.alloc(su, s);
  dV.alloc(sv, s);
  dU.zero(s);
  dV.zero(s);
  dk.alloc(nb, s);
  drp.alloc(nb * kmax, s);
  dcp.alloc(nb * kmax, s);
  cnt.alloc(1, s);
  cnt.zero(s);
  AcaJob J{};
  J.rl = dz.get();
  J.m = dm.get();
  J.cl = dz.get();
  J.nn = dn.get();
  J.order = dord.get();
  J.njobs = nb;
  J.u_off = duo.get();
  J.v_off = dvo.get();
  J.U = dU.get();
  J.V = dV.get();
  J.k_eff = dk.get();
  J.row_piv = drp.get();
  J.col_piv = dcp.get();
  J.kmax = static_cast<int>(kmax);
  J.has_eps = has_eps ? 1 : 0;
  J.eps_factor = eps * (1.0 - eta) / (1.0 + eps);
  J.counter = cnt.get();
  J.tile_shift = -1;
  J.dense = dA.get();
  J.dense_off = ddo.get();
  KernelEntry<1> E{nullptr, 0, 1, KernelParams{0, 1, 0.0}};
  aca_kernel<1, true><<<static_cast<unsigned>(std::min<long long>(nb, 1024)), kAcaThreads, 0, s>>>(J, E);
  HM_LAUNCH_CHECK();
  std::vector<int> hk(nb), hrp(nb * kmax), hcp(nb * kmax);
  std::vector<double> hu(su), hv(sv);
  HM_CUDA(cudaMemcpyAsync(hk.data(), dk.get(), sizeof(int) * nb, cudaMemcpyDeviceToHost, s));
  HM_CUDA(cudaMemcpyAsync(hrp.data(), drp.get(), sizeof(int) * nb * kmax, cudaMemcpyDeviceToHost, s));
  HM_CUDA(cudaMemcpyAsync(hcp.data(), dcp.get(), sizeof(int) * nb * kmax, cudaMemcpyDeviceToHost, s));
  HM_CUDA(cudaMemcpyAsync(hu.data(), dU.get(), sizeof(double) * su, cudaMemcpyDeviceToHost, s));
  HM_CUDA(cudaMemcpyAsync(hv.data(), dV.get(), sizeof(double) * sv, cudaMemcpyDeviceToHost, s));
  HM_CUDA(cudaStreamSynchronize(s));
  for (long long b = 0; b < nb; ++b) {
    const long long m = hm[b], n = hn[b];
    k_eff_out[b] = hk[b];
    for (long long l = 0; l < kmax; ++l) {
      row_piv_out[b * kmax + l] = hrp[b * kmax + l];
      col_piv_out[b * kmax + l] = hcp[b * kmax + l];
      const bool live = l < hk[b];
      for (long long i = 0; i < m; ++i) u_host[uoff[b] + l * m + i] = live ? hu[uoff[b] + l * m + i] : 0.0;
      for (long long j = 0; j < n; ++j) v_host[voff[b] + l * n + j] = live ? hv[voff[b] + j * kmax + l] : 0.0;
    }
  }
}

}  // namespace hmb

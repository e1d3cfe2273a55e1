// multi.cu -- H-MVP with R right-hand sides per pass.
//
// Semantics: column r of Z = H(A) X[:, r], exactly the reference mvp() applied to each
// right-hand side (hmatrix.cpp:66-123).  One pass streams (or recomputes) every
// operator entry ONCE and applies it to all R vectors:
//
//   exact mode  every (row, rhs) pair keeps the reference's sequential folds
//               (dense_blocks.cpp:101-116, aca.cpp:597-619), so column r is bitwise
//               equal to a single-RHS product of X[:, r];
//   DMMA mode   (recompute near field, R a multiple of 8) the dense-leaf contractions
//               A_leaf(8x4) X(4x8) run on the FP64 tensor cores (mma.sync m8n8k4 f64):
//               each lane evaluates its own A-fragment entry, so a kernel entry is
//               evaluated once and feeds R/8 DMMAs.  Leaves are still accumulated in
//               leaf order (z += y_leaf, hmatrix.cpp:80-104); only the order inside a
//               leaf changes (relative error ~1e-15).
//
// Layouts: vectors are rhs-major (x[r * n + i], Morton order inside the engine); the
// low-rank coefficients t[(b - t_base) * k + l) * R + r] are chunk-relative so the
// recompute mode's workspace scales with the chunk, not with the whole far field.
#include <algorithm>
#include <vector>

#include "hmatrix.h"
#include "primitives.h"

namespace hmb {

namespace {

constexpr int kMaxR = 16;

__global__ void gather_multi_kernel(const double* __restrict__ X, long long ldx, const long long* __restrict__ perm,
                                    long long n, int R, double* __restrict__ xm, double* __restrict__ xt) {
  const long long tot = n * R;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < tot;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = e / n, i = e - r * n;
    const double v = X[r * ldx + perm[i]];  // permute_vector Forward (core.cpp:167-177)
    xm[e] = v;
    xt[i * kMaxR + r] = v;                  // interleaved copy: the R values of point i contiguous
  }
}

__global__ void scatter_multi_kernel(const double* __restrict__ zm, const long long* __restrict__ perm, long long n,
                                     int R, double* __restrict__ Z, long long ldz) {
  const long long tot = n * R;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < tot;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = e / n, i = e - r * n;
    Z[r * ldz + perm[i]] = zm[e];  // permute_vector Inverse
  }
}

// t[b, l, r] = v_l . x_r(sigma_b), reference left fold starting at the first product
// (aca.cpp:613-614).  A group of G lanes (G = 16 for k <= 16, else 32) per leaf, lane l
// owns rank l; the R folds of a lane are independent chains fed by one V load.
template <int RM>
__global__ void __launch_bounds__(256) t_multi_kernel(const int* __restrict__ order, long long njobs,
                                                      const int* __restrict__ cl, const int* __restrict__ nn,
                                                      const int* __restrict__ k_eff,
                                                      const long long* __restrict__ v_off, long long v_base,
                                                      const double* __restrict__ V, const double* __restrict__ xt,
                                                      long long n_total, int kmax, int R, int G, long long t_base,
                                                      int* __restrict__ counter, double* __restrict__ t) {
  const int lane = threadIdx.x & 31, g = lane / G, l = lane % G;
  const int groups = 32 / G;
  for (;;) {
    long long job0 = 0;
    if (lane == 0) job0 = static_cast<long long>(atomicAdd(counter, 1)) * groups;
    job0 = __shfl_sync(0xffffffffu, job0, 0);
    if (job0 >= njobs) return;
    const long long job = job0 + g;
    if (job < njobs && l < kmax) {
      const int b = order[job];
      const int ke = k_eff[b], n = nn[b];
      double* tb = t + ((static_cast<long long>(b) - t_base) * kmax + l) * R;
      if (l >= ke) {
        for (int r = 0; r < R; ++r) tb[r] = 0.0;
      } else {
        // x interleaved (xt[j * 16 + r]): the R values of column j are one 128-byte line,
        // read as double2; v rows 4 columns ahead, so the loads of a group are in flight
        // together (the folds stay sequential in j, aca.cpp:613-614)
        const double* v = V + (v_off[b] - v_base) + l;
        const double2* x2 = reinterpret_cast<const double2*>(xt + static_cast<long long>(cl[b]) * kMaxR);
        double acc[RM];
        {
          const double v0 = v[0];
#pragma unroll
          for (int r2 = 0; r2 < RM / 2; ++r2) {
            const double2 xv = __ldg(x2 + r2);
            acc[2 * r2] = hmul(v0, xv.x);
            acc[2 * r2 + 1] = hmul(v0, xv.y);
          }
        }
        int j = 1;
        for (; j + 4 <= n; j += 4) {
          double vj[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) vj[u] = v[static_cast<long long>(j + u) * kmax];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int r2 = 0; r2 < RM / 2; ++r2) {
              const double2 xv = __ldg(x2 + static_cast<long long>(j + u) * (kMaxR / 2) + r2);
              acc[2 * r2] = hadd(acc[2 * r2], hmul(vj[u], xv.x));
              acc[2 * r2 + 1] = hadd(acc[2 * r2 + 1], hmul(vj[u], xv.y));
            }
          }
        }
        for (; j < n; ++j) {
          const double vj = v[static_cast<long long>(j) * kmax];
#pragma unroll
          for (int r2 = 0; r2 < RM / 2; ++r2) {
            const double2 xv = __ldg(x2 + static_cast<long long>(j) * (kMaxR / 2) + r2);
            acc[2 * r2] = hadd(acc[2 * r2], hmul(vj, xv.x));
            acc[2 * r2 + 1] = hadd(acc[2 * r2 + 1], hmul(vj, xv.y));
          }
        }
#pragma unroll
        for (int r = 0; r < RM; ++r)
          if (r < R) tb[r] = acc[r];
      }
    }
  }
}

struct MArgs {
  long long n, row_begin, row_end;
  int R;
  const double* coords;
  int d;
  KernelParams kp;
  const double* xm;  // R x n
  double* zm;        // R x n
  int z_acc;         // 1: accumulate into zm (recompute-mode far chunks)
  // dense leaves
  const int *d_rl, *d_m, *d_cl, *d_n;
  const long long* d_off;
  const double* d_vals;
  const double* part;  // symmetric near field: part[((L * S) + i) * R + r]
  int S;
  // admissible leaves in [a_lo, a_hi)
  const int *a_rl, *a_m, *a_keff;
  const long long* a_uoff;
  long long a_ubase;
  const double* U;
  int tile_shift, kmax;
  const double* t;
  long long t_base;
  long long a_lo, a_hi;
  // canonical spans per deepest row cluster
  const int *row_cluster, *dspan_ptr, *dspans, *aspan_ptr, *aspans;
};

// One thread per Morton row, R accumulators: the single-RHS row product
// (mvp.cu rows_kernel) with every entry applied to all R vectors.
// NEAR: 0 none, 1 recompute, 2 stored (full), 3 symmetric partials.
template <int DIM, int NEAR, bool FAR, int RM>
__global__ void __launch_bounds__(128) rows_multi_kernel(MArgs a) {
  const long long i = a.row_begin + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= a.row_end) return;
  const int R = a.R;
  const int c = __ldg(a.row_cluster + i);
  double z[RM], y[RM];
#pragma unroll
  for (int r = 0; r < RM; ++r) z[r] = (r < R && a.z_acc) ? a.zm[r * a.n + i] : 0.0;
  if constexpr (NEAR != 0) {
    double yi[DIM > 0 ? DIM : 20];
    if constexpr (NEAR == 1) {
      const int dd = DIM > 0 ? DIM : a.d;
      for (int q = 0; q < dd; ++q) yi[q] = a.coords[q * a.n + i];
    }
    const int p1 = __ldg(a.dspan_ptr + c + 1);
    for (int p = __ldg(a.dspan_ptr + c); p < p1; ++p) {
      const int rs = __ldg(a.dspans + 2 * p), re = __ldg(a.dspans + 2 * p + 1);
      for (int L = rs; L < re; ++L) {
        const int r0 = a.d_rl[L], mb = a.d_m[L], c0 = a.d_cl[L], nb = a.d_n[L];
        if constexpr (NEAR == 3) {
          const double* pp = a.part + (static_cast<long long>(L) * a.S + (i - r0)) * R;
#pragma unroll
          for (int r = 0; r < RM; ++r)
            if (r < R) z[r] = hadd(z[r], pp[r]);
          continue;
        }
#pragma unroll
        for (int r = 0; r < RM; ++r) y[r] = 0.0;
        const double* col = NEAR == 2 ? a.d_vals + a.d_off[L] + (i - r0) : nullptr;
        for (int j = 0; j < nb; ++j) {
          double av;
          if constexpr (NEAR == 2) {
            av = __ldcs(col + static_cast<long long>(j) * mb);
          } else {
            double r2 = 0.0;
            const int dd = DIM > 0 ? DIM : a.d;
#pragma unroll
            for (int q = 0; q < (DIM > 0 ? DIM : 20); ++q) {
              if (q >= dd) break;
              const double dx = hsub(yi[q], __ldg(a.coords + q * a.n + c0 + j));
              r2 = hadd(r2, hmul(dx, dx));
            }
            av = phi_r2(a.kp, r2);
          }
#pragma unroll
          for (int r = 0; r < RM; ++r)
            if (r < R) y[r] = hadd(y[r], hmul(av, __ldg(a.xm + r * a.n + c0 + j)));
        }
#pragma unroll
        for (int r = 0; r < RM; ++r)
          if (r < R) z[r] = hadd(z[r], y[r]);
      }
    }
  }
  if constexpr (FAR) {
    const int tsh = a.tile_shift, kmax = a.kmax;
    const int p1 = __ldg(a.aspan_ptr + c + 1);
    for (int p = __ldg(a.aspan_ptr + c); p < p1; ++p) {
      const int rs = static_cast<int>(max(static_cast<long long>(__ldg(a.aspans + 2 * p)), a.a_lo));
      const int re = static_cast<int>(min(static_cast<long long>(__ldg(a.aspans + 2 * p + 1)), a.a_hi));
      for (int L = rs; L < re; ++L) {
        const int r0 = __ldg(a.a_rl + L), mb = __ldg(a.a_m + L), ke = __ldg(a.a_keff + L);
        const double* u = a.U + (__ldg(a.a_uoff + L) - a.a_ubase);
        const long long ii = i - r0;
        const double* tl = a.t + (static_cast<long long>(L) - a.t_base) * kmax * R;
#pragma unroll
        for (int r = 0; r < RM; ++r) y[r] = 0.0;
        if (R == RM && kmax == 16 && RM % 2 == 0) {
          // all u_l of the row issued at once (HBM latency paid once per leaf, not per rank);
          // t_l as double2 (R values contiguous per rank)
          double uv[16];
#pragma unroll
          for (int l = 0; l < 16; ++l) {
            const long long ui = tsh < 0 ? static_cast<long long>(l) * mb + ii
                                         : (((ii >> tsh) * 16 + l) << tsh) + (ii & ((1ll << tsh) - 1));
            uv[l] = l < ke ? __ldcs(u + ui) : 0.0;
          }
          const double2* t2 = reinterpret_cast<const double2*>(tl);
#pragma unroll
          for (int l = 0; l < 16; ++l) {
            if (l < ke) {
#pragma unroll
              for (int r2 = 0; r2 < RM / 2; ++r2) {
                const double2 tv = __ldg(t2 + l * (RM / 2) + r2);
                y[2 * r2] = hadd(y[2 * r2], hmul(uv[l], tv.x));  // ((0 + u_0 t_0) + ...) aca.cpp:616
                y[2 * r2 + 1] = hadd(y[2 * r2 + 1], hmul(uv[l], tv.y));
              }
            }
          }
        } else {
          for (int l = 0; l < ke; ++l) {
            const long long ui = tsh < 0 ? static_cast<long long>(l) * mb + ii
                                         : (((ii >> tsh) * kmax + l) << tsh) + (ii & ((1ll << tsh) - 1));
            const double uv = __ldcs(u + ui);
#pragma unroll
            for (int r = 0; r < RM; ++r)
              if (r < R) y[r] = hadd(y[r], hmul(uv, __ldg(tl + l * R + r)));  // ((0 + u_0 t_0) + ...) aca.cpp:616
          }
        }
#pragma unroll
        for (int r = 0; r < RM; ++r)
          if (r < R) z[r] = hadd(z[r], y[r]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < RM; ++r)
    if (r < R) a.zm[r * a.n + i] = z[r];
}

// Far field only, 16 right-hand sides: TWO threads per row, each owning 8 of them (the
// register footprint of 16 accumulators + 16 leaf partials per thread held the one-thread-
// per-row kernel to 8 warps per SM).  Per leaf the thread's u_l are issued 4 ranks ahead;
// the folds are the reference's: y_r = ((0 + u_0 t_0r) + u_1 t_1r) + ..., z_r += y_r in
// leaf order (aca.cpp:616, hmatrix.cpp:96-113) -- bitwise the one-thread version.
__global__ void __launch_bounds__(128, 4) rows_multi_far16_kernel(MArgs a) {
  constexpr int RH = 8;
  const long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long i = a.row_begin + (g >> 1);
  const int half = static_cast<int>(g & 1);
  if (i >= a.row_end) return;
  const int c = __ldg(a.row_cluster + i);
  double z[RH];
#pragma unroll
  for (int r = 0; r < RH; ++r) z[r] = a.z_acc ? a.zm[(half * RH + r) * a.n + i] : 0.0;
  const int tsh = a.tile_shift;
  const int p1 = __ldg(a.aspan_ptr + c + 1);
  for (int p = __ldg(a.aspan_ptr + c); p < p1; ++p) {
    const int rs = static_cast<int>(max(static_cast<long long>(__ldg(a.aspans + 2 * p)), a.a_lo));
    const int re = static_cast<int>(min(static_cast<long long>(__ldg(a.aspans + 2 * p + 1)), a.a_hi));
    for (int L = rs; L < re; ++L) {
      const int r0 = __ldg(a.a_rl + L), mb = __ldg(a.a_m + L), ke = __ldg(a.a_keff + L);
      const double* u = a.U + (__ldg(a.a_uoff + L) - a.a_ubase);
      const long long ii = i - r0;
      auto uidx = [&](int l) -> long long {
        return tsh < 0 ? static_cast<long long>(l) * mb + ii : (((ii >> tsh) * 16 + l) << tsh) + (ii & ((1ll << tsh) - 1));
      };
      const double2* t2 = reinterpret_cast<const double2*>(a.t + (static_cast<long long>(L) - a.t_base) * 16 * 16) +
                          half * (RH / 2);
      double y[RH];
#pragma unroll
      for (int r = 0; r < RH; ++r) y[r] = 0.0;
      for (int l0 = 0; l0 < ke; l0 += 4) {
        // the group's u and t loads all issued before the first fold step (one latency per
        // group instead of one per rank)
        double uv[4];
        double2 tv[4][RH / 2];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uv[q] = l0 + q < ke ? __ldcs(u + uidx(l0 + q)) : 0.0;
#pragma unroll
          for (int r2 = 0; r2 < RH / 2; ++r2)
            tv[q][r2] = l0 + q < ke ? __ldg(t2 + (l0 + q) * 8 + r2) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (l0 + q < ke) {
#pragma unroll
            for (int r2 = 0; r2 < RH / 2; ++r2) {
              y[2 * r2] = hadd(y[2 * r2], hmul(uv[q], tv[q][r2].x));
              y[2 * r2 + 1] = hadd(y[2 * r2 + 1], hmul(uv[q], tv[q][r2].y));
            }
          }
        }
      }
#pragma unroll
      for (int r = 0; r < RH; ++r) z[r] = hadd(z[r], y[r]);
    }
  }
#pragma unroll
  for (int r = 0; r < RH; ++r) a.zm[(half * RH + r) * a.n + i] = z[r];
}

// Column-ordered fold schedule for the multi-RHS V^T X pass: per chunk its leaves sorted
// by column cluster start, so the x segments (16 values per point, 128 B) of consecutive
// leaves coincide and stay in L2.  Any order gives the same t (independent folds).
__global__ void col_keys_kernel(const int* __restrict__ cl, long long lo, long long cnt,
                                const long long* __restrict__ starts, int nchunks,
                                unsigned long long* __restrict__ keys, unsigned* __restrict__ vals) {
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < cnt;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long b = lo + q;
    int a0 = 0, z = nchunks;
    while (z - a0 > 1) {
      const int mid = (a0 + z) >> 1;
      if (starts[mid] <= b) a0 = mid;
      else z = mid;
    }
    keys[q] = (static_cast<unsigned long long>(a0) << 54) | (static_cast<unsigned long long>(cl[b]) << 27) |
              static_cast<unsigned long long>(b - starts[a0]);
    vals[q] = static_cast<unsigned>(b);
  }
}

// Symmetric stored near field, R right-hand sides: one CTA of S threads per stored
// S x S block B, staged once into a padded shared tile; thread t folds row t of B
// against x_sigma (leaf (tau, sigma)) and column t against x_tau (leaf (sigma, tau)),
// for every r, each in the reference's sequential order.
template <int S, int RM>
__global__ void __launch_bounds__(S) pair_multi_kernel(const int* __restrict__ list, const int* __restrict__ mirror,
                                                       long long cnt, const int* __restrict__ rl,
                                                       const int* __restrict__ cl, const long long* __restrict__ off,
                                                       const double* __restrict__ vals, const double* __restrict__ xm,
                                                       long long n, int R, double* __restrict__ part) {
  extern __shared__ double pm_smem[];
  double* sB = pm_smem;                  // S x (S+1), padded
  double* sxs = sB + S * (S + 1);        // R x S
  double* sxt = sxs + RM * S;            // R x S
  const int tid = threadIdx.x;
  for (long long q = blockIdx.x; q < cnt; q += gridDim.x) {
    const int L = list[q], M = mirror[q];
    const double* B = vals + off[L];
    for (int j = 0; j < S; ++j) sB[j * (S + 1) + tid] = B[j * S + tid];
    for (int r = 0; r < R; ++r) {
      sxs[r * S + tid] = xm[r * n + cl[L] + tid];
      sxt[r * S + tid] = xm[r * n + rl[L] + tid];
    }
    __syncthreads();
    double y[RM], y2[RM];
#pragma unroll
    for (int r = 0; r < RM; ++r) y[r] = y2[r] = 0.0;
    for (int j = 0; j < S; ++j) {
      const double b1 = sB[j * (S + 1) + tid];  // B(tid, j)
      const double b2 = sB[tid * (S + 1) + j];  // B(j, tid)
#pragma unroll
      for (int r = 0; r < RM; ++r) {
        if (r < R) {
          y[r] = hadd(y[r], hmul(b1, sxs[r * S + j]));
          if (M >= 0) y2[r] = hadd(y2[r], hmul(b2, sxt[r * S + j]));
        }
      }
    }
    double* p1 = part + (static_cast<long long>(L) * S + tid) * R;
    for (int r = 0; r < R; ++r) p1[r] = y[r];
    if (M >= 0) {
      double* p2 = part + (static_cast<long long>(M) * S + tid) * R;
      for (int r = 0; r < R; ++r) p2[r] = y2[r];
    }
    __syncthreads();
  }
}

// ---- DMMA near field (recompute): FP64 tensor cores, mma.sync.m8n8k4 ----------------
// Fragment layouts (PTX ISA, .f64 m8n8k4): A 8x4 row-major, lane holds A[lane/4][lane%4];
// B 4x8, lane holds B[lane%4][lane/4]; C/D 8x8, lane holds D[lane/4][2*(lane%4) + {0,1}].
__device__ __forceinline__ void dmma_m8n8k4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// One warp per 8-row tile of a deepest row cluster; for every dense leaf of the row
// (canonical order) it evaluates the leaf's 8 x n entries directly in A-fragment layout
// and contracts them with X (R/8 n-tiles), then adds the leaf's 8 x R product into
// the tile's accumulators (z += y_leaf, leaf order).
template <int DIM, int NT /* R / 8 */>
__global__ void __launch_bounds__(128) near_dmma_kernel(MArgs a, const long long* __restrict__ tiles,
                                                        long long ntiles) {
  const int lane = threadIdx.x & 31;
  const long long w = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
  if (w >= ntiles) return;
  const long long i0 = tiles[w];  // first row of the tile (inside one deepest cluster)
  const int c = __ldg(a.row_cluster + i0);
  const int ar = lane >> 2, ak = lane & 3;  // A fragment: row, k
  const long long ia = i0 + ar;            // this lane's row for A
  const bool rowok = ia < a.row_end && __ldg(a.row_cluster + (ia < a.n ? ia : i0)) == c;
  double yi[DIM > 0 ? DIM : 20];
  const int dd = DIM > 0 ? DIM : a.d;
  for (int q = 0; q < dd; ++q) yi[q] = rowok ? a.coords[q * a.n + ia] : 0.0;
  double z0[NT], z1[NT];
#pragma unroll
  for (int q = 0; q < NT; ++q) z0[q] = z1[q] = 0.0;
  const int p1 = __ldg(a.dspan_ptr + c + 1);
  for (int p = __ldg(a.dspan_ptr + c); p < p1; ++p) {
    const int rs = __ldg(a.dspans + 2 * p), re = __ldg(a.dspans + 2 * p + 1);
    for (int L = rs; L < re; ++L) {
      const int c0 = a.d_cl[L], nb = a.d_n[L];
      double y0[NT], y1[NT];
#pragma unroll
      for (int q = 0; q < NT; ++q) y0[q] = y1[q] = 0.0;
      for (int k0 = 0; k0 < nb; k0 += 4) {
        const int j = k0 + ak;
        double av = 0.0;
        if (rowok && j < nb) {
          double r2 = 0.0;
#pragma unroll
          for (int q = 0; q < (DIM > 0 ? DIM : 20); ++q) {
            if (q >= dd) break;
            const double dx = hsub(yi[q], __ldg(a.coords + q * a.n + c0 + j));
            r2 = hadd(r2, hmul(dx, dx));
          }
          av = phi_r2(a.kp, r2);
        }
        // B fragment: X[k0 + lane%4][8q + lane/4]
        const int bj = k0 + (lane & 3);
#pragma unroll
        for (int q = 0; q < NT; ++q) {
          const double bv = bj < nb ? __ldg(a.xm + static_cast<long long>(8 * q + (lane >> 2)) * a.n + c0 + bj) : 0.0;
          dmma_m8n8k4(y0[q], y1[q], av, bv);
        }
      }
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        z0[q] = hadd(z0[q], y0[q]);
        z1[q] = hadd(z1[q], y1[q]);
      }
    }
  }
  // D fragment: row lane/4, rhs 8q + 2*(lane%4) + {0,1}
  const long long iz = i0 + (lane >> 2);
  if (iz < a.row_end && __ldg(a.row_cluster + iz) == c) {
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      const int r = 8 * q + 2 * (lane & 3);
      a.zm[static_cast<long long>(r) * a.n + iz] = z0[q];
      a.zm[static_cast<long long>(r + 1) * a.n + iz] = z1[q];
    }
  }
}

// first rows of the 8-row tiles of every deepest cluster in [row_begin, row_end)
__global__ void tile_count_kernel(const long long* __restrict__ lo, const long long* __restrict__ hi, long long ncl,
                                  long long rb, long long re, long long* __restrict__ cnt) {
  for (long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; c < ncl;
       c += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long a = max(lo[c], rb), b = min(hi[c], re);
    cnt[c] = b > a ? (b - a + 7) / 8 : 0;
  }
}
__global__ void tile_fill_kernel(const long long* __restrict__ lo, const long long* __restrict__ hi, long long ncl,
                                 long long rb, long long re, const long long* __restrict__ start,
                                 long long* __restrict__ tiles) {
  for (long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; c < ncl;
       c += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long a = max(lo[c], rb), b = min(hi[c], re);
    for (long long i = a, q = start[c]; i < b; i += 8, ++q) tiles[q] = i;
  }
}

template <int DIM, int RM>
void launch_rows_multi(const MArgs& a, int near, bool far, cudaStream_t s) {
  const long long rows = a.row_end - a.row_begin;
  if (rows <= 0) return;
  const unsigned grid = grid_for(rows, 128);
#define HM_RM(NEAR, FAR) rows_multi_kernel<DIM, NEAR, FAR, RM><<<grid, 128, 0, s>>>(a)
  if (near == 3) {
    if (far) HM_RM(3, true);
    else HM_RM(3, false);
  } else if (near == 2) {
    if (far) HM_RM(2, true);
    else HM_RM(2, false);
  } else if (near == 1) {
    if (far) HM_RM(1, true);
    else HM_RM(1, false);
  } else {
    if (far) HM_RM(0, true);
  }
#undef HM_RM
  HM_LAUNCH_CHECK();
}

template <int DIM>
void dispatch_rows_multi_r(const MArgs& a, int near, bool far, cudaStream_t s) {
  if (a.R <= 4) launch_rows_multi<DIM, 4>(a, near, far, s);
  else if (a.R <= 8) launch_rows_multi<DIM, 8>(a, near, far, s);
  else launch_rows_multi<DIM, 16>(a, near, far, s);
}

void dispatch_rows_multi(const HMatrix& h, const MArgs& a, int near, bool far, cudaStream_t s) {
  if (near == 0 && far && a.R == 16 && a.kmax == 16) {
    const long long rows = a.row_end - a.row_begin;
    if (rows > 0) {
      rows_multi_far16_kernel<<<grid_for(2 * rows, 128), 128, 0, s>>>(a);
      HM_LAUNCH_CHECK();
    }
    return;
  }
  switch (h.d) {
    case 1: dispatch_rows_multi_r<1>(a, near, far, s); break;
    case 2: dispatch_rows_multi_r<2>(a, near, far, s); break;
    case 3: dispatch_rows_multi_r<3>(a, near, far, s); break;
    case 4: dispatch_rows_multi_r<4>(a, near, far, s); break;
    default: dispatch_rows_multi_r<0>(a, near, far, s); break;
  }
}

long long lower_bound_rows_m(const HostVec<int>& rl, long long v) {
  return std::lower_bound(rl.begin(), rl.end(), v, [](int x, long long y) { return x < y; }) - rl.begin();
}

MArgs base_margs(HMatrix& h, int R) {
  MArgs a{};
  a.n = h.n;
  a.row_begin = h.row_begin;
  a.row_end = h.row_end;
  a.R = R;
  a.coords = h.coords.get();
  a.d = h.d;
  a.kp = h.kp;
  a.xm = h.xmR.get();
  a.zm = h.zmR.get();
  a.d_rl = h.dense.rl.get();
  a.d_m = h.dense.m.get();
  a.d_cl = h.dense.cl.get();
  a.d_n = h.dense.n.get();
  a.d_off = h.dense_off.get();
  a.d_vals = h.dense_vals.get();
  a.part = h.partR.get();
  a.S = static_cast<int>(h.n >> h.dmax_leaf);
  a.a_rl = h.aca.rl.get();
  a.a_m = h.aca.m.get();
  a.a_keff = h.k_eff.get();
  a.a_uoff = h.u_off.get();
  a.U = h.U.get();
  a.tile_shift = h.u_tile_shift;
  a.kmax = static_cast<int>(h.cfg.k);
  a.t = h.tR.get();
  a.row_cluster = h.row_cluster.get();
  a.dspan_ptr = h.dspan_ptr.get();
  a.dspans = h.dspans.get();
  a.aspan_ptr = h.aspan_ptr.get();
  a.aspans = h.aspans.get();
  return a;
}

void launch_t_multi(HMatrix& h, const int* order, long long njobs, long long v_base, long long t_base, int R,
                    cudaStream_t s) {
  if (njobs <= 0) return;
  const int kmax = static_cast<int>(h.cfg.k);
  if (kmax > 32) raise(kEinval, "k > 32 not supported by the low-rank apply");
  const int G = kmax <= 16 ? 16 : 32;
  int sms = 0;
  HM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h.device));
  HM_CUDA(cudaMemsetAsync(h.counter.get(), 0, sizeof(int), s));
  const unsigned grid = static_cast<unsigned>(std::min<long long>((njobs * G / 32 + 8) / 8 + 1, sms * 8ll));
#define HM_T(RM)                                                                                                   \
  t_multi_kernel<RM><<<grid, 256, 0, s>>>(order, njobs, h.aca.cl.get(), h.aca.n.get(), h.k_eff.get(),              \
                                          h.v_off.get(), v_base, h.V.get(), h.xmT.get(), h.n, kmax, R, G, t_base, \
                                          h.counter.get(), h.tR.get())
  if (R <= 4) HM_T(4);
  else if (R <= 8) HM_T(8);
  else HM_T(16);
#undef HM_T
  HM_LAUNCH_CHECK();
}

template <int SS, int RM>
void launch_pair_multi(HMatrix& h, int R, unsigned grid, cudaStream_t s) {
  const size_t smem = sizeof(double) * (SS * (SS + 1) + 2 * RM * SS);
  HM_CUDA(cudaFuncSetAttribute(pair_multi_kernel<SS, RM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  pair_multi_kernel<SS, RM><<<grid, SS, smem, s>>>(h.pair_leaf.get(), h.pair_mirror.get(), h.n_pairs,
                                                  h.dense.rl.get(), h.dense.cl.get(), h.dense_off.get(),
                                                  h.dense_vals.get(), h.xmR.get(), h.n, R, h.partR.get());
}

void near_dmma(HMatrix& h, const MArgs& a, cudaStream_t s) {
  // 8-row tiles of the own deepest clusters
  const int D = h.dmax_leaf;
  const long long ncl = 1ll << D;
  const long long base = h.depth_base[D];
  // the tile list depends only on the tree: built by the first DMMA product, then reused
  if (h.n_dmma_tiles < 0) {
    DevBuf<long long> cnt, start;
    cnt.alloc(ncl + 1, s);
    start.alloc(ncl + 1, s);
    tile_count_kernel<<<grid_for(ncl, 256, 1 << 16), 256, 0, s>>>(h.slot_lo.get() + base, h.slot_hi.get() + base, ncl,
                                                                  h.row_begin, h.row_end, cnt.get());
    HM_LAUNCH_CHECK();
    const long long nt = exclusive_scan_i64(cnt.get(), start.get(), ncl, s);
    if (nt > 0) {
      h.dmma_tiles.alloc(nt, s);
      tile_fill_kernel<<<grid_for(ncl, 256, 1 << 16), 256, 0, s>>>(h.slot_lo.get() + base, h.slot_hi.get() + base,
                                                                   ncl, h.row_begin, h.row_end, start.get(),
                                                                   h.dmma_tiles.get());
      HM_LAUNCH_CHECK();
    }
    h.n_dmma_tiles = nt;
  }
  const long long ntiles = h.n_dmma_tiles;
  if (ntiles <= 0) return;
  const unsigned grid = grid_for(ntiles * 32, 128);
#define HM_DM(DIM)                                                                                          \
  if (a.R == 8) near_dmma_kernel<DIM, 1><<<grid, 128, 0, s>>>(a, h.dmma_tiles.get(), ntiles);              \
  else near_dmma_kernel<DIM, 2><<<grid, 128, 0, s>>>(a, h.dmma_tiles.get(), ntiles)
  switch (h.d) {
    case 1: HM_DM(1); break;
    case 2: HM_DM(2); break;
    case 3: HM_DM(3); break;
    case 4: HM_DM(4); break;
    default: HM_DM(0); break;
  }
#undef HM_DM
  HM_LAUNCH_CHECK();
}

}  // namespace

// the column-ordered schedule (built by the first multi-RHS product; falls back to the
// size-ordered schedule when the packed key does not fit)
static const int* multi_fold_order(HMatrix& h, long long lo, long long hi, cudaStream_t s) {
  const long long cnt = hi - lo;
  const int nch = static_cast<int>(h.chunks.size());
  if (cnt <= 0 || nch == 0 || nch > 1000 || cnt >= (1ll << 27) || h.n >= (1ll << 27)) return h.sched_order.get();
  if (h.sched_corder.size() < static_cast<size_t>(cnt)) {
    std::vector<long long> starts(nch + 1);
    for (int c = 0; c < nch; ++c) starts[c] = h.chunks[c].c0;
    starts[nch] = h.chunks.back().c1;
    DevBuf<long long> ds;
    DevBuf<unsigned long long> keys;
    ds.alloc(nch + 1, s);
    keys.alloc(cnt, s);
    h.sched_corder.alloc(cnt, s);
    HM_CUDA(cudaMemcpyAsync(ds.get(), starts.data(), sizeof(long long) * (nch + 1), cudaMemcpyHostToDevice, s));
    col_keys_kernel<<<grid_for(cnt, 256, 1 << 16), 256, 0, s>>>(h.aca.cl.get(), lo, cnt, ds.get(), nch, keys.get(),
                                                                 reinterpret_cast<unsigned*>(h.sched_corder.get()));
    HM_LAUNCH_CHECK();
    radix_sort_pairs(keys.get(), reinterpret_cast<unsigned*>(h.sched_corder.get()), cnt, s);
    HM_CUDA(cudaStreamSynchronize(s));  // the key buffers are released on return
  }
  return h.sched_corder.get();
}

// Morton-ordered product of R right-hand sides: h.xmR -> h.zmR (own rows).// Morton-ordered product of R right-hand sides: h.xmR -> h.zmR (own rows).
void mvp_multi_morton(HMatrix& h, int R, int flags, cudaStream_t s) {
  if (R < 1 || R > kMaxR) raise(kEinval, "mvp_multi: 1 <= nrhs <= 16 per pass");
  const bool dmma = (flags & 1) != 0;
  if (dmma && (h.cfg.near_stored || (R != 8 && R != 16)))
    raise(kEinval, "mvp_multi: the DMMA near field needs the recompute near field and nrhs 8 or 16");
  MArgs a = base_margs(h, R);
  const long long alo = lower_bound_rows_m(h.aca.h_rl, h.row_begin), ahi = lower_bound_rows_m(h.aca.h_rl, h.row_end);
  const long long kmax = h.cfg.k;
  int near = h.cfg.near_stored ? (h.near_sym ? 3 : 2) : 1;
  if (h.cfg.precompute_aca) {
    if (near == 3 && h.n_pairs > 0) {
      const int S = static_cast<int>(h.n >> h.dmax_leaf);
      int sms = 0;
      HM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h.device));
      const unsigned grid = static_cast<unsigned>(std::min<long long>(h.n_pairs, sms * 8ll));
      if (S == 64) {
        if (R <= 8) launch_pair_multi<64, 8>(h, R, grid, s);
        else launch_pair_multi<64, 16>(h, R, grid, s);
      } else {
        if (R <= 8) launch_pair_multi<32, 8>(h, R, grid, s);
        else launch_pair_multi<32, 16>(h, R, grid, s);
      }
      HM_LAUNCH_CHECK();
    }
    const AcaChunk c0c = h.chunks.empty() ? AcaChunk{} : h.chunks.front();
    const long long ub = c0c.ub, vb = c0c.vb;
    launch_t_multi(h, multi_fold_order(h, alo, ahi, s) + c0c.sched_off, ahi - alo, vb, 0, R, s);
    a.a_ubase = ub;
    a.a_lo = alo;
    a.a_hi = ahi;
    a.t_base = 0;
    dispatch_rows_multi(h, a, near, true, s);
    return;
  }
  // recompute mode: near field first (exact rows or DMMA tiles), then ACA chunk by chunk
  if (dmma) near_dmma(h, a, s);
  else dispatch_rows_multi(h, a, near, false, s);
  reset_aca_rejections(h, s);
  const int* corder = multi_fold_order(h, alo, ahi, s);
  for (const AcaChunk& c : h.chunks) {
    const long long c0 = c.c0, c1 = c.c1;
    if (h.U.size() < static_cast<size_t>(c.ue - c.ub)) h.U.alloc(c.ue - c.ub, s);
    if (h.V.size() < static_cast<size_t>(c.ve - c.vb)) h.V.alloc(c.ve - c.vb, s);
    if (h.tR.size() < static_cast<size_t>((c1 - c0) * kmax * R)) h.tR.alloc((c1 - c0) * kmax * R, s);
    compute_aca(h, c, s);
    launch_t_multi(h, corder + c.sched_off, c1 - c0, c.vb, c0, R, s);
    MArgs b = base_margs(h, R);
    b.z_acc = 1;
    b.a_ubase = c.ub;
    b.a_lo = c0;
    b.a_hi = c1;
    b.row_begin = std::max<long long>(h.row_begin, c.row_lo);
    b.row_end = std::min<long long>(h.row_end, c.row_hi);
    b.t_base = c0;
    b.U = h.U.get();
    b.t = h.tR.get();
    dispatch_rows_multi(h, b, 0, true, s);
  }
  h.keff_known = true;
}

// workspaces for R right-hand sides (precompute mode: t for every own leaf)
void ensure_multi(HMatrix& h, int R, cudaStream_t s) {
  const size_t nv = static_cast<size_t>(h.n) * R;
  if (h.xmR.size() < nv) h.xmR.alloc(nv, s);
  if (h.xmT.size() < static_cast<size_t>(h.n) * kMaxR) {  // interleaved copy, padded to 16 per point
    h.xmT.alloc(static_cast<size_t>(h.n) * kMaxR, s);
    h.xmT.zero(s);
  }
  if (h.zmR.size() < nv) h.zmR.alloc(nv, s);
  if (h.cfg.precompute_aca) {
    const size_t nt = static_cast<size_t>(std::max(h.aca.count, 1ll)) * h.cfg.k * R;
    if (h.tR.size() < nt) h.tR.alloc(nt, s);
  }
  if (h.near_sym) {
    const size_t np = static_cast<size_t>(std::max(h.dense.count, 1ll)) * (h.n >> h.dmax_leaf) * R;
    if (h.partR.size() < np) h.partR.alloc(np, s);
  }
  if (h.counter.size() < 1) h.counter.alloc(1, s);
}

void gather_multi(HMatrix& h, const double* X, long long ldx, int R, cudaStream_t s) {
  gather_multi_kernel<<<grid_for(h.n * R, 256, 1 << 16), 256, 0, s>>>(X, ldx, h.perm.get(), h.n, R, h.xmR.get(),
                                                                       h.xmT.get());
  HM_LAUNCH_CHECK();
}

void scatter_multi(HMatrix& h, double* Z, long long ldz, int R, cudaStream_t s) {
  scatter_multi_kernel<<<grid_for(h.n * R, 256, 1 << 16), 256, 0, s>>>(h.zmR.get(), h.perm.get(), h.n, R, Z, ldz);
  HM_LAUNCH_CHECK();
}

}  // namespace hmb

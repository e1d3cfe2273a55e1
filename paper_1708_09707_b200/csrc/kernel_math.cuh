// kernel_math.cuh -- kernel functions phi(r^2) with the reference's exact
// operation order (host + device).
//
//   Gaussian:  exp(-r2)                       core.hpp:71-74
//   Matern:    r2 == 0 ? norm : K1(r)*r*norm  core.cpp:130-134, r = sqrt(r2)
//   r2 = ((0 + dx0*dx0) + dx1*dx1) + ...     core.hpp:103-110 (axis order, no FMA)
//
// Both kernels are bit-exact with the reference: exp and log are ports of the
// glibc FMA variants (glibc_exp.h, glibc_log.h), sqrt/div are IEEE, and no
// product/sum is contracted.
#pragma once
#include "glibc_exp.h"
#include "glibc_log.h"

namespace hmb {

enum KernelKind : int { kGaussian = 0, kMatern = 1 };

struct KernelParams {
  int kind;
  int dim;
  double matern_norm;  // 1 / (2^(beta-1) Gamma(beta)), computed on the host with glibc pow/tgamma
};

HM_HD double hm_log(double x) { return glibc_log(x); }
HM_HD double hm_sqrt(double x) {
#ifdef __CUDA_ARCH__
  return __dsqrt_rn(x);
#else
  return std::sqrt(x);
#endif
}
HM_HD double hm_div(double a, double b) {
#ifdef __CUDA_ARCH__
  return __ddiv_rn(a, b);
#else
  return a / b;
#endif
}

// Loop-invariant constants of the series (bessel_k1_tables.inc, gen_k1_tables.py): the
// device loop reads psi_a(j) + psi_b(j) from a table (the reference's own sequential
// folds, bitwise) and divides by the exact integer (j+1)(j+2) through its correctly
// rounded reciprocal: q = a*y, r = fma(-q, den, a) (exact), q' = fma(r, y, q) is the
// correctly rounded a/den (Markstein's correction with y = RN(1/den); checked bit for
// bit by tests/cpp/div_const_check.c) -- 3 FP64 instructions instead of the ~15 of a
// general IEEE division, the dominant cost of every Matern entry.
struct K1Tables {
  double inv1[64], inv2[64], den[64], rden[64], psi[64];
};
#ifdef __CUDACC__
static __constant__ K1Tables kK1Dev =
#include "bessel_k1_tables.inc"
    ;
#endif

#ifdef __CUDACC__
__device__ __forceinline__ double div_by_const(double a, double den, double rden) {
  const double q = __dmul_rn(a, rden);
  const double r = __fma_rn(-q, den, a);
  return __fma_rn(r, rden, q);
}
#endif

#ifdef __CUDACC__
// The series' exit test `next < 1e-19 * (sum_i1 + 1.0)` (core.cpp:41).  (A branchy variant
// that skips the two FP64 operations outside [1.99e-19, 2.7e-19) -- exact, since sum_i1 is
// in [1, 1.591) on the series branch -- removed 12% of the FP64 instructions but measured
// 7% slower at config 3: the loop is latency-bound, and the branches cost more.)
__device__ __forceinline__ bool k1_series_exit(double next, double sum_i1) {
  return next < hmul(1e-19, hadd(sum_i1, 1.0));
}
#endif

// core.cpp:28-47
HM_HD double bessel_k1_series(double x) {
  const double kEulerGamma = 0.57721566490153286060651209008240243;
  const double q = hmul(hmul(0.25, x), x);
  double term = 1.0;
  double sum_i1 = 0.0;
  double sum_k = 0.0;
#ifdef __CUDA_ARCH__
  for (int j = 0; j < 64; ++j) {
    sum_i1 = hadd(sum_i1, term);
    sum_k = hadd(sum_k, hmul(kK1Dev.psi[j], term));
    const double next = div_by_const(hmul(term, q), kK1Dev.den[j], kK1Dev.rden[j]);
    if (k1_series_exit(next, sum_i1)) break;
    term = next;
  }
#else
  double psi_a = -kEulerGamma;
  double psi_b = 1.0 - kEulerGamma;
  for (int j = 0; j < 64; ++j) {
    sum_i1 = hadd(sum_i1, term);
    sum_k = hadd(sum_k, hmul(hadd(psi_a, psi_b), term));
    const double next = hm_div(hmul(term, q), hmul(j + 1.0, j + 2.0));
    if (next < hmul(1e-19, hadd(sum_i1, 1.0))) break;
    term = next;
    psi_a = hadd(psi_a, hm_div(1.0, j + 1.0));
    psi_b = hadd(psi_b, hm_div(1.0, j + 2.0));
  }
  (void)kEulerGamma;
#endif
  const double i1 = hmul(hmul(0.5, x), sum_i1);
#ifdef __CUDA_ARCH__
  const double inv_x = __drcp_rn(x);  // IEEE round-to-nearest 1/x, = the reference's 1.0 / x
#else
  const double inv_x = hm_div(1.0, x);
#endif
  return hsub(hadd(inv_x, hmul(hm_log(hmul(0.5, x)), i1)), hmul(hmul(0.25, x), sum_k));
}

// core.cpp:51-81
HM_HD double bessel_k1_cf(double x) {
  double b = hmul(2.0, hadd(1.0, x));
  double d = hm_div(1.0, b);
  double h = d;
  double delh = d;
  double q1 = 0.0;
  double q2 = 1.0;
  const double a1 = 0.25;
  double q = a1;
  double c = a1;
  double a = -a1;
  double s = hadd(1.0, hmul(q, delh));
  for (int i = 2; i <= 2000; ++i) {
    a = hsub(a, hmul(2.0, static_cast<double>(i - 1)));
    c = hm_div(hmul(-a, c), static_cast<double>(i));
    const double qnew = hm_div(hsub(q1, hmul(b, q2)), a);
    q1 = q2;
    q2 = qnew;
    q = hadd(q, hmul(c, qnew));
    b = hadd(b, 2.0);
    d = hm_div(1.0, hadd(b, hmul(a, d)));
    delh = hmul(hsub(hmul(b, d), 1.0), delh);
    h = hadd(h, delh);
    const double dels = hmul(q, delh);
    s = hadd(s, dels);
    if (std::fabs(hm_div(dels, s)) < 1e-17) break;
  }
  h = hmul(a1, h);
  const double k0 = hm_div(hmul(hm_sqrt(hm_div(M_PI, hmul(2.0, x))), glibc_exp(-x)), s);
  return hm_div(hmul(k0, hsub(hadd(0.5, x), h)), x);
}

HM_HD double bessel_k1(double x) { return x <= 2.0 ? bessel_k1_series(x) : bessel_k1_cf(x); }

// KernelEvaluator::from_squared_distance (core.hpp:71-74) + matern (core.cpp:130-134)
HM_HD double phi_r2(const KernelParams& kp, double r2) {
  if (kp.kind == kGaussian) return glibc_exp(-r2);
  if (r2 == 0.0) return kp.matern_norm;
  const double r = hm_sqrt(r2);
  return hmul(hmul(bessel_k1(r), r), kp.matern_norm);
}

// ---------------------------------------------------------------------------------
// Two independent entries at once (device).  Each value goes through exactly the
// operations of the scalar function above (bitwise identical results); the two
// instruction streams are merged so the FP64 dependency chains overlap: the main paths
// are straight-line for both values, the rare special cases are fixed up afterwards,
// and the K1 series runs both loops in one with per-value exit masks.
#ifdef __CUDACC__
// glibc exp main path (|x| in [2^-54, 512)); anything else takes glibc_exp afterwards
__device__ __forceinline__ double exp_main(double x) {
  const GlibcExpData& D = kExpDataDev;
  double kd = hfma(x, D.invln2N, D.shift);
  const unsigned long long ki = as_u64(kd);
  kd = hsub(kd, D.shift);
  double r = hfma(kd, D.negln2hiN, x);
  r = hfma(kd, D.negln2loN, r);
  const int idx = static_cast<int>(2u * (ki & 127u));
  const unsigned long long top = ki << 45;
  const double tail = as_double(exp_tab(idx));
  const unsigned long long sbits = exp_tab(idx + 1) + top;
  const double t1 = hfma(r, D.C3, D.C2);
  const double s = hadd(r, tail);
  const double r2 = hmul(r, r);
  const double t2 = hfma(r, D.C5, D.C4);
  const double p = hfma(t1, r2, s);
  const double r4 = hmul(r2, r2);
  const double tmp = hfma(r4, t2, p);
  const double scale = as_double(sbits);
  return hfma(scale, tmp, scale);
}
__device__ __forceinline__ bool exp_main_ok(double x) {
  const unsigned abstop = static_cast<unsigned>(as_u64(x) >> 52) & 0x7ffu;
  return abstop - 969u <= 62u;
}
__device__ __forceinline__ void glibc_exp_x2(double x0, double x1, double& e0, double& e1) {
  e0 = exp_main(x0);
  e1 = exp_main(x1);
  if (!exp_main_ok(x0)) e0 = glibc_exp(x0);
  if (!exp_main_ok(x1)) e1 = glibc_exp(x1);
}

// glibc log main path (not within [1 - 2^-4, 1 + 0x1.09p-4], positive normal)
__device__ __forceinline__ double log_main(double x) {
  const GlibcLogData& D = kLogDataDev;
  const unsigned long long ix = as_u64(x);
  const unsigned long long tmp = ix - 0x3fe6000000000000ull;
  const int i = static_cast<int>((tmp >> 45) & 127u);
  const int k = static_cast<int>(static_cast<long long>(tmp) >> 52);
  const unsigned long long iz = ix - (tmp & (0xfffull << 52));
  const double invc = log_tab(2 * i);
  const double logc = log_tab(2 * i + 1);
  const double z = as_double(iz);
  const double kd = static_cast<double>(k);
  const double w = hfma(kd, D.ln2hi, logc);
  const double r = hfma(z, invc, -1.0);
  const double p1 = hfma(r, D.A[2], D.A[1]);
  const double hi = hadd(r, w);
  const double r2 = hmul(r, r);
  double lo = hadd(hsub(w, hi), r);
  lo = hfma(kd, D.ln2lo, lo);
  const double r3 = hmul(r, r2);
  const double p2 = hfma(r, D.A[4], D.A[3]);
  const double t = hfma(r2, D.A[0], lo);
  const double q = hfma(p2, r2, p1);
  const double y = hfma(r3, q, t);
  return hadd(y, hi);
}
__device__ __forceinline__ bool log_main_ok(double x) {
  const unsigned long long ix = as_u64(x);
  const unsigned top = static_cast<unsigned>(ix >> 48);
  return !(ix - 0x3fee000000000000ull <= 0x308ffffffffffull) && !(top - 0x10u > 0x7fdfu);
}

// two K1 series (core.cpp:28-47) in one loop; a value stops updating at its own exit
__device__ __forceinline__ void bessel_k1_series_x2(double x0, double x1, double& k0, double& k1) {
  const double q0 = hmul(hmul(0.25, x0), x0), q1 = hmul(hmul(0.25, x1), x1);
  double t0 = 1.0, t1 = 1.0, si0 = 0.0, si1 = 0.0, sk0 = 0.0, sk1 = 0.0;
  // Branch-free body: a value whose series has stopped gets term 0, so its further steps
  // add +-0 to sums that are already nonzero (sum_i1 >= 1; sum_k gets -0 only at j = 0,
  // where the term is 1) and keep the term at 0 -- bitwise the reference's `break`.
#pragma unroll 1
  for (int j = 0; j < 64 && (t0 != 0.0 || t1 != 0.0); ++j) {
    const double psi = kK1Dev.psi[j], den = kK1Dev.den[j], rden = kK1Dev.rden[j];
    si0 = hadd(si0, t0);
    si1 = hadd(si1, t1);
    sk0 = hadd(sk0, hmul(psi, t0));
    sk1 = hadd(sk1, hmul(psi, t1));
    const double nx0 = div_by_const(hmul(t0, q0), den, rden), nx1 = div_by_const(hmul(t1, q1), den, rden);
    t0 = k1_series_exit(nx0, si0) ? 0.0 : nx0;
    t1 = k1_series_exit(nx1, si1) ? 0.0 : nx1;
  }
  const double i10 = hmul(hmul(0.5, x0), si0), i11 = hmul(hmul(0.5, x1), si1);
  const double h0 = hmul(0.5, x0), h1 = hmul(0.5, x1);
  double l0 = log_main(h0), l1 = log_main(h1);
  if (!log_main_ok(h0)) l0 = glibc_log(h0);
  if (!log_main_ok(h1)) l1 = glibc_log(h1);
  k0 = hsub(hadd(__drcp_rn(x0), hmul(l0, i10)), hmul(hmul(0.25, x0), sk0));
  k1 = hsub(hadd(__drcp_rn(x1), hmul(l1, i11)), hmul(hmul(0.25, x1), sk1));
}

// V K1 series in one loop (V = 4: two pivot-row entries + two look-ahead column entries)
template <int V>
__device__ __forceinline__ void bessel_k1_series_xv(const double (&x)[V], double (&kv)[V]) {
  double q[V], t[V], si[V], sk[V];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    q[v] = hmul(hmul(0.25, x[v]), x[v]);
    t[v] = 1.0;
    si[v] = 0.0;
    sk[v] = 0.0;
  }
  bool any = true;
#pragma unroll 1
  for (int j = 0; j < 64 && any; ++j) {  // branch-free body, as bessel_k1_series_x2
    const double psi = kK1Dev.psi[j], den = kK1Dev.den[j], rden = kK1Dev.rden[j];
    any = false;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      si[v] = hadd(si[v], t[v]);
      sk[v] = hadd(sk[v], hmul(psi, t[v]));
      const double nx = div_by_const(hmul(t[v], q[v]), den, rden);
      t[v] = k1_series_exit(nx, si[v]) ? 0.0 : nx;
      any |= t[v] != 0.0;
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const double i1 = hmul(hmul(0.5, x[v]), si[v]);
    const double h = hmul(0.5, x[v]);
    double l = log_main(h);
    if (!log_main_ok(h)) l = glibc_log(h);
    kv[v] = hsub(hadd(__drcp_rn(x[v]), hmul(l, i1)), hmul(hmul(0.25, x[v]), sk[v]));
  }
}

// phi for V squared distances at once (bitwise V scalar evaluations)
template <int KIND, int V>
__device__ __forceinline__ void phi_xv(const KernelParams& kp, const double (&r2)[V], double (&f)[V]) {
  if constexpr (KIND == 0) {
    double e[V];
#pragma unroll
    for (int v = 0; v < V; ++v) e[v] = exp_main(-r2[v]);
#pragma unroll
    for (int v = 0; v < V; ++v) f[v] = exp_main_ok(-r2[v]) ? e[v] : glibc_exp(-r2[v]);
  } else {
    double r[V];
    bool series = true;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      r[v] = hm_sqrt(r2[v]);
      series &= r[v] <= 2.0;
    }
    if (series) {
      double kv[V];
      bessel_k1_series_xv<V>(r, kv);
#pragma unroll
      for (int v = 0; v < V; ++v) f[v] = r2[v] == 0.0 ? kp.matern_norm : hmul(hmul(kv[v], r[v]), kp.matern_norm);
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v)
        f[v] = r2[v] == 0.0 ? kp.matern_norm : hmul(hmul(bessel_k1(r[v]), r[v]), kp.matern_norm);
    }
  }
}

// phi for two squared distances (core.hpp:71-74, core.cpp:130-134); KIND 0 Gaussian, 1 Matern
template <int KIND>
__device__ __forceinline__ void phi_x2(const KernelParams& kp, double r2a, double r2b, double& fa, double& fb) {
  if constexpr (KIND == 0) {
    glibc_exp_x2(-r2a, -r2b, fa, fb);
  } else {
    const double ra = hm_sqrt(r2a), rb = hm_sqrt(r2b);
    if (ra <= 2.0 && rb <= 2.0) {
      double ka, kb;
      bessel_k1_series_x2(ra, rb, ka, kb);
      fa = hmul(hmul(ka, ra), kp.matern_norm);
      fb = hmul(hmul(kb, rb), kp.matern_norm);
    } else {
      fa = r2a == 0.0 ? kp.matern_norm : hmul(hmul(bessel_k1(ra), ra), kp.matern_norm);
      fb = r2b == 0.0 ? kp.matern_norm : hmul(hmul(bessel_k1(rb), rb), kp.matern_norm);
      return;
    }
    if (r2a == 0.0) fa = kp.matern_norm;
    if (r2b == 0.0) fb = kp.matern_norm;
  }
}
#endif

// r2 over d axes of SoA coordinates (stride = n), reference axis order.
template <int DIM>
HM_HD double r2_soa(const double* __restrict__ c, long long n, long long i, long long j, int dim) {
  double r2 = 0.0;
  if constexpr (DIM > 0) {
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      const double dx = hsub(c[a * n + i], c[a * n + j]);
      r2 = hadd(r2, hmul(dx, dx));
    }
  } else {
    for (int a = 0; a < dim; ++a) {
      const double dx = hsub(c[a * n + i], c[a * n + j]);
      r2 = hadd(r2, hmul(dx, dx));
    }
  }
  return r2;
}

// r2 between a point held in registers (yi[DIM]) and SoA point j.
template <int DIM>
HM_HD double r2_reg(const double* yi, const double* __restrict__ c, long long n, long long j) {
  double r2 = 0.0;
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    const double dx = hsub(yi[a], c[a * n + j]);
    r2 = hadd(r2, hmul(dx, dx));
  }
  return r2;
}

}  // namespace hmb

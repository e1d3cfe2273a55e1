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

#ifdef __CUDA_ARCH__
__device__ __forceinline__ double div_by_const(double a, double den, double rden) {
  const double q = __dmul_rn(a, rden);
  const double r = __fma_rn(-q, den, a);
  return __fma_rn(r, rden, q);
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
    if (next < hmul(1e-19, hadd(sum_i1, 1.0))) break;
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

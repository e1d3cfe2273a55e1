// glibc_exp.h -- bit-exact port of glibc 2.39 x86-64 `__exp_fma` (host + device).
//
// Why: the reference evaluates every Gaussian entry as std::exp(-r2)
// (proj/include/hmat/core.hpp:71-74).  In d=2 the ACA pivots are chosen by
// argmax among near-ties at the noise floor, so 1-ulp entry differences flip
// pivots and move the product by >1e-8.  CUDA's exp() is not
// glibc's; this port reproduces the operation sequence of the FMA variant that
// the IFUNC resolver selects on FMA/AVX2 hosts, instruction by instruction
// (libm.so.6 @0x79b60, decoded from the objdump listing):
//
//   kd  = fma(x, InvLn2N, Shift); ki = bits(kd); kd -= Shift;
//   r   = fma(kd, NegLn2hiN, x);  r = fma(kd, NegLn2loN, r);
//   t1  = fma(r, C3, C2);  s = r + tail;  r2 = r*r;  t2 = fma(r, C5, C4);
//   p   = fma(t1, r2, s);  r4 = r2*r2;    tmp = fma(r4, t2, p);
//   exp = fma(scale, tmp, scale)
//
// plus the |x|<2^-54 branch (1+x), the |x|>=512 special case and the
// overflow/underflow/inf/nan exits.  Data (constants + 2^(i/128) table) is
// extracted from the same libm at build time by gen_glibc_exp.py.
//
// Every other operation is written so that nvcc cannot contract it (the
// library is compiled with -fmad=false); the FMAs are explicit.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>

#ifdef __CUDACC__
#define HM_HD __host__ __device__ __forceinline__
#else
#define HM_HD inline
#endif

namespace hmb {

struct GlibcExpData {
  double invln2N, shift, negln2hiN, negln2loN, C2, C3, C4, C5;
  unsigned long long tab[256];
};

// one copy per translation unit (no relocatable device code needed)
#ifdef __CUDACC__
static __device__ const GlibcExpData kExpDataDev =
#include "glibc_exp_data.inc"
    ;
#endif
static const GlibcExpData kExpDataHost =
#include "glibc_exp_data.inc"
    ;

HM_HD double as_double(unsigned long long u) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double(static_cast<long long>(u));
#else
  double d;
  std::memcpy(&d, &u, 8);
  return d;
#endif
}
HM_HD unsigned long long as_u64(double d) {
#ifdef __CUDA_ARCH__
  return static_cast<unsigned long long>(__double_as_longlong(d));
#else
  unsigned long long u;
  std::memcpy(&u, &d, 8);
  return u;
#endif
}
HM_HD double hfma(double a, double b, double c) {
#ifdef __CUDA_ARCH__
  return __fma_rn(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}
// explicit non-contracted ops (IEEE round-to-nearest)
HM_HD double hmul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
HM_HD double hadd(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
HM_HD double hsub(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}

HM_HD const GlibcExpData& exp_data() {
#ifdef __CUDA_ARCH__
  return kExpDataDev;
#else
  return kExpDataHost;
#endif
}

HM_HD unsigned long long exp_tab(int i) {
#ifdef __CUDA_ARCH__
  return __ldg(&kExpDataDev.tab[i]);
#else
  return kExpDataHost.tab[i];
#endif
}

// specialcase (e_exp.c), FMA-variant instruction order (libm @0x79c60..0x79d27)
HM_HD double glibc_exp_special(double tmp, unsigned long long sbits, unsigned long long ki) {
  if ((ki & 0x80000000ull) == 0) {
    sbits -= 1009ull << 52;
    const double scale = as_double(sbits);
    const double y = hfma(scale, tmp, scale);
    return hmul(y, 0x1p1009);
  }
  sbits += 1022ull << 52;
  const double scale = as_double(sbits);
  const double st = hmul(scale, tmp);
  double y = hadd(scale, st);
  if (y < 1.0) {
    const double hi = hadd(y, 1.0);
    const double lo = hadd(hsub(scale, y), st);
    double t = hsub(1.0, hi);
    t = hadd(t, y);
    t = hadd(t, lo);
    t = hadd(t, hi);
    y = hsub(t, 1.0);
    if (y == 0.0) y = 0.0;
  }
  return hmul(y, 0x1p-1022);
}

// Bit-exact glibc exp(x) (x86-64 __exp_fma).
HM_HD double glibc_exp(double x) {
  const GlibcExpData& D = exp_data();
  const unsigned long long ix = as_u64(x);
  unsigned abstop = static_cast<unsigned>(ix >> 52) & 0x7ffu;
  if (abstop - 969u > 62u) {                      // outside [2^-54, 512)
    if (static_cast<int>(abstop - 969u) < 0) return hadd(x, 1.0);  // tiny (includes +-0)
    if (abstop >= 1033u) {                         // |x| >= 1024, inf, nan
      if (ix == 0xfff0000000000000ull) return 0.0;
      if (abstop >= 0x7ffu) return hadd(x, 1.0);
      if (ix >> 63) return 0.0;                    // __math_uflow(0): 0x1p-767 * 0x1p-767
      return as_double(0x7ff0000000000000ull);     // __math_oflow(0)
    }
    abstop = 0;                                    // 512 <= |x| < 1024: special case below
  }
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
  if (abstop == 0) return glibc_exp_special(tmp, sbits, ki);
  const double scale = as_double(sbits);
  return hfma(scale, tmp, scale);
}

}  // namespace hmb

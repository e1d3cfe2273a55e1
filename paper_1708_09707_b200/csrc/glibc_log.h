// glibc_log.h -- bit-exact port of glibc 2.39 x86-64 `__log_fma` (host + device).
//
// The Matern kernel's K1 series evaluates log(0.5 x) (proj/src/core.cpp:46); in d=2 the
// ACA pivots are chaotic at the ulp level, so, like exp, log must match
// glibc bit for bit.  Operation sequence decoded from the FMA variant the IFUNC selects
// on FMA/AVX2 hosts (libm.so.6 @0x79d50):
//
//   main:   tmp = ix - OFF; i = (tmp >> 45) % 128; k = tmp >> 52; z = asdouble(ix - (tmp & 0xfff<<52))
//           w  = fma(kd, Ln2hi, logc);  r = fma(z, invc, -1)
//           p1 = fma(r, A2, A1);  hi = r + w;  r2 = r*r;  lo = fma(kd, Ln2lo, (w - hi) + r)
//           r3 = r*r2;  p2 = fma(r, A4, A3);  t = fma(r2, A0, lo);  q = fma(p2, r2, p1)
//           y  = fma(r3, q, t) + hi
//   |x-1| < 0x1.09p-4 (1 - 2^-4 <= x): polynomial B with the rhi/rlo split (fma forms)
//   special: 0 -> -inf, inf -> inf, negative/nan -> nan, subnormal -> renormalise.
#pragma once
#include "glibc_exp.h"

namespace hmb {

struct GlibcLogData {
  double ln2hi, ln2lo;
  double A[5];
  double B[11];
  double tab[256];  // {invc, logc} x 128
};

#ifdef __CUDACC__
static __device__ const GlibcLogData kLogDataDev =
#include "glibc_log_data.inc"
    ;
#endif
static const GlibcLogData kLogDataHost =
#include "glibc_log_data.inc"
    ;

HM_HD const GlibcLogData& log_data() {
#ifdef __CUDA_ARCH__
  return kLogDataDev;
#else
  return kLogDataHost;
#endif
}

HM_HD double log_tab(int i) {
#ifdef __CUDA_ARCH__
  return __ldg(&kLogDataDev.tab[i]);
#else
  return kLogDataHost.tab[i];
#endif
}

HM_HD double glibc_log(double x) {
  const GlibcLogData& D = log_data();
  unsigned long long ix = as_u64(x);
  const unsigned top = static_cast<unsigned>(ix >> 48);
  // close to 1.0: (ix - LO) < (HI - LO), LO = asuint64(1 - 0x1p-4), HI = asuint64(1 + 0x1.09p-4)
  if (ix - 0x3fee000000000000ull <= 0x308ffffffffffull) {
    if (ix == 0x3ff0000000000000ull) return 0.0;
    const double r = hsub(x, 1.0);
    const double r2 = hmul(r, r);
    const double q1 = hfma(r2, D.B[3], hfma(r, D.B[2], D.B[1]));
    const double q2 = hfma(r2, D.B[6], hfma(r, D.B[5], D.B[4]));
    const double r3 = hmul(r, r2);
    const double q3 = hfma(r3, D.B[10], hfma(r2, D.B[9], hfma(r, D.B[8], D.B[7])));
    const double P = hfma(hfma(q3, r3, q2), r3, q1);
    const double t = hfma(r, 0x1p27, r);
    const double rhi = hfma(-0x1p27, r, t);
    const double rr = hmul(rhi, rhi);
    const double rlo = hsub(r, rhi);
    const double hi = hfma(rr, D.B[0], r);
    double lo = hfma(rr, D.B[0], hsub(r, hi));
    lo = hfma(hmul(D.B[0], rlo), hadd(r, rhi), lo);
    const double y = hfma(P, r3, lo);
    return hadd(hi, y);
  }
  if (top - 0x10u > 0x7fdfu) {
    if ((ix << 1) == 0) return -as_double(0x7ff0000000000000ull);  // __math_divzero(1)
    if (ix == 0x7ff0000000000000ull) return x;                      // log(inf) = inf
    if ((top & 0x8000u) || ((~top) & 0x7ff0u) == 0) {
      return as_double(0x7ff8000000000000ull);                      // __math_invalid
    }
    ix = as_u64(hmul(x, 0x1p52)) - (52ull << 52);                   // subnormal
  }
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

}  // namespace hmb

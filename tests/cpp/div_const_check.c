/* div_const_check.c -- checks the device K1 series' division by the loop constant
 * den_j = (j+1)(j+2) (kernel_math.cuh): with y = RN(1/den), q = RN(a*y),
 * r = fma(-q, den, a) (exact), q' = fma(r, y, q) must equal RN(a/den) bit for bit.
 * The quotient's correctness depends only on a's significand (the exponent scales
 * exactly), so random significands over a few binades plus the binade edges cover it.
 * Usage: div_const_check [samples_per_divisor]; exit 0 = no mismatch. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static uint64_t s_state = 0x9E3779B97F4A7C15ull;
static uint64_t next_u64(void) { /* SplitMix64 */
  uint64_t z = (s_state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static double from_bits(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }

int main(int argc, char** argv) {
  const long long samples = argc > 1 ? atoll(argv[1]) : 2000000;
  long long bad = 0, total = 0;
  for (int j = 0; j < 64; ++j) {
    const double den = (j + 1.0) * (j + 2.0);
    const double y = 1.0 / den;
    for (long long t = 0; t < samples + 64; ++t) {
      uint64_t mant;
      if (t < 32) mant = (uint64_t)t;                         /* just above a power of two */
      else if (t < 64) mant = (1ull << 52) - 1 - (uint64_t)(t - 32); /* just below the next */
      else mant = next_u64() & ((1ull << 52) - 1);
      const uint64_t ex = 1023 - 80 + (next_u64() % 84);       /* 2^-80 .. 2^3 */
      const double a = from_bits((ex << 52) | mant);
      const double q = a * y;
      const double r = fma(-q, den, a);
      const double q1 = fma(r, y, q);
      const double want = a / den;
      ++total;
      if (memcmp(&q1, &want, 8) != 0) {
        if (bad < 5) printf("mismatch j=%d a=%a got %a want %a\n", j, a, q1, want);
        ++bad;
      }
    }
  }
  /* general divisors (the ACA pivot, aca.cpp:466-470): y = RN(1/p), both operands in
   * [2^-500, 2^500] as the device fast path requires */
  for (long long t = 0; t < 64 * samples; ++t) {
    const uint64_t ea = 1023 - 60 + (next_u64() % 64), ep = 1023 - 60 + (next_u64() % 64);
    uint64_t ma = next_u64() & ((1ull << 52) - 1), mp = next_u64() & ((1ull << 52) - 1);
    if ((t & 1023) < 8) mp = (1ull << 52) - 1 - (uint64_t)(t & 7);  /* significand of p all ones */
    const double a = from_bits((ea << 52) | ma) * ((t & 2) ? -1.0 : 1.0);
    const double p = from_bits((ep << 52) | mp) * ((t & 4) ? -1.0 : 1.0);
    const double y = 1.0 / p;
    const double q = a * y;
    const double r = fma(-q, p, a);
    const double q1 = fma(r, y, q);
    const double want = a / p;
    ++total;
    if (memcmp(&q1, &want, 8) != 0) {
      if (bad < 5) printf("mismatch (general) a=%a p=%a got %a want %a\n", a, p, q1, want);
      ++bad;
    }
  }
  printf("{\"checked\": %lld, \"mismatches\": %lld}\n", total, bad);
  return bad ? 1 : 0;
}
